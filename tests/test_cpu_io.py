"""PARSVD01 files and column-batch readers (io.py:1-153), byte-compatible with the
reference (tests/golden/sample_37x11.parsvd was written by the live reference)."""
import os

import numpy as np
import pytest

from paper_2108_08845_b200 import io as pio
from paper_2108_08845_b200.errors import MatrixFormatError

SAMPLE = os.path.join(os.path.dirname(__file__), "golden", "sample_37x11.parsvd")


def _sample():
    return np.random.Generator(np.random.Philox(77)).standard_normal((37, 11))


def test_reader_and_writer_match_reference_bytes(tmp_path):
    a = _sample()
    assert pio.read_matrix_header(SAMPLE) == (37, 11)
    assert np.array_equal(pio.read_matrix(SAMPLE), a)
    out = tmp_path / "m.parsvd"
    pio.write_matrix(out, a)
    assert out.read_bytes() == open(SAMPLE, "rb").read()


def test_submatrix_and_batches(tmp_path):
    a = _sample()
    assert np.array_equal(pio.read_submatrix(SAMPLE, 0, 37, 3, 9), a[:, 3:9])
    assert np.array_equal(pio.read_submatrix(SAMPLE, 5, 20, 2, 11), a[5:20, 2:11])
    assert pio.read_submatrix(SAMPLE, 4, 4, 0, 3).shape == (0, 3)
    src = pio.BatchSource.from_file(SAMPLE, 4)
    got = list(src)
    assert len(src) == 3 and [b.shape[1] for b in got] == [4, 4, 3]
    assert np.array_equal(np.concatenate(got, axis=1), a)
    part = list(pio.BatchSource(4, path=SAMPLE, rows=(10, 30)))
    assert np.array_equal(np.concatenate(part, axis=1), a[10:30])
    assert all(np.array_equal(x, y) for x, y in zip(pio.BatchSource.from_matrix(a, 5), [a[:, :5], a[:, 5:10], a[:, 10:]]))
    with pytest.raises(ValueError):
        pio.read_submatrix(SAMPLE, 0, 38, 0, 1)
    with pytest.raises(ValueError):
        pio.BatchSource(0, path=SAMPLE)
    with pytest.raises(ValueError):
        pio.BatchSource(2)


def test_format_errors(tmp_path):
    raw = open(SAMPLE, "rb").read()
    cases = {"short": raw[:10], "magic": b"PARSVD02" + raw[8:], "trunc": raw[:-8], "garbage": raw + b"x"}
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(MatrixFormatError):
            pio.read_matrix(p)
    p = tmp_path / "trunc2"
    p.write_bytes(raw[:-8])
    with pytest.raises(MatrixFormatError):
        pio.read_submatrix(p, 0, 37, 0, 11)
    with pytest.raises(ValueError):
        pio.write_matrix(tmp_path / "nan", np.array([[np.nan]]))
