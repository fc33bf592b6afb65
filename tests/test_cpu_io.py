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


def test_text_emitters_match_reference_bytes(tmp_path):
    """io.py:156-270: sigma / modes / history CSV and the mode SVG, byte for byte against files
    the live reference wrote (tests/golden/make_golden.py outputs()), and their readers."""
    g = os.path.join(os.path.dirname(__file__), "golden")
    rng = np.random.Generator(np.random.Philox(78))
    grid = np.linspace(0.0, 1.0, 33)
    modes = rng.standard_normal((33, 4))
    sigma = np.sort(np.abs(rng.standard_normal(6)))[::-1] * 1e3
    hist = np.abs(rng.standard_normal((5, 3)))
    cases = [("out_sigma.csv", lambda p: pio.write_singular_values_csv(p, sigma)),
             ("out_modes.csv", lambda p: pio.write_modes_csv(p, grid, modes)),
             ("out_history.csv", lambda p: pio.write_history_csv(p, hist)),
             ("out_modes.svg", lambda p: pio.write_mode_svg(p, grid, modes[:, :3])),
             ("out_flat.svg", lambda p: pio.write_mode_svg(p, np.arange(5.0), np.ones((5, 2))))]
    for name, write in cases:
        out = tmp_path / name
        write(out)
        assert out.read_bytes() == open(os.path.join(g, name), "rb").read(), name
    assert np.array_equal(pio.read_singular_values_csv(os.path.join(g, "out_sigma.csv")), sigma)
    gb, mb = pio.read_modes_csv(os.path.join(g, "out_modes.csv"))
    assert np.array_equal(gb, grid) and np.array_equal(mb, modes)
    with pytest.raises(ValueError):
        pio.write_modes_csv(tmp_path / "x.csv", np.zeros(3), np.zeros((4, 2)))
    junk = tmp_path / "junk.csv"
    junk.write_text("time,value\n0,1\n")
    with pytest.raises(MatrixFormatError):
        pio.read_singular_values_csv(junk)
    with pytest.raises(MatrixFormatError):
        pio.read_modes_csv(junk)
