"""`parsvd decompose` on the device (cli.py:248-359): the four modes read a
PARSVD01 file, run the per-rank body of cli.py:_rank_work on the library, and write the reference's
five output files; the values and modes in them match the oracle on the same bytes."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _p():
    import paper_2108_08845_b200 as p
    return p


@pytest.mark.parametrize("mode", ["serial-stream", "parallel-stream", "serial-batch", "parallel-batch"])
def test_decompose_outputs_match_oracle(tmp_path, mode):
    p = _p()
    a = oracle.burgers_matrix(4096, 800)
    path = str(tmp_path / "burgers.parsvd")
    p.write_matrix(path, a)
    out = str(tmp_path / mode)
    p.decompose(path, out, mode=mode, k=10, ff=0.95, batch=200, r1=40, r2=30)
    for f in ("singular_values.csv", "modes.csv", "modes.svg", "summary.txt"):
        assert os.path.exists(os.path.join(out, f)), f
    s = p.read_singular_values_csv(os.path.join(out, "singular_values.csv"))
    _, m = p.read_modes_csv(os.path.join(out, "modes.csv"))
    if mode in ("serial-stream", "parallel-stream"):
        rm, rs, rh = oracle.ref_stream_all([a[:, c:c + 200] for c in range(0, 800, 200)], 10, 0.95)
        hist = np.loadtxt(os.path.join(out, "singular_value_history.csv"), delimiter=",", skiprows=1)[:, 1:]
        assert hist.shape == (4, 10)
        for h, r in zip(hist, rh):
            assert oracle.sigma_rel_err(h, r) <= 1e-10
    elif mode == "serial-batch":
        ru, rsf, _ = oracle.ref_svd(a, want_vt=False)
        rm, rs = ru[:, :10], rsf[:10]
    else:
        rm, rs = oracle.ref_apmos([a], 40, 30, 10)
    assert oracle.sigma_rel_err(s, rs) <= 1e-10
    assert np.max(oracle.mode_angles(m, rm)) <= 1e-8
    assert np.all(np.sum(m * rm, axis=0) > 0)
    summary = open(os.path.join(out, "summary.txt")).read()
    assert f"mode={mode}" in summary and "rows=4096" in summary and "cols=800" in summary
