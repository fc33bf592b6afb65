"""PyParSVD's class surface (PAPER.md listings 1-2) over the function API: construction,
configuration and call-order checks (no device work; the numerics are in test_gpu_stream.py)."""
import pytest

import paper_2108_08845_b200 as p


def test_serial_class_config_and_defaults():
    s = p.Parsvd_Serial(10, 0.9)
    assert s.config == p.StreamConfig(k_modes=10, forget_factor=0.9, batch_columns=1)
    assert s.iteration == 0 and s.modes is None and s.singular_values is None and s.state is None
    r = p.Parsvd_Serial(7, low_rank=True)
    assert r.config.sketch == p.RandomSketchConfig(target_rank=7, oversampling=10, power_iterations=1, seed=0)
    sk = p.RandomSketchConfig(target_rank=7, oversampling=4, power_iterations=0, seed=3)
    assert p.Parsvd_Serial(7, sketch=sk).config.sketch is sk


@pytest.mark.parametrize("kw", [dict(K=0), dict(K=5, ff=0.0), dict(K=5, ff=1.5)])
def test_class_validation_follows_stream_config(kw):
    with pytest.raises(ValueError):
        p.Parsvd_Serial(**kw)
    with pytest.raises(ValueError):
        p.Parsvd_Parallel(**kw)


def test_incorporate_before_initialize_raises():
    with pytest.raises(ValueError, match="initialize"):
        p.Parsvd_Serial(3).incorporate_data([[1.0, 2.0], [3.0, 4.0]])
    par = p.Parsvd_Parallel(3)
    assert par.rank == 0 and par.nprocs == 1 and par.ulocal is None and par.modes is None
    with pytest.raises(ValueError, match="initialize"):
        par.incorporate_data([[1.0]])
    with pytest.raises(ValueError, match="initialize"):
        par.gather_modes()
