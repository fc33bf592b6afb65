"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/psvd.h declares; host-side config validation mirrors the
reference; the product package fails loudly without a GPU (no fallback)."""

import ctypes
import os

import numpy as np
import pytest

import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat


def test_library_exports_header_symbols():
    names = nat.header_symbols()
    assert "psvd_stream_update" in names and "psvd_gram" in names
    lib = ctypes.CDLL(nat.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(nat._SIGS) == set(names)  # ctypes table covers exactly the header
    assert nat.lib().psvd_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        p.StreamConfig(k_modes=0)
    with pytest.raises(ValueError):
        p.StreamConfig(k_modes=2, forget_factor=0.0)
    with pytest.raises(ValueError):
        p.StreamConfig(k_modes=2, forget_factor=1.5)
    with pytest.raises(ValueError):
        p.StreamConfig(k_modes=2, batch_columns=0)
    assert p.StreamConfig(k_modes=2).forget_factor == 0.95
    with pytest.raises(ValueError):
        p.RandomSketchConfig(target_rank=0)
    with pytest.raises(ValueError):
        p.RandomSketchConfig(target_rank=2, oversampling=-1)
    with pytest.raises(ValueError):
        p.RandomSketchConfig(target_rank=2, power_iterations=-1)
    with pytest.raises(ValueError):
        p.RandomSketchConfig(target_rank=2, seed=-1)
    assert p.RandomSketchConfig(target_rank=3, oversampling=4).sketch_width == 7


def test_partition_bounds_matches_oracle():
    import oracle
    for rows, world in [(10, 3), (2 ** 20, 8), (1038240, 8), (9, 9), (17, 4)]:
        assert p.partition_bounds(rows, world) == oracle.partition_bounds(rows, world)
    with pytest.raises(ValueError):
        p.partition_bounds(3, 4)
    with pytest.raises(ValueError):
        p.partition_bounds(3, 0)


def test_host_burgers_matches_oracle_bytes():
    import oracle
    assert np.array_equal(p.burgers_matrix(1024, 64), oracle.burgers_matrix(1024, 64))
    assert np.array_equal(p.burgers_matrix(1024, 64, rows=(5, 99), cols=(3, 17)),
                          oracle.burgers_matrix(1024, 64)[5:99, 3:17])


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError):
        p.stream_initialize(np.eye(4), p.StreamConfig(k_modes=2))


def test_product_never_imports_oracle():
    root = os.path.dirname(p.__file__)
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_apmos_config_validation():
    """ApmosConfig checks of dsvd.py:52-68 (host logic, no GPU)."""
    import pytest
    from paper_2108_08845_b200 import ApmosConfig, RandomSketchConfig
    with pytest.raises(ValueError):
        ApmosConfig(local_rank=0, global_rank=2, k_modes=1)
    with pytest.raises(ValueError):
        ApmosConfig(local_rank=4, global_rank=2, k_modes=3)
    with pytest.raises(ValueError):
        ApmosConfig(local_rank=4, global_rank=4, k_modes=2, sketch=RandomSketchConfig(target_rank=2))
    assert ApmosConfig(local_rank=4, global_rank=4, k_modes=2).use_randomized is False


def _kind_c(param):
    """Category of a C parameter declaration from include/psvd.h."""
    t = param.strip()
    if "*" in t or t.split()[0].endswith("_fn"):
        return "ptr"
    base = " ".join(t.split()[:-1]).replace("const ", "")
    return {"int": "i32", "int64_t": "i64", "long long": "i64", "double": "f64"}[base]


def _kind_ctypes(tp):
    if tp in (ctypes.c_int, ctypes.c_int32):
        return "i32"
    if tp in (ctypes.c_int64, ctypes.c_longlong):
        return "i64"
    if tp is ctypes.c_double:
        return "f64"
    return "ptr"


def test_ctypes_signatures_match_the_header():
    """Every ctypes argtypes list has the header's arity and argument kinds (32 / 64-bit integer,
    double, pointer): a drifted signature would pass wrong bits through the ABI silently."""
    import re
    hdr = open(os.path.join(os.path.dirname(nat.LIB_PATH), "..", "..", "include", "psvd.h")).read()
    protos = re.findall(r"^(?:int|long long|const char\s*\*)\s+(psvd_\w+)\s*\(([^;]*?)\)\s*;", hdr, re.M | re.S)
    assert len(protos) == len(nat._SIGS)
    for name, params in protos:
        params = " ".join(params.split())
        want = [] if params in ("", "void") else [_kind_c(x) for x in params.split(",")]
        got = [_kind_ctypes(t) for t in nat._SIGS[name][1]]
        assert got == want, (name, got, want)
