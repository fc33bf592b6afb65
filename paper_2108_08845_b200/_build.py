"""Build libpsvd.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels)."""

import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libpsvd.so")
SOURCES = ["psvd_tall.cu", "psvd_pass_tma.cu", "psvd_gemm.cu", "psvd_small.cu", "psvd_subspace.cu", "psvd_rand.cu",
           "psvd_api.cu", "psvd_stream.cu", "psvd_rand_api.cu", "psvd_dense.cu", "psvd_big.cu", "psvd_accurate.cu", "psvd_nccl.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC"]


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "psvd.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, defines=(), variant=None):
    """defines: extra -D flags; variant: build lib/libpsvd.<variant>.so instead (A/B timing)."""
    out = LIB if variant is None else os.path.join(LIBDIR, "libpsvd." + variant + ".so")
    if variant is None and not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = out + ".tmp"
    with tempfile.TemporaryDirectory(prefix="psvd_build_") as obj:
        # one nvcc per translation unit, in parallel; then one link
        cmds = [[nvcc()] + NVCC_FLAGS + ["-D" + d for d in defines] +
                ["-c", os.path.join(CSRC, s), "-o", os.path.join(obj, s + ".o")] for s in SOURCES]
        link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a"] + \
            [c[-1] for c in cmds] + ["-ldl", "-o", tmp]

        def run(cmd):
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True, cwd=CSRC)

        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
            for f in [ex.submit(run, c) for c in cmds]:
                f.result()
        run(link)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import sys
    # python -m paper_2108_08845_b200._build [VARIANT NAME=VALUE ...]
    if len(sys.argv) > 1:
        print(build(verbose=True, variant=sys.argv[1], defines=sys.argv[2:]))
    else:
        print(build(force=True, verbose=True))
