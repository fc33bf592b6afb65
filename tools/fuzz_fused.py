"""Random shapes through psvd_fused_pass mode 1 (the split-ring kernel) against fp64 matrix products
(tests/test_gpu_fused.py: _run); shapes the kernel refuses are counted, any mismatch raises.
    python tools/fuzz_fused.py [seed] [count]"""
import sys, random
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_fused as t
random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ok = refused = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 60):
    M = 16 * random.randint(2, 600)
    K = random.randint(1, 24)
    Kc = random.choice([0, K, random.randint(1, 24)])
    B = random.randint(max(K, 1), 256)
    Bn = random.randint(1, 256)
    noff = random.choice([0, 1, 3])
    try:
        t._run(M, Kc, B, Bn, K, 1, noff, seed=it)
        ok += 1
    except ValueError as e:
        refused += 1
    except AssertionError as e:
        print("FAIL", (M, Kc, B, Bn, K, noff), e)
        raise
    except Exception as e:
        print("ERROR", (M, Kc, B, Bn, K, noff), repr(e))
        raise
print("ok", ok, "refused", refused)
