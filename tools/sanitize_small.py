"""A five-second tour of every kernel family on small shapes: the TMA passes (rows a multiple of 16), the cp.async
passes (odd rows), the split-ring fused pass, the pipelined and per-update deterministic / randomized streams, the
wide GEMM route, the accurate routes, the any-width dense kernels, apmos and the Burgers generator.  Written for
   compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_small.py
(compute-sanitizer is closed on this GPU pool, so it has only run plain here; bad accesses are hunted with the
fuzzers against the oracle instead)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p

rng = np.random.default_rng(0)


def lowrank(m, n, r=12, noise=1e-9):
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (u * 2.0 ** -np.arange(r)) @ v.T + noise * rng.standard_normal((m, n))


def batches(a, w):
    return [np.asfortranarray(a[:, i:i + w]) for i in range(0, a.shape[1], w)]


done = 0
for m, k, w, nb in [(2048, 10, 200, 4), (4096, 4, 64, 3), (1000, 7, 33, 4), (37, 3, 9, 3), (2048, 20, 120, 3)]:
    a = lowrank(m, w * nb)
    cfg = p.StreamConfig(k_modes=k, forget_factor=0.95, batch_columns=w)
    st, _ = p.stream_all(batches(a, w), cfg)                       # pipelined window (fused / narrow passes)
    s2 = p.stream_initialize(a[:, :w], cfg)                        # per-update entry points
    s2 = p.stream_incorporate(s2, a[:, w:2 * w], cfg)
    for q in (0, 1):
        if k + 6 > w:
            continue
        sk = p.RandomSketchConfig(target_rank=k, oversampling=6, power_iterations=q, seed=1)
        cr = p.StreamConfig(k_modes=k, forget_factor=0.95, batch_columns=w, sketch=sk)
        p.stream_all(batches(a, w), cr)                            # pipelined randomized (narrow) / wide route (k = 20)
        p.stream_incorporate(p.stream_initialize(a[:, :w], cr), a[:, w:2 * w], cr)
    done += 1
# accurate routes: steep kept spectrum (deterministic gate), steep sketch (randomized gate)
u, _ = np.linalg.qr(rng.standard_normal((1024, 30)))
v, _ = np.linalg.qr(rng.standard_normal((120, 30)))
steep = (u * 1e-9 ** (np.arange(30) / 29)) @ v.T
p.stream_all(batches(steep, 60), p.StreamConfig(k_modes=20, forget_factor=1.0, batch_columns=60))
p.stream_all(batches(steep, 60), p.StreamConfig(k_modes=8, forget_factor=1.0, batch_columns=60,
                                                sketch=p.RandomSketchConfig(target_rank=8, oversampling=8,
                                                                            power_iterations=0, seed=0)))
# dense boundary: one-CTA and any-width kernels, wide and graded inputs
for m, n in [(300, 40), (500, 130), (600, 230), (40, 90), (230, 230)]:
    x = rng.standard_normal((m, n))
    p.qr_factor(x)
    p.svd_full(x)
p.svd_full(rng.standard_normal((400, 180)) * 1e-30 ** (np.arange(180)[::-1] / 179))
p.qr_factor(lowrank(800, 60, r=20, noise=0.0))                     # rank-deficient: the robust route
p.low_rank_svd(lowrank(900, 80), p.RandomSketchConfig(target_rank=6, oversampling=6, power_iterations=2, seed=2))
p.randomized_range(rng.standard_normal((300, 50)), p.RandomSketchConfig(target_rank=5, oversampling=5, seed=3))
# one-shot APMOS (single rank) and the Burgers generator
p.apmos(p.RankContext(), lowrank(700, 50), p.ApmosConfig(local_rank=12, global_rank=10, k_modes=5))
p.generate_right_vectors(rng.standard_normal((300, 20)), 8, method="gram")
p.burgers_device(1000, 40)
import torch
torch.cuda.synchronize()
print("sanitize tour ok:", done, "stream shapes + accurate routes + dense + apmos")
