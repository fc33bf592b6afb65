"""Randomized stream through the public stream_all (diagnostics)."""
import os, sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
for q in (0, 1):
    cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B,
                         sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0))
    for _ in range(3): p.stream_all(batches, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): p.stream_all(batches, cfg)
    e1.record(); torch.cuda.synchronize()
    print(f"q={q}: {e0.elapsed_time(e1)/5:.3f} ms")
