"""One deterministic and one randomized (q = 0) config-2 stream inside a cudaProfilerStart/Stop range
(ncu --profile-from-start off): the narrow-pass launches of both paths, warm."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
det = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B)
rnd = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B,
                     sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=0, seed=0))
for cfg in (det, rnd):
    p.stream_all(batches, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for cfg in (det, rnd):
    p.stream_all(batches, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
