"""Two config-4 updates (reduced rows) inside a cudaProfilerStart/Stop range: the wide route's tall-skinny GEMMs."""
import math, sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, B, K = 1 << 20, 512, 100
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(2)
sig = torch.arange(1, 201, dtype=torch.float64, device=dev) ** -1.5
Ut = torch.randn((200, M), generator=g, dtype=torch.float64, device=dev).div_(math.sqrt(M))
batches = []
for j in range(3):
    vb = torch.randn((B, 200), generator=g, dtype=torch.float64, device=dev).mul_(sig / math.sqrt(4096))
    at = vb @ Ut
    at.add_(torch.randn(at.shape, generator=g, dtype=torch.float64, device=dev), alpha=1e-4)
    batches.append(at.T)
cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B,
                     sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=1, seed=0))
p.stream_all(batches, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
p.stream_all(batches[:2], cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
