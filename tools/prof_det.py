"""One deterministic config-2 stream inside a cudaProfilerStart/Stop range (ncu --profile-from-start off)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
det = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B)
p.stream_all(batches, det)
torch.cuda.synchronize()
torch.cuda.profiler.start()
p.stream_all(batches, det)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
