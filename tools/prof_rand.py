"""One randomized (q from argv, default 0) config-2 stream inside a cudaProfilerStart/Stop range."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
q = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
rnd = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B,
                     sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0))
p.stream_all(batches, rnd)
torch.cuda.synchronize()
torch.cuda.profiler.start()
p.stream_all(batches, rnd)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
