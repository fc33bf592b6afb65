"""Timeline of the pipelined randomized stream (PSVD_TRACE=1 stamps), config 2, q from argv."""
import os, sys
os.environ["PSVD_TRACE"] = "1"
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
q = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda", 0)
pad = int(os.environ.get("LD_PAD", "0"))
buf = torch.empty((S, M + pad), dtype=torch.float64, device=dev)
from paper_2108_08845_b200 import _native as nat
D = p.burgers_device(M, S, device=dev, out=nat.DevMat(buf[:, :M].T, M + pad))
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B,
                     sketch=p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0))
for i in range(3):
    print(f"---- run {i}", file=sys.stderr, flush=True)
    p.stream_all(batches, cfg)
    torch.cuda.synchronize()
