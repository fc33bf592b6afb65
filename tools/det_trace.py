"""Timeline of the pipelined deterministic stream (PSVD_TRACE=1 stamps), config 2."""
import os, sys
os.environ["PSVD_TRACE"] = "1"
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B, K = 1 << 20, 800, 200, 10
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
batches = [D.view[:, i:i + B] for i in range(0, S, B)]
cfg = p.StreamConfig(k_modes=K, forget_factor=0.95, batch_columns=B)
for i in range(3):
    print(f"---- run {i}", file=sys.stderr, flush=True)
    p.stream_all(batches, cfg)
    torch.cuda.synchronize()
