"""bench.e2e: first call in a process vs later calls (diagnostics)."""
import sys, time, types, os
import torch
sys.path.insert(0, ".")
import bench
import paper_2108_08845_b200 as p
from paper_2108_08845_b200.dsvd import RankContext
bench.load_peaks()
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
a = types.SimpleNamespace(rows=1 << 20, steps=3, warmup=3)
D = p.burgers_device(a.rows, bench.SNAPS, device=dev)
if os.environ.get("PREPIN"):
    h = torch.empty((bench.SNAPS, a.rows), dtype=torch.float64, pin_memory=True)
    h.fill_(0.0)
    del h
s0 = torch.cuda.memory_stats(dev)
r = bench.e2e(a, p, D, a.rows, dev, 1, RankContext())
s1 = torch.cuda.memory_stats(dev)
print("e2e first", r["value"], "device cudaMallocs", s1.get("num_device_alloc", 0) - s0.get("num_device_alloc", 0))
s0 = torch.cuda.memory_stats(dev)
r = bench.e2e(a, p, D, a.rows, dev, 1, RankContext())
s1 = torch.cuda.memory_stats(dev)
print("e2e second", r["value"], "device cudaMallocs", s1.get("num_device_alloc", 0) - s0.get("num_device_alloc", 0))
