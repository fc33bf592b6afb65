"""Per-iteration e2e time from a fresh process (pinned host batches -> stream_all -> to_host)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
M, S, B = 1 << 20, 800, 200
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
host = torch.empty((S, M), dtype=torch.float64, pin_memory=True)
host.copy_(D.view.T)
batches = [host[i:i + B].T for i in range(0, S, B)]
cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=B)
t_start = time.perf_counter()
for it in range(14):
    torch.cuda.synchronize(); t = time.perf_counter()
    st, _ = p.stream_all(batches, cfg, device=dev)
    st.to_host()
    torch.cuda.synchronize()
    print(f"iter {it:2d} at {time.perf_counter()-t_start:6.2f} s: {(time.perf_counter()-t)*1e3:7.1f} ms")
