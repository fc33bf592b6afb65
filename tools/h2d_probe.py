"""Host->device bandwidth from pinned memory (diagnostics for the e2e leg)."""
import time
import torch
n = 1 << 20
h = torch.empty((200, n), dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty((200, n), dtype=torch.float64, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D contiguous {h.numel()*8/dt/1e9:.1f} GB/s")
hv = h.T  # column-major view
dv = torch.empty((n, 200), dtype=torch.float64, device="cuda").T.contiguous().T
for it in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    dv.copy_(hv, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D col-major view {h.numel()*8/dt/1e9:.1f} GB/s", dv.stride(), hv.stride())
for it in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"D2H contiguous {h.numel()*8/dt/1e9:.1f} GB/s")
