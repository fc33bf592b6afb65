"""Where the end-to-end time goes: uploads alone, stream_all on device batches, stream_all on pinned batches."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2108_08845_b200 as p
from paper_2108_08845_b200 import _native as nat
M, S, B = 1 << 20, 800, 200
dev = torch.device("cuda", 0)
D = p.burgers_device(M, S, device=dev)
host = torch.empty((S, M), dtype=torch.float64, pin_memory=True)
host.copy_(D.view.T)
pin = [host[i:i + B].T for i in range(0, S, B)]
devb = [D.view[:, i:i + B] for i in range(0, S, B)]
cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=B)

def timeit(f, n=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3

def uploads():
    return [nat.upload_async(b, dev)[0] for b in pin]

print("uploads only    %.1f ms" % timeit(uploads))
print("stream_all dev  %.1f ms" % timeit(lambda: p.stream_all(devb, cfg)))
print("stream_all pin  %.1f ms" % timeit(lambda: p.stream_all(pin, cfg)))
def full():
    st, _ = p.stream_all(pin, cfg)
    st.to_host()
print("e2e (with D2H)  %.1f ms" % timeit(full))
