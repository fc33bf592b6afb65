"""Where the end-to-end step's time goes (config 2, pinned host batches): raw H2D of the four
batches (one stream / two streams), D2H of the modes, and stream_all with and without to_host."""
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
dbuf = torch.empty((S, M), dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def h2d_one():
    with torch.cuda.stream(s1):
        for i in range(0, S, B):
            dbuf[i:i + B].copy_(host[i:i + B], non_blocking=True)


def h2d_two():
    for k, i in enumerate(range(0, S, B)):
        with torch.cuda.stream(s1 if k % 2 == 0 else s2):
            dbuf[i:i + B].copy_(host[i:i + B], non_blocking=True)


def full():
    st, _ = p.stream_all(batches, cfg, device=dev)
    st.to_host()


def no_d2h():
    st, _ = p.stream_all(batches, cfg, device=dev)


mh = torch.empty((10, M), dtype=torch.float64, pin_memory=True)
md = torch.empty((10, M), dtype=torch.float64, device=dev)
print(f"H2D 4 batches, one stream   {timed(h2d_one):7.2f} ms ({S * M * 8 / timed(h2d_one) / 1e6:.1f} GB/s)")
print(f"H2D 4 batches, two streams  {timed(h2d_two):7.2f} ms")
print(f"D2H modes (84 MB)           {timed(lambda: mh.copy_(md, non_blocking=True)):7.2f} ms")
print(f"stream_all, no to_host      {timed(no_d2h):7.2f} ms")
print(f"stream_all + to_host        {timed(full):7.2f} ms")
D2 = [D.view[:, i:i + B] for i in range(0, S, B)]
print(f"stream_all device batches   {timed(lambda: p.stream_all(D2, cfg, device=dev)):7.2f} ms")
