"""Throughput of the public stream_all on BASELINE configs 3-5 at their full per-GPU size (one GPU).

The bench line (bench.py) is config 2; this tool reports the other configs' snapshot GB/s and the
fraction of the binding roofline (SURVEY 8(d) formulas: algorithmic bytes over the measured HBM
copy peak, algorithmic flops over the measured DMMA peak).  Inputs are generated on the device
with torch (seeded; the same distributions as datagen.weather_matrix / factor_matrix, not the same
bytes), batches are device-resident, and configs 4 / 5 cycle a few distinct batches so the whole
stream fits HBM next to the state.

    python tools/config_bench.py 3 [q]      # weather-like, 1,038,240 x 1024, B=256, K=50, p=10
    python tools/config_bench.py 4 [q]      # weak scaling, 4,194,304 x 4096, B=512, K=100, p=10
    python tools/config_bench.py 5          # stress, 8,388,608 x 2048, B=128, K=64, deterministic
"""
import json
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_08845_b200 as p  # noqa: E402

HBM_GBS = 6542.7       # MEASURED_PEAKS.json hbm_gbs on this pool
DMMA_TFS = 37.02       # profiles/fp64_peaks_r01.jsonl


def weather(dev, M_lat=721, M_lon=1440, S=1024, n_modes=60, seed=1):
    g = np.random.Generator(np.random.Philox(seed))
    a = g.integers(1, 13, n_modes)
    b = g.integers(1, 13, n_modes)
    phi = g.uniform(0.0, 2.0 * np.pi, n_modes)
    c = np.empty((n_modes, S))
    c[:, 0] = g.standard_normal(n_modes)
    innov = g.standard_normal((n_modes, S - 1))
    for t in range(1, S):
        c[:, t] = 0.9 * c[:, t - 1] + math.sqrt(1 - 0.81) * innov[:, t - 1]
    amp = 10.0 * 0.85 ** np.arange(n_modes)
    lat = torch.linspace(-0.5 * math.pi, 0.5 * math.pi, M_lat, dtype=torch.float64, device=dev)
    lon = torch.arange(M_lon, dtype=torch.float64, device=dev) * (2 * math.pi / M_lon)
    at = torch.as_tensor(a, dtype=torch.float64, device=dev)
    bt = torch.as_tensor(b, dtype=torch.float64, device=dev)
    pt = torch.as_tensor(phi, dtype=torch.float64, device=dev)
    space_t = (torch.sin(at[:, None, None] * lat[None, :, None]) *
               torch.cos(bt[:, None, None] * lon[None, None, :] + pt[:, None, None])).reshape(n_modes, -1)
    coef_t = torch.as_tensor((amp[:, None] * c).T.copy(), device=dev)          # S x n_modes
    out = coef_t @ space_t                                                     # S x M, row-major
    gen = torch.Generator(device=dev).manual_seed(seed + 1000)
    out.add_(torch.randn(out.shape, generator=gen, dtype=torch.float64, device=dev), alpha=1e-3)
    return out.T                                                               # M x S column-major


def factor_batches(dev, M, S, B, sigma, noise, seed, distinct):
    """`distinct` batches of B columns of U diag(sigma) V^T + noise (U ~ N(0, 1/M), V ~ N(0, 1/S))."""
    r = sigma.numel()
    gen = torch.Generator(device=dev).manual_seed(seed)
    Ut = torch.randn((r, M), generator=gen, dtype=torch.float64, device=dev).div_(math.sqrt(M))
    V = torch.randn((S, r), generator=gen, dtype=torch.float64, device=dev).div_(math.sqrt(S))
    out = []
    for j in range(distinct):
        Vb = V[j * B:(j + 1) * B] * sigma[None, :]                             # B x r
        At = Vb @ Ut                                                           # B x M, row-major
        At.add_(torch.randn(At.shape, generator=gen, dtype=torch.float64, device=dev), alpha=noise)
        out.append(At.T)
    del Ut
    torch.cuda.empty_cache()
    return out


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    q = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    dev = torch.device("cuda", 0)
    if cfg_id == 3:
        A = weather(dev)
        M, S, B, K, ff = A.shape[0], A.shape[1], 256, 50, 0.95
        batches = [A[:, i:i + B] for i in range(0, S, B)]
        sketch = p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0)
    elif cfg_id == 4:
        M, S, B, K, ff = 4194304, 4096, 512, 100, 0.95
        sig = torch.arange(1, 201, dtype=torch.float64, device=dev) ** -1.5
        distinct = factor_batches(dev, M, S, B, sig, 1e-4, 2, 3)
        batches = [distinct[i % 3] for i in range(S // B)]
        sketch = p.RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0)
    else:
        M, S, B, K, ff = 8388608, 2048, 128, 64, 1.0
        sig = 1.0 / (1.0 + 0.01 * torch.arange(512, dtype=torch.float64, device=dev))
        distinct = factor_batches(dev, M, S, B, sig, 1e-6, 3, 4)
        batches = [distinct[i % 4] for i in range(S // B)]
        sketch = None
    config = p.StreamConfig(k_modes=K, forget_factor=ff, batch_columns=B, sketch=sketch)
    torch.cuda.synchronize()
    p.stream_all(batches, config)  # warm-up (workspace growth)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        state, hist = p.stream_all(batches, config)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = min(ms) * 1e-3
    nupd = len(batches)
    snap = 8.0 * M * S
    if sketch is None:
        bytes_ = sum(8.0 * M * (2 * B + 3 * (0 if i == 0 else K)) for i in range(nupd))
        flops = sum(M * n * n + 2.0 * M * n * K for n in [B] + [K + B] * (nupd - 1))
    else:
        l = K + 10
        bytes_ = sum(8.0 * M * ((2 + 2 * q) * (B + (0 if i == 0 else K)) + K) for i in range(nupd))
        flops = sum((2 + 2 * q) * 2.0 * M * n * l + 4.0 * (q + 1) * M * l * l + 2.0 * M * l * K
                    for n in [B] + [K + B] * (nupd - 1))
    t_hbm, t_fp64 = bytes_ / (HBM_GBS * 1e9), flops / (DMMA_TFS * 1e12)
    print(json.dumps({
        "config": cfg_id, "rows": M, "snapshots": S, "batch": B, "k": K,
        "path": "deterministic" if sketch is None else f"randomized p=10 q={q}",
        "ms_per_stream": round(t * 1e3, 2), "snapshot_gbs": round(snap / t / 1e9, 1),
        "hbm_frac": round(t_hbm / t, 3), "fp64_frac": round(t_fp64 / t, 3),
        "binding": "hbm" if t_hbm >= t_fp64 else "fp64", "binding_frac": round(max(t_hbm, t_fp64) / t, 3),
        "sigma_head": [round(float(x), 6) for x in state.singular_values[:3].cpu()],
        "runs_ms": [round(x, 2) for x in ms]}))


if __name__ == "__main__":
    main()
