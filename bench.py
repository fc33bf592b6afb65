#!/usr/bin/env python
"""bench.py — snapshot GB/s through the streaming-SVD update (BASELINE.json metric).

Workload (BASELINE.json configs[1], "config 2"): analytic Burgers snapshots,
2^20 grid rows x 800 snapshots, streamed in batches of 200 (init + 3
incorporates), K = 10 modes, forget factor 0.95, fp64, rows partitioned over
the GPUs with the reference's partition_bounds (strong scaling: total work
fixed).  One "step" = one full pass of the stream (4 updates, 6.7 GB of
snapshots).  Inputs (6.7 GB) are far larger than L2 (126 MB), so no flush is
needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--path det|rand] [--impl reference]

--impl reference times the reference algorithm's CPU implementation (the
numpy oracle port under oracle/, all host threads) on a bounded row sample of
the same workload; under torchrun only rank 0 runs it.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

if "reference" in sys.argv and "TORCHELASTIC_RUN_ID" in os.environ:
    # torchrun exports OMP_NUM_THREADS=1 to its workers and the BLAS reads it when numpy loads: the reference
    # arm uses every host thread at any N (blas_threads() below raises the pool again in any case)
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        if os.environ.get(_v) == "1":
            os.environ[_v] = str(len(os.sched_getaffinity(0)))

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID = 1 << 20
SNAPS = 800
BATCH = 200
K = 10
FF = 0.95
HBM_PEAK = None  # filled from MEASURED_PEAKS.json
FP64_PEAK_TFLOPS = 37.0  # measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peaks_r01.jsonl)


def load_peaks():
    global HBM_PEAK
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            HBM_PEAK = float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        HBM_PEAK = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks_r01.jsonl")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("test") == "dmma_peak":
                    globals()["FP64_PEAK_TFLOPS"] = max(FP64_PEAK_TFLOPS if d.get("warps_per_block") != 4 else 0,
                                                        d["tflops"])
    except Exception:
        pass


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="det", choices=["det", "rand"])
    ap.add_argument("--rows", type=int, default=GRID)
    ap.add_argument("--cpu-rows", type=int, default=1 << 17, help="row sample for the CPU baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rand", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--weak-rows", type=int, default=4194304, help="rows per GPU of the weak-scaling leg (config 4)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region:
    NVML every 2 ms on a thread (one sample at entry and exit at least), falling back
    to `nvidia-smi -lms 200` when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reasons)
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()

    def _nvml_sample(self):
        nv, h = self.nvml
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        reasons = {n for n, b in zip(self.NAMES, bits) if r & b}
        self.rows.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                          float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), reasons))

    def _nvml_loop(self):
        while not self._stop.is_set():
            try:
                self._nvml_sample()
            except Exception:
                return
            self._stop.wait(0.002)

    def __enter__(self):
        if os.environ.get("PSVD_NO_CLOCKS"):
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.index))
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._smi_read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _smi_read(self):
        for line in self.proc.stdout:
            parts = [q.strip() for q in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else 0.0,
                                  {n for n, v in zip(self.NAMES, parts[2:]) if v.lower() == "active"}))

    def __exit__(self, *a):
        if self.nvml is not None:
            self._stop.set()
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def sample_now(self):
        """One extra sample (call while the timed work is still queued on the GPU)."""
        if self.nvml is not None:
            try:
                self._nvml_sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "samples": len(self.rows), "source": "nvml" if self.nvml is not None else "nvidia-smi",
                "reasons": sorted(set().union(*[r[2] for r in self.rows]))}


# ------------------------------------------------------------------ CPU reference

def cpu_reference_gbs(rows, path, steps=1, warmup=0):
    """The reference algorithm's CPU implementation (oracle port, numpy/LAPACK,
    all host threads) on a `rows`-row sample of the workload.  Returns
    (GB/s, seconds per step)."""
    import oracle
    a = oracle.burgers_matrix(GRID, SNAPS, rows=(0, rows))  # the first `rows` grid rows of config 2
    batches = [np.ascontiguousarray(a[:, i:i + BATCH]) for i in range(0, SNAPS, BATCH)]

    def one():
        if path == "det":
            oracle.ref_stream_all(batches, K, FF)
        else:
            oracle.ref_rand_stream_all(batches, K, FF, 10, 1, 0)

    for _ in range(warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    return 8.0 * rows * SNAPS / dt / 1e9, dt


def host_config2(rows):
    """Config-2 host bytes (the first `rows` grid rows of Burgers 2^20 x 800, C-ordered as the
    reference generates them), generated in row slices on every core."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    a = np.empty((rows, SNAPS))
    edges = np.linspace(0, rows, 65).astype(np.int64)

    def fill(i):
        lo, hi = int(edges[i]), int(edges[i + 1])
        if hi > lo:
            a[lo:hi] = oracle.burgers_matrix(GRID, SNAPS, rows=(lo, hi))

    with ThreadPoolExecutor(os.cpu_count()) as ex:
        list(ex.map(fill, range(64)))
    return a


def blas_threads():
    """Give numpy's BLAS / LAPACK every host thread this process may use and return the count it runs with."""
    want = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        threadpool_limits(limits=want)
        got = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") in ("blas", "openmp")]
        return max(got) if got else want
    except Exception:
        return want


def run_reference(a):
    """The reference's CPU path (the oracle port of streaming.py / the R9 composition, numpy
    LAPACK on every host thread) on the SAME config as our arm: all 2^20 grid rows.  One step is
    one update of the stream at full size, cycling init, incorporate, incorporate, incorporate
    (so K steps cover K/4 full streams); warm-up steps run the same cycle on a 2^14-row slice
    (untimed; they only warm the BLAS threads)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    rows = a.rows
    full = host_config2(rows)
    small = full[: 1 << 14]
    nb = SNAPS // BATCH

    def cycle(mat):
        state = {"U": None, "s": None, "b": 0}

        def one():
            b = state["b"]
            blk = mat[:, b * BATCH:(b + 1) * BATCH]
            if a.path == "det":
                if b == 0:
                    state["U"], state["s"] = oracle.ref_stream_init(blk, K)
                else:
                    state["U"], state["s"] = oracle.ref_stream_update(state["U"], state["s"], blk, K, FF)
            else:
                if b == 0:
                    state["U"], state["s"] = oracle.ref_rand_stream_init(blk, K, 10, 1, 0)
                else:
                    state["U"], state["s"] = oracle.ref_rand_stream_update(state["U"], state["s"], blk, K, FF, 10,
                                                                           1, 0)
            state["b"] = (b + 1) % nb
        return one

    cores = blas_threads()
    warm = cycle(small)
    for _ in range(a.warmup):
        warm()
    step = cycle(full)
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    value = 8.0 * rows * BATCH / dt / 1e9  # snapshot bytes of one batch per step
    line = {
        "impl": "reference", "metric": metric_name(a.path), "value": round(value, 4), "unit": "GB/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(dt * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic Burgers, host-generated)", "config": config_dict(a, rows),
        "same_config": rows == GRID,
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"all {rows} grid rows; one step = one update (200 columns) of the 4-update stream, "
                                   f"cycled (oracle/core.py, numpy {np.__version__} LAPACK/BLAS, all {cores} host "
                                   "threads)"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(path):
    return ("snapshot GB/s through streaming-SVD update (Burgers 2^20 x 800, B=200, K=10, ff=0.95, "
            + ("deterministic" if path == "det" else "randomized p=10 q=1") + ")")


def config_dict(a, rows=None):
    return {"workload": f"config2-burgers-2^20x800-{a.path}", "rows": rows or a.rows, "snapshots": SNAPS,
            "batch": BATCH, "k": K, "ff": FF, "path": "deterministic" if a.path == "det" else "randomized",
            "parallelism": f"row-partition x{a.gpus}", "l2": "inputs 6.7 GB >> 126 MB L2, no flush"}


# ------------------------------------------------------------------ our arm

def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2108_08845_b200 as p
    from paper_2108_08845_b200 import _native as nat
    from paper_2108_08845_b200.dsvd import RankContext, allreduce_ordered

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PSVD_BENCH_SHARED_GPU=1 (flow check only, not a measurement): every rank on GPU 0 with gloo
    # through the host, so the N > 1 path runs on a one-GPU box
    shared = os.environ.get("PSVD_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    ctxr = RankContext()
    lo, hi = p.partition_bounds(a.rows, world)[rank]
    M = hi - lo
    D = p.burgers_device(a.rows, SNAPS, rows=(lo, hi), device=dev)  # M x 800 col-major, resident in HBM
    c = nat.context(dev)
    stream = torch.cuda.current_stream(dev)
    st = nat._vp(stream.cuda_stream)
    ld = D.ld

    def col_ptr(j):
        return nat._vp(D.data_ptr() + 8 * ld * j)

    Ubuf = [nat.DevMat.empty(M, K, dev) for _ in range(2)]
    Gloc = {n: torch.empty((n, n), dtype=torch.float64, device=dev) for n in (BATCH, K + BATCH)}

    nb = SNAPS // BATCH
    Aptr = (nat._vp * nb)(*[col_ptr(b * BATCH) for b in range(nb)])
    Ald = (ctypes.c_int64 * nb)(*([ld] * nb))
    Bc = (ctypes.c_int * nb)(*([BATCH] * nb))
    hist = torch.empty((nb, K), dtype=torch.float64, device=dev)
    fin = ctypes.c_int(0)

    ex = None
    if world > 1:
        # the pipelined stream with the library's exchange (dsvd.exchange_hooks): on NCCL the library
        # issues its own in-stream ncclAllGather + rank-ordered sum of the streaming Gram and of U^T U
        # per update (gloo in the shared-GPU flow check: torch.distributed callbacks)
        from paper_2108_08845_b200.dsvd import exchange_hooks
        ex = exchange_hooks(ctxr, dev, lo).__enter__()

    def step(record=False):
        # whole stream through psvd_stream_run (look-ahead A^T A on a second stream); no drift
        # rescue when row-partitioned (dsvd.py:220-242 has none)
        nat.call("psvd_stream_run", c, M, nat._vp(0), 0, nat._vp(0), 0, nb, Aptr, Ald, Bc, K, FF, int(world == 1),
                 nat._vp(Ubuf[0].data_ptr()), nat._vp(Ubuf[1].data_ptr()), Ubuf[0].ld, nat.ptr(hist),
                 ctypes.byref(fin), None, st)
        return Ubuf[fin.value], hist[nb - 1]

    def gram_probe():
        """The dominant kernel on its own: the batch Gram A^T A (M x B, the look-ahead pass of
        psvd_stream_run; psvd_gram with Kc = 0 runs the same TMA-fed Gram kernel in one launch)."""
        n = BATCH
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            nat.call("psvd_gram", c, M, nat._vp(0), 0, nat._vp(0), FF, 0,
                     col_ptr(BATCH), ld, BATCH, nat.ptr(Gloc[n]), st)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 5, M * n * (n + 1)

    def fused_probe():
        """The step's second kernel on its own: the split-ring fused pass over [U | A_b | A_next]
        (psvd_fused_pass mode 1, three Gram tiles offloaded as in the step; the state from the last run)."""
        Wp = torch.randn((K, K + BATCH), dtype=torch.float64, device=dev)
        uu = torch.empty((K, K), dtype=torch.float64, device=dev)
        au = torch.empty((K, BATCH), dtype=torch.float64, device=dev)
        nb32 = (BATCH + 31) // 32
        off = torch.empty((nb32 * nb32, 32, 32), dtype=torch.float64, device=dev)

        def call():
            nat.call("psvd_fused_pass", c, M, nat._vp(Ubuf[0].data_ptr()), Ubuf[0].ld, K, col_ptr(BATCH), ld, BATCH,
                     col_ptr(2 * BATCH), ld, BATCH, nat.ptr(Wp), K, nat._vp(Ubuf[1].data_ptr()), Ubuf[1].ld,
                     nat.ptr(uu), nat.ptr(au), 1, 3, nat.ptr(off), st)
        try:
            call()
        except ValueError:
            return None  # shapes outside the split-ring kernel (the step then runs the narrow TMA pass)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        byts = 8.0 * M * (2 * BATCH + 2 * K)  # reads U, A_b, A_next, writes U
        # DMMA issued per 32 rows: Y = [U | A_b] W, A_next^T Y, Y^T Y on 8-column blocks, 3 offloaded tiles
        ncb = (K + 7) // 8
        kst = ((K + 7) // 8 * 8 + BATCH + 3) // 4
        dm = 4 * ncb * kst + 8 * ncb * ((BATCH + 7) // 8) + 8 * ncb * ncb + 3 * 128
        return {"kernel": "fused_split_kernel (U_b = [U | A_b] W, U_b^T U_b, U_b^T A_next and 3 tiles of "
                          "A_next^T A_next in one read of the panel; 32-row 3-D TMA boxes, two column-group rings)",
                "ms": round(ms, 4), "hbm_gbs": round(byts / (ms * 1e-3) / 1e9, 1),
                "hbm_frac": round(byts / (ms * 1e-3) / 1e9 / HBM_PEAK[0], 4),
                "dmma_tflops_issued": round(dm * 512.0 * (M / 32.0) / (ms * 1e-3) / 1e12, 2),
                "dmma_frac_issued": round(dm * 512.0 * (M / 32.0) / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                "note": "standalone probe; both roofs at once: bytes 8*M*(2B+2K) over the measured HBM peak, DMMA "
                        "issued (8-column padding included) over the measured DMMA peak"}

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    status = nat.read_status(c)
    assert not (status & nat.ST_NONFINITE), "non-finite input"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2108_08845_b200.dsvd import exchange_stats
    launches0 = nat.lib().psvd_launch_count(c)
    ex0 = exchange_stats(dev)
    gt = (ctypes.c_double * 3)()
    with ClockSampler(local) as clk:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        nat.call("psvd_gram_timing", c, 1, gt)  # event pairs around every in-step A^T A Gram
        t0.record(stream)
        for _ in range(a.steps):
            step(record=True)
        t1.record(stream)
        clk.sample_now()  # the queued steps are still running
        barrier()
    nat.call("psvd_gram_timing", c, 0, gt)
    launches = nat.lib().psvd_launch_count(c) - launches0
    ex1 = exchange_stats(dev)
    if ex is not None:
        ex.suspend()
    ms = t0.elapsed_time(t1)
    if world > 1:
        ms = max_over_ranks(ms, dev)
    ms_step = ms / a.steps
    snap_bytes = 8.0 * a.rows * SNAPS  # whole job, all ranks
    value = snap_bytes / (ms_step * 1e-3) / 1e9

    # the dominant kernel IN the step: the look-ahead A^T A Gram launches of psvd_stream_run, timed by
    # event pairs on the library's low-priority stream (they share SMs with the high-priority fused
    # pass, so this is the in-step rate, below the kernel's standalone rate: gram_probe)
    g_ms_sum, g_launches, g_flops = gt[0], int(gt[1]), gt[2]
    g_ach = g_flops / (g_ms_sum * 1e-3) / 1e12 if g_ms_sum > 0 else 0.0
    gms, gfl = gram_probe()
    g_probe = gfl / (gms * 1e-3) / 1e12
    nbu = SNAPS // BATCH
    alg_bytes_step = sum(8.0 * M * (2 * BATCH + 3 * (0 if b == 0 else K)) for b in range(nbu))
    hbm_ach = alg_bytes_step / (ms_step * 1e-3) / 1e9  # per GPU
    gram_share = g_ms_sum / ms
    # SURVEY 8(d) Gram-route flops per update: M n^2 + 2 M n K (n = Kc + B), per GPU
    flops_step = sum(M * (BATCH + (0 if b == 0 else K)) ** 2 + 2.0 * M * (BATCH + (0 if b == 0 else K)) * K
                     for b in range(nbu))
    t_fp64 = flops_step / (FP64_PEAK_TFLOPS * 1e12)
    t_hbm = alg_bytes_step / (HBM_PEAK[0] * 1e9)
    binding = "fp64" if t_fp64 >= t_hbm else "hbm"
    binding_frac = max(t_fp64, t_hbm) / (ms_step * 1e-3)

    traffic = None
    for name in ("ncu_gram_r02.json", "ncu_gram_r01.json"):  # the newest ncu --set full capture of the kernel
        tp = os.path.join(ROOT, "profiles", name)
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    traffic = json.load(f).get("dram_bytes_per_launch")
                break
            except Exception:
                traffic = None

    line = {
        "metric": metric_name(a.path), "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic Burgers, device-generated; same formula as the host generator)",
        "config": config_dict(a),
        "roofline": {"bound": "tensor",
                     "kernel": "gram_tma_kernel (batch Gram A^T A on DMMA, TMA-fed): the in-step look-ahead launches "
                               "of psvd_stream_run, CUDA events on the library's low-priority stream",
                     "achieved": round(g_ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(g_ach / FP64_PEAK_TFLOPS, 4), "traffic": traffic,
                     "peak_source": "measured DMMA.8x8x4 peak (profiles/fp64_peaks_r01.jsonl); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "flops_per_launch": "M*B*(B+1) (upper triangle of A^T A, B = 200) less 2*M*32*32 per 32 x 32 tile "
                                         "the split-ring fused pass of the previous update computes instead (3 of 28 "
                                         "tiles for batches 1..3); traffic = mean DRAM bytes per launch over the "
                                         "step's four launches (profiles/ncu_gram_r02.json)",
                     "launches_timed": g_launches, "share_of_step": round(gram_share, 4),
                     "standalone_probe_tflops": round(g_probe, 3)},
        "hbm_roofline": {"achieved": round(hbm_ach, 1), "peak": HBM_PEAK[0], "unit": "GB/s",
                         "frac": round(hbm_ach / HBM_PEAK[0], 4), "peak_source": HBM_PEAK[1],
                         "bytes_per_step": "sum over updates of 8*M*(2B+3K) per GPU"},
        "binding_roofline": {"bound": binding, "frac": round(binding_frac, 4),
                             "fp64_flops_per_step": flops_step, "t_fp64_ms": round(t_fp64 * 1e3, 3),
                             "t_hbm_ms": round(t_hbm * 1e3, 3),
                             "flops": "sum over updates of M n^2 + 2 M n K (Gram route, SURVEY 8(d)), per GPU"},
        "gpu_launches": int(launches),
    }
    if world == 1:
        fp = fused_probe()
        if fp is not None:
            line["fused_pass"] = fp
    if world > 1:
        upd = a.steps * nbu
        line["exchange"] = {"collectives_per_update": round((ex1[0] - ex0[0]) / upd, 2),
                            "bytes_received_per_update_per_rank": int((ex1[1] - ex0[1]) / upd),
                            "data_plane": "library NCCL (in-stream allgather + rank-ordered sum)"
                            if (ex is not None and ex.nccl) else "torch.distributed callbacks"}
    line["parity"] = self_check(hist[nb - 1], a, world)
    line["clocks"] = clk.summary()

    # ---- end to end through the public API with host (pinned) buffers
    if not a.no_e2e:
        line["e2e"] = e2e(a, p, D, M, dev, world, ctxr)

    if world == 1 and not a.no_rand:
        line["randomized"] = {f"q{qq}": time_randomized(a, D, M, dev, c, stream, qq) for qq in (0, 1)}

    if not a.no_weak:
        del D
        torch.cuda.empty_cache()
        try:
            line["weak_scaling"] = weak_scaling(a, p, dev, world, rank, ctxr)
        except Exception as e:  # reported, never fatal to the headline line
            line["weak_scaling"] = {"error": repr(e)[:300]}

    if world == 1 and rank == 0 and not a.no_cpu:
        cores = blas_threads()
        g, dt = cpu_reference_gbs(a.cpu_rows, a.path)  # bounded row sample; --impl reference runs all rows
        line["cpu_baseline"] = {"value": round(g, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                                "sample": f"first {a.cpu_rows} grid rows x {SNAPS} snapshots, init + 3 incorporates"
                                          f" ({dt:.1f} s; oracle/core.py numpy LAPACK, {cores} threads)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def time_randomized(a, D, M, dev, c, stream, q):
    """Device-resident randomized stream (R9: low_rank_svd of [ff U S | A_i] per
    batch, p = 10, seed 0) over the same 4 batches; snapshot GB/s."""
    import torch
    from paper_2108_08845_b200 import _native as nat
    from paper_2108_08845_b200.linalg import RandomSketchConfig, device_omega
    sk = RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=q, seed=0)
    l = sk.sketch_width
    st = nat._vp(stream.cuda_stream)
    nb = SNAPS // BATCH
    om = {n: device_omega(n, sk, dev) for n in (BATCH, K + BATCH)}
    Uo = nat.DevMat.empty(M, K, dev)
    hist = torch.empty((nb, K), dtype=torch.float64, device=dev)
    Aptr = (nat._vp * nb)(*[nat._vp(D.data_ptr() + 8 * D.ld * b * BATCH) for b in range(nb)])
    Ald = (ctypes.c_int64 * nb)(*([D.ld] * nb))
    Bc = (ctypes.c_int * nb)(*([BATCH] * nb))
    Om = (nat._vp * nb)(*[nat._vp(om[(0 if b == 0 else K) + BATCH].data_ptr()) for b in range(nb)])

    def step():
        # the whole stream through psvd_rand_stream_run (pipelined: the next batch's sketch
        # A Omega[K:] overlaps the small solves; U written once at the end)
        nat.call("psvd_rand_stream_run", c, M, nat._vp(0), 0, nat._vp(0), 0, nb, Aptr, Ald, Bc, K, l, q, FF, Om,
                 nat._vp(Uo.data_ptr()), Uo.ld, nat.ptr(hist), None, st)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(a.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    passes = 2 * (q + 1)
    alg = sum(8.0 * M * (passes * (BATCH + (0 if b == 0 else K)) + K) for b in range(SNAPS // BATCH))
    # FP64 flops of the R9 composition per update and sketch round: C Omega and C^T Q (2 M n l each), the two
    # orthonormalization Grams (M l^2 each, symmetric) and Y T (2 M l^2); U = Q W (2 M l K) once per stream
    flops = sum((q + 1) * M * (4.0 * (BATCH + (0 if b == 0 else K)) * l + 4.0 * l * l) for b in range(nb)) \
        + 2.0 * M * l * K
    return {"value": round(8.0 * a.rows * SNAPS / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "sketch": f"K={K} p=10 q={q} seed=0", "hbm_frac": round(alg / (ms * 1e-3) / 1e9 / HBM_PEAK[0], 4),
            "fp64_frac": round(flops / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
            "fp64_frac_issued": round(flops * 24.0 / l / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
            "note": "both roofs at once: algorithmic bytes over the measured HBM peak, useful FP64 flops over the "
                    "measured DMMA peak; issued = with the sketch's 20 columns padded to three 8-wide DMMA tiles"}


def self_check(sigma_dev, a, world):
    """The timed run's final singular values against the live reference's own full-size run of
    the same config (tests/golden/fullsize_fingerprints.npz, written by make_fullsize.py; the
    device-generated Burgers bytes differ from the host's by a few ulp)."""
    import oracle
    path = os.path.join(ROOT, "tests", "golden", "fullsize_fingerprints.npz")
    if a.rows != GRID or a.path != "det" or not os.path.exists(path):
        return {"checked": False}
    ref = np.load(path)["c2_det_sigma"]
    err = oracle.sigma_rel_err(sigma_dev.cpu().numpy(), ref)
    return {"checked": True, "sigma_rel_err_vs_reference": float(f"{err:.3e}"), "ok": bool(err <= 1e-10),
            "reference": "live reference stream_all at 2^20 rows (fullsize_fingerprints.npz)"}


def weak_scaling(a, p, dev, world, rank, ctxr):
    """BASELINE config 4 (the north star's >= 85% weak-scaling target): 4,194,304 rows per GPU,
    batches of 512 snapshots, 8 updates, K = 100, randomized p = 10, q = 1, through the
    public stream_all (N = 1) / parallel_stream_all (N > 1: every sketch Gram / projection summed
    over the ranks by the library's NCCL exchange).  Data: rank-200 Gaussian-factor signal with
    sigma_i = i^-1.5 plus N(0, 1e-4) noise, generated on the device (seeded; the datagen
    distribution, not its bytes); 3 distinct batches per GPU cycle through the 8 updates so the
    stream fits HBM next to the state.  Timed on the device, max over ranks."""
    import math
    import torch
    import torch.distributed as dist
    M, S, B, KK = a.weak_rows, 4096, 512, 100
    sig = torch.arange(1, 201, dtype=torch.float64, device=dev) ** -1.5
    gen = torch.Generator(device=dev).manual_seed(2 + 7919 * rank)  # this rank's rows of U_f
    Ut = torch.randn((200, M), generator=gen, dtype=torch.float64, device=dev).div_(math.sqrt(M * world))
    gv = torch.Generator(device=dev).manual_seed(2)  # V_f is shared by every rank
    V = torch.randn((S, 200), generator=gv, dtype=torch.float64, device=dev).div_(math.sqrt(S))
    distinct = []
    for j in range(3):
        At = (V[j * B:(j + 1) * B] * sig[None, :]) @ Ut  # B x M row-major = M x B column-major
        At.add_(torch.randn(At.shape, generator=gen, dtype=torch.float64, device=dev), alpha=1e-4)
        distinct.append(At.T)
    del Ut, V
    torch.cuda.empty_cache()
    batches = [distinct[i % 3] for i in range(S // B)]
    sk = p.RandomSketchConfig(target_rank=KK, oversampling=10, power_iterations=1, seed=0)
    cfg = p.StreamConfig(k_modes=KK, forget_factor=0.95, batch_columns=B, sketch=sk)
    stream = torch.cuda.current_stream(dev)

    def one():
        if world == 1:
            return p.stream_all(batches, cfg, device=dev)[0].singular_values
        return p.parallel_stream_all(ctxr, batches, cfg, device=dev)[0].singular_values

    one()  # warm-up (workspaces, Omega uploads)
    steps = max(2, min(a.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        s_last = one()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if world > 1:
        ms = max_over_ranks(ms, dev)
    l = KK + 10
    per_upd_bytes = [8.0 * M * (4 * (B + (0 if u == 0 else KK)) + KK) for u in range(S // B)]
    per_upd_flops = [4 * 2.0 * M * (B + (0 if u == 0 else KK)) * l + 8.0 * M * l * l + 2.0 * M * l * KK
                     for u in range(S // B)]
    return {"config": f"config4: {M:,} rows per GPU x 4096 snapshots, B=512, K=100, p=10, q=1",
            "n_gpus": world, "rows_total": M * world, "ms_per_stream": round(ms, 2),
            "value": round(8.0 * M * world * S / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "per_gpu_gbs": round(8.0 * M * S / (ms * 1e-3) / 1e9, 2),
            "hbm_frac": round(sum(per_upd_bytes) / (ms * 1e-3) / 1e9 / HBM_PEAK[0], 4),
            "fp64_frac": round(sum(per_upd_flops) / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
            "steps": steps, "scaling": "weak", "sigma_head": [round(float(x), 6) for x in s_last[:3].cpu()],
            "data": "device-generated Gaussian factors (datagen.weak_scaling_matrix distribution)"}


def max_over_ranks(x, dev):
    """Max of a host scalar over ranks (on the device under NCCL, through the host under gloo)."""
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    tt = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def e2e(a, p, D, M, dev, world, ctxr):
    """Same metric through the public API (stream_all at N = 1, parallel_stream_* at
    N > 1) with the snapshot batches in pinned host memory: every step copies its
    batches host->device (overlapped with the updates on a side stream) and reads
    the modes + sigma back (StreamState.to_host: one dense copy into pinned memory)."""
    import torch
    import torch.distributed as dist

    host = torch.empty((SNAPS, M), dtype=torch.float64, pin_memory=True)  # column-major M x 800
    host.copy_(D.view.T)
    cfg = p.StreamConfig(k_modes=K, forget_factor=FF, batch_columns=BATCH)
    batches = [host[i:i + BATCH].T for i in range(0, SNAPS, BATCH)]

    def one():
        if world == 1:
            # stream_all: pinned batches upload on a side stream, overlapping the pipelined updates
            st, _ = p.stream_all(batches, cfg, device=dev)
            return st.to_host()
        else:  # row-partitioned pipelined stream (exchange hooks on NCCL)
            st, _ = p.parallel_stream_all(ctxr, batches, cfg, device=dev)
            m, s = st.modes, st.singular_values
        return m.cpu(), s.cpu()

    # same warm-up count as the device-timed leg, and the same allocation pattern as the timed loop:
    # holding the previous result while the next one is produced makes the second pinned host block
    # (StreamState.to_host) get allocated here, not inside the timed region
    out = None
    for _ in range(max(2, getattr(a, "warmup", 3))):
        ti = time.perf_counter()
        out = one()
        if os.environ.get("PSVD_E2E_VERBOSE"):
            torch.cuda.synchronize()
            print(f"e2e warm-up {(time.perf_counter() - ti) * 1e3:.1f} ms", file=sys.stderr)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n = max(3, min(a.steps, 10))
    verbose = os.environ.get("PSVD_E2E_VERBOSE")
    import gc
    gc.collect()
    gc.disable()  # no collector pauses inside the wall-clock region
    t0 = time.perf_counter()
    for _ in range(n):
        ti = time.perf_counter()
        out = one()
        if verbose:
            torch.cuda.synchronize()
            print(f"e2e iteration {(time.perf_counter() - ti) * 1e3:.1f} ms", file=sys.stderr)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    gc.enable()
    if world > 1:
        dt = max_over_ranks(dt, dev)
    return {"value": round(8.0 * a.rows * SNAPS / dt / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(8 * M * SNAPS), "d2h_bytes_per_step": int(out[0].numel() * 8 + out[1].numel() * 8),
            "ms_per_step": round(dt * 1e3, 2), "steps": n,
            "path": "public API stream_all (N=1) / parallel_stream_all (N>1) from pinned host batches"}


def main():
    a = args_()
    load_peaks()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
