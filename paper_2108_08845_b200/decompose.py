"""The reference's `parsvd decompose` body on the device (cli.py:248-359).

`decompose(...)` is one rank's share of the four modes of cli.py, with the same inputs (a
PARSVD01 matrix file), the same per-rank work (`_rank_work`, cli.py:248-289: the rank's row
block read with `read_submatrix`, streamed through `parallel_stream_initialize` /
`parallel_stream_incorporate`, or the one-shot `apmos`) and the same output files
(`_write_outputs`, cli.py:292-319: singular_values.csv, modes.csv, modes.svg,
singular_value_history.csv, summary.txt).  The transport is torch.distributed (one process per
GPU, e.g. under torchrun) instead of the reference's thread simulator / TCP star; the
summary's byte counters come from the library's exchange accounting (psvd_exchange_stats, the
analogue of CommStats, comm.py:74-88).  Argument parsing and config-file precedence (the rest
of cli.py) stay out of scope.

    python -m paper_2108_08845_b200.decompose INPUT OUTDIR --mode parallel-stream -k 10 --batch 200
    torchrun --nproc-per-node 8 -m paper_2108_08845_b200.decompose INPUT OUTDIR --mode parallel-stream ...
"""

from __future__ import annotations

import argparse
import os

import numpy as np
import torch

from . import io as pio
from .dsvd import RankContext, exchange_stats, gather_modes, parallel_stream_incorporate, parallel_stream_initialize
from .errors import ConfigError
from .linalg import RandomSketchConfig, low_rank_svd, svd_full
from .oneshot import ApmosConfig, apmos
from .streaming import StreamConfig, stream_all

MODES = ("serial-batch", "serial-stream", "parallel-stream", "parallel-batch")


def _sketch(k, oversampling, power_iterations, seed):
    return RandomSketchConfig(target_rank=k, oversampling=oversampling, power_iterations=power_iterations, seed=seed)


def rank_work(ctx, path, mode, k, ff=0.95, batch=100, r1=None, r2=None, randomized=False, oversampling=10,
              power_iterations=1, seed=0, device=None):
    """cli.py:248-289 for one rank: returns the root's result dict (None on other ranks)."""
    rows, cols = pio.read_matrix_header(path)
    lo, hi = __import__("paper_2108_08845_b200").partition_bounds(rows, ctx.world_size)[ctx.rank]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    calls0, bytes0 = exchange_stats(dev)
    history = None
    if mode == "parallel-batch":
        block = pio.read_submatrix(path, lo, hi, 0, cols)
        sk = _sketch(r2, oversampling, power_iterations, seed) if randomized else None
        state = apmos(ctx, block, ApmosConfig(local_rank=r1, global_rank=r2, k_modes=k, use_randomized=randomized,
                                              sketch=sk))
    else:
        cfg = StreamConfig(k_modes=k, forget_factor=ff, batch_columns=batch)
        state, history = None, []
        for start in range(0, cols, batch):
            block = pio.read_submatrix(path, lo, hi, start, min(start + batch, cols))
            state = (parallel_stream_initialize(ctx, block, cfg) if state is None
                     else parallel_stream_incorporate(ctx, state, block, cfg))
            history.append(state.singular_values.cpu().numpy().copy())
        if state is None:
            raise ConfigError(f"{path} has no columns to stream")
    stacked = gather_modes(ctx, state)
    calls1, bytes1 = exchange_stats(dev)
    if ctx.rank != 0:
        return None
    return {"modes": stacked.cpu().numpy(), "values": state.singular_values.cpu().numpy(), "history": history,
            "rows": rows, "cols": cols, "exchange_calls": calls1 - calls0, "bytes_received": bytes1 - bytes0}


def write_outputs(outdir, mode, k, world_size, seed, result):
    """cli.py:292-319: the same five files, byte-compatible emitters (io.py)."""
    os.makedirs(outdir, exist_ok=True)
    modes = np.asarray(result["modes"])
    grid = np.arange(modes.shape[0], dtype=np.float64)
    pio.write_singular_values_csv(os.path.join(outdir, "singular_values.csv"), np.asarray(result["values"]))
    pio.write_modes_csv(os.path.join(outdir, "modes.csv"), grid, modes)
    pio.write_mode_svg(os.path.join(outdir, "modes.svg"), grid, modes)
    history = result.get("history")
    if history is not None:
        pio.write_history_csv(os.path.join(outdir, "singular_value_history.csv"), np.vstack(history))
    lines = [f"mode={mode}", f"rows={result['rows']}", f"cols={result['cols']}", f"k={k}",
             f"world_size={world_size}", f"seed={seed}",
             f"iterations={len(history) if history is not None else 1}",
             f"rank0_exchange_collectives={result.get('exchange_calls', 0)}",
             f"rank0_bytes_received={result.get('bytes_received', 0)}"]
    with open(os.path.join(outdir, "summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")


def decompose(path, outdir, mode="serial-stream", k=10, ff=0.95, batch=100, r1=None, r2=None, randomized=False,
              oversampling=10, power_iterations=1, seed=0, ctx=None, device=None):
    """cli.py:322-359 `_cmd_decompose` for this process (one rank of the world under torchrun)."""
    if mode not in MODES:
        raise ConfigError(f"unknown mode {mode!r}; expected one of {MODES}")
    ctx = ctx or RankContext()
    rows, cols = pio.read_matrix_header(path)
    if mode == "serial-batch":
        a = pio.read_matrix(path)
        if k > min(a.shape):
            raise ConfigError(f"k {k} exceeds min(rows, cols) = {min(a.shape)}")
        res = (low_rank_svd(a, _sketch(k, oversampling, power_iterations, seed), device) if randomized
               else svd_full(a, want_vt=False, device=device))
        result = {"modes": res.u[:, :k].cpu().numpy(), "values": res.s[:k].cpu().numpy(), "history": None,
                  "rows": rows, "cols": cols}
    elif mode == "serial-stream":
        source = pio.BatchSource.from_file(path, batch)
        state, history = stream_all(source, StreamConfig(k_modes=k, forget_factor=ff, batch_columns=batch),
                                    device=device)
        m, s = state.numpy()
        result = {"modes": m, "values": s, "history": [h.cpu().numpy() for h in history], "rows": rows,
                  "cols": cols}
    else:
        if mode == "parallel-batch" and (r1 is None or r2 is None):
            raise ConfigError("parallel-batch needs r1 and r2")
        result = rank_work(ctx, path, mode, k, ff, batch, r1, r2, randomized, oversampling, power_iterations, seed,
                           device)
    if ctx.rank == 0:
        write_outputs(outdir, mode, k, ctx.world_size, seed, result)
    return result


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2108_08845_b200.decompose")
    ap.add_argument("input")
    ap.add_argument("outdir")
    ap.add_argument("--mode", default="serial-stream", choices=MODES)
    ap.add_argument("-k", type=int, default=10)
    ap.add_argument("--ff", type=float, default=0.95)
    ap.add_argument("--batch", type=int, default=100)
    ap.add_argument("--r1", type=int)
    ap.add_argument("--r2", type=int)
    ap.add_argument("--randomized", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    decompose(a.input, a.outdir, a.mode, a.k, a.ff, a.batch, a.r1, a.r2, a.randomized, seed=a.seed)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    print(f"wrote results for {a.mode} to {a.outdir}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
