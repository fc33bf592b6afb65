"""Random row-partitioned streams (parallel_stream_all, deterministic and randomized; processes sharing one GPU
over gloo) against the serial oracle: row counts that leave short / uneven blocks, K up to 40, ragged widths,
windows chained through the state.  python tools/fuzz_parallel.py [seed] [count] [world]"""
import os, random, socket, sys
import numpy as np
sys.path.insert(0, ".")


def cases(seed, count):
    random.seed(seed)
    rng = np.random.Generator(np.random.Philox(seed))
    for _ in range(count):
        M = random.choice([random.randint(40, 400), 16 * random.randint(20, 300), random.randint(300, 5000)])
        K = random.choice([random.randint(1, 16), random.randint(17, 40)])
        if os.environ.get("FUZZ_BIG_K") and random.random() < 0.5:   # the wide cores and panels
            K = random.randint(41, 150)
            M = max(M, K + 10)
        nb = random.randint(2, 7)
        win = random.choice([2, 3, 8])
        widths = [random.randint(max(K, 8), max(K, 8) + random.choice([100, 240])) for _ in range(nb)] if K > 40 else \
            [random.randint(max(K, 8), random.choice([100, 240])) for _ in range(nb)]
        ff = random.choice([1.0, 0.95, 0.8])
        rand = random.random() < 0.4
        q = random.randint(0, 1)
        over = min(random.choice([8, 12]), min(widths) - K)
        cols = sum(widths)
        r = min(random.choice([40, 90]), cols, M)
        U, _ = np.linalg.qr(rng.standard_normal((M, r)))
        V, _ = np.linalg.qr(rng.standard_normal((cols, r)))
        kind = random.choice(["decay", "decay", "steep", "gauss"])
        if kind == "decay":
            a = (U * (2.0 ** -np.arange(r))) @ V.T + 1e-9 * rng.standard_normal((M, cols))
        elif kind == "steep":   # spans that trip the conditioning gates (the accurate routes across ranks)
            a = (U * (random.choice([1e-6, 1e-9, 1e-12]) ** (np.arange(r) / max(r - 1, 1)))) @ V.T
        else:
            a = rng.standard_normal((M, cols))
        per_update = random.random() < 0.3
        batches, c0 = [], 0
        for w in widths:
            batches.append(np.asfortranarray(a[:, c0:c0 + w]))
            c0 += w
        yield dict(M=M, K=K, widths=widths, ff=ff, rand=rand, q=q, over=over, win=win, kind=kind, per_update=per_update), batches


def worker(rank, world, port, seed, count, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2108_08845_b200 as p
    ctx = p.RankContext()
    worst_s = worst_a = 0.0
    done = 0
    try:
        for c, batches in cases(seed, count):
            K, ff = c["K"], c["ff"]
            sk = None
            if c["rand"]:
                sk = p.RandomSketchConfig(target_rank=K, oversampling=max(c["over"], 0), power_iterations=c["q"],
                                          seed=seed)
                if sk.sketch_width > min(c["M"], min(c["widths"])):
                    continue
            p.streaming.STREAM_WINDOW = p.streaming.STREAM_WINDOW_RESIDENT = c["win"]
            cfg = p.StreamConfig(k_modes=K, forget_factor=ff, batch_columns=c["widths"][0], sketch=sk)
            lo, hi = p.partition_bounds(c["M"], world)[rank]
            if c["per_update"]:
                st = p.parallel_stream_initialize(ctx, batches[0][lo:hi], cfg)
                hist = [st.singular_values]
                for b in batches[1:]:
                    st = p.parallel_stream_incorporate(ctx, st, b[lo:hi], cfg)
                    hist.append(st.singular_values)
            else:
                st, hist = p.parallel_stream_all(ctx, [b[lo:hi] for b in batches], cfg)
            full = p.gather_modes(ctx, st)
            done += 1
            if rank:
                continue
            if sk is None:
                ref_m, ref_s, _ = oracle.ref_stream_all(batches, K, ff)
            else:
                ref_m, ref_s, _ = oracle.ref_rand_stream_all(batches, K, ff, sk.oversampling, c["q"], seed)
            m, s = full.cpu().numpy(), st.singular_values.cpu().numpy()
            es = float(np.max(np.abs(s - ref_s) / ref_s - 100 * np.finfo(float).eps * ref_s[0] / ref_s))
            gaps = np.array([min(abs(ref_s[j] - ref_s[i]) for i in range(K) if i != j) / ref_s[j] if K > 1 else 1.0
                             for j in range(K)])
            sel = (gaps > 1e-3) & (ref_s > 1e-6 * ref_s[0])
            ang = oracle.mode_angles(m, ref_m)
            ea = float(np.max(ang[sel])) if sel.any() else 0.0
            if (es > 1e-10 or ea > 1e-8) and len(hist) == len(batches):
                # the case's own conditioning (tools/fuzz_stream.py): the oracle against itself on inputs perturbed
                # by one ulp; flat or rank-exhausted spectra with a sketch amplify rounding from update to update
                pert = np.random.default_rng(1)
                b2 = [b * (1.0 + 2.2e-16 * pert.standard_normal(b.shape)) for b in batches]
                m2, s2, _ = (oracle.ref_stream_all(b2, K, ff) if sk is None else
                             oracle.ref_rand_stream_all(b2, K, ff, sk.oversampling, c["q"], seed))
                cs = float(np.max(np.abs(s2 - ref_s) / ref_s))
                ca = float(np.max(oracle.mode_angles(m2, ref_m)[sel])) if sel.any() else 0.0
                if es <= max(1e-10, 100 * cs) and ea <= max(1e-8, 100 * ca):
                    print(f"  ill-posed case ({c['kind']}, rand={c['rand']}, K={K}): ours {es:.1e} / {ea:.1e}, the oracle "
                          f"under a 1-ulp input perturbation {cs:.1e} / {ca:.1e}", flush=True)
                    continue
            worst_s, worst_a = max(worst_s, es), max(worst_a, ea)
            if es > 1e-10 or ea > 1e-8 or len(hist) != len(batches):
                print("FAIL", c, es, ea, flush=True)
                out.put("fail")
                os._exit(1)
        if rank == 0:
            print(f"{done} streams over {world} ranks ok: worst sigma {worst_s:.2e}, worst angle {worst_a:.2e}",
                  flush=True)
        out.put("ok")
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    world = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    mpc = mp.get_context("spawn")
    out = mpc.Queue()
    procs = [mpc.Process(target=worker, args=(r, world, port, seed, count, out)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=1500)
    sys.exit(0 if all(pr.exitcode == 0 for pr in procs) else 1)
