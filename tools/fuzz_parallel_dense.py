"""Random shapes, conditionings and rank counts through the row-partitioned dense calls — parallel_qr
(dsvd.py:176-202) and apmos (dsvd.py:39-173) — on processes sharing one GPU over gloo, against the oracle:
short blocks (fewer rows than columns on a rank), steep and rank-deficient inputs included.
python tools/fuzz_parallel_dense.py [seed] [count] [world]"""
import os, random, socket, sys
import numpy as np
sys.path.insert(0, ".")
EPS = np.finfo(float).eps


def cases(seed, count, world):
    random.seed(seed)
    rng = np.random.Generator(np.random.Philox(seed))
    for _ in range(count):
        n = random.choice([random.randint(2, 40), random.randint(41, 230)])
        if os.environ.get("FUZZ_BIG_N") and random.random() < 0.5:   # the global-memory Cholesky / multi-CTA Jacobi
            n = random.randint(231, 420)
        m = random.choice([random.randint(max(n, world), 3 * n + world), random.randint(n, 4000),
                           16 * random.randint(n // 16 + 1, 300)])
        kind = random.choice(["gauss", "decay", "steep", "deficient", "graded"])
        rnk = n
        if kind == "gauss":
            a = rng.standard_normal((m, n))
        elif kind == "graded":   # column norms over up to 60 orders, either direction
            d = random.choice([1e-8, 1e-30, 1e-60]) ** (np.arange(n) / max(n - 1, 1))
            a = rng.standard_normal((m, n)) * (d if random.random() < 0.5 else d[::-1])
        else:
            u, _ = np.linalg.qr(rng.standard_normal((m, n)))
            v, _ = np.linalg.qr(rng.standard_normal((n, n)))
            sv = {"decay": 1e-4, "steep": 1e-11, "deficient": 1e-3}[kind] ** (np.arange(n) / max(n - 1, 1))
            if kind == "deficient":
                rnk = random.randint(1, n)
                sv[rnk:] = 0.0
            a = (u * sv) @ v.T
        r1 = random.randint(1, max(1, min(n, 48, m // world)))
        r2 = random.randint(1, r1)
        k = random.randint(1, min(r2, rnk))   # modes beyond the rank divide by a rounding-level value
        yield dict(m=m, n=n, kind=kind, r1=r1, r2=r2, k=k), a


def worker(rank, world, port, seed, count):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2108_08845_b200 as p
    ctx = p.RankContext()
    worst = dict(orth=0.0, rec=0.0, r=0.0, sig=0.0, ang=0.0)
    nq = na = 0
    try:
        for c, a in cases(seed, count, world):
            m, n = a.shape
            bounds = p.partition_bounds(m, world)
            lo, hi = bounds[rank]
            # ---- parallel_qr
            res = p.parallel_qr(ctx, a[lo:hi])
            dist.all_gather_object(obj := [None] * world, res.q.cpu().numpy())
            rr = [None] * world
            dist.all_gather_object(rr, res.r.cpu().numpy())
            if rank == 0:
                q, r = np.concatenate(obj, axis=0), rr[0]
                assert all(np.array_equal(r, x) for x in rr[1:]), ("r differs between ranks", c)
                an = np.linalg.norm(a, 2)
                orth = float(np.max(np.abs(q.T @ q - np.eye(n))))
                rec = float(np.max(np.abs(q @ r - a)) / an)
                assert np.all(np.diag(r) >= 0) and np.max(np.abs(np.tril(r, -1))) == 0.0, ("r shape", c)
                _, r0 = oracle.ref_qr(a)
                # rows of r whose pivot is resolved: |dr| <= c eps |a|^2 / r_kk (the bar DESIGN states for qr)
                piv = np.abs(np.diag(r0))
                okrow = piv >= 1e-6 * piv[0]
                bound = 64 * EPS * an * an / np.maximum(piv, 1e-300)
                dr = float(np.max((np.max(np.abs(r - r0), axis=1) / bound)[okrow]))
                if c["kind"] == "graded":   # Householder-level: every column of r relative to that column's norm
                    cn = np.linalg.norm(a, axis=0)
                    dr = float(np.max(np.abs(r - r0) / cn[None, :]) / 1e-12)
                    rec = float(np.max(np.abs(q @ r - a) / cn[None, :]))
                worst.update(orth=max(worst["orth"], orth), rec=max(worst["rec"], rec), r=max(worst["r"], dr))
                if orth > 1e-12 or rec > 1e-13 or dr > 1.0:
                    print("FAIL parallel_qr", c, orth, rec, dr, flush=True)
                    os._exit(1)
            nq += 1
            # ---- apmos
            if min(hi - lo for lo, hi in bounds) < 1:
                continue
            cfg = p.ApmosConfig(local_rank=c["r1"], global_rank=c["r2"], k_modes=c["k"])
            try:
                loc = p.apmos(ctx, a[lo:hi], cfg)
            except p.DegenerateModeError:
                loc = None
            full = None if loc is None else p.gather_modes(ctx, loc)
            if rank == 0:
                try:
                    rm, rs = oracle.ref_apmos([a[b[0]:b[1]] for b in bounds], c["r1"], c["r2"], c["k"])
                except Exception as e:
                    assert loc is None, ("the oracle raised, the device did not", c, repr(e))
                    continue
                assert loc is not None, ("the device raised DegenerateModeError, the oracle did not", c)
                rm = np.concatenate(rm, axis=0) if isinstance(rm, (list, tuple)) else rm
                gs, gm, k = loc.singular_values.cpu().numpy(), full.cpu().numpy(), c["k"]
                es = float(np.max(np.abs(gs - rs) / rs - 100 * EPS * rs[0] / rs))
                gaps = np.array([min([abs(rs[j] - rs[i]) for i in range(k) if i != j] + [rs[j]]) / rs[j]
                                 for j in range(k)])
                sel = (gaps > 1e-3) & (rs > 1e-6 * rs[0])
                ea = float(np.max(oracle.mode_angles(gm, rm)[sel])) if sel.any() else 0.0
                worst.update(sig=max(worst["sig"], es), ang=max(worst["ang"], ea))
                if es > 1e-10 or ea > 1e-8:
                    print("FAIL apmos", c, es, ea, flush=True)
                    os._exit(1)
            na += 1
        if rank == 0:
            print(f"{nq} parallel_qr and {na} apmos cases over {world} ranks ok:",
                  {k: f"{v:.1e}" for k, v in worst.items()}, flush=True)
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
    procs = [mpc.Process(target=worker, args=(r, world, port, seed, count)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=1500)
    sys.exit(0 if all(pr.exitcode == 0 for pr in procs) else 1)
