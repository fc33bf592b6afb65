"""Debug: the row-partitioned pipelined randomized stream vs the serial one (2 gloo ranks on one GPU)."""
import os, sys, socket
import numpy as np
sys.path.insert(0, ".")


def worker(rank, world, port, nb, qit, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2108_08845_b200 as p
    a = oracle.burgers_matrix(6001, 1000)[:, :100 * nb]
    lo, hi = p.partition_bounds(a.shape[0], world)[rank]
    cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=100,
                         sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=qit, seed=0))
    st, hist = p.parallel_stream_all(p.RankContext(), [a[lo:hi, c:c + 100] for c in range(0, 100 * nb, 100)], cfg)
    full = p.gather_modes(p.RankContext(), st)
    if rank == 0:
        q.put((full.cpu().numpy(), [h.cpu().numpy() for h in hist]))
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    import oracle
    import paper_2108_08845_b200 as p
    for nb, qit in ((1, 0), (2, 0), (3, 0), (6, 0), (10, 0), (3, 1)):
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        ctx = mp.get_context("spawn"); q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, port, nb, qit, q)) for r in range(2)]
        for pr in ps: pr.start()
        m, h = q.get(timeout=300)
        for pr in ps: pr.join()
        a = oracle.burgers_matrix(6001, 1000)[:, :100 * nb]
        cfg = p.StreamConfig(k_modes=10, forget_factor=0.95, batch_columns=100,
                             sketch=p.RandomSketchConfig(target_rank=10, oversampling=10, power_iterations=qit, seed=0))
        st, hs = p.stream_all([a[:, c:c + 100] for c in range(0, 100 * nb, 100)], cfg)
        ms, ss = st.numpy()
        print(nb, qit, "sigma", max(oracle.sigma_rel_err(x, y.cpu().numpy()) for x, y in zip(h, hs)),
              "angles", np.max(oracle.mode_angles(m, ms)), flush=True)
