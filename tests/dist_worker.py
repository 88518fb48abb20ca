"""One rank of the world-size-N sharded step, launched by
paper_1704_07468_b200.parallel.launch (torch.distributed.run): the launcher and
ShardedStep that bench.py uses, with the gloo backend and the CPU test double
(tests/mock_plan.py) in place of libgakco.so. Rank 0 assembles the packed
slices of every rank and compares them with the oracle.

    python -m torch.distributed.run ... tests/dist_worker.py RESULT_PATH
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from paper_1704_07468_b200 import parallel
    from synth import corpus as sc
    from tests.mock_plan import MockPlan
    out_path = sys.argv[1]
    gpu = len(sys.argv) > 2 and sys.argv[2] == "gpu"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    if gpu:  # the real library on cuda:0 (every rank), collectives staged through host
        from paper_1704_07468_b200 import gakco
        cfg = sc.CONFIGS["tiny"]
        cp, g, k, M = sc.make("tiny"), cfg.g, cfg.k, cfg.M
        plan = gakco.Plan(cp.sigma, g, k, M, 0)
        plan.set_shard(rank, world)
        dev = "cuda:0"
    else:
        g, k, M = 6, 3, 3
        cp = sc.random_small(np.random.default_rng(11), 4, n_max=9, l_max=30)
        plan = MockPlan(cp, g, k, M, rank, world)
        dev = "cpu"
    N = cp.n_seq
    nmax = int(max(0, max(int(l) - g + 1 for l in cp.lengths())))
    exch = sys.argv[3] if len(sys.argv) > 3 else "auto"
    st = parallel.ShardedStep(plan, N, g, k, M, nmax, dev, exchange=exch)
    C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
    for _ in range(2 if gpu else 1):  # (twice on the GPU: both receive buffers)
        b, e = st.step(cp.codes, cp.offsets, C)
    if gpu:
        torch.cuda.synchronize()
    mine = {"b": b, "e": e, "Cp": st.complete_C().cpu(), "Nm": st.Nm[:, : e - b].cpu(),
            "K": st.K[: e - b].cpu(), "Kn": st.Knorm[: e - b].cpu()}
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank == 0:
        import oracle
        ref = oracle.compute(cp, g, k, M)
        T = parallel.tri_size(N)
        Cp = np.zeros((M + 1, T), np.int64)
        Nm = np.zeros((M + 1, T), np.int64)
        K = np.zeros(T, np.int64)
        Kn = np.zeros(T, np.float64)
        for r in got:
            Cp[:, r["b"]:r["e"]] = r["Cp"].numpy()
            Nm[:, r["b"]:r["e"]] = r["Nm"].numpy()
            K[r["b"]:r["e"]] = r["K"].numpy()
            Kn[r["b"]:r["e"]] = r["Kn"].numpy()
        iu = np.triu_indices(N)
        ok = (np.array_equal(Cp, ref["C"][:, iu[0], iu[1]])
              and np.array_equal(Nm, ref["Nm"][:, iu[0], iu[1]])
              and np.array_equal(K, ref["K"][iu])
              and np.allclose(Kn, ref["Knorm"][iu], rtol=1e-12, atol=0)
              and sorted((r["b"], r["e"]) for r in got)[-1][1] == T)
        with open(out_path, "w") as f:
            f.write(f"ok world={world} N={N} exchange={st.exchange}" if ok else "mismatch")
    st.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
