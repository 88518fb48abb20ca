"""World-size-2 gloo test of the mask-sharded path on CPU (-m "not gpu").

Each rank emulates gakco_accumulate for its mask shard with the literal
Algorithm 1 reference (tests/refs.py, test-only), the partial int64 C are
reduced to rank 0 through torch.distributed (gloo here, NCCL on B200s), and rank
0 checks the full C against the oracle. The shard rule is the one the C library
uses (paper_1704_07468_b200.parallel).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _partial_C(cp, g, M, my_masks):
    from collections import Counter
    from tests.refs import gmers
    N = cp.n_seq
    C = np.zeros((M + 1, N, N), dtype=np.int64)
    per_seq = [gmers(cp.seq(i), g) for i in range(N)]
    for m, removed in my_masks:
        kept = [p for p in range(g) if p not in removed]
        groups = {}
        for s in range(N):
            for gm in per_seq[s]:
                groups.setdefault(tuple(gm[p] for p in kept), Counter())[s] += 1
        for cnt in groups.values():
            for a, ca in cnt.items():
                for b, cb in cnt.items():
                    if b >= a:  # upper triangle, as gakco_accumulate
                        C[m, a, b] += ca * cb
    return C


def _worker(rank, world, port, result_path):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1704_07468_b200 import parallel
    from synth import corpus as sc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, k, M = 6, 3, 3
    rng = np.random.default_rng(5)
    cp = sc.random_small(rng, 4, n_max=7, l_max=30)
    N = cp.n_seq
    mine = parallel.shard_masks(g, M, rank, world)
    C = torch.zeros((M + 1, N, N), dtype=torch.int64)
    out = {}

    def acc(Ct):
        Ct += torch.from_numpy(_partial_C(cp, g, M, mine))

    def fin(Ct):
        out["C"] = Ct.numpy().copy()

    acc(C)
    dist.reduce(C, dst=0, op=dist.ReduceOp.SUM)
    if rank == 0:
        fin(C)
        import oracle
        ref = oracle.compute(cp, g, k, M)["C"]
        upper = np.triu(np.ones((N, N), dtype=bool))
        ok = np.array_equal(out["C"][:, upper], ref[:, upper])
        with open(result_path, "w") as f:
            f.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


def test_shard_rule_partitions_masks():
    from paper_1704_07468_b200 import parallel
    from math import comb
    g, M = 10, 5
    allm = parallel.masks(g, M)
    assert len(allm) == sum(comb(g, m) for m in range(M + 1)) == 638
    for world in (1, 2, 3, 8):
        shards = [parallel.shard_masks(g, M, r, world) for r in range(world)]
        flat = [mk for s in shards for mk in s]
        assert sorted(flat) == sorted(allm)
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_reduce(tmp_path, oracle_lib):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    res = tmp_path / "res.txt"
    mp.start_processes(_worker, args=(2, port, str(res)), nprocs=2, join=True,
                       start_method="spawn")
    assert res.read_text() == "ok"


@pytest.mark.parametrize("world", [2, 3])
def test_launcher_sharded_step_gloo(tmp_path, oracle_lib, world):
    """The launcher (parallel.launch -> torch.distributed.run) and the ShardedStep
    that bench.py uses for --gpus N > 1, world 2 and 3 on CPU with gloo: per-level
    packed reduce-scatter, diagonal all-reduce and per-rank slice epilogue (through
    the CPU test double); the assembled slices equal the oracle's C, N_m, K, Knorm."""
    from paper_1704_07468_b200 import parallel
    res = tmp_path / "res.txt"
    rc = parallel.launch(world, os.path.join(ROOT, "tests", "dist_worker.py"), [str(res)],
                         env={"CUDA_VISIBLE_DEVICES": "", "OMP_NUM_THREADS": "1"})
    assert rc == 0
    assert res.read_text().startswith("ok"), res.read_text()


def test_tri_slices_cover_triangle():
    from paper_1704_07468_b200 import parallel
    for N in (1, 2, 7, 50, 20000):
        T = parallel.tri_size(N)
        for world in (1, 2, 3, 8):
            sl = [parallel.tri_slice(N, r, world) for r in range(world)]
            assert sl[0][1] == 0 and sl[-1][2] == T
            assert all(sl[i][2] == sl[i + 1][1] for i in range(world - 1))
            assert all(e - b <= c for c, b, e in sl)
    # packed index: row starts and the last entry
    N = 9
    assert parallel.tri_index(0, 0, N) == 0 and parallel.tri_index(N - 1, N - 1, N) == parallel.tri_size(N) - 1
    assert parallel.tri_index(1, 1, N) == N
