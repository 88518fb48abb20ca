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

    r = parallel.sharded_kernel_matrix(C, N, acc, fin)
    if r == 0:
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
