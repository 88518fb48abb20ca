"""CPU test double of gakco.Plan for the sharded-step wiring tests (-m "not gpu").

It stands in for libgakco.so on a machine without a GPU so that
paper_1704_07468_b200.parallel.ShardedStep and its launcher can be exercised
across real processes with the gloo backend. Its accumulate is the literal
Algorithm 1 restatement of tests/refs.py restricted to the rank's masks (the
shard rule of gakco_set_shard); pack / diag / finalize restate the C-ABI
contracts of include/gakco.h in numpy. It is never used by the product.
"""
from __future__ import annotations

from collections import Counter
from math import comb

import numpy as np

from tests.refs import gmers


class MockPlan:
    def __init__(self, corpus, g, k, M, rank, world):
        from paper_1704_07468_b200 import parallel
        self.cp, self.g, self.k, self.M = corpus, g, k, M
        self.mine = parallel.shard_masks(g, M, rank, world)

    def zero_upper(self, C, N, levels, stream=None):
        """gakco_zero_upper: the upper triangles (Y >= X) of `levels` N x N matrices."""
        iu = np.triu_indices(N)
        for lv in range(levels):
            C[lv][iu] = 0

    def accumulate(self, codes, offsets, N, C, stream=None):
        """Upper triangle (Y >= X) of this shard's C_m, Algorithm 1."""
        per_seq = [gmers(self.cp.seq(i), self.g) for i in range(N)]
        acc = np.zeros((self.M + 1, N, N), dtype=np.int64)
        for m, removed in self.mine:
            kept = [p for p in range(self.g) if p not in removed]
            groups = {}
            for s in range(N):
                for gm in per_seq[s]:
                    groups.setdefault(tuple(gm[p] for p in kept), Counter())[s] += 1
            for cnt in groups.values():
                for a, ca in cnt.items():
                    for b, cb in cnt.items():
                        if b >= a:
                            acc[m, a, b] += ca * cb
        C += __import__("torch").from_numpy(acc)

    def level_order(self):
        return list(range(self.M + 1))

    def stream_wait_level(self, m, stream=None):
        pass

    def pack_upper(self, C, N, levels, begin, end, out, out_bytes, stream=None):
        iu = np.triu_indices(N)  # row-major: the packed order of include/gakco.h
        src = C.numpy().reshape(levels, N, N) if levels > 1 else C.numpy()[None]
        o = out.numpy().reshape(levels, -1)
        for lv in range(levels):
            o[lv, : end - begin] = src[lv][iu][begin:end]

    def diag(self, C, N, levels, out, stream=None):
        c = C.numpy()
        for lv in range(levels):
            out[lv] = __import__("torch").from_numpy(np.diagonal(c[lv]).copy())

    def finalize_packed(self, Cp, in_bytes, ld, N, begin, end, Cdiag, Nm=None, K=None, Knorm=None,
                        stream=None):
        g, k, M = self.g, self.k, self.M
        h = [comb(g - m, k) if m <= g - k else 0 for m in range(M + 1)]

        def eq9(c):  # Eq. 9 on stacked columns
            n = np.zeros_like(c)
            for m in range(M + 1):
                n[m] = c[m] - sum(comb(g - j, m - j) * n[j] for j in range(m))
            return n
        kd_n = eq9(Cdiag.numpy().astype(np.int64))
        kdiag = sum(h[m] * kd_n[m] for m in range(M + 1))
        cnt = end - begin
        c = Cp.numpy()[:, :cnt].astype(np.int64)
        nm = eq9(c)
        kv = sum(h[m] * nm[m] for m in range(M + 1))
        iu = np.triu_indices(N)
        X, Y = iu[0][begin:end], iu[1][begin:end]
        a, b = kdiag[X].astype(np.float64), kdiag[Y].astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            kn = np.where((a > 0) & (b > 0), kv / np.sqrt(a * b), 0.0)
        kn = np.where((X == Y) & (a > 0), 1.0, kn)
        if Nm is not None:
            Nm.numpy()[:, :cnt] = nm
        if K is not None:
            K.numpy()[:cnt] = kv
        if Knorm is not None:
            Knorm.numpy()[:cnt] = kn
