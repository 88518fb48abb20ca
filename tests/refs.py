"""Small, independent pure-Python references used only to PIN the oracle.

None of these is the oracle and none is the CUDA path; each restates one
passage of the paper (PAPER.md = P) in the most literal way, for tiny inputs.
"""
from __future__ import annotations

from collections import Counter
from itertools import combinations
from math import comb

import numpy as np


def gmers(seq, g):
    """g-mers with start positions 0..l-g (reading A7)."""
    s = [int(c) for c in seq]
    return [tuple(s[i:i + g]) for i in range(len(s) - g + 1)]


def feature_map_kernel(corpus, g, k):
    """Eq. 4: K = sum over gapped k-mers gamma of c_x(gamma) c_x'(gamma).
    A gapped k-mer is (k kept positions of the g-window, symbols there); every
    g-mer of x contributes one count to each of its C(g,k) gapped k-mers."""
    feats = []
    for i in range(corpus.n_seq):
        c = Counter()
        for gm in gmers(corpus.seq(i), g):
            for pos in combinations(range(g), k):
                c[(pos, tuple(gm[p] for p in pos))] += 1
        feats.append(c)
    N = corpus.n_seq
    K = np.zeros((N, N), dtype=np.int64)
    for a in range(N):
        for b in range(N):
            fa, fb = feats[a], feats[b]
            if len(fb) < len(fa):
                fa, fb = fb, fa
            K[a, b] = sum(v * fb.get(key, 0) for key, v in fa.items())
    return K


def spectrum_kernel(corpus, g):
    """Eq. 3 with k-mers of length g: sum_gamma c_x(gamma) c_x'(gamma)."""
    cs = [Counter(gmers(corpus.seq(i), g)) for i in range(corpus.n_seq)]
    N = corpus.n_seq
    K = np.zeros((N, N), dtype=np.int64)
    for a in range(N):
        for b in range(N):
            K[a, b] = sum(v * cs[b].get(key, 0) for key, v in cs[a].items())
    return K


def mask_sort_count(corpus, g, M):
    """Algorithm 1 MISMATCHPROFILE with a Counter for sort-and-count:
    for every m and every one of the C(g,m) removed-position sets, drop those
    positions from every g-mer, group equal (g-m)-mers and add c_X*c_Y to C_m."""
    N = corpus.n_seq
    C = np.zeros((M + 1, N, N), dtype=np.int64)
    per_seq = [gmers(corpus.seq(i), g) for i in range(N)]
    for m in range(M + 1):
        for removed in combinations(range(g), m):
            kept = [p for p in range(g) if p not in removed]
            groups = {}
            for s in range(N):
                for gm in per_seq[s]:
                    key = tuple(gm[p] for p in kept)
                    groups.setdefault(key, Counter())[s] += 1
            for cnt in groups.values():
                for a, ca in cnt.items():
                    for b, cb in cnt.items():
                        C[m, a, b] += ca * cb
    return C


def eq9_recursion(C, g):
    """Eq. 9 exactly as Algorithm 1 lines 18-21."""
    Nm = np.zeros_like(C)
    for m in range(C.shape[0]):
        Nm[m] = C[m]
        for j in range(m):
            Nm[m] -= comb(g - j, m - j) * Nm[j]
    return Nm


# ----------------------------------------------------------------- digest
_M1 = np.uint64(0xbf58476d1ce4e5b9)
_M2 = np.uint64(0x94d049bb133111eb)


def _mix(z):
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def digest_np(a, rows=False, chunk_rows=512):
    """Numpy restatement of the oracle's order-independent digest:
    sum over entries of mix(idx ^ mix(bits)) mod 2^64, idx = r*ncols + c."""
    a = np.ascontiguousarray(a)
    ncols = a.shape[-1]
    bits = a.reshape(-1, ncols).view(np.uint64)
    total = np.uint64(0)
    rd = np.zeros(bits.shape[0], dtype=np.uint64)
    for r0 in range(0, bits.shape[0], chunk_rows):
        blk = bits[r0:r0 + chunk_rows]
        idx = (np.arange(r0, r0 + blk.shape[0], dtype=np.uint64)[:, None] * np.uint64(ncols)
               + np.arange(ncols, dtype=np.uint64)[None, :])
        t = _mix(idx ^ _mix(blk))
        with np.errstate(over="ignore"):
            rs = t.sum(axis=1, dtype=np.uint64)
        rd[r0:r0 + blk.shape[0]] = rs
        with np.errstate(over="ignore"):
            total = total + rs.sum(dtype=np.uint64)
    return (int(total), rd) if rows else int(total)
