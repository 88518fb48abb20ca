"""Python face of the CPU oracle (oracle/gakco_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product path
(paper_1704_07468_b200/) never imports it and shares no code with it.

Each function names the paper passage (PAPER.md = P) its C routine follows;
see the header of gakco_oracle.c for the full statement.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gakco_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ERRORS = {1: "bad argument", 2: "int64 overflow", 3: "out of memory",
          4: "histogram total != n_X*n_Y"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        L.gko_binom.restype = i64
        L.gko_binom.argtypes = [ci, ci]
        L.gko_h.restype = i64
        L.gko_h.argtypes = [ci, ci, ci]
        for f in (L.gko_hist_pair, L.gko_hist_pair_direct):
            f.restype = ci
            f.argtypes = [P, i64, P, i64, ci, P]
        L.gko_profiles.restype = ci
        L.gko_profiles.argtypes = [P, P, i64, ci, ci, ci, P]
        L.gko_cumulative.restype = ci
        L.gko_cumulative.argtypes = [P, i64, ci, ci, P]
        L.gko_kernel.restype = ci
        L.gko_kernel.argtypes = [P, i64, ci, ci, ci, P]
        L.gko_normalize.restype = None
        L.gko_normalize.argtypes = [P, i64, P]
        L.gko_digest_u64.restype = ctypes.c_uint64
        L.gko_digest_u64.argtypes = [P, i64, i64, P]
        L.gko_pairs.restype = ci
        L.gko_pairs.argtypes = [P, P, i64, ci, ci, P, P, i64, ci, P]
        L.gko_digests.restype = ci
        L.gko_digests.argtypes = [P, P, i64, ci, ci, ci, ci, i64, i64, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc:
        raise RuntimeError(f"oracle {what}: {ERRORS.get(rc, rc)}")


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def binom(n: int, r: int) -> int:
    return int(lib().gko_binom(n, r))


def h(g: int, k: int, m: int) -> int:
    """Eq. 6."""
    return int(lib().gko_h(g, k, m))


def hist_pair(x, y, g: int, direct: bool = False) -> np.ndarray:
    """Hamming-distance histogram of all g-mer pairs of x and y (Def. 1, Eq. 5)."""
    x = np.ascontiguousarray(x, dtype=np.uint8)
    y = np.ascontiguousarray(y, dtype=np.uint8)
    out = np.zeros(g + 1, dtype=np.int64)
    f = lib().gko_hist_pair_direct if direct else lib().gko_hist_pair
    _check(f(_ptr(x), x.size, _ptr(y), y.size, g, _ptr(out)), "hist_pair")
    return out


def _corpus_arrays(corpus):
    codes = np.ascontiguousarray(corpus.codes, dtype=np.uint8)
    if codes.size == 0:
        codes = np.zeros(1, dtype=np.uint8)
    offsets = np.ascontiguousarray(corpus.offsets, dtype=np.int64)
    return codes, offsets


def profiles(corpus, g: int, M: int, threads: int | None = None) -> np.ndarray:
    """N_m(X,Y) for m = 0..M, shape (M+1, N, N) (Def. 1; Eq. 5)."""
    codes, offsets = _corpus_arrays(corpus)
    N = offsets.size - 1
    out = np.zeros((M + 1, N, N), dtype=np.int64)
    _check(lib().gko_profiles(_ptr(codes), _ptr(offsets), N, g, M,
                              threads or default_threads(), _ptr(out)), "profiles")
    return out


def cumulative(Nm: np.ndarray, g: int) -> np.ndarray:
    """C_m = sum_{j<=m} C(g-j, m-j) N_j (Eq. 8)."""
    Nm = np.ascontiguousarray(Nm, dtype=np.int64)
    M = Nm.shape[0] - 1
    out = np.zeros_like(Nm)
    _check(lib().gko_cumulative(_ptr(Nm), Nm.shape[1], g, M, _ptr(out)), "cumulative")
    return out


def kernel(Nm: np.ndarray, g: int, k: int) -> np.ndarray:
    """K = sum_{m<=min(M,g-k)} h_m N_m (Eq. 6-7)."""
    Nm = np.ascontiguousarray(Nm, dtype=np.int64)
    M = Nm.shape[0] - 1
    out = np.zeros(Nm.shape[1:], dtype=np.int64)
    _check(lib().gko_kernel(_ptr(Nm), Nm.shape[1], g, k, M, _ptr(out)), "kernel")
    return out


def normalize(K: np.ndarray) -> np.ndarray:
    """K(X,Y)/sqrt(K(X,X)K(Y,Y)); 0 if a diagonal is 0; diagonal 1 (reading A5)."""
    K = np.ascontiguousarray(K, dtype=np.int64)
    out = np.zeros(K.shape, dtype=np.float64)
    lib().gko_normalize(_ptr(K), K.shape[0], _ptr(out))
    return out


def compute(corpus, g: int, k: int, M: int, threads: int | None = None) -> dict:
    """All outputs of the path: C (M+1,N,N), Nm (M+1,N,N), K (N,N), Knorm (N,N)."""
    Nm = profiles(corpus, g, M, threads)
    C = cumulative(Nm, g)
    K = kernel(Nm, g, k)
    return {"C": C, "Nm": Nm, "K": K, "Knorm": normalize(K)}


def digest(a: np.ndarray, rows: bool = False):
    """Order-independent 64-bit digest of a 2-D (or stacked) matrix's bits."""
    a = np.ascontiguousarray(a)
    bits = a.view(np.uint64).reshape(-1, a.shape[-1])
    rd = np.zeros(bits.shape[0], dtype=np.uint64) if rows else None
    d = int(lib().gko_digest_u64(_ptr(bits), bits.shape[0], bits.shape[1],
                                 _ptr(rd) if rows else None))
    return (d, rd) if rows else d


def pairs(corpus, g: int, M: int, X, Y, threads: int | None = None) -> np.ndarray:
    """N_m(X_i, Y_i), m = 0..M, for a list of sequence pairs; shape (P, M+1)."""
    codes, offsets = _corpus_arrays(corpus)
    X = np.ascontiguousarray(X, dtype=np.int64)
    Y = np.ascontiguousarray(Y, dtype=np.int64)
    out = np.zeros((X.size, M + 1), dtype=np.int64)
    _check(lib().gko_pairs(_ptr(codes), _ptr(offsets), offsets.size - 1, g, M,
                           _ptr(X), _ptr(Y), X.size, threads or default_threads(),
                           _ptr(out)), "pairs")
    return out


def pair_outputs(nm_rows: np.ndarray, g: int, k: int) -> dict:
    """Eq. 8 and Eq. 7 applied to histogram rows (P, M+1) -> C (P,M+1), K (P,)."""
    M = nm_rows.shape[1] - 1
    C = np.zeros_like(nm_rows)
    for m in range(M + 1):
        for j in range(m + 1):
            C[:, m] += binom(g - j, m - j) * nm_rows[:, j]
    K = np.zeros(nm_rows.shape[0], dtype=np.int64)
    for m in range(min(M, g - k) + 1):
        K += h(g, k, m) * nm_rows[:, m]
    return {"C": C, "K": K}


def normalize_rect(K: np.ndarray, kd_rows: np.ndarray, kd_cols: np.ndarray) -> np.ndarray:
    """K(X,Y)/sqrt(K(X,X)K(Y,Y)) for a rectangular block (reading A5): 0 where a
    diagonal is <= 0; computed as (double)K / sqrt((double)Kxx * (double)Kyy)."""
    out = np.zeros(K.shape, dtype=np.float64)
    for i in range(K.shape[0]):
        for j in range(K.shape[1]):
            a, b = int(kd_rows[i]), int(kd_cols[j])
            if a > 0 and b > 0:
                out[i, j] = float(K[i, j]) / np.sqrt(float(a) * float(b))
    return out


def rect(corpus, NA: int, g: int, k: int, M: int, threads: int | None = None) -> dict:
    """Train x test block: rows X < NA, columns Y = NA..N-1 of
    the concatenated corpus's C_m, N_m, K, Knorm (the same definitions as compute():
    Def. 1 / Eq. 5 histograms per pair, Eq. 8, Eq. 6-7, reading A5), and
    Kdiag[X] = K(X,X) for all N (Eq. 1 needs K(x_i, x))."""
    N = int(np.asarray(corpus.offsets).size - 1)
    NB = N - NA
    X = np.repeat(np.arange(NA, dtype=np.int64), NB)
    Y = np.tile(np.arange(NA, N, dtype=np.int64), NA)
    nm = pairs(corpus, g, M, X, Y, threads)
    po = pair_outputs(nm, g, k)
    d = np.arange(N, dtype=np.int64)
    kd = pair_outputs(pairs(corpus, g, M, d, d, threads), g, k)["K"]
    K = po["K"].reshape(NA, NB)
    return {"C": po["C"].T.reshape(M + 1, NA, NB).copy(),
            "Nm": nm.T.reshape(M + 1, NA, NB).copy(),
            "K": K, "Knorm": normalize_rect(K, kd[:NA], kd[NA:]), "Kdiag": kd}


def digests(corpus, g: int, k: int, M: int, threads: int | None = None,
            row_begin: int = 0, row_end: int | None = None, rows: bool = True):
    """Digests of C_0..C_M, N_0..N_M, K, Knorm without materialising them."""
    codes, offsets = _corpus_arrays(corpus)
    N = offsets.size - 1
    row_end = N if row_end is None else row_end
    nmat = 2 * (M + 1) + 2
    md = np.zeros(nmat, dtype=np.uint64)
    rd = np.zeros((nmat, N), dtype=np.uint64) if rows else None
    _check(lib().gko_digests(_ptr(codes), _ptr(offsets), N, g, k, M,
                             threads or default_threads(), row_begin, row_end,
                             _ptr(md), _ptr(rd) if rows else None), "digests")
    return md, rd


def matrix_names(M: int):
    return ([f"C{m}" for m in range(M + 1)] + [f"N{m}" for m in range(M + 1)]
            + ["K", "Knorm"])
