"""Seeded synthetic corpora shaped like the paper's workloads.

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (tests, bench, smoke). It holds NONE of the method's arithmetic:
it only draws symbol codes. Each recipe below is the BASELINE.json `configs`
entry it stands in for; SURVEY.md §8(d) fixes the details BASELINE.json leaves
open (DESIGN.md "Input recipe" restates them):

* the paper's real datasets (ENCODE DNA, SCOP protein, WebKB / Sentiment text;
  PAPER.md:254-277, Table 3, Supp. §S:3.2) are not in the
  container; these generators stand in for them;
* a "substitution" always draws a *different* symbol;
* codes are 0..Σ−1; unknown-character handling is the caller's
  job, so no UNK code is produced.

A corpus is CSR: ``codes`` uint8[offsets[-1]] and ``offsets`` int64[N+1].
Random numbers come from ``numpy.random.default_rng(seed)`` (PCG64); the
default seed of config i is i (1..5).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Corpus:
    sigma: int
    codes: np.ndarray    # uint8, concatenated sequences
    offsets: np.ndarray  # int64, N+1, offsets[0] == 0

    @property
    def n_seq(self) -> int:
        return int(self.offsets.shape[0] - 1)

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def seq(self, i: int) -> np.ndarray:
        return self.codes[self.offsets[i]:self.offsets[i + 1]]

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64(self.sigma).tobytes())
        h.update(np.ascontiguousarray(self.offsets, dtype="<i8").tobytes())
        h.update(np.ascontiguousarray(self.codes, dtype=np.uint8).tobytes())
        return h.hexdigest()


@dataclass(frozen=True)
class Config:
    name: str
    index: int          # 1-based position in BASELINE.json `configs`
    sigma: int
    g: int
    k: int
    M: int
    description: str


# BASELINE.json `configs`, in order.
CONFIGS = {
    "tiny": Config("tiny", 1, 4, 7, 5, 2,
                   "Σ=4, N=50, l=100 iid uniform; g=7, k=5 (M=2)"),
    "dna": Config("dna", 2, 4, 10, 6, 4,
                  "Σ=4, N=4000, l=101 iid uniform + planted 10-mer motif "
                  "(≤2 substitutions) in half the sequences; g=10, k=6 (M=4)"),
    "protein": Config("protein", 3, 20, 8, 4, 4,
                      "Σ=20, N=3312, l~U[50,400], 30 families "
                      "(ancestor + p=0.2 substitution); g=8, k=4 (M=4)"),
    "text": Config("text", 4, 36, 10, 5, 5,
                   "Σ=36, N=2000, l~U[1000,5000], iid Zipf(s=1) over 36 ranks; "
                   "g=10, k=5 (M=5)"),
    "scale": Config("scale", 5, 20, 10, 5, 5,
                    "Σ=20, N=20000, l=300, 200 families "
                    "(ancestor + p=0.2 substitution); g=10, k=5 (M=5)"),
}


def _from_list(sigma: int, seqs) -> Corpus:
    lens = np.array([len(s) for s in seqs], dtype=np.int64)
    offsets = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    codes = (np.concatenate([np.asarray(s, dtype=np.uint8) for s in seqs])
             if len(seqs) and offsets[-1] > 0 else np.zeros(0, dtype=np.uint8))
    return Corpus(sigma, codes, offsets)


def from_sequences(sigma: int, seqs) -> Corpus:
    """Build a corpus from a list of code sequences (lists/arrays of ints)."""
    for s in seqs:
        a = np.asarray(s)
        if a.size and (a.min() < 0 or a.max() >= sigma):
            raise ValueError("code outside 0..sigma-1")
    return _from_list(sigma, seqs)


def from_strings(alphabet: str, strings) -> Corpus:
    """Map characters through `alphabet` (index = code). Fig. 2 uses 'ACGT'."""
    table = {c: i for i, c in enumerate(alphabet)}
    return _from_list(len(alphabet), [[table[c] for c in s] for s in strings])


def _substitute(rng, seq: np.ndarray, p: float, sigma: int) -> np.ndarray:
    """Each residue independently, w.p. p, becomes a *different* symbol."""
    hit = rng.random(seq.shape[0]) < p
    shift = rng.integers(1, sigma, size=seq.shape[0])
    out = seq.astype(np.int64)
    out[hit] = (out[hit] + shift[hit]) % sigma
    return out.astype(np.uint8)


def uniform(n_seq: int, length: int, sigma: int, seed: int) -> Corpus:
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, sigma, size=n_seq * length, dtype=np.int64).astype(np.uint8)
    offsets = np.arange(n_seq + 1, dtype=np.int64) * length
    return Corpus(sigma, codes, offsets)


def gen_tiny(seed: int = 1) -> Corpus:
    return uniform(50, 100, 4, seed)


def gen_dna(seed: int = 2, n_seq: int = 4000, length: int = 101) -> Corpus:
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 4, size=(n_seq, length), dtype=np.int64)
    motif = rng.integers(0, 4, size=10, dtype=np.int64)
    for i in range(0, n_seq, 2):          # the even-index half
        copy = motif.copy()
        s = int(rng.integers(0, 3))        # 0, 1 or 2 substitutions
        pos = rng.choice(10, size=s, replace=False)
        for p in pos:
            copy[p] = (copy[p] + int(rng.integers(1, 4))) % 4
        q = int(rng.integers(0, length - 10 + 1))
        codes[i, q:q + 10] = copy
    offsets = np.arange(n_seq + 1, dtype=np.int64) * length
    return Corpus(4, codes.reshape(-1).astype(np.uint8), offsets)


def gen_families(seed: int, n_seq: int, n_fam: int, anc_len: int,
                 min_len: int, max_len: int, sigma: int = 20,
                 p_sub: float = 0.2) -> Corpus:
    rng = np.random.default_rng(seed)
    anc = rng.integers(0, sigma, size=(n_fam, anc_len), dtype=np.int64).astype(np.uint8)
    seqs = []
    for i in range(n_seq):
        fam = anc[i % n_fam]
        L = int(rng.integers(min_len, max_len + 1))
        start = int(rng.integers(0, anc_len - L + 1))
        seqs.append(_substitute(rng, fam[start:start + L], p_sub, sigma))
    return _from_list(sigma, seqs)


def gen_protein(seed: int = 3) -> Corpus:
    return gen_families(seed, 3312, 30, 400, 50, 400)


def gen_scale(seed: int = 5, n_seq: int = 20000) -> Corpus:
    return gen_families(seed, n_seq, 200, 300, 300, 300)


def gen_text(seed: int = 4, n_seq: int = 2000, min_len: int = 1000,
             max_len: int = 5000) -> Corpus:
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, 37, dtype=np.float64)
    p = (1.0 / ranks) / np.sum(1.0 / ranks)   # Zipf(s=1): code r-1 ∝ 1/r
    lens = rng.integers(min_len, max_len + 1, size=n_seq)
    offsets = np.zeros(n_seq + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    codes = rng.choice(36, size=int(offsets[-1]), p=p).astype(np.uint8)
    return Corpus(36, codes, offsets)


GENERATORS = {
    "tiny": gen_tiny,
    "dna": gen_dna,
    "protein": gen_protein,
    "text": gen_text,
    "scale": gen_scale,
}


def make(name: str, seed: int | None = None) -> Corpus:
    """Corpus of BASELINE.json config `name` (seed defaults to its index)."""
    cfg = CONFIGS[name]
    return GENERATORS[name](cfg.index if seed is None else seed)


def random_small(rng: np.random.Generator, sigma: int, n_max: int = 12,
                 l_max: int = 40) -> Corpus:
    """Tiny random corpus for sweeps: N in [1,n_max], lengths in [0,l_max]."""
    n = int(rng.integers(1, n_max + 1))
    seqs = [rng.integers(0, sigma, size=int(rng.integers(0, l_max + 1)))
            for _ in range(n)]
    return from_sequences(sigma, seqs)
