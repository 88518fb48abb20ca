"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: the paper's printed Fig. 2
numbers, brute force on tiny inputs, the explicit feature map of Eq. 4, the
literal Algorithm 1 with a Counter, closed forms, invariants and invariances.
"""
import json
import os
from math import comb

import numpy as np
import pytest

from synth import corpus as sc
from tests import refs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fig2():
    with open(os.path.join(GOLDEN, "fig2.json")) as f:
        return json.load(f)


def test_fig2_printed_values(oracle_lib):
    """PAPER.md:106 (Fig. 2): N_0(S,T)=2, C_1(S,T)=9, N_1(S,T)=3."""
    fx = _fig2()
    cp = sc.from_strings(fx["alphabet"], fx["sequences"])
    r = oracle_lib.compute(cp, fx["g"], 2, 1)
    p = fx["printed"]
    assert r["Nm"][0, 0, 1] == p["N0_ST"]
    assert r["C"][1, 0, 1] == p["C1_ST"]
    assert r["Nm"][1, 0, 1] == p["N1_ST"]
    # printed g-mer lists of the caption
    S, T = fx["sequences"]
    assert ["".join("ACGT"[c] for c in gm) for gm in refs.gmers(cp.seq(0), 3)] == p["gmers_S"]
    assert ["".join("ACGT"[c] for c in gm) for gm in refs.gmers(cp.seq(1), 3)] == p["gmers_T"]


def test_fig2_hand_enumeration(oracle_lib):
    fx = _fig2()
    d = fx["derived_by_hand"]
    cp = sc.from_strings(fx["alphabet"], fx["sequences"])
    assert list(oracle_lib.hist_pair(cp.seq(0), cp.seq(1), 3)) == d["hist_ST"]
    assert list(oracle_lib.hist_pair(cp.seq(0), cp.seq(0), 3)) == d["hist_SS"]
    assert list(oracle_lib.hist_pair(cp.seq(1), cp.seq(1), 3)) == d["hist_TT"]
    r = oracle_lib.compute(cp, 3, 2, 1)
    assert r["C"][1].tolist() == d["C1"]
    assert r["K"].tolist() == d["K_k2"]
    assert r["Knorm"][0, 1] == pytest.approx(d["Knorm_ST_k2"], rel=1e-15)
    assert r["Knorm"][0, 0] == 1.0 and r["Knorm"][1, 1] == 1.0
    r3 = oracle_lib.compute(cp, 3, 3, 0)
    assert r3["K"][0, 1] == d["K_k3_ST"]


def test_diagonal_walk_equals_double_loop(oracle_lib):
    """Brute force: the diagonal walk equals the literal Eq. 5 double loop."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(1, 9))
        x = rng.integers(0, sigma, size=int(rng.integers(0, 40)))
        y = rng.integers(0, sigma, size=int(rng.integers(0, 40)))
        a = oracle_lib.hist_pair(x, y, g)
        b = oracle_lib.hist_pair(x, y, g, direct=True)
        assert a.tolist() == b.tolist()
        nx, ny = max(0, len(x) - g + 1), max(0, len(y) - g + 1)
        assert a.sum() == nx * ny


def test_against_python_hamming(oracle_lib):
    """Brute force in pure Python (Def. 1): Hamming distance of every pair."""
    rng = np.random.default_rng(12)
    for _ in range(60):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(1, 7))
        cp = sc.random_small(rng, sigma, n_max=5, l_max=15)
        Nm = oracle_lib.profiles(cp, g, g)
        for a in range(cp.n_seq):
            for b in range(cp.n_seq):
                h = [0] * (g + 1)
                for u in refs.gmers(cp.seq(a), g):
                    for v in refs.gmers(cp.seq(b), g):
                        h[sum(p != q for p, q in zip(u, v))] += 1
                assert Nm[:, a, b].tolist() == h


def test_feature_map_equivalence(oracle_lib):
    """Eq. 4: explicit gapped k-mer feature vectors give the same K."""
    rng = np.random.default_rng(13)
    n = 0
    while n < 60:
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(1, 7))
        cp = sc.random_small(rng, sigma, n_max=6, l_max=18)
        for k in range(1, g + 1):
            r = oracle_lib.compute(cp, g, k, g - k)
            assert np.array_equal(r["K"], refs.feature_map_kernel(cp, g, k)), (g, k)
            n += 1


def test_algorithm1_counter_equivalence(oracle_lib):
    """Algorithm 1 literally, with a Counter as sort-and-count,
    gives the oracle's C_m (so Eq. 8's coefficients are pinned), and Eq. 9's
    recursion applied to it gives the oracle's N_m."""
    rng = np.random.default_rng(14)
    for _ in range(120):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(1, 8))
        M = int(rng.integers(0, g + 1))
        cp = sc.random_small(rng, sigma, n_max=7, l_max=25)
        r_nm = oracle_lib.profiles(cp, g, M)
        C_ref = refs.mask_sort_count(cp, g, M)
        assert np.array_equal(oracle_lib.cumulative(r_nm, g), C_ref)
        assert np.array_equal(refs.eq9_recursion(C_ref, g), r_nm)


def test_invariants_random(oracle_lib):
    """Closed-form identities: sum_m N_m = n_X n_Y (M=g);
    C_g = n_X n_Y; K = C_{g-k}; symmetry; PSD; |Knorm| <= 1."""
    rng = np.random.default_rng(15)
    for _ in range(200):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(1, 9))
        k = int(rng.integers(1, g + 1))
        cp = sc.random_small(rng, sigma)
        n = np.maximum(cp.lengths() - g + 1, 0)
        r = oracle_lib.compute(cp, g, k, g)
        nn = np.outer(n, n)
        assert np.array_equal(r["Nm"].sum(axis=0), nn)
        assert np.array_equal(r["C"][g], nn)
        assert np.array_equal(r["K"], r["C"][g - k])
        for mat in (r["C"], r["Nm"]):
            assert np.array_equal(mat, mat.transpose(0, 2, 1))
        assert np.array_equal(r["K"], r["K"].T)
        if cp.n_seq <= 20 and r["K"].any():
            ev = np.linalg.eigvalsh(r["K"].astype(np.float64))
            assert ev.min() >= -1e-9 * np.trace(r["K"])
        assert np.all(np.abs(r["Knorm"]) <= 1.0 + 1e-15)
        diag = np.diag(r["K"])
        assert np.array_equal(np.diag(r["Knorm"]), (diag > 0).astype(np.float64))


def test_cap_truncates_kernel(oracle_lib):
    """M < g-k truncates Eq. 7; M > g-k adds nothing (h_m = 0, Eq. 6)."""
    rng = np.random.default_rng(16)
    cp = sc.random_small(rng, 4, n_max=6, l_max=30)
    g, k = 6, 2
    full = oracle_lib.compute(cp, g, k, g - k)["K"]
    over = oracle_lib.compute(cp, g, k, g)["K"]
    assert np.array_equal(full, over)
    Nm = oracle_lib.profiles(cp, g, g)
    for M in range(g - k + 1):
        Kc = oracle_lib.compute(cp, g, k, M)["K"]
        assert np.array_equal(Kc, sum(comb(g - m, k) * Nm[m] for m in range(M + 1)))


@pytest.mark.parametrize("g", range(2, 8))
def test_closed_forms(oracle_lib, g):
    """Homopolymers, disjoint homopolymers, alternating strings, short rows."""
    lx, ly = 3 * g + 1, 2 * g + 5
    nx, ny = lx - g + 1, ly - g + 1
    cp = sc.from_sequences(3, [[0] * lx, [0] * ly, [1] * ly, [0, 1] * g + [0],
                               [0, 1] * (g + 2), [0] * (g - 1)])
    Nm = oracle_lib.profiles(cp, g, g)
    # a^lx vs a^ly: every pair at distance 0
    assert Nm[0, 0, 1] == nx * ny and Nm[1:, 0, 1].sum() == 0
    # a vs b: every pair at distance g
    assert Nm[g, 0, 2] == nx * ny and Nm[:g, 0, 2].sum() == 0
    # (ab)^*: distance 0 when start parities agree, g otherwise
    a = np.array(cp.seq(3)); b = np.array(cp.seq(4))
    na, nb = len(a) - g + 1, len(b) - g + 1
    same = sum(1 for i in range(na) for j in range(nb) if (i - j) % 2 == 0)
    assert Nm[0, 3, 4] == same and Nm[g, 3, 4] == na * nb - same
    assert Nm[1:g, 3, 4].sum() == 0
    # shorter than g: zero row
    assert Nm[:, 5, :].sum() == 0 and Nm[:, :, 5].sum() == 0
    for k in range(1, g + 1):
        K = oracle_lib.compute(cp, g, k, g - k)["K"]
        assert K[0, 1] == comb(g, k) * nx * ny
        assert K[0, 2] == 0


def test_spectrum_special_case(oracle_lib):
    """k = g (M = 0): K is the g-spectrum kernel (Eq. 3)."""
    rng = np.random.default_rng(17)
    for _ in range(40):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(1, 7))
        cp = sc.random_small(rng, sigma)
        assert np.array_equal(oracle_lib.compute(cp, g, g, 0)["K"], refs.spectrum_kernel(cp, g))


def test_invariances(oracle_lib):
    """Relabelling symbols keeps K; reversing every sequence keeps N_m;
    permuting sequences permutes rows and columns; a duplicate row has Knorm 1."""
    rng = np.random.default_rng(18)
    for _ in range(40):
        sigma = int(rng.choice([4, 20]))
        g = int(rng.integers(2, 7))
        k = int(rng.integers(1, g + 1))
        cp = sc.random_small(rng, sigma)
        base = oracle_lib.compute(cp, g, k, g - k)
        perm_sym = rng.permutation(sigma)
        relab = sc.Corpus(sigma, perm_sym[cp.codes].astype(np.uint8), cp.offsets)
        assert np.array_equal(oracle_lib.compute(relab, g, k, g - k)["K"], base["K"])
        rev = sc.from_sequences(sigma, [cp.seq(i)[::-1] for i in range(cp.n_seq)])
        assert np.array_equal(oracle_lib.profiles(rev, g, g - k), base["Nm"])
        p = rng.permutation(cp.n_seq)
        perm = sc.from_sequences(sigma, [cp.seq(i) for i in p])
        assert np.array_equal(oracle_lib.compute(perm, g, k, g - k)["K"], base["K"][np.ix_(p, p)])
        dup = sc.from_sequences(sigma, [cp.seq(0), cp.seq(0)])
        Kn = oracle_lib.compute(dup, g, k, g - k)["Knorm"]
        if base["K"][0, 0] > 0:
            assert Kn[0, 1] == 1.0


def test_eq9_closed_form_inverse():
    """The epilogue's closed form N_m = sum_j (-1)^(m-j) C(g-j,m-j) C_j inverts
    Eq. 8 (pure integer algebra; pins the reading used by the CUDA epilogue)."""
    for g in range(1, 16):
        for m in range(g + 1):
            for j in range(m + 1):
                # coefficient of N_j in sum_i (-1)^(m-i) C(g-i,m-i) C_i with C_i = sum_j C(g-j,i-j) N_j
                coef = sum((-1) ** (m - i) * comb(g - i, m - i) * comb(g - j, i - j)
                           for i in range(j, m + 1))
                assert coef == (1 if j == m else 0)


def test_pairs_and_streaming_digests(oracle_lib):
    """The sampled-pair and streaming-digest entry points agree with the dense ones."""
    cp = sc.make("tiny")
    g, k, M = 7, 5, 2
    r = oracle_lib.compute(cp, g, k, M)
    md, rd = oracle_lib.digests(cp, g, k, M)
    mats = [r["C"][m] for m in range(M + 1)] + [r["Nm"][m] for m in range(M + 1)] + [r["K"], r["Knorm"]]
    for i, mat in enumerate(mats):
        d, rows = refs.digest_np(mat, rows=True)
        assert d == int(md[i]) == oracle_lib.digest(mat)
        assert np.array_equal(rows, rd[i])
    rng = np.random.default_rng(19)
    X = rng.integers(0, cp.n_seq, 50)
    Y = rng.integers(0, cp.n_seq, 50)
    out = oracle_lib.pairs(cp, g, M, X, Y)
    assert np.array_equal(out, r["Nm"][:, X, Y].T)
    po = oracle_lib.pair_outputs(out, g, k)
    assert np.array_equal(po["C"], r["C"][:, X, Y].T)
    assert np.array_equal(po["K"], r["K"][X, Y])


def test_overflow_is_an_error(oracle_lib):
    """Eq. 7/8 overflow raises (SPEC S:149 'error, not silent wraparound')."""
    Nm = np.full((2, 1, 1), 2 ** 62, dtype=np.int64)
    with pytest.raises(RuntimeError):
        oracle_lib.cumulative(Nm, 3)


def test_rect_is_block_of_full(oracle_lib):
    """NEXT-2 oracle: the train x test block assembled pair by pair equals the
    corresponding block of the full oracle on the concatenated corpus (every
    output, incl. Knorm from the full diagonal), for several splits."""
    rng = np.random.default_rng(31)
    for _ in range(6):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(2, 8))
        k = int(rng.integers(1, g + 1))
        M = int(rng.integers(0, g + 1))
        cp = sc.random_small(rng, sigma, n_max=14, l_max=30)
        N = cp.n_seq
        if N < 2:
            continue
        full = oracle_lib.compute(cp, g, k, M)
        for NA in sorted({1, N // 2, N - 1}):
            r = oracle_lib.rect(cp, NA, g, k, M)
            assert np.array_equal(r["C"], full["C"][:, :NA, NA:])
            assert np.array_equal(r["Nm"], full["Nm"][:, :NA, NA:])
            assert np.array_equal(r["K"], full["K"][:NA, NA:])
            assert np.array_equal(r["Kdiag"], np.diag(full["K"]))
            np.testing.assert_allclose(r["Knorm"], full["Knorm"][:NA, NA:], rtol=1e-15, atol=0)
