"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar: C_m, N_m, K bit-exact (int64); Knorm within 1e-12
relative (BASELINE.json north_star), with the diagonal exactly 1.0.
"""
import json
import os

import numpy as np
import pytest

from synth import corpus as sc
from tests import refs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KNORM_RTOL = 1e-12


@pytest.fixture(scope="module")
def gk():
    from paper_1704_07468_b200 import build, gakco
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return gakco


def run(gk, cp, g, k, M, **opts):
    plan = gk.Plan(cp.sigma, g, k, M)
    for opt, val in opts.items():
        plan.set_option(getattr(gk, "GAKCO_OPT_" + opt.upper()), val)
    r = gk.kernel_matrix(cp.codes, cp.offsets, cp.sigma, g, k, M, plan=plan)
    out = {key: v.cpu().numpy() for key, v in r.items()}
    out["stats"] = plan.stats()
    plan.close()
    return out


def assert_parity(gpu, ref):
    assert np.array_equal(gpu["C"], ref["C"])
    assert np.array_equal(gpu["Nm"], ref["Nm"])
    assert np.array_equal(gpu["K"], ref["K"])
    assert_knorm(gpu["Knorm"], ref["Knorm"])


def assert_knorm(a, b):
    assert a.shape == b.shape
    np.testing.assert_allclose(a, b, rtol=KNORM_RTOL, atol=0)
    d = np.diag(b)
    assert np.array_equal(np.diag(a), d)


def test_fig2_through_abi(gk, oracle_lib):
    """N_0(S,T)=2, C_1(S,T)=9, N_1(S,T)=3; K=[[15,9],[9,13]]."""
    cp = sc.from_strings("ACGT", ["ACACA", "AAACA"])
    r = run(gk, cp, 3, 2, 1)
    assert r["Nm"][0, 0, 1] == 2 and r["C"][1, 0, 1] == 9 and r["Nm"][1, 0, 1] == 3
    assert r["K"].tolist() == [[15, 9], [9, 13]]
    assert r["Knorm"][0, 1] == pytest.approx(9 / np.sqrt(195), rel=1e-15)
    assert_parity(r, oracle_lib.compute(cp, 3, 2, 1))


def test_tiny_config(gk, oracle_lib):
    cfg = sc.CONFIGS["tiny"]
    cp = sc.make("tiny")
    assert_parity(run(gk, cp, cfg.g, cfg.k, cfg.M), oracle_lib.compute(cp, cfg.g, cfg.k, cfg.M))


def test_random_sweep(gk, oracle_lib):
    """Seeded random corpora: Σ in {2,4,20,36}, ragged lengths (incl. < g and 0)."""
    rng = np.random.default_rng(101)
    for it in range(40):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(1, 11))
        k = int(rng.integers(1, g + 1))
        M = int(rng.integers(0, g + 1))
        cp = sc.random_small(rng, sigma, n_max=40, l_max=120)
        assert_parity(run(gk, cp, g, k, M), oracle_lib.compute(cp, g, k, M))


def test_several_tiles_ragged(gk, oracle_lib):
    """Enough g-mers to span many sort tiles (4096 keys) with a ragged tail."""
    rng = np.random.default_rng(102)
    seqs = [rng.integers(0, 4, size=int(rng.integers(0, 700))) for _ in range(60)]
    cp = sc.from_sequences(4, seqs)
    for (g, k, M) in [(6, 3, 3), (9, 5, 4), (12, 8, 4)]:
        assert_parity(run(gk, cp, g, k, M), oracle_lib.compute(cp, g, k, M))


def test_heavy_light_equivalence(gk, oracle_lib):
    """Forced all-heavy (tensor-core Gram for every multi-sequence group) ==
    forced all-light == default == oracle (SURVEY §8c GPU-internal pins)."""
    rng = np.random.default_rng(103)
    cases = [(sc.make("tiny"), 7, 5, 2)]
    for _ in range(12):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(2, 10))
        k = int(rng.integers(1, g + 1))
        cases.append((sc.random_small(rng, sigma, n_max=300, l_max=90), g, k, g - k))
    # more than 256 rows and columns of tiles, counts up to 255+ (light fallback)
    cases.append((sc.from_sequences(2, [[0] * 300] + [list(rng.integers(0, 2, 60))
                                                     for _ in range(520)]), 6, 3, 3))
    for cp, g, k, M in cases:
        ref = oracle_lib.compute(cp, g, k, M)
        heavy = run(gk, cp, g, k, M, heavy_min_seqs=2)
        assert_parity(heavy, ref)
        assert_parity(run(gk, cp, g, k, M, heavy_min_seqs=2, gram_pair=0), ref)
        assert_parity(run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=0), ref)
        assert_parity(run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=1), ref)
        assert_parity(run(gk, cp, g, k, M, heavy_min_seqs=1 << 50), ref)
        assert_parity(run(gk, cp, g, k, M), ref)


def test_e2m1_gram_large_sums(gk, oracle_lib):
    """the e2m1 Gram (tcgen05 kind::mxf4, f32 accumulators) is exact only
    if the tensor core keeps every bit of sums up to 2^24 within one flush. Here the
    per-cell sums of one flush reach ~2^20 with every count <= 4: four copies of a
    period-16 sequence (n = 64 g-mers, each masked key 4 times per sequence),
    g = 16, M = 6 (level 6: 8008 masks, flushes of (2^24 - 1) / 64^2 = 4095 masks,
    each adding up to 16 keys * 4 * 4 = 256 per mask and cell). e2m1 forced ==
    u8 / s32 == oracle."""
    rng = np.random.default_rng(141)
    period = list(rng.integers(0, 4, 16))
    rep = (period * 6)[:79]
    seqs = [rep] * 4 + [list(rng.integers(0, 4, 79)) for _ in range(4)]
    cp = sc.from_sequences(4, seqs)
    g, k, M = 16, 10, 6
    ref = oracle_lib.compute(cp, g, k, M)
    # the premise: one flush of level 6 carries a cell sum near 2^20
    assert ref["C"][6, 0, 1] - ref["C"][5, 0, 1] > 0
    r4 = run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=1)
    assert r4["stats"]["gram_fp4"] == (1 << (M + 1)) - 1
    assert r4["stats"]["heavy_macs_fp4"] > 0
    assert_parity(r4, ref)
    assert_parity(run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=0), ref)
    # the largest single-level cell value (a bound on any flush's partial sum there)
    assert ref["C"][6, 0, 1] > (1 << 20)


def _fp4_levels(cp, g, M):
    """The documented auto policy (include/gakco.h GAKCO_OPT_GRAM_FP4): level m uses
    e2m1 when n_max * p_max^(g-m) <= 1/8."""
    lens = np.diff(cp.offsets)
    nmax = int(max(0, (lens - g + 1).max())) if len(lens) else 0
    pmax = np.bincount(cp.codes, minlength=256).max() / max(1, len(cp.codes))
    return sum(1 << m for m in range(M + 1) if nmax * pmax ** (g - m) <= 0.125)


def test_gram_format_per_level(gk, oracle_lib):
    """Auto Gram operand format is chosen per level: e2m1 where keys are rare within a
    sequence, u8 where counts > 4 are common (few effective keys: high m on DNA, Zipf
    text). Mixed plans keep parity; host and device codes choose the same formats."""
    import torch
    rng = np.random.default_rng(131)
    dna = sc.uniform(300, 90, 4, 5)
    zipf = sc.gen_text(7, 260, 60, 120)
    for cp, g, k, M in [(dna, 8, 2, 6), (zipf, 6, 1, 5)]:
        ref = oracle_lib.compute(cp, g, k, M)
        want = _fp4_levels(cp, g, M)
        assert 0 < want < (1 << (M + 1)) - 1  # a mixed plan
        r = run(gk, cp, g, k, M, heavy_min_seqs=2)
        assert_parity(r, ref)
        assert r["stats"]["gram_fp4"] == want
        assert 0 < r["stats"]["heavy_macs_fp4"] < r["stats"]["heavy_macs"]
        # device-resident codes: histogram on the device, same choice
        plan = gk.Plan(cp.sigma, g, k, M)
        plan.set_option(gk.GAKCO_OPT_HEAVY_MIN_SEQS, 2)
        rd = gk.kernel_matrix(torch.from_numpy(cp.codes).cuda(), cp.offsets, cp.sigma, g, k,
                              M, plan=plan)
        assert plan.stats()["gram_fp4"] == want
        plan.close()
        assert np.array_equal(rd["C"].cpu().numpy(), ref["C"])
        # forced formats
        assert run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=0)["stats"]["gram_fp4"] == 0
        assert run(gk, cp, g, k, M, heavy_min_seqs=2, gram_fp4=1)["stats"]["gram_fp4"] == \
            (1 << (M + 1)) - 1
    del rng


def test_light_flat_threshold(gk, oracle_lib):
    """Light groups enumerated flattened across a warp (s <= flat) or from
    registers one group per warp: every threshold gives the oracle's result."""
    rng = np.random.default_rng(111)
    for _ in range(6):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(3, 9))
        k = int(rng.integers(1, g + 1))
        cp = sc.random_small(rng, sigma, n_max=150, l_max=90)
        ref = oracle_lib.compute(cp, g, k, g - k)
        for flat in (1, 5, 32):
            assert_parity(run(gk, cp, g, k, g - k, light_flat=flat, heavy_min_seqs=1 << 50), ref)


def test_xl_compaction_families(gk, oracle_lib):
    """Cross-level mask-trie chain with compacted parents (GAKCO_OPT_XL_COMPACT): family
    corpora (groups of many sizes, repeated keys within a sequence, Σ = 4 and 20),
    segments of many tiles, several batches per level (ragged device counts reused),
    relabelled or not; == the uncompacted chain == oracle."""
    cases = [(sc.gen_families(41, 60, 4, 2000, 1500, 2000, sigma=20), 8, 4, 4),
             (sc.gen_families(42, 80, 8, 900, 600, 900, sigma=4), 9, 5, 4),
             (sc.from_sequences(4, [[0, 1] * 700, [0, 1] * 650, [1, 0] * 500] +
                                [list(np.random.default_rng(43).integers(0, 4, 1200))
                                 for _ in range(20)]), 6, 2, 4)]
    for cp, g, k, M in cases:
        ref = oracle_lib.compute(cp, g, k, M)
        for opts in ({}, {"batch_keys": 70000}, {"light_relabel": 1}, {"xl_compact": 0},
                     {"leaf_fuse": 0}):
            assert_parity(run(gk, cp, g, k, M, sort=6, **opts), ref)


def test_leaf_fused_big_groups(gk, oracle_lib):
    """Fused last pass + run-length (leaf.cu, GAKCO_OPT_LEAF_FUSE): groups of the pass
    before larger than a CTA's tile (2048) are split into the overflow slot and taken
    by the segment kernel -- periodic sequences make groups of ~10^4 g-mers next to
    small random ones, in the trie and the compacted chain, several batches per
    level; == the unfused path == oracle."""
    rng = np.random.default_rng(44)
    seqs = [[0, 1, 2] * 900 for _ in range(4)] + [[1, 2, 0, 3] * 600 for _ in range(3)]
    seqs += [list(rng.integers(0, 4, int(rng.integers(200, 1500)))) for _ in range(40)]
    cp = sc.from_sequences(4, seqs)
    for g, k, M in [(7, 3, 4), (8, 4, 3)]:
        ref = oracle_lib.compute(cp, g, k, M)
        r = run(gk, cp, g, k, M, sort=6)
        assert_parity(r, ref)
        assert_parity(run(gk, cp, g, k, M, sort=6, batch_keys=90000), ref)
        assert_parity(run(gk, cp, g, k, M, sort=6, light_relabel=1), ref)
        r0 = run(gk, cp, g, k, M, sort=6, leaf_fuse=0)
        assert_parity(r0, ref)
        assert r["stats"]["triples"] == r0["stats"]["triples"]
        assert r["stats"]["groups_multi"] == r0["stats"]["groups_multi"]


def test_far_pair_records(gk, oracle_lib):
    """Far-pair records (GAKCO_OPT_FAR_NEAR): with the relabelled accumulator past
    96 MB (N = 7200: 104 MB), light pairs whose labels are >= near apart are
    appended as records and added per accumulator block after each batch. Default
    (256), every pair a record (1), none (2^30), off (0), and many batches (record
    buffer reused) all equal the oracle; the stats count the records."""
    cp = sc.gen_families(31, 7200, 72, 70, 50, 70, sigma=20)
    g, k, M = 7, 4, 3
    ref = oracle_lib.compute(cp, g, k, M)
    r = run(gk, cp, g, k, M)
    assert r["stats"]["far_records"] > 0
    assert_parity(r, ref)
    r1 = run(gk, cp, g, k, M, far_near=1)
    assert r1["stats"]["far_records"] > r["stats"]["far_records"]
    assert_parity(r1, ref)
    assert run(gk, cp, g, k, M, far_near=1 << 30)["stats"]["far_records"] == 0
    r0 = run(gk, cp, g, k, M, far_near=0)
    assert r0["stats"]["far_records"] == 0
    assert_parity(r0, ref)
    assert_parity(run(gk, cp, g, k, M, far_near=64, batch_keys=400000, light_window=0), ref)
    assert_parity(run(gk, cp, g, k, M, far_bytes=8), ref)


def test_light_relabel(gk, oracle_lib):
    """Light accumulator relabelled after the first level by best-partner clusters
    (forced on; automatic only for accumulators far beyond L2) == oracle, on
    family-structured and random corpora, M >= 1 so later levels use the labels."""
    rng = np.random.default_rng(113)
    cases = [(sc.gen_families(7, 90, 6, 60, 30, 60, sigma=20), 6, 3, 3),
             (sc.gen_families(8, 150, 10, 80, 80, 80, sigma=4), 8, 5, 3),
             (sc.gen_families(9, 400, 4, 100, 100, 100, sigma=20), 7, 4, 3),
             (sc.gen_families(10, 300, 150, 60, 60, 60, sigma=20), 6, 3, 3)]
    for _ in range(4):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(3, 9))
        k = int(rng.integers(1, g))
        cases.append((sc.random_small(rng, sigma, n_max=120, l_max=90), g, k, g - k))
    for cp, g, k, M in cases:
        ref = oracle_lib.compute(cp, g, k, M)
        assert_parity(run(gk, cp, g, k, M, light_relabel=1), ref)
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, heavy_min_seqs=1 << 50), ref)
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, light_window=0), ref)
        # far-pair records forced at small N (every pair >= 3 labels apart a record),
        # 4- and 8-byte records
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, far_near=3), ref)
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, far_near=3, far_bytes=8), ref)
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, relabel_host=1), ref)
        # single-mask trie with cross-level reuse: relabelling puts level 0 first
        assert_parity(run(gk, cp, g, k, M, light_relabel=1, sort=6), ref)


def test_light_window_gram(gk, oracle_lib):
    """Window Gram (relabelled accumulator; groups inside one window of 256 labels
    -> u8 columns of that window's block on the tensor cores) == oracle: every
    multi-sequence group a candidate (flat 1, window min 2), windows straddling the
    end of the label range (N not a multiple of 128), counts > 1, several windows."""
    rng = np.random.default_rng(131)
    cases = [(sc.gen_families(11, 300, 12, 70, 40, 70, sigma=20), 6, 3, 3),
             (sc.gen_families(12, 517, 9, 90, 90, 90, sigma=4), 7, 4, 3),
             (sc.gen_families(13, 700, 40, 60, 60, 60, sigma=20), 6, 2, 4),
             (sc.random_small(rng, 4, n_max=300, l_max=120), 5, 2, 3)]
    for cp, g, k, M in cases:
        ref = oracle_lib.compute(cp, g, k, M)
        r = run(gk, cp, g, k, M, light_window=1, light_flat=1, window_min=2,
                heavy_min_seqs=1 << 50)
        assert_parity(r, ref)
        r2 = run(gk, cp, g, k, M, light_window=1)
        assert_parity(r2, ref)
        if cp.n_seq > 300:
            assert r["stats"]["win_groups"] > 0 and r["stats"]["win_macs"] > 0


def test_light_binning(gk, oracle_lib):
    """Binned light updates (forced, tiny accumulator blocks so records span many
    buckets and some buckets overflow to direct atomics) == oracle."""
    rng = np.random.default_rng(107)
    for _ in range(6):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(2, 9))
        k = int(rng.integers(1, g + 1))
        cp = sc.random_small(rng, sigma, n_max=120, l_max=80)
        ref = oracle_lib.compute(cp, g, k, g - k)
        for cells in (7, 1000):
            assert_parity(run(gk, cp, g, k, g - k, light_bins=cells, heavy_min_seqs=1 << 50), ref)


def test_batch_size_invariance(gk, oracle_lib):
    """Different mask batch sizes give identical results (integer sums), with the
    two-stream batch pipeline (default) and on one stream."""
    cp = sc.make("tiny")
    ref = oracle_lib.compute(cp, 7, 5, 2)
    for bk in (1, 4700, 3 * 4700 + 5, 1 << 20):
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=1), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=3), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=4), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=6), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=6, heavy_min_seqs=2), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, sort=7), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, pipeline=0), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, level_order=0), ref)
        assert_parity(run(gk, cp, 7, 5, 2, batch_keys=bk, heavy_min_seqs=2), ref)


def test_sort_modes_ragged(gk, oracle_lib):
    """The chunked LSD passes (v1; v2 with bulk-copied tiles, atomicOr or match.any
    ranking) and the onesweep pass give identical results on segments spanning many
    tiles, with ragged tails and odd alignments (u32 and u64 composites)."""
    rng = np.random.default_rng(104)
    seqs = [rng.integers(0, 20, size=int(rng.integers(0, 3000))) for _ in range(37)]
    cp = sc.from_sequences(20, seqs)
    ref = oracle_lib.compute(cp, 8, 4, 4)
    for bk in (0, 50001, 4097 * 3):
        for mode in (0, 1, 3, 4, 5, 6, 7):
            assert_parity(run(gk, cp, 8, 4, 4, batch_keys=bk, sort=mode), ref)
        # the mask trie on the generic 8-bit radix pass instead of trie.cu's, and the
        # cross-level chain without compaction
        assert_parity(run(gk, cp, 8, 4, 4, batch_keys=bk, sort=6, trie_pass=0), ref)
        assert_parity(run(gk, cp, 8, 4, 4, batch_keys=bk, sort=6, xl_compact=0), ref)
    cp4 = sc.from_sequences(4, [rng.integers(0, 4, size=int(rng.integers(0, 5000)))
                                for _ in range(23)])
    ref4 = oracle_lib.compute(cp4, 6, 3, 3)
    for bk in (0, 12289):
        for mode in (0, 3, 4, 5, 7):
            r = run(gk, cp4, 6, 3, 3, batch_keys=bk, sort=mode)
            assert r["stats"]["keys32"] > 0
            assert_parity(r, ref4)


def test_grouping_modes(gk, oracle_lib):
    """Every grouping path == oracle: chunked LSD sort (0; v2: 3-5), onesweep (1),
    hash partition (2), mask trie (6), batched mask trie (7, the default for masks
    below 2M g-mers); the stats report which path ran."""
    rng = np.random.default_rng(108)
    for it in range(10):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(2, 11))
        k = int(rng.integers(1, g + 1))
        M = int(rng.integers(0, g + 1))
        cp = sc.random_small(rng, sigma, n_max=200, l_max=300)
        ref = oracle_lib.compute(cp, g, k, M)
        for mode in (0, 1, 2, 3, 4, 5, 6, 7):
            r = run(gk, cp, g, k, M, sort=mode)
            assert_parity(r, ref)
            if r["stats"]["keys"] > 0:
                assert r["stats"]["grouping"] == {6: 3, 7: 4}.get(mode, mode if mode < 3 else 0)
        assert_parity(run(gk, cp, g, k, M, sort=6, trie_pass=0), ref)
        assert_parity(run(gk, cp, g, k, M, sort=6, xl_compact=0), ref)
        r = run(gk, cp, g, k, M)
        if r["stats"]["keys"] > 0:  # auto: the batched trie where one word holds the composite
            bits = max(1, int(np.ceil(np.log2(max(sigma, 2)))))
            sb = int(np.ceil(np.log2(cp.n_seq))) if cp.n_seq > 1 else 0
            assert r["stats"]["grouping"] == (4 if g * bits + sb <= 64 else 0)


def test_hash_big_buckets(gk, oracle_lib):
    """Buckets far above the shared-memory capacity (4096 keys) take the
    global-table path: few distinct keys (Σ = 2, g = 4; Σ = 1) over many g-mers,
    mixed with ordinary buckets (Σ = 4 background)."""
    rng = np.random.default_rng(109)
    cases = [
        (sc.from_sequences(2, [rng.integers(0, 2, size=3000) for _ in range(12)]), 4, 2, 2),
        (sc.from_sequences(1, [[0] * 2500, [0] * 1800, [0] * 3]), 5, 3, 2),
        (sc.from_sequences(4, [[0] * 6000] + [rng.integers(0, 4, size=2000) for _ in range(20)]),
         6, 3, 3),
    ]
    for cp, g, k, M in cases:
        ref = oracle_lib.compute(cp, g, k, M)
        for hm in (0, 1 << 50):
            assert_parity(run(gk, cp, g, k, M, sort=2, heavy_min_seqs=hm), ref)


def test_hash_batch_size_invariance(gk, oracle_lib):
    """Hash grouping over different mask batch sizes (bucket counts, chunk sizes
    and masks per CTA change with the batch) gives identical results."""
    rng = np.random.default_rng(110)
    seqs = [rng.integers(0, 20, size=int(rng.integers(0, 2500))) for _ in range(41)]
    cp = sc.from_sequences(20, seqs)
    ref = oracle_lib.compute(cp, 8, 4, 4)
    for bk in (1, 50001, 1 << 22):
        assert_parity(run(gk, cp, 8, 4, 4, batch_keys=bk, sort=2), ref)


def test_edge_cases(gk, oracle_lib):
    cases = [
        (sc.from_sequences(4, [[0, 1, 2, 3, 0, 1]]), 3, 2, 1),      # N = 1
        (sc.from_sequences(4, [[], [1, 2], [0] * 20]), 3, 1, 2),     # empty and short rows
        (sc.from_sequences(4, [[], []]), 3, 1, 2),                   # no g-mers at all
        (sc.from_sequences(1, [[0] * 30, [0] * 7]), 5, 2, 5),        # Σ = 1, M = g
        (sc.from_sequences(255, [list(range(255)), list(range(254, -1, -1))]), 4, 2, 2),
        (sc.from_sequences(4, [[0, 1] * 40, [1, 0] * 33]), 8, 8, 0),  # k = g, M = 0
        (sc.from_sequences(36, [[5] * 200, [5] * 150, [7] * 90]), 10, 5, 10),
    ]
    for cp, g, k, M in cases:
        assert_parity(run(gk, cp, g, k, M), oracle_lib.compute(cp, g, k, M))


def test_shard_emulation(gk, oracle_lib):
    """P shards accumulated into one C equal the 1-GPU result (mask sharding), also
    with the single-mask / batched tries (a shard's masks miss some parents)."""
    cp = sc.make("tiny")
    g, k, M = 7, 5, 2
    ref = oracle_lib.compute(cp, g, k, M)
    N = cp.n_seq
    for world, sort in ((2, -1), (3, -1), (8, -1), (40, -1), (2, 6), (3, 6), (3, 7)):
        C = torch.zeros((M + 1, N, N), dtype=torch.int64, device="cuda")
        total = 0
        for rank in range(world):
            plan = gk.Plan(cp.sigma, g, k, M)
            plan.set_option(gk.GAKCO_OPT_SORT, sort)  # (6: cross-level trie, parents in other shards)
            plan.set_shard(rank, world)
            total += plan.num_masks(shard_only=True)
            plan.accumulate(cp.codes, cp.offsets, N, C)
            plan.close()
        assert total == 29
        plan = gk.Plan(cp.sigma, g, k, M)
        Nm = torch.empty_like(C)
        K = torch.empty((N, N), dtype=torch.int64, device="cuda")
        Kn = torch.empty((N, N), dtype=torch.float64, device="cuda")
        plan.finalize(C, N, Nm, K, Kn)
        plan.close()
        assert_parity({"C": C.cpu().numpy(), "Nm": Nm.cpu().numpy(), "K": K.cpu().numpy(),
                       "Knorm": Kn.cpu().numpy()}, ref)


def test_shard_rule_matches_library(gk):
    """gakco_set_shard(r, P) accumulates exactly the masks parallel.shard_masks
    lists (checked against the literal Algorithm 1 reference per shard)."""
    from tests.test_multirank import _partial_C
    from paper_1704_07468_b200 import parallel
    rng = np.random.default_rng(105)
    cp = sc.random_small(rng, 4, n_max=6, l_max=30)
    g, k, M, N = 6, 3, 3, cp.n_seq
    for world in (3, 5):
        for rank in range(world):
            C = torch.zeros((M + 1, N, N), dtype=torch.int64, device="cuda")
            plan = gk.Plan(cp.sigma, g, k, M)
            plan.set_shard(rank, world)
            plan.accumulate(cp.codes if cp.codes.size else np.zeros(1, np.uint8), cp.offsets, N, C)
            plan.close()
            ref = _partial_C(cp, g, M, parallel.shard_masks(g, M, rank, world))
            assert np.array_equal(C.cpu().numpy(), ref)


def test_host_buffers_e2e(gk, oracle_lib):
    """Host (pinned) inputs and host outputs through gakco_kernel (the e2e path)."""
    cp = sc.make("tiny")
    g, k, M = 7, 5, 2
    N = cp.n_seq
    ref = oracle_lib.compute(cp, g, k, M)
    codes = torch.from_numpy(cp.codes).pin_memory()
    offs = torch.from_numpy(cp.offsets).pin_memory()
    K = torch.empty((N, N), dtype=torch.int64).pin_memory()
    Kn = torch.empty((N, N), dtype=torch.float64).pin_memory()
    plan = gk.Plan(cp.sigma, g, k, M)
    plan.kernel(codes, offs, N, None, None, K, Kn)
    plan.close()
    assert np.array_equal(K.numpy(), ref["K"])
    assert_knorm(Kn.numpy(), ref["Knorm"])


def test_k_only_fast_path(gk, oracle_lib):
    """NEXT-1: gakco_kernel_k (level g-k masks only) gives the oracle's K and
    Knorm; refused when M < g-k."""
    rng = np.random.default_rng(106)
    cases = [(sc.make("tiny"), 7, 5)]
    for _ in range(10):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(1, 10))
        k = int(rng.integers(1, g + 1))
        cases.append((sc.random_small(rng, sigma, n_max=60, l_max=100), g, k))
    for cp, g, k in cases:
        ref = oracle_lib.compute(cp, g, k, g - k)
        N = cp.n_seq
        K = torch.empty((N, N), dtype=torch.int64, device="cuda")
        Kn = torch.empty((N, N), dtype=torch.float64, device="cuda")
        codes = cp.codes if cp.codes.size else np.zeros(1, np.uint8)
        for opts in ({}, {"light_relabel": 1, "batch_keys": 3000},
                     {"light_relabel": 1, "batch_keys": 3000, "light_window": 1, "sort": 6}):
            plan = gk.Plan(cp.sigma, g, k, g - k)
            for opt, val in opts.items():  # (relabelled after the level's first batch)
                plan.set_option(getattr(gk, "GAKCO_OPT_" + opt.upper()), val)
            plan.kernel_k(codes, cp.offsets, N, K, Kn)
            plan.close()
            assert np.array_equal(K.cpu().numpy(), ref["K"])
            assert_knorm(Kn.cpu().numpy(), ref["Knorm"])
    plan = gk.Plan(4, 7, 5, 1)
    with pytest.raises(gk.GakcoError):
        plan.kernel_k(cases[0][0].codes, cases[0][0].offsets, 50, K, Kn)
    plan.close()


def test_k_only_dna_digest(gk):
    """K-only on the full DNA config matches the oracle's committed K digest."""
    gold = _golden("dna")
    cfg = sc.CONFIGS["dna"]
    cp = sc.make("dna")
    N = cp.n_seq
    K = torch.empty((N, N), dtype=torch.int64, device="cuda")
    plan = gk.Plan(cfg.sigma, cfg.g, cfg.k, cfg.M)
    plan.kernel_k(cp.codes, cp.offsets, N, K, None)
    plan.close()
    assert refs.digest_np(K.cpu().numpy()) == int(gold["digests"]["K"])


def test_zero_upper(gk):
    """gakco_zero_upper zeroes exactly the upper triangles (Y >= X) of each level,
    odd and even N (16-byte vector body, scalar head and tail); the lower triangles
    keep their values."""
    import torch
    plan = gk.Plan(4, 5, 3, 2)
    for N, L in ((1, 1), (7, 3), (64, 2), (333, 3)):
        C = torch.randint(1, 1 << 40, (L, N, N), dtype=torch.int64, device="cuda")
        ref = C.clone().cpu().numpy()
        plan.zero_upper(C, N, L)
        torch.cuda.synchronize()
        got = C.cpu().numpy()
        iu = np.triu_indices(N)
        for lv in range(L):
            ref[lv][iu] = 0
        assert np.array_equal(got, ref)
    plan.close()


def test_stage_timeline(gk, oracle_lib):
    """gakco_stage_timeline (GAKCO_OPT_TIMING, pipeline on and off): every stage event
    of the last call as (stage, t0, t1), 0 <= t0 <= t1, stages 0..7, and per stage the
    same totals as the stats' ms_* fields; the results stay exact."""
    cp = sc.gen_families(61, 120, 8, 200, 120, 200, sigma=20)
    g, k, M = 8, 4, 3
    ref = oracle_lib.compute(cp, g, k, M)
    names = ["encode", "sort", "segment", "light", "heavy", "epilogue", "dense", "far"]
    for pipe in (0, 1):
        plan = gk.Plan(cp.sigma, g, k, M)
        plan.set_option(gk.GAKCO_OPT_TIMING, 1)
        plan.set_option(gk.GAKCO_OPT_PIPELINE, pipe)
        r = gk.kernel_matrix(cp.codes, cp.offsets, cp.sigma, g, k, M, plan=plan)
        assert_parity({key: v.cpu().numpy() for key, v in r.items()}, ref)
        tl = plan.stage_timeline()
        st = plan.stats()
        plan.close()
        assert tl and all(0 <= s < 8 and 0.0 <= a <= b for s, a, b in tl)
        tot = {}
        for s, a, b in tl:
            tot[names[s]] = tot.get(names[s], 0.0) + (b - a)
        for nm, v in tot.items():
            assert abs(v - st["ms_" + nm]) <= 1e-3 * max(1.0, v)


def test_errors(gk):
    with pytest.raises(gk.GakcoError) as e:
        gk.Plan(4, 3, 4, 0)
    assert e.value.status == gk.GAKCO_E_ARG
    cp = sc.from_sequences(4, [[0, 1, 2, 3]])
    bad = cp.codes.copy()
    bad[1] = 9
    with pytest.raises(gk.GakcoError) as e:
        gk.kernel_matrix(bad, cp.offsets, 4, 3, 2, 1)
    assert e.value.status == gk.GAKCO_E_SYMBOL
    # device codes: checked on the device, reported by finalize; the plan recovers
    plan = gk.Plan(4, 3, 2, 1)
    with pytest.raises(gk.GakcoError) as e:
        gk.kernel_matrix(torch.from_numpy(bad).cuda(), cp.offsets, 4, 3, 2, 1, plan=plan)
    assert e.value.status == gk.GAKCO_E_SYMBOL
    ok = gk.kernel_matrix(torch.from_numpy(cp.codes).cuda(), cp.offsets, 4, 3, 2, 1, plan=plan)
    assert ok["K"][0, 0].item() == 2 * 3  # two 3-mers, h_0 = C(3,2) = 3, one self-pair each
    plan.close()
    with pytest.raises(gk.GakcoError) as e:
        gk.kernel_matrix(cp.codes, np.array([0, 5, 4]), 4, 3, 2, 1)
    assert e.value.status == gk.GAKCO_E_ARG
    # 36^12 keys and 11 bits of sequence id do not fit 64 bits at m = 0
    long = sc.from_sequences(36, [[1] * 20] * 2000)
    with pytest.raises(gk.GakcoError) as e:
        gk.kernel_matrix(long.codes, long.offsets, 36, 13, 12, 1)
    assert e.value.status == gk.GAKCO_E_RANGE


def _golden(name):
    with open(os.path.join(GOLDEN, f"oracle_{name}.json")) as f:
        return json.load(f)


def _check_digests(name, r, which=None):
    """Every C_m, N_m and K of r (device tensors) against the committed oracle
    digests (digests taken on the device, tests/digest_gpu.py); Knorm against the
    oracle's normalisation of the verified K (1e-12, diagonal exact)."""
    from tests.digest_gpu import digest_torch
    gold = _golden(name)
    cfg = sc.CONFIGS[name]
    d = gold["digests"]
    for m in range(cfg.M + 1):
        if which is None or "C" in which:
            assert digest_torch(r["C"][m]) == int(d[f"C{m}"]), f"{name} C{m}"
        if r.get("Nm") is not None and (which is None or "Nm" in which):
            assert digest_torch(r["Nm"][m]) == int(d[f"N{m}"]), f"{name} N{m}"
    assert digest_torch(r["K"]) == int(d["K"]), f"{name} K"
    if r.get("Knorm") is not None:
        _knorm_from_k(r["K"], r["Knorm"])


def _knorm_from_k(K, Kn):
    """Reading A5 recomputed from the verified K on the device in fp64 with the
    oracle's formula (K / sqrt(Kxx * Kyy), 0 when a diagonal is 0, diagonal 1)
    and compared at 1e-12 relative, row blocks at a time."""
    kd = K.diagonal().to(torch.float64)
    N = K.shape[0]
    for r0 in range(0, N, 2048):
        kb = K[r0:r0 + 2048].to(torch.float64)
        a = kd[r0:r0 + 2048, None]
        ref = kb / torch.sqrt(a * kd[None, :])
        ref = torch.where((a > 0) & (kd[None, :] > 0), ref, torch.zeros_like(ref))
        got = Kn[r0:r0 + 2048]
        assert torch.allclose(got, ref, rtol=KNORM_RTOL, atol=0)
    dg = Kn.diagonal()
    assert torch.equal(dg, torch.where(kd > 0, torch.ones_like(dg), torch.zeros_like(dg)))


def test_digest_gpu_matches_numpy(gk):
    """tests/digest_gpu.py (device) == tests/refs.digest_np (numpy restatement)."""
    from tests.digest_gpu import digest_torch
    rng = np.random.default_rng(3)
    a = rng.integers(-2 ** 62, 2 ** 62, size=(301, 257)).astype(np.int64)
    b = rng.random((129, 77))
    assert digest_torch(torch.from_numpy(a).cuda()) == refs.digest_np(a)
    assert digest_torch(torch.from_numpy(b).cuda()) == refs.digest_np(b)


@pytest.mark.parametrize("name", ["tiny", "dna", "protein", "text", "scale"])
def test_full_config_digests(gk, name):
    """All five BASELINE.json configs at full size, in bench's launch configuration
    (default options), against the oracle's committed digests of every output
    matrix (tests/golden/oracle_<name>.json, written by oracle/make_digests.py)."""
    gold = _golden(name)
    cfg = sc.CONFIGS[name]
    cp = sc.make(name)
    assert cp.sha256() == gold["corpus_sha256"], "generator drifted"
    r = gk.kernel_matrix(cp.codes, cp.offsets, cfg.sigma, cfg.g, cfg.k, cfg.M)
    _check_digests(name, r)
    del r
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,opts", [
    ("text", {"sort": 0}), ("text", {"heavy_min_seqs": 1 << 50}),
    ("scale", {"light_relabel": 0, "light_window": 0}), ("scale", {"sort": 0}),
    ("scale", {"heavy_min_seqs": 1 << 50, "light_window": 0}),
])
def test_large_config_paths_digests(gk, name, opts):
    """Text / Scale at full size through the non-default paths (LSD sort instead of
    the mask trie, no relabelling / window Gram, all-light) against the same
    committed oracle digests of C_m and K: a bug confined to one path's windows,
    tiles or batches shows up here."""
    cfg = sc.CONFIGS[name]
    cp = sc.make(name)
    plan = gk.Plan(cfg.sigma, cfg.g, cfg.k, cfg.M)
    for opt, val in opts.items():
        plan.set_option(getattr(gk, "GAKCO_OPT_" + opt.upper()), val)
    N = cp.n_seq
    C = torch.zeros((cfg.M + 1, N, N), dtype=torch.int64, device="cuda")
    K = torch.empty((N, N), dtype=torch.int64, device="cuda")
    plan.kernel(cp.codes, cp.offsets, N, C, None, K, None)
    plan.close()
    _check_digests(name, {"C": C, "K": K}, which=("C",))
    del C, K
    torch.cuda.empty_cache()


def test_dna_digests_hash_grouping(gk):
    """The hash-partition grouping (GAKCO_OPT_SORT 2, the NEXT-4 ablation) on the
    full DNA config also matches the committed digests (the default is LSD)."""
    gold = _golden("dna")
    cfg = sc.CONFIGS["dna"]
    cp = sc.make("dna")
    plan = gk.Plan(cfg.sigma, cfg.g, cfg.k, cfg.M)
    plan.set_option(gk.GAKCO_OPT_SORT, 2)
    r = gk.kernel_matrix(cp.codes, cp.offsets, cfg.sigma, cfg.g, cfg.k, cfg.M, plan=plan)
    assert plan.stats()["grouping"] == 2
    plan.close()
    assert refs.digest_np(r["K"].cpu().numpy()) == int(gold["digests"]["K"])
    for m in range(cfg.M + 1):
        assert refs.digest_np(r["C"][m].cpu().numpy()) == int(gold["digests"][f"C{m}"])


@pytest.mark.parametrize("name", ["text", "scale"])
def test_large_config_sampled_pairs(gk, oracle_lib, name):
    """Text / Scale at full size: sampled entries recomputed one by one by the
    oracle (all diagonal entries of a sample of rows, random off-diagonal pairs,
    and the highest-K pairs), plus the Knorm recomputation from K."""
    cfg = sc.CONFIGS[name]
    cp = sc.make(name)
    N = cp.n_seq
    r = gk.kernel_matrix(cp.codes, cp.offsets, cfg.sigma, cfg.g, cfg.k, cfg.M)
    C = r["C"]
    K = r["K"]
    rng = np.random.default_rng(7)
    X = rng.integers(0, N, 160)
    Y = rng.integers(0, N, 160)
    d = rng.integers(0, N, 40)
    Kd = K.diagonal().cpu().numpy()
    # the largest off-diagonal entries of a few rows (the most-updated cells)
    rows = rng.integers(0, N, 8)
    Kr = K[torch.as_tensor(rows, device=K.device)].clone()
    Kr[torch.arange(8), torch.as_tensor(rows, device=K.device)] = -1
    top = Kr.argmax(dim=1).cpu().numpy()
    X = np.concatenate([X, d, rows])
    Y = np.concatenate([Y, d, top])
    nm = oracle_lib.pairs(cp, cfg.g, cfg.M, X, Y)
    po = oracle_lib.pair_outputs(nm, cfg.g, cfg.k)
    Xt = torch.as_tensor(X, device=C.device)
    Yt = torch.as_tensor(Y, device=C.device)
    assert np.array_equal(r["Nm"][:, Xt, Yt].cpu().numpy().T, nm)
    assert np.array_equal(C[:, Xt, Yt].cpu().numpy().T, po["C"])
    assert np.array_equal(K[Xt, Yt].cpu().numpy(), po["K"])
    # properties at any size: symmetry, K == C_{g-k}
    assert torch.equal(K, K.T)
    assert torch.equal(K, C[cfg.g - cfg.k])
    # Knorm from the (spot-verified) K, rows sampled
    import oracle
    sub = np.unique(np.concatenate([X, Y]))[:64]
    Ks = K[torch.as_tensor(sub, device=K.device)][:, torch.as_tensor(sub, device=K.device)]
    ref = oracle.normalize(Ks.cpu().numpy())
    got = r["Knorm"][torch.as_tensor(sub, device=K.device)][:, torch.as_tensor(sub, device=K.device)]
    assert_knorm(got.cpu().numpy(), ref)
    assert np.array_equal(Kd[d], po["K"][160:200])


def _run_rect(gk, cp, NA, g, k, M, **opts):
    plan = gk.Plan(cp.sigma, g, k, M)
    for opt, val in opts.items():
        plan.set_option(getattr(gk, "GAKCO_OPT_" + opt.upper()), val)
    r = gk.kernel_matrix_rect(cp.codes, cp.offsets, NA, cp.sigma, g, k, M, plan=plan)
    plan.close()
    return {key: v.cpu().numpy() for key, v in r.items()}


def _assert_rect(got, ref):
    for key in ("C", "Nm", "K", "Kdiag"):
        assert np.array_equal(got[key], ref[key]), key
    np.testing.assert_allclose(got["Knorm"], ref["Knorm"], rtol=KNORM_RTOL, atol=0)


def test_rect_train_test(gk, oracle_lib):
    """NEXT-2: the train x test block through gakco_kernel_rect == the oracle's
    block (pair-by-pair histograms), over splits, alphabets and the light, heavy
    (tensor-core Gram, rectangular tiles) and default paths."""
    rng = np.random.default_rng(112)
    for it in range(12):
        sigma = int(rng.choice([2, 4, 20, 36]))
        g = int(rng.integers(2, 10))
        k = int(rng.integers(1, g + 1))
        M = int(rng.integers(0, g + 1))
        cp = sc.random_small(rng, sigma, n_max=120, l_max=100)
        N = cp.n_seq
        if N < 2:
            continue
        NA = int(rng.integers(1, N))
        ref = oracle_lib.rect(cp, NA, g, k, M)
        _assert_rect(_run_rect(gk, cp, NA, g, k, M), ref)
        _assert_rect(_run_rect(gk, cp, NA, g, k, M, heavy_min_seqs=2), ref)
        _assert_rect(_run_rect(gk, cp, NA, g, k, M, heavy_min_seqs=2, gram_fp4=0), ref)
        _assert_rect(_run_rect(gk, cp, NA, g, k, M, heavy_min_seqs=1 << 50), ref)


def test_rect_is_block_of_full_dna(gk):
    """At the DNA config's full size (bench launch configuration), the rectangular
    block equals the block of the full-matrix path (whose K is digest-verified in
    test_full_config_digests), for an uneven split (tiles ragged on both sides)."""
    cfg = sc.CONFIGS["dna"]
    cp = sc.make("dna")
    NA = 2731
    full = gk.kernel_matrix(cp.codes, cp.offsets, cfg.sigma, cfg.g, cfg.k, cfg.M)
    r = gk.kernel_matrix_rect(cp.codes, cp.offsets, NA, cfg.sigma, cfg.g, cfg.k, cfg.M)
    assert torch.equal(r["K"], full["K"][:NA, NA:])
    assert torch.equal(r["C"], full["C"][:, :NA, NA:])
    assert torch.equal(r["Kdiag"], full["K"].diagonal())
    assert torch.equal(r["Knorm"], full["Knorm"][:NA, NA:])


# ------------------------------------------------------------ sharded step
def _assemble_packed(N, M, slices):
    T = N * (N + 1) // 2
    out = {"C": np.zeros((M + 1, T), np.int64), "Nm": np.zeros((M + 1, T), np.int64),
           "K": np.zeros(T, np.int64), "Knorm": np.zeros(T, np.float64)}
    for b, e, d in slices:
        for key in out:
            out[key][..., b:e] = d[key]
    return out


def _assert_packed(got, ref, N):
    iu = np.triu_indices(N)
    assert np.array_equal(got["C"], ref["C"][:, iu[0], iu[1]])
    assert np.array_equal(got["Nm"], ref["Nm"][:, iu[0], iu[1]])
    assert np.array_equal(got["K"], ref["K"][iu])
    np.testing.assert_allclose(got["Knorm"], ref["Knorm"][iu], rtol=KNORM_RTOL, atol=0)
    dg = iu[0] == iu[1]
    assert np.array_equal(got["Knorm"][dg], np.diag(ref["Knorm"]))


def test_sharded_packed_emulation(gk, oracle_lib):
    """The device side of the P-GPU step on one GPU: P shards accumulate into their
    own C (gakco_set_shard), each level is packed (gakco_pack_upper, 32- and 64-bit
    words), the packs and diagonals (gakco_diag) are summed as the collectives
    would, and every rank's slice is finalised (gakco_finalize_packed); the
    assembled slices equal the oracle's upper triangles. Also checks that every
    level is reported complete (gakco_level_order) and waitable."""
    from paper_1704_07468_b200 import parallel
    rng = np.random.default_rng(131)
    cases = [(sc.make("tiny"), 7, 5, 2)]
    for _ in range(4):
        sigma = int(rng.choice([2, 4, 20]))
        g = int(rng.integers(2, 9))
        k = int(rng.integers(1, g + 1))
        cases.append((sc.random_small(rng, sigma, n_max=70, l_max=90), g, k, int(rng.integers(0, g + 1))))
    for cp, g, k, M in cases:
        N = cp.n_seq
        ref = oracle_lib.compute(cp, g, k, M)
        codes = cp.codes if cp.codes.size else np.zeros(1, np.uint8)
        T = N * (N + 1) // 2
        for world, wb in ((2, 8), (3, 4), (5, 8)):
            chunk = -(-T // world)
            dt = torch.int32 if wb == 4 else torch.int64
            packs = torch.zeros((M + 1, chunk * world), dtype=dt, device="cuda")
            D = torch.zeros((M + 1, N), dtype=torch.int64, device="cuda")
            for rank in range(world):
                plan = gk.Plan(cp.sigma, g, k, M)
                plan.set_shard(rank, world)
                C = torch.zeros((M + 1, N, N), dtype=torch.int64, device="cuda")
                plan.accumulate(codes, cp.offsets, N, C)
                assert sorted(plan.level_order()) == list(range(M + 1))
                p1 = torch.zeros_like(packs)
                s = torch.cuda.current_stream()
                for m in plan.level_order():
                    plan.stream_wait_level(m, s)
                    plan.pack_upper(C[m], N, 1, 0, T, p1[m], wb, s)
                d1 = torch.empty_like(D)
                plan.diag(C, N, M + 1, d1, s)
                packs += p1
                D += d1
                plan.close()
            slices = []
            for rank in range(world):
                _, b, e = parallel.tri_slice(N, rank, world)
                Cp = packs[:, rank * chunk:(rank + 1) * chunk].contiguous()
                Nm = torch.empty((M + 1, chunk), dtype=torch.int64, device="cuda")
                K = torch.empty((chunk,), dtype=torch.int64, device="cuda")
                Kn = torch.empty((chunk,), dtype=torch.float64, device="cuda")
                plan = gk.Plan(cp.sigma, g, k, M)
                plan.finalize_packed(Cp, wb, chunk, N, b, e, D, Nm, K, Kn)
                plan.close()
                slices.append((b, e, {"C": Cp[:, : e - b].long().cpu().numpy(),
                                      "Nm": Nm[:, : e - b].cpu().numpy(),
                                      "K": K[: e - b].cpu().numpy(),
                                      "Knorm": Kn[: e - b].cpu().numpy()}))
            _assert_packed(_assemble_packed(N, M, slices), ref, N)


@pytest.mark.parametrize("exchange", ["p2p", "collective"])
def test_sharded_step_two_ranks_one_gpu(gk, oracle_lib, tmp_path, exchange):
    """parallel.launch + ShardedStep with the real library: two ranks on cuda:0, Tiny
    config, two steps (both receive buffers); the assembled packed slices equal the
    oracle. p2p: the fused pack writes into the other rank's receive buffer through a
    CUDA IPC mapping (on one GPU the 'peer' memory is local), the epilogue sums the
    contributions; collective: pack + reduce-scatter (gloo, staged through host
    memory; NCCL on a multi-GPU box). Multi-GPU boxes are not available to this
    build."""
    from paper_1704_07468_b200 import parallel
    res = tmp_path / "res.txt"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rc = parallel.launch(2, os.path.join(root, "tests", "dist_worker.py"), [str(res), "gpu", exchange])
    assert rc == 0
    assert res.read_text().startswith("ok"), res.read_text()
    assert f"exchange={exchange}" in res.read_text()


def test_k_sweep_parity(gk, oracle_lib):
    """NEXT-3, reduced k-sweep (Fig. 4 shape): g = 10, M = g - k =
    1..9 (up to 1013 masks) on a DNA-like and a Zipf text-like corpus of 300
    sequences of length 100. The oracle's Hamming histograms are computed once per
    corpus with M = g; each point's expected C_m (Eq. 8), N_m, K (Eq. 7) and Knorm
    follow from them; full path and K-only path must match."""
    g = 10
    for cp in (sc.uniform(300, 100, 4, 21), sc.gen_text(22, 300, 100, 100)):
        hist = oracle_lib.profiles(cp, g, g)
        for M in range(1, g):
            k = g - M
            nm = np.ascontiguousarray(hist[: M + 1])
            ref = {"Nm": nm, "C": oracle_lib.cumulative(nm, g), "K": oracle_lib.kernel(nm, g, k)}
            ref["Knorm"] = oracle_lib.normalize(ref["K"])
            assert_parity(run(gk, cp, g, k, M), ref)
            N = cp.n_seq
            K = torch.empty((N, N), dtype=torch.int64, device="cuda")
            plan = gk.Plan(cp.sigma, g, k, M)
            plan.kernel_k(cp.codes, cp.offsets, N, K, None)
            plan.close()
            assert np.array_equal(K.cpu().numpy(), ref["K"])
