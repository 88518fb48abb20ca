"""compute-sanitizer driver: one small invocation of every path through the C-ABI.

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize.py

Each case runs gakco_kernel on a small seeded corpus with one option set and
checks C / K against the oracle (so a sanitizer run that perturbs results fails
too). Paths: default (batched trie), mask trie + cross-level chain with
compaction, generic radix pass, LSD v1 / v2 / onesweep, hash grouping, all heavy
(e2m1 and u8 Gram, CTA pair and one SM), all light, pipeline off, relabelling +
window Gram + far-pair records, train x test, K-only, the sharded step's
pack / diag / packed epilogue.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import oracle
    from paper_1704_07468_b200 import gakco as gk
    from synth import corpus as sc
    cp = sc.gen_families(3, 160, 8, 120, 90, 120, sigma=20)
    g, k, M = 7, 4, 3
    ref = oracle.compute(cp, g, k, M)
    cases = [{}, {"sort": 6}, {"sort": 6, "xl_compact": 0}, {"sort": 6, "trie_pass": 0},
             {"sort": 0}, {"sort": 3}, {"sort": 1}, {"sort": 2},
             {"heavy_min_seqs": 2}, {"heavy_min_seqs": 2, "gram_fp4": 0},
             {"heavy_min_seqs": 2, "gram_pair": 0}, {"heavy_min_seqs": 1 << 50},
             {"pipeline": 0}, {"light_relabel": 1, "light_window": 1, "far_near": 2},
             {"light_relabel": 1, "sort": 6, "far_near": 4}, {"sort": 6, "leaf_fuse": 0},
             {"sort": 6, "light_relabel": 1, "batch_keys": 30000}]
    only = os.environ.get("SAN_CASES")
    for i, opts in enumerate(cases):
        if only and str(i) not in only.split(","):
            continue
        plan = gk.Plan(cp.sigma, g, k, M)
        for o, v in opts.items():
            plan.set_option(getattr(gk, "GAKCO_OPT_" + o.upper()), v)
        r = gk.kernel_matrix(cp.codes, cp.offsets, cp.sigma, g, k, M, plan=plan)
        plan.close()
        assert np.array_equal(r["C"].cpu().numpy(), ref["C"]), opts
        assert np.array_equal(r["K"].cpu().numpy(), ref["K"]), opts
        print("ok", opts, flush=True)
    # fused leaves with groups past a CTA's window (periodic sequences: groups of ~10^4
    # g-mers), both the queued 1024-thread split and the owner-CTA split
    rng = np.random.default_rng(44)
    seqs = [[0, 1, 2] * 900 for _ in range(4)] + [[1, 2, 0, 3] * 600 for _ in range(3)]
    seqs += [list(rng.integers(0, 4, int(rng.integers(200, 1500)))) for _ in range(40)]
    cpb = sc.from_sequences(4, seqs)
    refb = oracle.compute(cpb, 7, 3, 4)
    for opts in ({"sort": 6}, {"sort": 6, "batch_keys": 90000}):
        plan = gk.Plan(cpb.sigma, 7, 3, 4)
        for o, v in opts.items():
            plan.set_option(getattr(gk, "GAKCO_OPT_" + o.upper()), v)
        r = gk.kernel_matrix(cpb.codes, cpb.offsets, cpb.sigma, 7, 3, 4, plan=plan)
        plan.close()
        assert np.array_equal(r["C"].cpu().numpy(), refb["C"]), opts
        print("ok big groups", opts, flush=True)
    N = cp.n_seq
    # K-only and train x test
    plan = gk.Plan(cp.sigma, g, k, M)
    K = torch.empty((N, N), dtype=torch.int64, device="cuda")
    plan.kernel_k(cp.codes, cp.offsets, N, K, None)
    assert np.array_equal(K.cpu().numpy(), ref["K"])
    rr = gk.kernel_matrix_rect(cp.codes, cp.offsets, 70, cp.sigma, g, k, M, plan=plan)
    assert np.array_equal(rr["K"].cpu().numpy(), ref["K"][:70, 70:])
    plan.close()
    print("ok k-only / rect", flush=True)
    # sharded step device side (2 shards)
    from paper_1704_07468_b200 import parallel
    T = parallel.tri_size(N)
    chunk = -(-T // 2)
    packs = torch.zeros((M + 1, 2 * chunk), dtype=torch.int32, device="cuda")
    D = torch.zeros((M + 1, N), dtype=torch.int64, device="cuda")
    for rank in range(2):
        plan = gk.Plan(cp.sigma, g, k, M)
        plan.set_shard(rank, 2)
        C = torch.zeros((M + 1, N, N), dtype=torch.int64, device="cuda")
        plan.accumulate(cp.codes, cp.offsets, N, C)
        p1 = torch.zeros_like(packs)
        for m in plan.level_order():
            plan.stream_wait_level(m, torch.cuda.current_stream())
            plan.pack_upper(C[m], N, 1, 0, T, p1[m], 4)
        d1 = torch.empty_like(D)
        plan.diag(C, N, M + 1, d1)
        packs += p1
        D += d1
        plan.close()
    plan = gk.Plan(cp.sigma, g, k, M)
    Kp = torch.empty((chunk,), dtype=torch.int64, device="cuda")
    plan.finalize_packed(packs[:, :chunk].contiguous(), 4, chunk, N, 0, chunk, D, None, Kp, None)
    plan.close()
    iu = np.triu_indices(N)
    assert np.array_equal(Kp.cpu().numpy(), ref["K"][iu][:chunk])
    print("ok sharded", flush=True)


if __name__ == "__main__":
    main()
