"""NEXT-3: the paper's scaling shapes on the GPU path.

    python tools/sweep.py [--out profiles/sweeps_r01.json] [--quick]

* k-sweep (Fig. 4): fixed g, M = g - k = 1..g-1 (up to
  2^g - 1 masks), on DNA-like (Σ=4, g=10), protein-like (Σ=20, g=10) and
  text-like (Σ=36 Zipf, g=8) corpora of N=2000 sequences of length 100.
* N-sweep (Fig. 5(c)): l = 100, N in {100, 250, 500, 750} as in the paper
  plus {1500, 3000, 6000} (GPU scaling shape), at one (g, k) per alphabet.

Every point: the full path through gakco_kernel (C_m, N_m, K, Knorm on the
device; CUDA events, 1 warm-up + median of 3), and the K-only path (NEXT-1)
where M >= g-k. Every point is also PARITY-CHECKED: the oracle's Hamming
histograms are computed once per corpus with M = g (their cost does not depend
on M), and each point's expected C_m (Eq. 8), N_m, K (Eq. 7) and Knorm come from
them through oracle.cumulative / oracle.kernel / oracle.normalize; the GPU
outputs (full path and K-only) must be equal (Knorm within 1e-12), and each point
records `parity: true/false`. The oracle is timed beside the GPU at N <= 750 of
the N-sweep and once per k-sweep corpus. Synthetic inputs only
(synth/corpus.py); the paper's datasets are not in the container. Numbers are
context for the paper's shapes, not bench lines.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import corpus as sc  # noqa: E402

ALPHABETS = {
    # name: (sigma, generator(N, l, seed), g for the k-sweep, (g, k) for the N-sweep)
    "dna": (4, lambda N, l, s: sc.uniform(N, l, 4, s), 10, (10, 6)),
    "protein": (20, lambda N, l, s: sc.gen_families(s, N, max(1, N // 110), l, l, l), 10, (10, 1)),
    "text": (36, lambda N, l, s: sc.gen_text(s, N, l, l), 8, (8, 4)),
}


def time_gpu(gk, torch, cp, g, k, M, reps=3):
    N = cp.n_seq
    dev = torch.device("cuda", 0)
    plan = gk.Plan(cp.sigma, g, k, M, 0)
    codes = torch.from_numpy(cp.codes).to(dev)
    offs = torch.from_numpy(cp.offsets)
    C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
    Nm = torch.empty_like(C)
    K = torch.empty((N, N), dtype=torch.int64, device=dev)
    Kn = torch.empty((N, N), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)

    def run(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    full = run(lambda: plan.kernel(codes, offs, N, C, Nm, K, Kn, stream=s))
    st = plan.stats()
    outs = {"C": C.cpu().numpy(), "Nm": Nm.cpu().numpy(), "K": K.cpu().numpy(),
            "Knorm": Kn.cpu().numpy()}
    konly = None
    if M >= g - k:
        konly = run(lambda: plan.kernel_k(codes, offs, N, K, Kn, stream=s))
        outs["K_only"] = K.cpu().numpy()
        outs["Knorm_only"] = Kn.cpu().numpy()
    plan.close()
    return {"ms": full, "k_only_ms": konly, "masks": int(st["masks"]), "keys": int(st["keys"]),
            "light_pairs": int(st["light_pairs"]), "heavy_macs": int(st["heavy_macs"])}, outs


def oracle_hist(cp, g, Mmax=None):
    """N_m(X,Y) for m = 0..Mmax (default g; Def. 1 / Eq. 5), once per corpus (the
    direct Hamming count's cost does not depend on M)."""
    import oracle
    oracle.build()
    return oracle.profiles(cp, g, g if Mmax is None else Mmax)


def parity(hist, g, k, M, outs):
    """The point's expected outputs from the oracle histograms (Eq. 8, Eq. 7, reading
    A5) against the GPU's; True iff all equal (Knorm within 1e-12 relative)."""
    import oracle
    nm = np.ascontiguousarray(hist[: M + 1])
    C = oracle.cumulative(nm, g)
    K = oracle.kernel(nm, g, k)
    Kn = oracle.normalize(K)
    ok = (np.array_equal(outs["C"], C) and np.array_equal(outs["Nm"], nm)
          and np.array_equal(outs["K"], K)
          and np.allclose(outs["Knorm"], Kn, rtol=1e-12, atol=0))
    if "K_only" in outs:
        ok = ok and np.array_equal(outs["K_only"], K) and np.allclose(
            outs["Knorm_only"], Kn, rtol=1e-12, atol=0)
    return bool(ok)


def time_oracle(cp, g, k, M):
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    oracle.compute(cp, g, k, M)
    return (time.perf_counter() - t0) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweeps.json"))
    ap.add_argument("--quick", action="store_true", help="fewer points (smoke of the tool)")
    a = ap.parse_args()
    import torch
    from paper_1704_07468_b200 import gakco as gk
    out = {"k_sweep": [], "n_sweep": [], "host_cores": os.cpu_count(),
           "note": "GPU: gakco_kernel full path, CUDA events, median of 3 after 1 warm-up; "
                   "oracle: CPU, all host cores, one run"}
    for name, (sigma, gen, gk_g, _) in ALPHABETS.items():
        cp = gen(2000 if not a.quick else 300, 100, 11)
        Ms = range(1, gk_g) if not a.quick else (1, gk_g - 1)
        ora = time_oracle(cp, gk_g, gk_g - 1, 1) if not a.quick else None
        hist = oracle_hist(cp, gk_g)
        for M in Ms:
            k = gk_g - M
            r, outs = time_gpu(gk, torch, cp, gk_g, k, M)
            r.update({"alphabet": name, "sigma": sigma, "N": cp.n_seq, "l": 100, "g": gk_g,
                      "k": k, "M": M, "oracle_ms_any_M": ora,
                      "parity": parity(hist, gk_g, k, M, outs)})
            out["k_sweep"].append(r)
            print(json.dumps(r), flush=True)
    Ns = (100, 250, 500, 750, 1500, 3000, 6000) if not a.quick else (100, 500)
    for name, (sigma, gen, _, (g, k)) in ALPHABETS.items():
        for N in Ns:
            cp = gen(N, 100, 12)
            M = g - k
            r, outs = time_gpu(gk, torch, cp, g, k, M)
            r.update({"alphabet": name, "sigma": sigma, "N": N, "l": 100, "g": g, "k": k, "M": M,
                      "oracle_ms": time_oracle(cp, g, k, M) if N <= 750 else None,
                      "parity": parity(oracle_hist(cp, g, M), g, k, M, outs)})
            out["n_sweep"].append(r)
            print(json.dumps(r), flush=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    # markdown summary next to the JSON
    md = [f"# NEXT-3 sweeps (GPU full path; oracle on {out['host_cores']} host cores)", "",
          "## k-sweep (Fig. 4 shape): N=2000, l=100", "",
          "| alphabet | g | k | M | masks | GPU ms | K-only ms | oracle ms (any M) | parity |",
          "|---|---|---|---|---|---|---|---|---|"]
    for r in out["k_sweep"]:
        md.append(f"| {r['alphabet']} | {r['g']} | {r['k']} | {r['M']} | {r['masks']} | "
                  f"{r['ms']:.2f} | {r['k_only_ms'] if r['k_only_ms'] is None else round(r['k_only_ms'], 2)} | "
                  f"{r['oracle_ms_any_M'] if r['oracle_ms_any_M'] is None else round(r['oracle_ms_any_M'])} | "
                  f"{'bit-exact' if r['parity'] else 'MISMATCH'} |")
    md += ["", "## N-sweep (Fig. 5(c) shape): l=100", "",
           "| alphabet | g | k | N | GPU ms | oracle ms | parity |", "|---|---|---|---|---|---|---|"]
    for r in out["n_sweep"]:
        md.append(f"| {r['alphabet']} | {r['g']} | {r['k']} | {r['N']} | {r['ms']:.2f} | "
                  f"{'-' if r['oracle_ms'] is None else round(r['oracle_ms'])} | "
                  f"{'bit-exact' if r['parity'] else 'MISMATCH'} |")
    with open(os.path.splitext(a.out)[0] + ".md", "w") as f:
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
