"""Write tests/golden/oracle_<config>.json: oracle digests of every output.

Calls only oracle/ and the input generators (synth/). The digests are the
expected values the GPU parity tests compare against at full size; the corpus
SHA-256 is recorded so a drifting generator is detected.

usage: python -m oracle.make_digests CONFIG [--threads T]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import corpus as sc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=list(sc.CONFIGS))
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = sc.CONFIGS[a.config]
    cp = sc.make(a.config)
    t0 = time.time()
    md, _ = oracle.digests(cp, cfg.g, cfg.k, cfg.M, threads=a.threads, rows=False)
    dt = time.time() - t0
    names = oracle.matrix_names(cfg.M)
    out = {
        "config": a.config,
        "baseline_json_config": cfg.description,
        "written_by": "python -m oracle.make_digests " + a.config + " (calls only oracle/ and synth/)",
        "digest": "sum over entries of splitmix64(idx ^ splitmix64(bits)) mod 2^64, idx = X*N + Y",
        "corpus_sha256": cp.sha256(),
        "N": cp.n_seq, "sigma": cfg.sigma, "g": cfg.g, "k": cfg.k, "M": cfg.M,
        "digests": {n: str(int(d)) for n, d in zip(names, md)},
        "oracle_seconds": round(dt, 2), "threads": a.threads,
        "host": platform.node(), "cpu": platform.processor(),
    }
    path = a.out or os.path.join(ROOT, "tests", "golden", f"oracle_{a.config}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"config": a.config, "seconds": dt, "path": path}))


if __name__ == "__main__":
    main()
