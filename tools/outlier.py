"""Diagnosis of Scale's occasional slow steps: the pipelined step (two streams) with
per-stage events on, so each step's stage times (measured under contention) show which
stage grows in a slow step. Not a bench number."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1704_07468_b200 import gakco  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "scale"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
extra = [a.split("=") for a in sys.argv[3:]]
cfg, cp, masks, n = bench.workload(cfgname)
dev = torch.device("cuda", 0)
N, M = cp.n_seq, cfg.M
codes_d = torch.from_numpy(cp.codes).to(dev)
offs_h = torch.from_numpy(cp.offsets).pin_memory()
plan = gakco.Plan(cfg.sigma, cfg.g, cfg.k, M, 0)
plan.set_option(gakco.GAKCO_OPT_TIMING, 1)
plan.set_option(gakco.GAKCO_OPT_PIPELINE, 1)
for k, v in extra:
    plan.set_option(getattr(gakco, k), int(v))
C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
Nm = torch.empty_like(C)
K = torch.empty((N, N), dtype=torch.int64, device=dev)
Kn = torch.empty((N, N), dtype=torch.float64, device=dev)
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream(dev)
rows = []
for i in range(steps + 3):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    C.zero_()
    plan.accumulate(codes_d, offs_h, N, C, stream)
    plan.finalize(C, N, Nm, K, Kn, stream)
    e1.record(stream)
    st = plan.stats()
    torch.cuda.synchronize()
    r = {"step": round(e0.elapsed_time(e1), 1), "host": round(st["ms_host"], 1)}
    for k, v in st.items():
        if k.startswith("ms_") and k != "ms_host":
            r[k[3:]] = round(v, 1)
    r["n_far"] = st["n_far"]
    rows.append(r)
    print(json.dumps(r), flush=True)
