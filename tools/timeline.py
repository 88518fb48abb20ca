"""Stage timeline of one pipelined step (GAKCO_OPT_TIMING with the pipeline on):
per stream group the busy time, the idle gaps and the serial stretches where only one
stream works. Diagnostic only, not a bench number.

    python tools/timeline.py [config] [steps]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1704_07468_b200 import gakco  # noqa: E402

NAMES = ["encode", "sort", "segment", "light", "heavy", "epilogue", "dense", "far"]
STREAM = {0: "s", 1: "s", 2: "s", 5: "s", 3: "s2", 6: "s2", 4: "s2/s3", 7: "s3"}

cfgname = sys.argv[1] if len(sys.argv) > 1 else "scale"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg, cp, masks, n = bench.workload(cfgname)
dev = torch.device("cuda", 0)
N, M = cp.n_seq, cfg.M
codes_d = torch.from_numpy(cp.codes).to(dev)
offs_h = torch.from_numpy(cp.offsets).pin_memory()
plan = gakco.Plan(cfg.sigma, cfg.g, cfg.k, M, 0)
plan.set_option(gakco.GAKCO_OPT_TIMING, 1)
plan.set_option(gakco.GAKCO_OPT_PIPELINE, 1)
C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
Nm = torch.empty_like(C)
K = torch.empty((N, N), dtype=torch.int64, device=dev)
Kn = torch.empty((N, N), dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream(dev)
for it in range(steps):
    torch.cuda.synchronize()
    C.zero_()
    plan.accumulate(codes_d, offs_h, N, C, stream)
    plan.finalize(C, N, Nm, K, Kn, stream)
    tl = plan.stage_timeline()
    torch.cuda.synchronize()
end = max(b for _, _, b in tl)
print(f"step span (first stage event -> last): {end:.2f} ms, {len(tl)} stage events")
# per stage totals and per stream busy unions
tot = {}
for s, a, b in tl:
    tot[NAMES[s]] = tot.get(NAMES[s], 0.0) + (b - a)
print("stage sums (overlapped):", {k: round(v, 2) for k, v in tot.items()})


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


groups = {"s (encode/sort/segment/epilogue)": [0, 1, 2, 5], "s2 (light/dense)": [3, 6],
          "heavy": [4], "far": [7]}
busy = {}
for gname, ss in groups.items():
    u = union([(a, b) for s, a, b in tl if s in ss])
    busy[gname] = u
    print(f"{gname}: busy {sum(b - a for a, b in u):.2f} ms in {len(u)} runs")
# time where only the s group is busy, only s2 busy, both, none
grid = [i * 0.05 for i in range(int(end / 0.05) + 1)]


def on(u, t):
    lo, hi = 0, len(u)
    while lo < hi:
        mid = (lo + hi) // 2
        if u[mid][1] < t:
            lo = mid + 1
        else:
            hi = mid
    return lo < len(u) and u[lo][0] <= t <= u[lo][1]


cnt = {"only s": 0, "only s2": 0, "both": 0, "neither (far/heavy only or idle)": 0}
us, u2 = busy["s (encode/sort/segment/epilogue)"], busy["s2 (light/dense)"]
for t in grid:
    a, b = on(us, t), on(u2, t)
    k = "both" if a and b else "only s" if a else "only s2" if b else "neither (far/heavy only or idle)"
    cnt[k] += 1
print({k: round(v * 0.05, 1) for k, v in cnt.items()})
# the longest serial stretches of each kind
