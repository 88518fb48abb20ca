#!/usr/bin/env python
"""bench.py — the gapped k-mer kernel-matrix step on 1..8 B200s.

One STEP = the whole hot path of SURVEY.md §8(a) for one synthetic corpus, with
the corpus already resident in HBM:
  1 GPU:  zero C -> gakco_accumulate over all masks (encode, mask-trie sort,
          segment, light / heavy pair updates, diagonal) -> gakco_finalize (Eq. 9,
          Eq. 7, normalisation; full N x N outputs);
  P GPUs: one process per GPU (re-launched under torch.distributed.run when
          --gpus P > 1 is given without a torchrun environment); each rank
          accumulates its round-robin share of the masks, the packed upper
          triangles are reduce-scattered level by level over NCCL while later
          levels accumulate, the diagonals all-reduced, and each rank finalises its
          slice (parallel.ShardedStep). Total work is fixed as P grows ("strong").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config scale] [--impl reference]

Default workload: BASELINE.json configs[4] ("scale", the largest: 3.71e9 masked
keys, a 20000 x 20000 output, the config north_star names for 1/2/4/8 GPUs).
Prints ONE JSON line on rank 0. value = masked g-mer keys processed per second by
the whole job (c_gk * n / step time); ms_per_step is the gkm kernel-matrix time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import corpus as sc  # noqa: E402

METRIC = "gkm kernel-matrix time (s) at 1/2/4/8 B200; masked g-mer keys sorted/s; HBM %"
UNIT = "keys/s"


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="scale", choices=list(sc.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target seconds of oracle work per CPU sample")
    ap.add_argument("--heavy-min", type=int, default=0)
    ap.add_argument("--batch-keys", type=int, default=0)
    ap.add_argument("--sort", type=int, default=None, choices=[-1, 0, 1, 2, 3, 4, 5, 6, 7],
                    help="grouping: -1 auto, 0 chunked LSD sort, 1 onesweep LSD, 2 hash partition, "
                         "3/4/5 chunked LSD v2 (bulk-copy tiles; atomicOr / match.any / ballot ranking), "
                         "6 mask trie (shared leading-position passes), 7 batched mask trie")
    ap.add_argument("--sort-ctas", type=int, default=0)
    ap.add_argument("--light-flat", type=int, default=0,
                    help="light groups of <= this many sequences share a warp (1..32)")
    ap.add_argument("--light-window", type=int, default=None, choices=[-1, 0, 1],
                    help="window Gram of cluster-local light groups (-1 auto)")
    ap.add_argument("--gram-each", type=int, default=None, choices=[0, 1],
                    help="heavy Gram after every batch (1) or per level / full D (0)")
    ap.add_argument("--window-min", type=int, default=0,
                    help="smallest group for the window Gram (0: default)")
    ap.add_argument("--relabel", type=int, default=None, choices=[-1, 0, 1],
                    help="light accumulator relabelling: -1 auto, 0 off, 1 on")
    ap.add_argument("--fp4", type=int, default=None, choices=[-1, 0, 1],
                    help="heavy Gram operands: -1 auto (e2m1 where exact), 0 u8, 1 e2m1")
    ap.add_argument("--pipeline", type=int, default=None, choices=[0, 1],
                    help="two-stream batch pipeline (default 1)")
    ap.add_argument("--level-order", type=int, default=None, choices=[0, 1],
                    help="0: levels m = 0..M (default), 1: m = M..0")
    ap.add_argument("--gram-pair", type=int, default=None, choices=[0, 1],
                    help="heavy Gram kernel: 1 CTA pairs (default), 0 one SM per tile")
    ap.add_argument("--far-near", type=int, default=None,
                    help="far-pair records from this label distance (-1 auto, 0 off)")
    ap.add_argument("--trie-pass", type=int, default=None, choices=[0, 1],
                    help="mask-trie pass kernel: 1 symbol-digit (trie.cu), 0 generic radix")
    ap.add_argument("--xl-compact", type=int, default=None, choices=[0, 1],
                    help="cross-level trie chain with compacted parents (1, default) or full arrays")
    ap.add_argument("--light-ctas", type=int, default=None, choices=[3, 4, 6],
                    help="relabelled light kernel register budget (CTAs per SM)")
    ap.add_argument("--light-grid", type=int, default=None,
                    help="light kernel grid in CTAs per SM (0 = 8)")
    ap.add_argument("--no-timing", action="store_true",
                    help="no per-stage events (roofline then uses the last timed stages)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


def red_peaks():
    """Measured random u32 RED ceilings (tools/measure_peaks.py -> profiles/peaks_r02.json):
    G updates/s into an L2-resident (32 MB) and a DRAM-resident (800 MB) array."""
    p = os.path.join(ROOT, "profiles", "peaks_r02.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    out = {"source": "measured (tools/measure_peaks.py, profiles/peaks_r02.json)"}
    for r in d.get("red", []):
        if r["pattern"] == "random cells":
            out["l2" if r["array_MB"] <= 64 else "dram"] = r["G_updates_per_s"]
    out["int8_tops"] = d.get("int8_gemm", {}).get("TOPS")
    out["fp4_tflops"] = d.get("fp4_gemm", {}).get("TFLOPS")
    return out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload(cfg_name):
    cfg = sc.CONFIGS[cfg_name]
    cp = sc.make(cfg_name)
    from math import comb
    masks = sum(comb(cfg.g, m) for m in range(cfg.M + 1))
    n = int(sum(max(0, int(l) - cfg.g + 1) for l in cp.lengths()))
    return cfg, cp, masks, n


# --------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("BENCH_CLOCK_MS", "50")],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        # the sampler takes a moment to start: wait for its first line, so that the
        # timed region (which follows) is sampled from its first step
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 5.0:
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU baseline
def oracle_sample(cp, cfg, seconds, threads):
    """Time the oracle (as it stands) on rows [0, r) of the matrix; r is sized
    from a 1-row calibration so the sample takes about `seconds`. Returns
    (sample seconds, fraction of the full upper-triangle work, rows, fixed seconds):
    the oracle's digest routine first computes K(X,X) of all N sequences (a serial
    pass, independent of the row range), timed alone as `fixed` (rows [0, 0)), so the
    full-matrix time is fixed + (sample - fixed) / fraction."""
    import numpy as np
    import oracle
    n = np.maximum(cp.lengths() - cfg.g + 1, 0).astype(np.float64)
    suffix = np.cumsum(n[::-1])[::-1]             # sum_{y>=x} n_y
    row_work = n * suffix                          # window steps of row x (y >= x)
    total = row_work.sum()
    cum = np.cumsum(row_work)

    def run(r):
        t0 = time.perf_counter()
        oracle.digests(cp, cfg.g, cfg.k, cfg.M, threads=threads, row_begin=0, row_end=r,
                       rows=False)
        return time.perf_counter() - t0

    # the fixed part (K(X,X) of every sequence), then calibrate on a growing row count
    # and size the sample so that its row work takes about `seconds`
    fixed = run(0)
    r = max(1, min(cp.n_seq, threads))
    dt = run(r)
    while dt - fixed < 0.1 * seconds and r < cp.n_seq:
        r = min(cp.n_seq, r * 4)
        dt = run(r)
    if dt - fixed < 0.5 * seconds and r < cp.n_seq:
        rate = cum[r - 1] / max(dt - fixed, 1e-6)
        r = int(np.searchsorted(cum, rate * seconds)) + 1
        r = max(1, min(cp.n_seq, r))
        dt = run(r)
    frac = cum[r - 1] / total
    return dt, frac, r, fixed


def oracle_full_seconds(dt, frac, fixed):
    """Full-matrix oracle time from a row sample (fixed part + row work by pair work)."""
    return fixed + max(dt - fixed, 0.0) / frac


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on the host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    cfg, cp, masks, n = workload(a.config)
    threads = os.cpu_count() or 1
    per = max(2.0, min(a.cpu_seconds, 150.0 / max(1, a.steps + a.warmup)))
    for _ in range(a.warmup):
        oracle_sample(cp, cfg, per / 2, threads)
    times, fracs, rows = [], [], []
    for _ in range(a.steps):
        dt, frac, r, fixed = oracle_sample(cp, cfg, per, threads)
        times.append(oracle_full_seconds(dt, frac, fixed))   # extrapolated full-matrix seconds
        fracs.append(frac)
        rows.append(r)
    t = statistics.median(times)
    value = masks * n / t
    sample = (f"oracle rows [0,{rows[-1]}) x all Y>=X of the {a.config} corpus "
              f"({100 * fracs[-1]:.2f}% of the upper-triangle pair work), full-matrix time = "
              f"the K(X,X) pass (timed alone) + the sampled row work extrapolated by pair work; "
              f"digests of C_m, N_m, K, Knorm")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
           "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
           "data": "synthetic",
           "config": config_dict(a.config, cfg, cp, masks, n, 1),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "cpu": cpu_model(), "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def config_dict(name, cfg, cp, masks, n, world):
    return {"workload": name, "baseline_config": cfg.description, "N": cp.n_seq,
            "sigma": cfg.sigma, "g": cfg.g, "k": cfg.k, "M": cfg.M, "masks": masks,
            "gmers": n, "keys_per_step": masks * n,
            "parallelism": f"mask-sharded x{world}: per-level packed-triangle NCCL "
                           f"reduce-scatter + per-rank slice epilogue" if world > 1
            else "1 GPU, all masks",
            "l2": "flushed between timed steps (256 MiB write)"}


# ----------------------------------------------------------------- GPU arm
def stage_model(stats, cfg, N):
    """Algorithmic bytes / ops per stage: unit x count."""
    # composites are 8 B, or 4 B where key + sequence bits fit 32 (keys32)
    keys, passes = stats["keys"], stats["sort_passes"]
    k32, p32 = stats.get("keys32", 0), stats.get("sort_passes32", 0)
    kbytes = 8.0 * (keys - k32) + 4.0 * k32
    trip, grp = stats["triples"], stats["groups_multi"]
    M = cfg.M
    epi = N * N * ((M + 1) * 4 + (M + 1) * 4 + (M + 1) * 8 + 16) + N * (M + 1) * 8
    grouping = stats.get("grouping", 0)
    n_gm = keys / max(1, stats["masks"])  # g-mers per mask
    if grouping == 3:
        # mask trie (SoA): u64 window + u16 (N <= 65536) or u32 sequence id per element,
        # read + written per pass; no per-mask encode (the windows are packed once)
        esz = 8.0 + (2.0 if N <= 65536 else 4.0)
        # the compacted cross-level chain moves fewer elements than its capacities:
        # pass_keys (device count) when the trie.cu pass reports it
        pk = float(stats.get("pass_keys", 0) or 0) or float(passes)
        return {
            "encode": ("hbm", 8.0 * n_gm + 4.0 * n_gm),
            "sort": ("hbm", 2.0 * esz * pk),
            "segment": ("hbm", esz * min(float(keys), pk) + 8.0 * trip + 8.0 * grp),
            # far-pair records: written once, bucketed (hist read, read + write), added
            "far": ("hbm", 40.0 * float(stats.get("far_records", 0) or 0)),
            "light": ("hbm", 8.0 * stats["light_pairs"]),
            "heavy": ("tensor", 2.0 * (stats["heavy_macs"] + stats.get("win_macs", 0))),
            "dense": ("hbm", float(stats["heavy_groups"]) * float(stats.get("n_pad", 0))
                      + 256.0 * float(stats.get("win_groups", 0))),
            "epilogue": ("hbm", float(epi)),
        }
    if grouping == 4:
        # batched mask trie: one-word composites built once (root), read + written per
        # pass (sort_passes32 counts the 4-byte ones)
        enc = ("hbm", 12.0 * n_gm + (4.0 if k32 else 8.0) * n_gm)
        srt = ("hbm", 16.0 * (passes - p32) + 8.0 * p32)
    elif grouping == 2:
        # hash partition (bucket.cu): the count pass recomputes keys from the packed
        # windows (ALU work, windows re-read once per CTA mask group: L2);
        # the scatter pass writes every composite once; group reads it once
        enc = ("alu", float(keys))
        srt = ("hbm", kbytes)
    else:
        enc = ("hbm", kbytes + 4.0 * keys)     # write the key + read the 4 B seq id
        srt = ("hbm", 16.0 * (passes - p32) + 8.0 * p32)  # read + write per key per pass
    e2m1 = float(stats.get("gram_fp4", 0) or 0) > 0
    return {
        "encode": enc,
        "sort": srt,
        "segment": ("hbm", kbytes + 8.0 * trip + 8.0 * grp),  # read keys; write triples, groups
        "far": ("hbm", 40.0 * float(stats.get("far_records", 0) or 0)),
        "light": ("hbm", 8.0 * stats["light_pairs"]),  # u32 read-modify-write per update
        "heavy": ("tensor", 2.0 * (stats["heavy_macs"] + stats.get("win_macs", 0))),
        # one n_pad-byte u8 (n_pad/2 e2m1) column per heavy group, written once
        "dense": ("hbm", float(stats["heavy_groups"]) * float(stats.get("n_pad", 0))
                  * (0.5 if e2m1 and stats.get("heavy_macs_fp4", 0) == stats["heavy_macs"] else 1.0)
                  + 256.0 * float(stats.get("win_groups", 0))),
        "epilogue": ("hbm", float(epi)),
    }


def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_1704_07468_b200 import gakco

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, cp, masks, n = workload(a.config)
    N = cp.n_seq
    M = cfg.M
    codes_d = torch.from_numpy(cp.codes).to(dev)
    offs_h = torch.from_numpy(cp.offsets).pin_memory()
    plan = gakco.Plan(cfg.sigma, cfg.g, cfg.k, M, local)
    plan.set_shard(rank, world)
    # timed steps run without per-stage events; the stage split comes from separate
    # single-stream profiling steps below
    plan.set_option(gakco.GAKCO_OPT_TIMING, 0)
    if a.heavy_min:
        plan.set_option(gakco.GAKCO_OPT_HEAVY_MIN_SEQS, a.heavy_min)
    if a.batch_keys:
        plan.set_option(gakco.GAKCO_OPT_BATCH_KEYS, a.batch_keys)
    if a.sort is not None:
        plan.set_option(gakco.GAKCO_OPT_SORT, a.sort)
    if a.sort_ctas:
        plan.set_option(gakco.GAKCO_OPT_SORT_CTAS_PER_SM, a.sort_ctas)
    if a.light_flat:
        plan.set_option(gakco.GAKCO_OPT_LIGHT_FLAT, a.light_flat)
    if a.relabel is not None:
        plan.set_option(gakco.GAKCO_OPT_LIGHT_RELABEL, a.relabel)
    if a.light_window is not None:
        plan.set_option(gakco.GAKCO_OPT_LIGHT_WINDOW, a.light_window)
    if a.gram_each is not None:
        plan.set_option(gakco.GAKCO_OPT_GRAM_EACH, a.gram_each)
    if a.window_min:
        plan.set_option(gakco.GAKCO_OPT_WINDOW_MIN, a.window_min)
    if a.fp4 is not None:
        plan.set_option(gakco.GAKCO_OPT_GRAM_FP4, a.fp4)
    if a.pipeline is not None:
        plan.set_option(gakco.GAKCO_OPT_PIPELINE, a.pipeline)
    if a.level_order is not None:
        plan.set_option(gakco.GAKCO_OPT_LEVEL_ORDER, a.level_order)
    if a.gram_pair is not None:
        plan.set_option(gakco.GAKCO_OPT_GRAM_PAIR, a.gram_pair)
    if a.far_near is not None:
        plan.set_option(gakco.GAKCO_OPT_FAR_NEAR, a.far_near)
    if a.trie_pass is not None:
        plan.set_option(gakco.GAKCO_OPT_TRIE_PASS, a.trie_pass)
    if a.xl_compact is not None:
        plan.set_option(gakco.GAKCO_OPT_XL_COMPACT, a.xl_compact)
    if a.light_ctas is not None:
        plan.set_option(gakco.GAKCO_OPT_LIGHT_CTAS, a.light_ctas)
    if a.light_grid is not None:
        plan.set_option(gakco.GAKCO_OPT_LIGHT_GRID, a.light_grid)
    C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    from paper_1704_07468_b200 import parallel
    nmax = int(max(0, int(cp.lengths().max()) - cfg.g + 1))
    if world == 1:
        # one GPU: accumulate all masks, then the full-matrix epilogue (mirrored C,
        # N_m, K, Knorm as full N x N matrices)
        Nm = torch.empty_like(C)
        K = torch.empty((N, N), dtype=torch.int64, device=dev)
        Kn = torch.empty((N, N), dtype=torch.float64, device=dev)

        def step():
            plan.zero_upper(C, N, M + 1, stream)  # (accumulate adds into the upper triangles)
            plan.accumulate(codes_d, offs_h, N, C, stream)
            plan.finalize(C, N, Nm, K, Kn, stream)
    else:
        # P GPUs: this rank's masks, per-level packed reduce-scatter over NCCL
        # overlapping the later levels, diagonal all-reduce, epilogue of this rank's
        # slice of the packed triangle (parallel.ShardedStep)
        sh = parallel.ShardedStep(plan, N, cfg.g, cfg.k, M, nmax, dev)
        K = sh.K

        def step():
            sh.step(codes_d, offs_h, C, stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(a.warmup):
        step()
    barrier()
    clk = Clocks(local) if rank == 0 and os.environ.get("BENCH_CLOCK_MS") != "0" else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    stage_ms = {}
    launches = 0
    last = None
    host_ms, enq_ms, far_ov = [], [], []
    # (the host enqueues every step's ~3000 launches: no garbage-collector pauses while
    # the timed steps run)
    import gc
    gc.collect()
    gc.disable()
    barrier()
    for i in range(a.steps):
        flush.fill_(i)                      # L2 flush, outside the step's events
        ev[i][0].record(stream)
        t0 = time.perf_counter()
        step()
        host_ms.append((time.perf_counter() - t0) * 1e3)
        ev[i][1].record(stream)
        st = plan.stats()              # synchronises; after the end event
        enq_ms.append(st.get("ms_host", 0.0))
        far_ov.append(st.get("far_overflow", 0))
        launches += st["launches"]
        last = st
    barrier()
    gc.enable()
    clocks = clk.stop() if clk else None
    # stage split: single-stream profiling steps with per-stage CUDA events (the
    # timed steps overlap light / dense / Gram of batch b with batch b+1 on two
    # streams, so their per-stage events would measure contention, not kernels)
    prof_steps = 0 if a.no_timing else 2
    if prof_steps:
        plan.set_option(gakco.GAKCO_OPT_PIPELINE, 0)
        plan.set_option(gakco.GAKCO_OPT_TIMING, 1)
        for i in range(prof_steps):
            flush.fill_(i)
            step()
            st = plan.stats()
            for kk, v in st.items():
                if kk.startswith("ms_") and kk != "ms_host":
                    stage_ms[kk] = stage_ms.get(kk, 0.0) + v / prof_steps * a.steps
        plan.set_option(gakco.GAKCO_OPT_TIMING, 0)
        plan.set_option(gakco.GAKCO_OPT_PIPELINE, 1 if a.pipeline is None else a.pipeline)
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    mine = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    total_ms = float(mine.item())
    ms_per_step = total_ms / a.steps
    value = masks * n / (ms_per_step / 1e3)

    # ---- e2e through the public C-ABI with host (pinned) buffers
    e2e = None
    if not a.no_e2e:
        codes_h = torch.from_numpy(cp.codes).pin_memory()
        Kh = torch.empty((N, N), dtype=torch.int64).pin_memory() if rank == 0 else None
        Knh = torch.empty((N, N), dtype=torch.float64).pin_memory() if rank == 0 else None

        if world > 1:  # this rank's slice of K and Knorm, to pinned host memory
            Kh = torch.empty((sh.chunk,), dtype=torch.int64).pin_memory()
            Knh = torch.empty((sh.chunk,), dtype=torch.float64).pin_memory()

        def e2e_step():
            if world == 1:
                plan.kernel(codes_h, offs_h, N, C, None, Kh, Knh, stream)
            else:
                sh.step(codes_h, offs_h, C, stream)
                Kh.copy_(sh.K, non_blocking=True)
                Knh.copy_(sh.Knorm, non_blocking=True)
        for _ in range(2):
            e2e_step()
        barrier()
        ee = []
        for i in range(a.steps):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ee.append(e0.elapsed_time(e1))
        t = torch.tensor([sum(ee)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item()) / a.steps
        h2d = (cp.codes.nbytes + cp.offsets.nbytes) * world
        d2h = N * N * 16 if world == 1 else parallel.tri_size(N) * 16
        e2e = {"value": masks * n / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "gakco_kernel(host pinned codes/offsets -> host K, Knorm)" if world == 1
               else "gakco_accumulate(host inputs) + per-level NCCL reduce-scatter + "
                    "gakco_finalize_packed -> each rank's packed slice of K, Knorm to host"}

    # ---- K-only fast path (NEXT-1): K = C_{g-k} from the level-(g-k) masks only
    k_only = None
    if world == 1 and cfg.M >= cfg.g - cfg.k:
        from math import comb
        for _ in range(2):
            plan.kernel_k(codes_d, offs_h, N, K, Kn, stream)
        kt = []
        for i in range(a.steps):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan.kernel_k(codes_d, offs_h, N, K, Kn, stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            kt.append(e0.elapsed_time(e1))
        k_only = {"ms_per_step": sum(kt) / len(kt), "masks": comb(cfg.g, cfg.g - cfg.k),
                  "outputs": "K, Knorm (device)", "api": "gakco_kernel_k"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant stage (CUDA events on the launching stream)
    pk = peaks()
    model = stage_model(last, cfg, N)
    per_step = {k[3:]: v / a.steps for k, v in stage_ms.items()}
    if not any(per_step.values()):  # --no-timing: stage split unavailable
        per_step = {"sort": ms_per_step}
    dom = max((s_ for s_ in per_step if model[s_][0] != "alu") or per_step,
              key=lambda s_: per_step[s_])
    bound, algo = model[dom]
    t_dom = per_step[dom] / 1e3
    stages = {}
    for s_, ms in per_step.items():
        b_, alg = model[s_]
        if ms > 0 and b_ == "alu":
            stages[s_] = {"ms": round(ms, 4), "bound": b_,
                          "Gkeys/s": round(alg / (ms / 1e3) / 1e9, 2)}
        elif ms > 0:
            stages[s_] = {"ms": round(ms, 4), "bound": b_,
                          ("GB/s" if b_ == "hbm" else "TOPS"):
                              round(alg / (ms / 1e3) / (1e9 if b_ == "hbm" else 1e12), 2)}
    # per launch of a stage's kernels (the stage's launches per step come from the
    # plan); traffic = ncu dram bytes per launch (profiles/ncu_traffic.json)
    tr = {}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f).get(a.config, {})
    limiter = {
        "light": "L2 atomic throughput: random u32 REDs into the packed triangle "
                 "(ncu: RED sectors 54% of the L2 peak, lts 80% busy; profiles/)",
        "heavy": "tensor pipe (ncu: 89-94% tensor-pipe active on the large flushes)",
        "sort": "shared-memory ranking latency and bank conflicts (ncu: 27% of HBM)",
    }

    rp = red_peaks()

    def roof_of(st):
        b_, algo_ = model[st]
        t_ = per_step[st] / 1e3
        nl_ = max(1, int(last.get("n_" + st, 0) or 1))
        traffic_ = tr.get(st, {}).get("dram_bytes_per_launch_mean")
        if st == "light" and rp and rp.get("l2"):
            # the light updates are L2 atomics (REDs): achieved pair updates/s against
            # the measured random-RED ceiling into an L2-resident array (the near pairs;
            # far pairs go through records); the DRAM-resident ceiling is
            # what unrelabelled / record-less REDs into a triangle beyond L2 get
            ups = float(last["light_pairs"]) / t_ / 1e9 if t_ > 0 else 0.0
            return {"bound": "l2_atomics", "kernel": st, "achieved": ups, "peak": rp["l2"],
                    "unit": "G updates/s", "frac": ups / rp["l2"], "traffic": traffic_,
                    "algorithmic_updates_per_launch": float(last["light_pairs"]) / nl_,
                    "launches_per_step": nl_, "avg_launch_ms": per_step[st] / nl_,
                    "dram_resident_red_peak": rp.get("dram"),
                    "far_records": int(last.get("far_records", 0)),
                    "peak_source": rp["source"] + ": random u32 RED into 32 MB"}
        if b_ == "hbm":
            ach = algo_ / t_ / 1e9 if t_ > 0 else 0.0
            r = {"bound": "hbm", "kernel": st, "achieved": ach, "peak": pk["hbm_gbs"],
                 "unit": "GB/s", "frac": ach / pk["hbm_gbs"], "traffic": traffic_,
                 "algorithmic_bytes_per_launch": algo_ / nl_, "launches_per_step": nl_,
                 "avg_launch_ms": per_step[st] / nl_, "peak_source": pk["source"] + " hbm_gbs"}
        else:
            ach = algo_ / t_ / 1e12 if t_ > 0 else 0.0
            # int8 = 2x bf16 (nominal 4.5 vs 2.25 PFLOP/s); e2m1 (kind::mxf4) = 4x (9 vs 2.25)
            # the e2m1 / u8 levels mix (GAKCO_OPT_GRAM_FP4 per level): the peak is the
            # rate at which this MAC mix would run at the two nominal peaks
            macs = float(last.get("heavy_macs", 0) or 0)
            f4 = float(last.get("heavy_macs_fp4", 0) or 0) / macs if macs > 0 else 0.0
            ratio = 1.0 / (f4 / 4.0 + (1.0 - f4) / 2.0)
            peak_ = pk["bf16_tflops"] * ratio
            src_ = pk["source"] + " bf16_tflops x %.3g (e2m1 x4, int8 x2 nominal ratios, " \
                                  "weighted by the MAC mix)" % ratio
            if rp and rp.get("int8_tops") and rp.get("fp4_tflops"):
                # measured library GEMM peaks for the two operand types (cuBLASLt int8,
                # cuBLAS nvfp4), mixed by the MAC share
                peak_ = 1.0 / (f4 / rp["fp4_tflops"] + (1.0 - f4) / rp["int8_tops"])
                src_ = ("measured cuBLASLt int8 %.0f TOPS / nvfp4 %.0f TFLOPS "
                        "(profiles/peaks_r02.json), weighted by the MAC mix"
                        % (rp["int8_tops"], rp["fp4_tflops"]))
            r = {"bound": "tensor", "kernel": st, "achieved": ach, "peak": peak_,
                 "unit": "TFLOP/s", "frac": ach / peak_, "traffic": traffic_,
                 "algorithmic_ops_per_launch": algo_ / nl_, "launches_per_step": nl_,
                 "avg_launch_ms": per_step[st] / nl_, "e2m1_mac_share": round(f4, 4),
                 "peak_source": src_}
        if st in limiter:
            r["limiter"] = limiter[st]
        return r

    roof = roof_of(dom)
    # SURVEY §8(d) headline: encode + sort + segment against HBM at the algorithmic
    # floor of 38-44 B per masked key (encode write 8, one sort read + write 16,
    # segment read 8, triple write 6-12)
    ess_ms = sum(per_step.get(k_, 0.0) for k_ in ("encode", "sort", "segment"))
    keys_ = float(last["keys"])
    hbm_headline = None
    if ess_ms > 0:
        lo_, hi_ = 38.0 * keys_ / (ess_ms / 1e3) / 1e9, 44.0 * keys_ / (ess_ms / 1e3) / 1e9
        hbm_headline = {"floor_bytes_per_key": [38, 44], "keys": keys_,
                        "ms_encode_sort_segment": ess_ms,
                        "achieved_gbs": [lo_, hi_], "peak_gbs": pk["hbm_gbs"],
                        "frac": [lo_ / pk["hbm_gbs"], hi_ / pk["hbm_gbs"]],
                        "target_frac": 0.6,
                        "model_bytes_gbs": sum(model[k_][1] for k_ in ("encode", "sort", "segment")
                                               if model[k_][0] == "hbm") / (ess_ms / 1e3) / 1e9}
    roof["stage_times"] = ("single-stream profiling steps (pipeline off), CUDA events on the "
                           "launching stream; the timed steps overlap stages on two streams")
    others = {st: roof_of(st) for st in ("heavy", "sort", "light", "segment", "encode")
              if st in per_step and st != dom and per_step[st] > 0 and model[st][0] != "alu"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms_per_step,
           "step_ms_spread": {"min": min(step_ms), "median": statistics.median(step_ms),
                              "max": max(step_ms), "all": [round(x, 2) for x in step_ms],
                              "host_call_ms": [round(x, 1) for x in host_ms],
                              "host_accumulate_ms": [round(x, 1) for x in enq_ms],
                              "far_overflow_warps": far_ov}
           if step_ms else None,
           "kernel_matrix_seconds": ms_per_step / 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "config": config_dict(a.config, cfg, cp, masks, n, world),
           "roofline": roof, "roofline_other_stages": others, "stages": stages,
           "hbm_headline_encode_sort_segment": hbm_headline,
           "gpu_launches": int(launches),
           "clocks": clocks, "e2e": e2e, "k_only": k_only,
           "counters": {k: v for k, v in last.items() if not k.startswith("ms_")}}
    if world == 1 and not a.no_cpu_baseline:
        import oracle
        oracle.build()
        threads = os.cpu_count() or 1
        dt, frac, r, fixed = oracle_sample(cp, cfg, a.cpu_seconds, threads)
        out["cpu_baseline"] = {
            "value": masks * n / oracle_full_seconds(dt, frac, fixed), "unit": UNIT,
            "cores": threads, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"oracle rows [0,{r}) x all Y>=X ({100 * frac:.2f}% of the upper-triangle "
                      f"pair work, {dt:.1f} s incl. the {fixed:.1f} s K(X,X) pass), extrapolated to "
                      f"the full matrix by pair work"}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = args_()
    if a.impl == "ours" and a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        from paper_1704_07468_b200 import parallel
        sys.exit(parallel.launch(a.gpus, os.path.abspath(__file__), sys.argv[1:]))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
