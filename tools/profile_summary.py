"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/profile_summary.py --launches gpurun_out/launches.csv \
        --report gpurun_out/prof.ncu-rep --tag r01_dna --config dna

Writes profiles/<tag>_launches.md (per-kernel launch count, summed device time
and share of the step, from the `--metrics gpu__time_duration.sum` pass) and
profiles/<tag>_ncu.md (per-launch duration, DRAM bytes, throughputs from the
`--set full` capture), and merges per-stage DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = {"encode_kernel": "encode", "encode_win_kernel": "encode", "window_kernel": "encode",
         "radix_hist_kernel": "sort", "radix_scatter_kernel": "sort",
         "onesweep_kernel": "sort", "segment_kernel": "segment", "light_kernel": "light",
         "light_flush_kernel": "light", "light_flush_perm_kernel": "light",
         "best_partner_kernel": "light", "best_union_kernel": "light", "uf_roots_kernel": "light",
         "gram_kernel": "heavy", "gram2_kernel": "heavy", "gram4_kernel": "heavy",
         "fill_reset_kernel": "heavy", "build_dense_kernel": "dense",
         "build_dense2_kernel": "dense", "build_dense3_kernel": "dense",
         "fill_round_kernel": "dense", "epilogue_kernel": "epilogue", "kdiag_kernel": "epilogue",
         "diag_closed_form_kernel": "light", "gmer_index_kernel": "encode",
         "check_codes_kernel": "encode", "bk_pass_kernel": "encode", "bk_colscan_kernel": "sort",
         "bk_bscan_kernel": "sort", "bk_group_kernel": "segment",
         "radix_scatter2_kernel": "sort", "hist_scan_kernel": "sort", "seq16_kernel": "sort",
         "symbol_hist_kernel": "encode", "thresh_union_kernel": "light",
         "light_flush_rect_kernel": "light", "fill_reset4_kernel": "heavy",
         "trie_root_kernel": "encode", "window_build_kernel": "dense", "window_round_kernel": "dense",
         "window_reset_kernel": "heavy", "window_flush_kernel": "light",
         "tp_hist_kernel": "sort", "tp_scatter_kernel": "sort", "segment_rag_kernel": "segment",
         "far_add_kernel": "far", "far_gate_kernel": "far", "far_reset_kernel": "far", "fill_u32_kernel": "sort", "pack_upper_kernel": "exchange",
         "diag_kernel": "exchange", "epilogue_packed_kernel": "epilogue",
         "kdiag_rect_kernel": "epilogue", "leaf_kernel": "segment", "far_warm_kernel": "far",
         "far_offsets_kernel": "far", "far_scan_kernel": "far", "cluster_roots_kernel": "light",
         "relabel_keys_kernel": "light", "relabel_perm_kernel": "light"}


def short(name):
    n = name.strip()
    if n.startswith("void "):
        n = n[5:]
    n = n.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    cut = min([i for i in (n.find("<"), n.find("(")) if i >= 0] or [len(n)])
    return n[:cut].split("::")[-1]


def launches(path, tag, out_dir):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[i:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.OrderedDict()
    total = 0.0
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[ui]
        us = (v / 1e3 if unit in ("ns", "nsecond") else
              v * 1e3 if unit in ("ms", "msecond") else v)
        k = short(r[ki])
        c = per.setdefault(k, [0, 0.0])
        c[0] += 1
        c[1] += us
        total += us
    lines = [f"# {tag}: kernel launch list (ncu gpu__time_duration.sum, --clock-control none)",
             "", "Cold-cache, serialised replay: compare SHARES, not absolute times.", "",
             "| kernel | stage | launches | sum (us) | share |", "|---|---|---|---|---|"]
    for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {STAGE.get(k, 'torch/other')} | {n} | {us:.1f} | "
                     f"{100 * us / total:.1f}% |")
    lines.append(f"| **total** | | {sum(n for n, _ in per.values())} | {total:.1f} | 100% |")
    with open(os.path.join(out_dir, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return per


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__registers_per_thread"]


def report(paths, tag, config, out_dir):
    if isinstance(paths, str):
        paths = [paths]
    lines, traffic = None, {}
    for path in paths:
        lines, traffic = _report_one(path, tag, lines, traffic)
    with open(os.path.join(out_dir, f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(out_dir, "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt.setdefault(config, {})
    for st, v in traffic.items():
        allt[config][st] = {"dram_bytes_per_launch_mean": sum(v) / len(v), "launches": len(v),
                            "source": tag}
    json.dump(allt, open(tp, "w"), indent=1)


_SCALE = {"nsecond": ("us", 1e-3), "usecond": ("us", 1.0), "msecond": ("us", 1e3),
          "second": ("us", 1e6), "byte": ("MB", 1e-6), "Kbyte": ("MB", 1e-3),
          "Mbyte": ("MB", 1.0), "Gbyte": ("MB", 1e3), "ns": ("us", 1e-3), "us": ("us", 1.0),
          "ms": ("us", 1e3), "s": ("us", 1e6)}


def _report_one(path, tag, lines, traffic):
    # values normalised per report (ncu picks a unit per report): times in us, bytes in MB
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [m for m in METRICS if m in idx]

    def unit(m):
        u = units[idx[m]]
        return _SCALE[u][0] if u in _SCALE else u

    def val(r, m):
        u = units[idx[m]]
        try:
            return f"{float(r[idx[m]]) * _SCALE[u][1]:.6g}" if u in _SCALE else r[idx[m]]
        except ValueError:
            return r[idx[m]]

    if lines is None:
        lines = [f"# {tag}: ncu --set full --clock-control none captures (per launch; "
                 "cold caches: compare shares and counters, not absolute times)", "",
                 "| kernel | " + " | ".join(f"{m.split('.')[0]} [{unit(m)}]" for m in cols) + " |",
                 "|---|" + "---|" * len(cols)]
    for r in rows[2:]:
        k = short(r[idx["Kernel Name"]])
        lines.append(f"| {k} | " + " | ".join(val(r, m) for m in cols) + " |")
        try:
            rb = float(val(r, "dram__bytes_read.sum")) * 1e6
            wb = float(val(r, "dram__bytes_write.sum")) * 1e6
            traffic.setdefault(STAGE.get(k, k), []).append(rb + wb)
        except (KeyError, ValueError):
            pass
    return lines, traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report", action="append")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="dna")
    a = ap.parse_args()
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag, out)
    if a.report:
        report(a.report, a.tag, a.config, out)


if __name__ == "__main__":
    main()
