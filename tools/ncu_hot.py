"""Summaries of an ncu report (read here, on the CPU box).

    python tools/ncu_hot.py REPORT.ncu-rep [--kernel REGEX] [--launch I] [--top N]

Prints per-launch duration / DRAM bytes / throughputs, then the hottest SASS
instructions (warp-stall samples) of the selected launch.
"""
import argparse
import csv
import io
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--launch", type=int, default=-1)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--no-sass", action="store_true")
    a = ap.parse_args()
    filt = ["-k", "regex:" + a.kernel] if a.kernel else []
    raw = ncu(["-i", a.report, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)] + filt)
    rows = list(csv.reader(io.StringIO(raw)))
    if not rows:
        print("no data")
        return
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    units = rows[1]
    print("launch | kernel | " + " | ".join(f"{m.split('.')[0]}[{units[idx[m]]}]" for m in METRICS
                                              if m in idx))
    data = rows[2:]
    for i, r in enumerate(data):
        print(i, "|", r[idx["Kernel Name"]][:40], "|",
              " | ".join(r[idx[m]] for m in METRICS if m in idx))
    if a.no_sass or not data:
        return
    sel = data[a.launch]
    kid = sel[idx["ID"]] if "ID" in idx else None
    src = ncu(["-i", a.report, "--page", "source", "--csv", "--print-source", "sass"] + filt +
              (["--launch-skip", str(a.launch if a.launch >= 0 else len(data) + a.launch),
                "--launch-count", "1"]))
    srows = list(csv.reader(io.StringIO(src)))
    h2 = None
    out = []
    for r in srows:
        if len(r) > 3 and r[0] == "Address":
            h2 = {h: i for i, h in enumerate(r)}
            continue
        if h2 and len(r) > 3:
            try:
                out.append((int(r[h2["Warp Stall Sampling (All Samples)"]]), r[h2["Source"]].strip()))
            except (ValueError, KeyError):
                pass
    tot = sum(s for s, _ in out) or 1
    print(f"\nlaunch {a.launch} (ID {kid}): {tot} samples; top instructions:")
    for s, ins in sorted(out, reverse=True)[:a.top]:
        print(f"{100.0 * s / tot:5.1f}%  {ins}")


if __name__ == "__main__":
    main()
