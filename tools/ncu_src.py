"""Per-source-line warp-stall samples of an ncu report (read here, on the CPU box).

    python tools/ncu_src.py REPORT.ncu-rep [TOP]

Uses `ncu --page source --print-source cuda,sass`; prints the source lines with the
most warp-stall samples and their executed thread instructions."""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    res, fname, hdr = [], None, None
    tot = tinst = 0
    for r in csv.reader(out.splitlines()):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
            continue
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            ti = int(r[hdr.index("Thread Instructions Executed")])
        except ValueError:
            continue
        tot += s
        tinst += ti
        res.append((s, ti, fname, int(r[0]), r[1].strip()[:96]))
    res.sort(reverse=True)
    print(f"total samples {tot}, thread instructions {tinst / 1e6:.1f}M")
    for s, ti, f, ln, src in res[:top]:
        print(f"{100 * s / max(tot, 1):5.1f}% {ti / 1e6:8.2f}M  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
