"""Per-CUDA-source-line totals of an ncu --set full report (needs -lineinfo):
python tools/ncu_lines.py rep.ncu-rep [top] [kernel-regex] -> stall samples and executed warp instructions per line."""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kf = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", *kf],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg = "?", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].strip().isdigit():
            continue
        try:
            s = float(r[4] or 0)
            i = float(r[7] or 0)
        except ValueError:
            continue
        agg.append((s, i, f"{fname}:{r[0]}", r[1].strip()[:90]))
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    print(f"total stall samples {ts:.0f}, warp instructions {ti:.4g}")
    for s, i, loc, src in sorted(agg, key=lambda a: -a[0])[:top]:
        print(f"{100 * s / ts:6.2f}% samples {100 * i / ti:6.2f}% inst  {loc:<22} {src}")


if __name__ == "__main__":
    main()
