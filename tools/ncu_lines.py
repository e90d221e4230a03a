#!/usr/bin/env python3
"""Per-source-line hot spots of one kernel in an ncu report (development tool).

  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top 40]

Reads `ncu -i --page source --print-source cuda,sass --csv` and prints the
source lines ranked by warp-level instructions executed, with their share of
stall samples and the average active threads.
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + a.kernel], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    lines = {}
    fname = "?"
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")] or 0)
            thr = float(r[hdr.index("Thread Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        e = lines.setdefault(key, [0.0, 0.0, 0.0, r[1]])
        e[0] += inst
        e[1] += thr
        e[2] += st
    ti = sum(v[0] for v in lines.values()) or 1
    ts = sum(v[2] for v in lines.values()) or 1
    print(f"total warp inst {ti:.3e}  stall samples {ts:.0f}")
    for (f, ln), (i, t, s, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"{i / ti * 100:5.1f}% inst {s / ts * 100:5.1f}% stall thr/inst {t / max(i, 1):4.1f}  "
              f"{f}:{ln}  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
