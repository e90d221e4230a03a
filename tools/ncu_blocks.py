#!/usr/bin/env python3
"""Hottest straight-line SASS runs of one kernel in an ncu report (runs of
consecutive instructions with the same execution count = basic blocks):

  python tools/ncu_blocks.py report.ncu-rep firsthit [--top 30] [--dump A-B]

Prints each block's instruction count, executions and share of the
kernel's executed warp instructions; --dump prints the SASS of a range.
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess


def sass_rows(report: str, kernel: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Instructions Executed" in r)
    ia, src = hdr.index("Instructions Executed"), hdr.index("Source")
    data = [r for r in rows if len(r) > ia and r[ia].isdigit()]
    # a report with several launches of the kernel repeats the listing: keep the first
    n = len(data)
    for k in (2, 3, 4):
        if n % k == 0 and all(data[i][src] == data[i + n // k][src] for i in range(0, n // k, max(1, n // 200))):
            data = data[: n // k]
            break
    return [(int(r[ia]), r[src].strip()) for r in data]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--dump", help="print SASS rows A-B")
    a = ap.parse_args()
    rows = sass_rows(a.report, a.kernel)
    tot = sum(c for c, _ in rows)
    if a.dump:
        lo, hi = (int(x) for x in a.dump.split("-"))
        for i in range(lo, min(hi + 1, len(rows))):
            print(f"{i:5d} {rows[i][0]:9d}  {rows[i][1][:100]}")
        return
    runs = []
    for i, (c, _) in enumerate(rows):
        if runs and runs[-1][2] == c and runs[-1][1] == i - 1:
            runs[-1][1] = i
        else:
            runs.append([i, i, c])
    print(f"total warp instructions {tot:.4g} over {len(rows)} SASS rows")
    for lo, hi, c in sorted(runs, key=lambda r: -(r[1] - r[0] + 1) * r[2])[: a.top]:
        n = hi - lo + 1
        print(f"{lo:5d}-{hi:5d} n={n:4d} exec={c:9d} share={100.0 * n * c / tot:5.2f}%  {rows[lo][1][:48]}")


if __name__ == "__main__":
    main()
