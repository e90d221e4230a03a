#!/usr/bin/env python3
"""Executed warp-instructions and stall samples per SASS opcode of one kernel
in an ncu report (development tool).

  python tools/ncu_opmix.py REPORT.ncu-rep KERNEL_REGEX [--top 30]
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + a.kernel], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ii, si, ti = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Thread Instructions Executed")
    inst = collections.Counter()
    stall = collections.Counter()
    thr = collections.Counter()
    for r in rows:
        if len(r) <= ii or not r[0].startswith("0x"):
            continue
        src = r[1].strip()
        src = re.sub(r"^@!?U?P\w+\s+", "", src)
        op = src.split()[0] if src else "?"
        inst[op] += float(r[ii] or 0)
        stall[op] += float(r[si] or 0)
        thr[op] += float(r[ti] or 0)
    ti_ = sum(inst.values()) or 1
    ts = sum(stall.values()) or 1
    print(f"total warp inst {ti_:.3e} thread inst {sum(thr.values()):.3e} stall samples {ts:.0f}")
    for op, n in inst.most_common(a.top):
        print(f"{n / ti_ * 100:5.1f}% inst {stall[op] / ts * 100:5.1f}% stall  {op}")


if __name__ == "__main__":
    main()
