#!/usr/bin/env python3
"""Per-kernel share of device time from an ncu launch list
(--metrics gpu__time_duration.sum --csv --log-file ...).

  python tools/launch_shares.py launches.csv "command line" > profiles/rNN_launch_shares.txt
"""
import csv
import sys
from collections import defaultdict


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "?"
    note = sys.argv[3] if len(sys.argv) > 3 else ("includes warm-up, the brute-force counting frames, the "
                                                  "profiled frames and the side measurements")
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    head = rows[0]
    kn, mv, unit = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        name = r[kn].split("(")[0][:60]
        scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[unit], 1.0)
        tot[name] += float(r[mv].replace(",", "")) * scale
        cnt[name] += 1
    all_ns = sum(tot.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none, command: {cmd}")
    print(f"(cold-cache, serialised launches; {note})")
    print(f"{'kernel':62s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"{name:62s} {cnt[name]:8d} {tot[name] / cnt[name] / 1e3:10.1f} {tot[name] / all_ns * 100:6.1f}%")
    step = {k: v for k, v in tot.items() if "firsthit_kernel" in k or "shade_kernel" in k}
    if step:
        s_ns = sum(step.values())
        print("share of the frame's two kernels: " +
              ", ".join(f"{k.split('<')[0].split()[-1]} {v / s_ns * 100:.1f}%" for k, v in step.items()))


if __name__ == "__main__":
    main()
