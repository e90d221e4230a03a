#!/usr/bin/env python3
"""Summarise an ncu report (read here, no GPU): per kernel duration,
DRAM traffic, occupancy, issue and pipe utilisation; writes the per-launch
DRAM traffic used by bench.py's roofline.traffic to profiles/raycast_traffic.json.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json profiles/raycast_traffic.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
    # texture-path evidence (VC_SAMPLER_TEXTURE): texture data pipe and
    # filter wavefronts, L1TEX throughput, L2 hit rate of texture traffic
    "l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_tex_pipe_pct",
    "l1tex__f_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_filter_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_lsu_pipe_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_throughput_pct",
    "lts__average_t_sector_hit_rate_srcunit_tex_realtime.pct": "l2_hit_pct_tex_unit",
}


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
         "nsecond": 1.0, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9}


def to_float(v, unit=""):
    try:
        return float(v.replace(",", "")) * SCALE.get(unit, 1.0)
    except Exception:
        return None


def main():
    rep = sys.argv[1]
    out_json = None
    if "--json" in sys.argv:
        out_json = sys.argv[sys.argv.index("--json") + 1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    per = defaultdict(list)
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("<")[0]
        rec = {}
        for m, k in METRICS.items():
            # some columns carry a section prefix ("SM_A.TriageCompute.<metric>")
            for col in [i for i, h in enumerate(head) if h == m] + \
                    [i for i, h in enumerate(head) if h.endswith("." + m)]:
                v = to_float(r[col], units[col])
                if v is not None:
                    rec[k] = v
                    break
        per[short].append(rec)
    summary = {}
    for k, recs in per.items():
        agg = {}
        for key in recs[0]:
            vals = [x[key] for x in recs if x.get(key) is not None]
            agg[key] = sum(vals) / len(vals) if vals else None
        if agg.get("dram_read_bytes") is not None and agg.get("dram_write_bytes") is not None:
            agg["dram_bytes_per_launch"] = agg["dram_read_bytes"] + agg["dram_write_bytes"]
        agg["launches"] = len(recs)
        summary[k] = agg
    for k, v in summary.items():
        print(k, json.dumps({a: (round(b, 3) if isinstance(b, float) else b) for a, b in v.items()}))
    if out_json:
        with open(out_json, "w") as f:
            json.dump({"source": rep, "note": "ncu --set full, --cache-control all (cold caches), per launch",
                       **{("vc::" + k): v for k, v in summary.items()}}, f, indent=1)


if __name__ == "__main__":
    main()
