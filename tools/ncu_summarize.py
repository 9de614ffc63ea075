"""Summaries of ncu output for profiles/ (run here, on the imported report / launch csv).

  python tools/ncu_summarize.py launches <launches.csv> <out.txt> "<command line>"
  python tools/ncu_summarize.py full <report.ncu-rep> <out.json>
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed.sum": "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "regs_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct_peak",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_peak",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc_pipe_pct_peak",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_hmma_pct_peak",
    "sm__inst_executed_pipe_tc.sum": "tc_pipe_inst",
}


# to ns and bytes
SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path, out, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    with open(out, "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ (cold-cache, serialised launches)\n")
        f.write(f"command: {cmd}\n")
        f.write("kernel, launches, mean us, total us\n")
        for k, (n, t) in agg.items():
            f.write(f"{k}, {n}, {t / n:.1f}, {t:.1f}\n")


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()}
        for m, k in FULL_METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    d[k] = v
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(json.dumps(d))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3])
