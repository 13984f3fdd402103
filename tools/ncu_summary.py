"""Summarise `ncu --set full` captures into profiles/ncu_summary.json.

python tools/ncu_summary.py CLASS=path.ncu-rep[@i] [CLASS=path.ncu-rep ...] [--out profiles/ncu_summary.json]

@i selects the i-th captured launch of a report (default the first).

CLASS is the bench kernel class ("pass", "reopt", ...); bench.py reads
`dram_bytes_per_launch` of the dominant class as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_s",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__inst_executed.sum": "instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "dram__bytes.sum.per_second": "dram_bytes_per_s",
    "lts__t_bytes.sum.per_second": "l2_bytes_per_s",
    "l1tex__t_bytes.sum.per_second": "l1_bytes_per_s",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed":
        "tensor_pipe_elapsed_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active": "imma_pipe_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
SCALE = {"byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9,
         "Tbyte/second": 1e12, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}


def summarise(path):
    idx = 0
    if "@" in path:  # path@i: the i-th captured launch of the report
        path, i = path.rsplit("@", 1)
        idx = int(i)
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    d = {"kernel": vals[hdr.index("Kernel Name")], "source": os.path.basename(path)}
    for m, key in METRICS.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        d[key] = v * SCALE.get(units[i], 1.0)
    d["dram_bytes_per_launch"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
    if d.get("duration_s"):
        d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration_s"] / 1e9
    return d


def main():
    out = "profiles/ncu_summary.json"
    items = []
    for a in sys.argv[1:]:
        if a.startswith("--out="):
            out = a.split("=", 1)[1]
        elif "=" in a:
            items.append(a.split("=", 1))
    try:
        with open(out) as f:
            summary = json.load(f)
    except (OSError, ValueError):
        summary = {}
    for cls, path in items:
        summary[cls] = summarise(path)
        print(cls, json.dumps(summary[cls], indent=1))
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
