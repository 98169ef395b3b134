"""Summarise ncu reports: python tools/ncu_summary.py rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Cluster Size", "Dynamic Shared Memory Per Block",
        "Issue Slots Busy", "Mem Busy", "Max Bandwidth", "L2 Compression Success Rate", "Elapsed Cycles", "SM Frequency",
        "DRAM Frequency"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]


def run(args):
    return subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    print("==", rep)
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details"]))))
    if rows:
        h = rows[0]
        ki, ni, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        print("  kernel:", rows[1][ki][:100])
        seen = set()
        for r in rows[1:]:
            if r[ni] in KEEP and r[ni] not in seen:
                seen.add(r[ni])
                print(f"  {r[ni]:36s} {r[vi]:>14s} {r[ui]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw"]))))
    if raw:
        h = raw[0]
        for m in RAW:
            matches = [i for i, x in enumerate(h) if x == m]
            for i in matches:
                print(f"  {m:70s} {raw[2][i]:>14s} {raw[1][i]}")
