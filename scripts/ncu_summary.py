"""Summarise an exported ncu capture: key metrics + hottest SASS lines.
usage: python scripts/ncu_summary.py gpurun_out/prof_knn [top]"""
import csv, gzip, sys
base = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Block Limit Registers", "Block Limit Shared Mem", "SM Frequency",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Avg. Active Threads Per Warp", "Branch Instructions Ratio"]
rows = list(csv.reader(open(base + ".details.csv")))
h = rows[0]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:]:
    if r[mi] in want:
        print(f"{r[mi]:40s} {r[vi]:>14s} {r[ui]}")
try:
    raw = list(csv.reader(gzip.open(base + ".raw.csv.gz", "rt")))
    hdr, units, vals = raw[0], raw[1], raw[2]
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.sum",
            "sm__inst_executed_pipe_alu.sum", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.sum"]
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:75s} {vals[i]:>16s} {units[i]}")
except FileNotFoundError:
    pass
src = list(csv.reader(gzip.open(base + ".source.csv.gz", "rt")))
h = src[0]
print(h[:12])
def col(name):
    for i, c in enumerate(h):
        if c.strip() == name:
            return i
    return None
ci = col("Warp Stall Sampling (All Samples)")
ai = col("Address") or 0
si = col("Source")
if ci is not None:
    body = [r for r in src[1:] if len(r) > ci and r[ci].replace('.', '').isdigit()]
    tot = sum(float(r[ci]) for r in body) or 1
    body.sort(key=lambda r: -float(r[ci]))
    print("total samples", tot)
    for r in body[:top]:
        print(f"{float(r[ci])/tot*100:5.1f}%  {r[ai]:>6s}  {r[si][:110]}")
