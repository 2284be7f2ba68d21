"""Summarize an .ncu-rep into a small text file (run where ncu is; keeps reports out of
the 64 MiB gpurun pull).  python tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Executed Ipc Active",
        "Avg. Active Threads Per Warp", "Executed Instructions", "DRAM Throughput",
        "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Block Limit Registers", "Waves Per SM", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
ids = h.index("ID") if "ID" in h else None
cur = None
for r in rows[1:]:
    key = (r[ids] if ids is not None else "", r[ki])
    if key != cur:
        cur = key
        print(f"== [{key[0]}] {r[ki][:160]}")
    if r[mi] in WANT:
        print(f"   {r[mi]:42s} {r[vi]} {r[ui]}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if raw:
    hh = raw[0]
    stall = [(i, n) for i, n in enumerate(hh) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    for r in raw[2:]:
        print(f"-- raw [{r[hh.index('ID')] if 'ID' in hh else ''}] {r[hh.index('Kernel Name')][:100]}")
        for m in RAW:
            if m in hh:
                print(f"   {m:52s} {r[hh.index(m)]}")
        st = sorted(((float(r[i].replace(',', '') or 0), n[34:]) for i, n in stall), reverse=True)[:8]
        print("   stalls(pc samples): " + ", ".join(f"{n}={int(v)}" for v, n in st))
