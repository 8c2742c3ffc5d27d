"""Summarise an ncu --set full report (.ncu-rep) as markdown: launch metrics,
throughputs, occupancy, DRAM bytes, tensor-pipe activity, top SASS opcodes by
stall samples. Usage: python tools/ncu_summary.py report.ncu-rep [title]"""
import collections
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "No Eligible",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Instructions"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tc.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.sum", "lts__t_bytes.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = [f"## {title}", "", f"source: `{rep}` (ncu --set full --clock-control none)", ""]
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    if rows:
        h = rows[0]
        mi, vi, ui, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
        out.append(f"kernel: `{rows[1][ki][:120]}`")
        out += ["", "| metric | value |", "|---|---|"]
        seen = set()
        for r in rows[1:]:
            if r[mi] in WANT and r[mi] not in seen:
                seen.add(r[mi])
                out.append(f"| {r[mi]} | {r[vi]} {r[ui]} |")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) > 2:
        h, units, vals = raw[0], raw[1], raw[2]
        out += ["", "| raw counter | value |", "|---|---|"]
        for k in RAW:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {vals[i]} {units[i]} |")
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source=sass"))))
    if len(sass) > 2:
        h = sass[1]
        si, st, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        stall, inst = collections.Counter(), collections.Counter()
        for r in sass[2:]:
            if not r[si]:
                continue
            t = r[si].split()
            op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
            stall[op] += float(r[st] or 0)
            inst[op] += float(r[ie] or 0)
        ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
        out += ["", "| SASS opcode | stall samples | executed |", "|---|---|---|"]
        for op, v in stall.most_common(14):
            out.append(f"| {op} | {100 * v / ts:.1f}% | {100 * inst[op] / ti:.1f}% |")
    print("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
