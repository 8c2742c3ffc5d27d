"""Extract the counters the bench's roofline object cites from an ncu --set full
report of ONE kernel launch, as JSON (committed under profiles/ and read by
bench.py for roofline.traffic).

usage: python tools/ncu_counters.py REPORT.ncu-rep KERNEL_NAME "capture command" ["config"] > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_sectors.sum": "l2_sectors",
    "gpu__time_duration.sum": "duration",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed.sum.per_cycle_active": "ipc_per_sm_sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
}
SCALE = {"byte": 1, "":1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "us": 1e-6, "ms": 1e-3,
         "ns": 1e-9, "s": 1, "%": 1, "inst/cycle": 1}


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    # the last launch whose kernel name matches (reports may hold several
    # kernels / launches; later launches are past the warm-up)
    ki = h.index("Kernel Name") if "Kernel Name" in h else None
    match = [r for r in rows[2:] if ki is None or r[ki].startswith(kernel)]
    if not match:
        sys.exit(f"no launch of {kernel} in {rep}")
    vals = match[-1]
    res = {"kernel": kernel, "report": rep, "capture": cmd}
    if len(sys.argv) > 4:
        res["config"] = sys.argv[4]
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            v = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
            res[name] = v
    if "dram_read_bytes" in res and "dram_write_bytes" in res:
        res["dram_bytes"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    if "l2_sectors" in res:
        res["l2_bytes"] = res["l2_sectors"] * 32
        if "duration" in res:
            res["l2_gbs"] = res["l2_bytes"] / res["duration"] / 1e9
    if "dram_bytes" in res and "duration" in res:
        res["dram_gbs"] = res["dram_bytes"] / res["duration"] / 1e9
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
