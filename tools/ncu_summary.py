"""Summarise an ncu report (details page) into the handful of numbers we track."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "No Eligible",
        "Avg. Active Threads Per Warp"]


def summary(rep, kernel_filter=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if kernel_filter and kernel_filter not in d.get("Kernel Name", ""):
            continue
        if d["Metric Name"] in KEYS:
            res[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hdr, units, vals = rr[0], rr[1], rr[2]
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "smsp__inst_executed_pipe_fp64.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
                    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
                    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
                    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"):
            if key in hdr:
                k = hdr.index(key)
                res[key] = f"{vals[k]} {units[k]}".strip()
        # warp stall reasons (cycles stalled per issued instruction), largest first
        stalls = []
        for k, name in enumerate(hdr):
            if "issue_stalled" in name and name.endswith("_per_warp_active.pct"):
                try:
                    stalls.append((float(vals[k].replace(",", "")), name))
                except ValueError:
                    pass
        for v, name in sorted(stalls, reverse=True)[:6]:
            short = name.split("issue_stalled_")[1].replace("_per_warp_active.pct", "")
            res[f"stall {short}"] = f"{v:.1f} % of warp-active cycles"
    return res


if __name__ == "__main__":
    for k, v in summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None).items():
        print(f"{k}: {v}")
