"""Summarise an ncu report: headline sections + top stall reasons + hottest SASS."""
import csv
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(path, top=20):
    rows = list(csv.reader(run([path, "--page", "details", "--csv"]).splitlines()))
    h = rows[0]
    si, mi, vi, ui = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    keep = {"GPU Speed Of Light Throughput", "Occupancy", "Scheduler Statistics", "Compute Workload Analysis",
            "Memory Workload Analysis", "Launch Statistics"}
    names = {"Duration", "DRAM Throughput", "Compute (SM) Throughput", "SM Active Cycles", "Elapsed Cycles",
             "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM", "Registers Per Thread",
             "Grid Size", "Block Size", "Eligible Warps Per Scheduler", "No Eligible", "Memory Throughput",
             "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "SM Frequency"}
    for r in rows[1:]:
        if r[si] in keep and r[mi] in names:
            print(f"{r[mi]:36s} {r[vi]} {r[ui]}")
    raw = list(csv.reader(run([path, "--page", "raw", "--csv"]).splitlines()))
    hdr, val = raw[0], raw[2]
    stalls = []
    for k, v in zip(hdr, val):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum"):
            print(f"{k:36s} {v}")
    tot = sum(s for s, _ in stalls) or 1
    print("stalls:", ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    src = list(csv.reader(run([path, "--page", "source", "--csv"]).splitlines()))
    hh = src[1]
    sI, wI = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    body = [r for r in src[2:] if len(r) > wI and r[wI].isdigit()]
    body.sort(key=lambda r: -int(r[wI]))
    for r in body[:top]:
        print(f"{r[wI]:>6} {r[sI][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
