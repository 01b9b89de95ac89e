"""Summarise an ncu --set full report: stall reasons, pipe use, and the SASS
lines with the most warp-stall samples (with their neighbourhood).
usage: python tools/ncu_hot.py report.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
st = []
for n, val in zip(h, v):
    try:
        x = float(val.replace(",", ""))
    except ValueError:
        continue
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        st.append((x, n[len("smsp__pcsamp_warps_issue_stalled_"):]))
    if n.startswith("sm__inst_executed_pipe_") and n.endswith("pct_of_peak_sustained_active") and x > 1:
        print(f"pipe {n[len('sm__inst_executed_pipe_'):].split('.')[0]:12s} {x:6.1f} %")
tot = sum(x for x, _ in st)
for x, n in sorted(st, reverse=True)[:10]:
    print(f"stall {n:28s} {100 * x / tot:5.1f} %")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ia, isrc, iss, ie = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                          "Instructions Executed"))
R = [r for r in rows[2:] if r[iss].isdigit()]
tot = sum(int(r[iss]) for r in R)
print("samples", tot)
for r in sorted(R, key=lambda r: -int(r[iss]))[:ntop]:
    print(f"{r[ia][-5:]} {int(r[iss]):6d} {100 * int(r[iss]) / tot:5.1f}% x{r[ie]:>9s}  {r[isrc][:80]}")
