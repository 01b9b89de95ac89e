"""profiles/<tag>_traffic.json from a round's ncu captures (bench.py's 'traffic'):
K5 per launch inside the decode graph (single-pass DRAM metrics, no cache flush),
K5 cold, K1 and the prefill from their --set full reports.
  python tools/make_traffic.py r1e"""
import csv
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import traffic  # noqa: E402

tag = sys.argv[1]
P = "profiles"
U = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "B": 1, "KB": 1e3, "MB": 1e6}
rows = [r for r in csv.reader(open(f"{P}/{tag}_k5_traffic.csv")) if len(r) > 10]
h = rows[0]
ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = {}
for r in rows[1:]:
    if r[mi].startswith("dram__bytes"):
        per[r[ii]] = per.get(r[ii], 0.0) + float(r[vi].replace(",", "")) * U[r[ui]]
pl = [per[k] for k in sorted(per, key=int)]
prev = sorted(f for f in os.listdir(P) if f.endswith("_traffic.json") and not f.startswith(tag))
old = json.load(open(f"{P}/{prev[-1]}")) if prev else {}
out = {
    "K5": {"bytes": statistics.median(pl), "per_launch_bytes": pl, "report": f"{P}/{tag}_k5_traffic.csv",
           "how": "ncu --graph-profiling node --cache-control none, launches 150-154 of the decode graph "
                  "(tools/k5_graph_run.py, bench inputs): the compressed cache is L2-resident between launches; "
                  "algorithmic bytes per launch 46.5 MB"},
    "K5_cold": {**traffic(f"{P}/{tag}_k5.ncu-rep"), "report": f"{P}/{tag}_k5.ncu-rep",
                "how": "ncu --set full, caches flushed by ncu before the launch"},
    "K1": {**traffic(f"{P}/{tag}_k1.ncu-rep"), "report": f"{P}/{tag}_k1.ncu-rep",
           "how": "ncu --set full, exact-mode K1 on tools/profile_step.py GEN=1 (generator inputs); "
                  "algorithmic: keys 194 MB + Q 17 MB"},
}
if os.path.exists(f"{P}/{tag}_prefill.ncu-rep"):
    out["prefill"] = {**traffic(f"{P}/{tag}_prefill.ncu-rep"), "report": f"{P}/{tag}_prefill.ncu-rep",
                      "how": "ncu --set full, vlc_prefill on 4 layers of the M7B shapes (tools/prefill_once.py)"}
for k in ("K3", "K4"):
    if k in old:
        out[k] = old[k]
json.dump(out, open(f"{P}/{tag}_traffic.json", "w"), indent=1)
print(json.dumps({k: (v["bytes"], v.get("duration_us")) for k, v in out.items()}))
