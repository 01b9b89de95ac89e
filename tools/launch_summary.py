"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[vi]:
            agg[r[ki]].append(float(r[vi].replace(",", "")) / 1e3)   # ns -> us
    total = sum(sum(v) for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'mean us':>9s} {'total us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k[:70]:70s} {len(v):8d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {100*sum(v)/total:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
