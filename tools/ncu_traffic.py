"""dram read+write bytes per launch from ncu --set full reports -> JSON (bench.py 'traffic')."""
import csv
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def traffic(path):
    r = list(csv.reader(subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                                       capture_output=True, text=True).stdout.splitlines()))
    hdr, units, vals = r[0], r[1], r[2]
    out = {}
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(key)
        out[key] = float(vals[i].replace(",", "")) * UNIT[units[i]]
    i = hdr.index("gpu__time_duration.sum")
    out["duration_us"] = float(vals[i].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[units[i]]
    out["bytes"] = out["dram__bytes_read.sum"] + out["dram__bytes_write.sum"]
    return out


if __name__ == "__main__":
    res = {name: {**traffic(path), "report": path} for name, path in (a.split("=") for a in sys.argv[2:])}
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(res, indent=1))
