"""Executed warp instructions and stall samples per CUDA source line of an ncu
report captured with --import-source (cuda,sass view):
python tools/ncu_lines_inst.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=45):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, res = "", None, {}
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "File Name":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        try:
            ie = int(r[7] or 0)
            st = int(r[4] or 0)
        except ValueError:
            continue
        k = (fname, r[0])
        a = res.setdefault(k, [0, 0, r[1]])
        a[0] += ie
        a[1] += st
    tot = sum(v[0] for v in res.values()) or 1
    sst = sum(v[1] for v in res.values()) or 1
    print(f"total warp instructions {tot}, stall samples {sst}")
    for (f, ln), (ie, st, src) in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{ie:10d} {100 * ie / tot:5.1f}%  stall {100 * st / sst:5.1f}%  {f}:{ln:<5} {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
