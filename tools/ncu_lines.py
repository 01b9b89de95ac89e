"""Per-CUDA-source-line stall samples of an ncu report (needs -lineinfo and
--import-source at capture): python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    res, hdr, fname = {}, None, ""
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[0] == "-":
            continue
        try:
            n = int(r[4] or 0)
        except ValueError:
            continue
        if n:
            key = (fname, r[0])
            res[key] = (res.get(key, (0, ""))[0] + n, r[1])
    tot = sum(v[0] for v in res.values()) or 1
    for (f, ln), (n, src) in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{n:6d} {100 * n / tot:5.1f}%  {f}:{ln:<5} {src.strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
