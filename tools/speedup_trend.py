"""Decode speedup vs prompt length through run_bench (the reference's criterion-8
setting: default BenchSpec, batch 1), a few times, to see the run-to-run spread."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_23317_b200 as V  # noqa: E402

for rep in range(3):
    for r in (3, 7):
        sp = [V.run_bench(V.BenchSpec(prompt_len=m, repeats=r)).decode_speedup for m in (2048, 8192, 32768)]
        print(r, [round(x, 2) for x in sp], flush=True)
