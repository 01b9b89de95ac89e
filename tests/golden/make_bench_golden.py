"""Golden outputs of the reference's benchmark harness (bench.py) on bf16-rounded
generator traces: run_bench kept counts / memory accounting / report keys and the
compression pass's kept index sets for every policy x budget mode.
Run here:  python tests/golden/make_bench_golden.py  -> tests/golden/bench_golden.npz"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import bf16_round, load_reference  # noqa: E402

BASE = dict(prompt_len=320, n_output_tokens=4, num_layers=3, num_query_heads=4, num_kv_heads=2, head_dim=64,
            post_vision_len=64, stats_window=50, repeats=3, warmup=1, seed=5)
CASES = [("vlcache", "sparsity_aware", 0.1), ("h2o", "sparsity_aware", 0.1), ("sliding", "uniform", 0.2),
         ("streaming", "uniform", 0.1), ("vlcache", "uniform", 0.3), ("sliding", "sparsity_aware", 0.05)]
# (policy, budget, alpha, shape overrides): odd head dims, MHA, no post-vision rows
EXTRA = [("h2o", "uniform", 0.15, dict(head_dim=32, num_query_heads=2, num_kv_heads=2, post_vision_len=0)),
         ("sliding", "sparsity_aware", 0.1, dict(head_dim=96, post_vision_len=0, stats_window=40)),
         ("vlcache", "sparsity_aware", 0.25, dict(prompt_len=200, post_vision_len=24, stats_window=50))]


def main():
    vl = load_reference()
    from vlcache import bench as rb

    real_gen = rb.generate_trace

    def rounded(spec):
        tr, planted = real_gen(spec)
        return vl.AttentionTrace(header=tr.header, layout=tr.layout, queries=[bf16_round(x) for x in tr.queries],
                                 keys=[bf16_round(x) for x in tr.keys]), planted

    rb.generate_trace = rounded
    out, meta = {}, {}
    for i, (policy, budget, alpha, extra) in enumerate([c + ({},) for c in CASES] + EXTRA):
        spec = rb.BenchSpec(policy=policy, budget=budget, alpha=alpha, **{**BASE, **extra})
        rep = rb.run_bench(spec)
        out[f"c{i}_kept_counts"] = np.array(rep.kept_counts)
        out[f"c{i}_kv"] = np.array([rep.kv_bytes_full, rep.kv_bytes_compressed])
        trace, _ = rounded(spec.gen_spec())
        _, kept, _ = rb._compression_pass(trace, spec)
        for l, row in enumerate(kept):
            for kv, idx in enumerate(row):
                out[f"c{i}_kept_{l}_{kv}"] = np.asarray(idx)
        meta["report_keys"] = sorted(rep.to_dict())
        meta["estimate_bytes"] = rb.estimate_bytes(spec)
    np.savez_compressed(os.path.join(HERE, "bench_golden.npz"), **out)
    with open(os.path.join(HERE, "bench_golden.json"), "w") as f:
        json.dump({"base": BASE, "cases": [c + ({},) for c in CASES] + EXTRA, **meta}, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
