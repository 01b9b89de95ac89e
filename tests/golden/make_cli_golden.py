"""Golden outputs of the reference CLI's `compress`:
allocation.json and kept_sets.json as cli.py:195-203 writes them, for a few
policy x budget choices on bf16-rounded generator traces (the values K1
consumes on the B200).  The trace itself is not stored: the package's
generator is bit-identical to the reference's (tests/test_oracle_golden.py),
so the test regenerates it from the spec.

Run here (where /root/reference is mounted):  python tests/golden/make_cli_golden.py
Writes tests/golden/cli_golden.json; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import io
import json
import os
import sys
import tempfile
from contextlib import redirect_stdout

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_eval_golden import rounded_trace  # noqa: E402
from make_golden import load_reference  # noqa: E402

SPECS = {
    # tau = 64 > --stats-window 50: the CLI measures gamma on the last 50 rows but
    # scores the post-vision tokens over all 64 (cli.py:169-176 vs scoring.py:127-130)
    "tau64": dict(num_layers=3, num_query_heads=8, num_kv_heads=2, head_dim=64, prompt_len=700,
                  post_vision_len=64, decode_len=4, seed=21),
    "tau32": dict(num_layers=2, num_query_heads=8, num_kv_heads=8, head_dim=64, prompt_len=400,
                  post_vision_len=32, decode_len=4, seed=22),
}
RUNS = [
    ("tau64", []),
    ("tau64", ["--policy", "h2o", "--budget", "uniform"]),
    ("tau64", ["--policy", "sliding", "--budget", "pyramid", "--sliding-window", "40"]),
    ("tau64", ["--policy", "streaming", "--alpha", "0.2", "--recent-frac", "0.25"]),
    ("tau32", ["--alpha", "0.05", "--stats-window", "16"]),
]


def main():
    vl = load_reference()
    from vlcache import cli

    out = {"specs": SPECS, "runs": []}
    with tempfile.TemporaryDirectory() as tmp:
        for name, spec in SPECS.items():
            vl.write_trace(rounded_trace(vl, spec), os.path.join(tmp, f"{name}.vlct"))
        for i, (name, extra) in enumerate(RUNS):
            od = os.path.join(tmp, f"out{i}")
            buf = io.StringIO()
            with redirect_stdout(buf):
                rc = cli.main(["compress", "--trace", os.path.join(tmp, f"{name}.vlct"), "--out-dir", od, *extra])
            assert rc == 0, rc
            out["runs"].append({"trace": name, "args": extra, "stdout": buf.getvalue(),
                                "allocation.json": open(os.path.join(od, "allocation.json")).read(),
                                "kept_sets.json": open(os.path.join(od, "kept_sets.json")).read()})
    with open(os.path.join(HERE, "cli_golden.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(out["runs"]), "runs")


if __name__ == "__main__":
    main()
