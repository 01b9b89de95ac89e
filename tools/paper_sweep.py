"""The paper's efficiency sweep (compression overhead, prefill
"speedup", decode and end-to-end speedups at 10 % KV, 100 output tokens) run
through the reference-shaped harness (paper_2410_23317_b200.run_bench) at
LLaVA-1.6-Mistral-7B shapes on one B200.  Prints one JSON row per prompt length.
  python tools/paper_sweep.py [1024,2048,4096,8192,16384] [batch]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_23317_b200 as V  # noqa: E402

lens = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,2048,4096,8192,16384").split(",")]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for m in lens:
    spec = V.BenchSpec(prompt_len=m, batch_size=batch, n_output_tokens=100, alpha=0.1, num_layers=32,
                       num_query_heads=32, num_kv_heads=8, head_dim=128, post_vision_len=64, stats_window=50,
                       repeats=3, warmup=1, max_bytes=200 * 1024**3)
    r = V.run_bench(spec)
    print(json.dumps({"prompt_len": m, "batch": batch, "stats_overhead_ms": r.stats_overhead_time_s * 1e3,
                      "prefill_ms": r.prefill_time_s * 1e3, "decode_full_ms": r.decode_time_full_s * 1e3,
                      "decode_compressed_ms": r.decode_time_compressed_s * 1e3,
                      "prefill_speedup": r.prefill_speedup, "decode_speedup": r.decode_speedup,
                      "end_to_end_speedup": r.end_to_end_speedup, "kept_mean": sum(r.kept_counts) / len(r.kept_counts)}),
          flush=True)
