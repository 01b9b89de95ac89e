"""The path at every BASELINE.json configuration that fits one B200, on the
reference generator's recipe drawn on the device (trace.device_synthetic; the
host generator needs ~20 GB of fp32 at Y34B -- oracle parity at these shapes
is tests/test_gpu_configs.py), K1 in exact mode, the L2 flushed (512 MB
write + read) before every timed call, SM clocks and throttle reasons sampled
by NVML during the timed calls:

  M7B    LLaVA-1.6-Mistral-7B shapes, batch 1            (the bench.py workload)
  Y34B   LLaVA-1.6-34B shapes (L60, Hq56, Hkv8), batch 4 x 5 images x 2K visual
  VID    32 frames x 196 tokens on 7B shapes, batch 8
  SWEEP  7B shapes at 16K context, alpha 1/5/10/20/100 %, plus the full cache:
         decode speedup of the compressed cache vs the full cache

Per config: compress ms/prompt (K1..K4), K1 TFLOP/s, decode us/step (99 steps,
one CUDA graph, the compressed cache L2-resident when it fits), algorithmic GB/s
of K5, generated tok/s.  Checks: every slot keeps exactly k_l ascending in-range
indices, and decode step 0 of 8 sampled slots against a float64 torch reference.

  python tools/configs_bench.py [--only Y34B,VID] [--out profiles/r1b_configs.json]
"""
import argparse

EXACT = True
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402
from paper_2410_23317_b200.trace import GenSpec, device_synthetic  # noqa: E402

N_DEC = 99
CONFIGS = {
    "M7B": dict(B=1, L=32, Hq=32, Hkv=8, d=128, m=2960, tau=64, alphas=[0.1]),
    "Y34B": dict(B=4, L=60, Hq=56, Hkv=8, d=128, m=16 + 5 * 2048 + 64, tau=64, alphas=[0.1]),
    "VID": dict(B=8, L=32, Hq=32, Hkv=8, d=128, m=16 + 32 * 196 + 64, tau=64, alphas=[0.1]),
    "SWEEP": dict(B=1, L=32, Hq=32, Hkv=8, d=128, m=16384, tau=64, alphas=[0.01, 0.05, 0.1, 0.2, 1.0, "full"]),
}


FLUSH = None
CLOCKS = None


def timed(fn, reps=5):
    global FLUSH
    if FLUSH is None:
        FLUSH = (torch.empty(512 << 20, dtype=torch.uint8, device="cuda"),
                 torch.ones(512 << 20, dtype=torch.uint8, device="cuda"), torch.zeros(1, device="cuda"))
    ts = []
    for _ in range(reps):
        FLUSH[0].zero_()
        FLUSH[2].add_(FLUSH[1][::4096].float().sum())   # then a read: no dirty lines left in L2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with CLOCKS:
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[1:]))


def inputs(c, seed):
    spec = GenSpec(num_layers=c["L"], num_query_heads=c["Hq"], num_kv_heads=c["Hkv"], head_dim=c["d"],
                   prompt_len=c["m"], post_vision_len=c["tau"], decode_len=N_DEC, seed=seed)
    qw, qd, k, v = device_synthetic(spec, c["B"], c["tau"])
    return qw, k, v, qd


def check(eng, c, qd, k, v):
    """Kept sets well formed; decode step 0 of sampled slots vs float64 torch."""
    s = eng.shape
    counts = eng.kept_counts.view(s.B, s.L).cpu().numpy()
    off = eng.kept_off.cpu().numpy()
    idx = eng.kept_idx[: int(off[-1])].cpu().numpy()
    for sl in range(s.slots):
        kk = idx[off[sl]:off[sl + 1]]
        kl = counts[sl // (s.L * s.Hkv), (sl // s.Hkv) % s.L]
        assert kk.size == kl and (np.diff(kk) > 0).all() and kk[0] >= 0 and kk[-1] < s.m, sl
    out = eng.decode_step(qd, k, v, 0).view(s.B, s.L, s.Hq, s.d)
    rng = np.random.default_rng(0)
    worst = 0.0
    for sl in rng.choice(s.slots, size=min(8, s.slots), replace=False):
        b, l, kv = sl // (s.L * s.Hkv), (sl // s.Hkv) % s.L, sl % s.Hkv
        rows = torch.from_numpy(np.append(idx[off[sl]:off[sl + 1]], s.m)).cuda()
        kk, vv = k[b, l, kv, rows].double(), v[b, l, kv, rows].double()
        q = qd[b, l, kv * s.G:(kv + 1) * s.G, 0].double()
        p = torch.softmax(q @ kk.T / math.sqrt(s.d), dim=-1)
        ref = p @ vv
        got = out[b, l, kv * s.G:(kv + 1) * s.G].double()
        worst = max(worst, float(((got - ref).abs() / (ref.abs() + 1e-3)).max()))
    assert worst < 1e-3, worst
    return worst


def run(name, c):
    res = []
    qw, k, v, qd = inputs(c, 0)
    shape = Shape(c["B"], c["L"], c["Hq"], c["Hkv"], c["d"], c["m"], c["tau"])
    causal = c["tau"] * (c["m"] - c["tau"]) + c["tau"] * (c["tau"] + 1) // 2
    flops = 2 * c["d"] * c["Hq"] * causal * c["L"] * c["B"]
    for alpha in c["alphas"]:
        full = alpha == "full"
        global CLOCKS
        CLOCKS = bench.ClockSampler(torch.cuda.current_device())
        eng = VLCache(shape, alpha=1.0 if full else alpha, decode_steps=N_DEC, exact=EXACT)
        if full:
            zeros = torch.zeros((c["B"], c["L"]), dtype=torch.float64, device="cuda")
            comp = lambda: (eng.score_stats(qw, k), eng.allocate_from_gamma(zeros), eng.select(),  # noqa: E731
                            eng.gather(k, v))
        else:
            comp = lambda: eng.compress(qw, k, v)  # noqa: E731
        t_k1 = timed(lambda: eng.score_stats(qw, k))
        t_comp = timed(comp)
        eng.check()
        worst = check(eng, c, qd, k, v)
        comp()
        eng.decode(qd, k, v, graph=True)   # capture
        t_dec = timed(lambda: (comp(), eng.decode(qd, k, v, graph=True))) - t_comp
        counts = eng.kept_counts.cpu().numpy().reshape(-1)
        rows = c["Hkv"] * (counts.sum() * N_DEC + counts.size * N_DEC * (N_DEC + 1) // 2)
        by = rows * c["d"] * 2 * 2
        r = {"config": name, "alpha": alpha, "B": c["B"], "L": c["L"], "Hq": c["Hq"], "Hkv": c["Hkv"],
             "m": c["m"], "kept_mean": float(counts.mean()), "compress_ms_per_prompt": t_comp / c["B"],
             "k1_ms": t_k1, "k1_tflops": flops / (t_k1 / 1e3) / 1e12, "decode_us_per_step": t_dec * 1e3 / N_DEC,
             "k5_gbs": by / N_DEC / (t_dec / 1e3 / N_DEC) / 1e9, "tok_s": c["B"] * N_DEC / ((t_comp + t_dec) / 1e3),
             "decode_tok_s": c["B"] * N_DEC / (t_dec / 1e3), "decode_rel_err_vs_f64": worst,
             "exact_mode": eng.exact_stats() if EXACT else None, "clocks": CLOCKS.summary()}
        print(json.dumps(r), flush=True)
        res.append(r)
        del eng
        torch.cuda.empty_cache()
    if name == "SWEEP":
        full = next(r for r in res if r["alpha"] == "full")
        for r in res:
            r["decode_speedup_vs_full"] = full["decode_us_per_step"] / r["decode_us_per_step"]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(CONFIGS))
    ap.add_argument("--out", default=None)
    ap.add_argument("--fp32", action="store_true", help="K1 with plain fp32 decisions (exact mode off)")
    args = ap.parse_args()
    global EXACT
    EXACT = not args.fp32
    allres = []
    for name in args.only.split(","):
        allres += run(name, CONFIGS[name])
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"device": torch.cuda.get_device_name(),
                       "inputs": "reference generator recipe drawn on the device (trace.device_synthetic), bf16",
                       "l2": "flushed (512 MB write + read) before every timed call",
                       "k1_decisions": "exact mode" if EXACT else "fp32 (exact mode off: random logits)",
                       "results": allres}, f, indent=1)


if __name__ == "__main__":
    main()
