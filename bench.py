"""Benchmark of the VL-Cache compress + compressed-decode hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--batch B]

One step = one pass of the path over one batch of synthetic prompts at the
LLaVA-1.6-Mistral-7B shapes of BASELINE.json configs[1]: 32 layers, 32 Q / 8
KV heads, d = 128, m = 2,960 prompt tokens (16 text + 2,880 visual + 64
post-vision), tau = 64, alpha = 0.1, then 99 decode steps (100 output tokens,
reference bench.py:361).  Inputs come from the reference's own synthetic
generator (restated in paper_2410_23317_b200/trace.py), rounded to bf16.

value  = generated tokens / s over the whole step (compress + 99 decode steps),
         all ranks (weak scaling: each rank owns its own prompts).
e2e    = the same through the public API with host (pinned) inputs: H2D of the
         step's Q/K/V inside the timed region, D2H of the kept counts and the
         last decode output.
roofline: the dominant kernel of the step (K5 decode, HBM-bound, unless K1
         dominates): algorithmic bytes per launch / average launch duration in
         the timed region (the step's decode graph / 99), plus the same launch
         timed alone after an L2 flush ("cold").
cpu_baseline: the reference's own compiled kernels (oracle/_ref) or the C
         oracle, on a bounded sample of the same workload, all host threads.
--impl reference: that CPU arm as the headline line (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress ms/prompt + compressed-decode tokens/s @LLaVA-1.6-7B, 10% budget, % HBM roofline"
CFG = dict(layers=32, q_heads=32, kv_heads=8, head_dim=128, prompt_len=2960, tau=64, alpha=0.1,
           n_out=100, p=0.01, recent=0.10)
L2_FLUSH_BYTES = 512 << 20   # > 126 MB L2: written between timed steps


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["hbm_gbs"], pk["bf16_tflops"], "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback"


def m7b_config(batch, world):
    """The bench line's config for the M7B workload (both arms print it)."""
    return {"workload": "llava-1.6-mistral-7b shapes: L32 Hq32 Hkv8 d128 m2960 (16+2880+64) "
                        "tau64 alpha0.1, 99 decode steps", "global_batch": batch * world,
            "seq_len": CFG["prompt_len"], "parallelism": f"batch-sharded x{world} (no collective)",
            "l2": "flushed (512 MB write) before every timed step"}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` ("K1" / "K5") from the newest committed
    ncu --set full capture (profiles/r*_traffic.json, tools/ncu_traffic.py)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        data = json.load(f)
    if kernel not in data:
        return None, None
    return data[kernel]["bytes"], os.path.relpath(files[-1], ROOT)


def synth_inputs(batch, seed0, w, layers=None):
    """bf16-rounded host arrays [B, L, H, rows, d] from the reference generator
    (q_win holds the last w prompt rows; w = prompt_len keeps them all)."""
    from paper_2410_23317_b200.trace import GenSpec, iter_layers, round_to_bf16, synthesize_values

    c = CFG
    qw, qd, ks, vs = [], [], [], []
    for b in range(batch):
        spec = GenSpec(num_layers=layers or c["layers"], num_query_heads=c["q_heads"], num_kv_heads=c["kv_heads"],
                       head_dim=c["head_dim"], prompt_len=c["prompt_len"], post_vision_len=c["tau"],
                       decode_len=c["n_out"] - 1, seed=seed0 + b)
        k_l, qw_l, qd_l = [], [], []
        for k, q in iter_layers(spec, keep_prompt_rows=w):
            k_l.append(round_to_bf16(k))
            q = round_to_bf16(q)
            qw_l.append(q[:, :w])
            qd_l.append(q[:, w:])
        ks.append(np.stack(k_l))
        qw.append(np.stack(qw_l))
        qd.append(np.stack(qd_l))
        vs.append(np.stack([round_to_bf16(v) for v in synthesize_values(spec)]))
    return np.stack(qw), np.stack(qd), np.stack(ks), np.stack(vs)


class ClockSampler:
    """nvidia-smi style clock / throttle sampling (NVML) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - NVML optional
            self.nv = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):   # re-entrant: one sampler covers several timed regions
        self.stop.clear()
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU arm
def _as_layers(inputs):
    qw, qd, ks, vs = (x[0] for x in inputs)
    L = CFG["layers"]
    return tuple([np.ascontiguousarray(a[l], dtype=np.float32) for l in range(L)] for a in (qw, qd, ks, vs))


def cpu_path(threads, kernels_kind, layers_in):
    """One step of the reference CPU path over the WHOLE prompt (no sampling):
    the fused compression pass -- stats for every (layer, head) on `threads`
    host threads (the kernel releases the GIL, reference _core.pyx:234), the
    sparsity-aware allocation and the eviction (reference bench.py:245-323) --
    then the 99-step compressed decode (bench.py:356-372), its layers on
    `threads` threads.  Returns (compress_s, decode_s, kept_counts)."""
    from oracle import oracle as O

    c = CFG
    kern = O.Kernels(kernels_kind)
    qw_l, qd_l, k_l, v_l = layers_in
    g = c["q_heads"] // c["kv_heads"]
    t0 = time.perf_counter()
    res = O.compression_pass(qw_l, k_l, c["prompt_len"], g, p=c["p"], alpha=c["alpha"], recent_frac=c["recent"],
                             kernels=kern, threads=threads)
    t1 = time.perf_counter()
    O.decode_sequence(qd_l, k_l, v_l, res["kept"], c["prompt_len"], g, c["n_out"] - 1, kernels=kern,
                      collect=False, threads=threads)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, res["kept_counts"]


def cpu_extras(threads, kernels_kind, layers_in):
    """The rest of BASELINE.md's CPU plan, measured once: the compression pass
    on ONE thread, and the 99-step decode over the FULL (uncompressed) cache."""
    from oracle import oracle as O

    c = CFG
    kern = O.Kernels(kernels_kind)
    qw_l, qd_l, k_l, v_l = layers_in
    g = c["q_heads"] // c["kv_heads"]
    t0 = time.perf_counter()
    O.compression_pass(qw_l, k_l, c["prompt_len"], g, p=c["p"], alpha=c["alpha"], recent_frac=c["recent"],
                       kernels=kern, threads=1)
    t1 = time.perf_counter()
    O.decode_sequence(qd_l, k_l, v_l, None, c["prompt_len"], g, c["n_out"] - 1, kernels=kern, collect=False,
                      threads=threads)
    t2 = time.perf_counter()
    return {"compress_ms_per_prompt_1thread": (t1 - t0) * 1e3,
            "full_cache_decode_tokens_per_s": (c["n_out"] - 1) / (t2 - t1),
            "full_cache_decode_threads": threads}


def cpu_kind():
    from oracle import oracle as O

    return "reference" if O.ref_module() is not None else "port"


def cpu_env(threads, kind):
    return {"cores": threads, "kind": kind,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset"),
            "backend": "oracle/_ref: the reference's compiled _core.pyx" if kind == "reference"
            else "oracle/liboracle.so (C restatement)"}


def cpu_sample_desc(threads):
    return (f"the whole M7B prompt, no sampling: 32 layers x 32 heads of stats on {threads} threads + "
            f"sparsity-aware allocation + eviction (reference bench.py:245-323), then 99 compressed decode "
            f"steps (bench.py:356-372), layers on {threads} threads")


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    kind = cpu_kind()
    kk = "reference" if kind == "reference" else "oracle"
    layers_in = _as_layers(synth_inputs(1, 0, CFG["tau"]))
    for _ in range(args.warmup):
        cpu_path(threads, kk, layers_in)
    times = []
    for _ in range(args.steps):
        tc, td, _ = cpu_path(threads, kk, layers_in)
        times.append((tc, td))
    tc = statistics.median(t[0] for t in times)
    td = statistics.median(t[1] for t in times)
    step = statistics.median(t[0] + t[1] for t in times)
    value = (CFG["n_out"] - 1) / step
    extras = cpu_extras(threads, kk, layers_in)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference trace generator, bf16-rounded; seed = rank*B + b)",
        "config": m7b_config(1, 1),   # the b200 arm's config at N = 1 (same workload)
        "compress_ms_per_prompt": tc * 1e3, "decode_tokens_per_s": (CFG["n_out"] - 1) / td,
        "cpu_baseline": {"value": value, "unit": "tok/s", **cpu_env(threads, kind),
                         "sample": cpu_sample_desc(threads), **extras},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm
def decode_bytes_per_step(kept_counts, step, hkv=None, hq=None, d=None):
    """Algorithmic HBM bytes of one K5 launch: every cached K
    and V row of every slot read once (k + step + 1 rows), the appended row
    read + written, Q read, output written.  kept_counts: k_l per (prompt,
    layer); hkv / hq: the KV / query heads this rank decodes."""
    c = CFG
    d = d or c["head_dim"]
    hkv = hkv or c["kv_heads"]
    hq = hq or c["q_heads"]
    rows = hkv * (kept_counts + step + 1).sum()
    return (rows * d * 2 * 2 + kept_counts.size * hkv * d * 2 * 2 * 2
            + kept_counts.size * hq * d * (2 + 4))


def k1_flops(batch):
    c = CFG
    m, tau = c["prompt_len"], c["tau"]
    causal = tau * (m - tau) + tau * (tau + 1) // 2
    return 2 * c["head_dim"] * c["q_heads"] * causal * c["layers"] * batch


def k1_mufu_floor(batch, torch):
    """ex2 count of K1 (two per causal entry: row pass and column pass) over the
    device's SFU rate at its max SM clock: the epilogue's floor in microseconds."""
    c = CFG
    m, tau = c["prompt_len"], c["tau"]
    exps = 2 * (tau * (m - tau) + tau * (tau + 1) // 2) * c["q_heads"] * c["layers"] * batch
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    sms = props.multi_processor_count
    mhz = None
    try:
        import pynvml

        pynvml.nvmlInit()
        mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()),
                                               pynvml.NVML_CLOCK_SM)
    except Exception:  # noqa: BLE001
        mhz = 1965
    return {"exps": exps, "floor_us": exps / (sms * 16 * mhz * 1e6) * 1e6}


def k5_hbm_probe(batch, dev_inputs, shape1, hbm_peak, flush, torch, reps=5):
    """K5 where the compressed cache cannot live in L2: the same M7B prompt
    replicated `batch` times (the reference bench replicates one trace across
    its batch, bench.py:377) into distinct buffers -- `batch` x ~39 MB of cache
    per step, well above the 126 MB L2 -- then the 99-launch decode graph
    timed with CUDA events (L2 flushed before each replay).  Per launch:
    algorithmic bytes / (graph time / 99), the HBM-honest K5 figure."""
    from paper_2410_23317_b200.engine import Shape, VLCache

    c = CFG
    n_dec = c["n_out"] - 1
    rep = lambda t: t.expand(batch, *t.shape[1:]).contiguous()  # noqa: E731
    qw, qd, k, v = (rep(t[:1]) for t in dev_inputs)
    sh = Shape(batch, shape1.L, shape1.Hq, shape1.Hkv, shape1.d, shape1.m, shape1.w)
    eng = VLCache(sh, alpha=c["alpha"], p=c["p"], recent_frac=c["recent"], decode_steps=n_dec)
    eng.compress(qw, k, v)
    st = torch.cuda.current_stream()
    eng.decode(qd, k, v, graph=True)          # capture + warm
    times = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.decode(qd, k, v, graph=True)
        b.record(st)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    eng.check()
    counts = eng.kept_counts.cpu().numpy()
    by = float(np.mean([decode_bytes_per_step(counts, s_) for s_ in range(n_dec)]))
    launch_us = float(np.median(times)) * 1e3 / n_dec
    ach = by / (launch_us / 1e6) / 1e9
    traffic, tsrc = ncu_traffic("K5_b%d" % batch)
    del eng
    return {"batch": batch, "bytes_per_launch": by, "launch_us": launch_us, "achieved": ach, "peak": hbm_peak,
            "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic, "traffic_source": tsrc,
            "how": f"M7B prompt replicated x{batch} into distinct buffers ({by / 1e6:.0f} MB per launch > 126 MB L2), "
                   f"99-launch decode graph, median of {reps} replays, L2 flushed before each"}


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2410_23317_b200.engine import Shape, VLCache

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CFG
    B, n_dec = args.batch, c["n_out"] - 1
    qw, qd, ks, vs = synth_inputs(B, seed0=rank * B, w=c["tau"])
    dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
    d_qw, d_qd, d_k, d_v = dev(qw), dev(qd), dev(ks), dev(vs)
    shape = Shape(B, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"])
    eng = VLCache(shape, alpha=c["alpha"], p=c["p"], recent_frac=c["recent"], decode_steps=n_dec)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def step(timers=None):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timers is not None else None
        if e: e[0].record(st)
        eng.score_stats(d_qw, d_k)
        if e: e[1].record(st)
        eng.allocate(); eng.select(); eng.gather(d_k, d_v)
        if e: e[2].record(st)
        eng.decode(d_qd, d_k, d_v, graph=True)
        if e: e[3].record(st)
        if timers is not None:
            timers.append(e)

    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step([])
    torch.cuda.synchronize()
    eng.check()
    timers = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()   # L2 flush between timed steps (outside the events)
            step(timers)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    k1 = [t[0].elapsed_time(t[1]) for t in timers]
    k234 = [t[1].elapsed_time(t[2]) for t in timers]
    dec = [t[2].elapsed_time(t[3]) for t in timers]
    step_ms = float(np.mean([a + b + d for a, b, d in zip(k1, k234, dec)]))
    t_step = torch.tensor([step_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    step_ms = float(t_step.item())
    tokens = B * n_dec * world
    value = tokens / (step_ms / 1e3)

    # K5 per launch.  In the timed region each step's 99 K5 launches run as one
    # CUDA graph; their average duration is the decode time / 99 (events on the
    # launching stream around the graph).  Within a step the compressed cache
    # stays in L2 from launch to launch (L2 is flushed only between steps), so
    # ncu's DRAM traffic per launch (profiles/) is far below the algorithmic
    # bytes.  "cold" re-times every launch alone after an L2 flush: all bytes
    # from HBM, the kernel's pure-HBM figure.
    counts = eng.kept_counts.view(B, c["layers"]).cpu().numpy()
    eng.score_stats(d_qw, d_k); eng.allocate(); eng.select(); eng.gather(d_k, d_v)
    per = []
    # cold flush: the 512 MB write, then a 512 MB read, so L2 holds clean lines
    # only (a write alone leaves ~126 MB of dirty lines whose write-back would
    # be charged to the launch: +4 us, tools/k5_cold.py)
    rd = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.int64, device="cuda")
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s_ in range(n_dec):
        flush.zero_()
        sink.add_(rd.sum())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.decode_step(d_qd, d_k, d_v, s_)
        b.record(st)
        per.append((a, b))
    torch.cuda.synchronize()
    k5_cold_ms = [a.elapsed_time(b) for a, b in per]
    k5_bytes = [decode_bytes_per_step(counts.reshape(-1), s_) for s_ in range(n_dec)]
    hbm_peak, tc_peak, src = peaks()
    k5_cold_gbs = float(np.mean([by / (ms / 1e3) for by, ms in zip(k5_bytes, k5_cold_ms)])) / 1e9
    k1_ms = float(np.mean(k1))
    k1_tflops = k1_flops(B) / (k1_ms / 1e3) / 1e12
    dec_ms = float(np.mean(dec))
    k5_launch_us = dec_ms * 1e3 / n_dec
    k5_achieved = float(np.mean(k5_bytes)) / (k5_launch_us / 1e6) / 1e9
    if dec_ms >= k1_ms:
        traffic, tsrc = ncu_traffic("K5")
        roof = {"kernel": "K5 decode_step (99 launches per step, CUDA graph, timed region)", "bound": "hbm",
                "achieved": k5_achieved, "peak": hbm_peak, "unit": "GB/s", "frac": k5_achieved / hbm_peak,
                "traffic": traffic, "traffic_source": tsrc, "peak_source": src,
                "bytes_per_launch": float(np.mean(k5_bytes)), "launch_us": k5_launch_us,
                "l2_resident": True,
                "memory_level": "L2: the batch-1 compressed cache (~39 MB) stays in the 126 MB L2 between the "
                                "launches of a step, so this fraction is of L2-fed bytes, not HBM",
                "cold": {"launch_us": float(np.mean(k5_cold_ms)) * 1e3, "achieved": k5_cold_gbs,
                         "frac": k5_cold_gbs / hbm_peak,
                         "how": "each launch alone after a 512 MB L2 flush (write, then read: clean "
                                "lines only) -- all bytes from HBM"}}
        if args.hbm_batch > 1 and world == 1:
            roof["hbm"] = k5_hbm_probe(args.hbm_batch, (d_qw, d_qd, d_k, d_v), shape, hbm_peak, flush, torch)
    else:
        traffic, tsrc = ncu_traffic("K1")
        roof = {"kernel": "K1 score_stats", "bound": "tensor", "achieved": k1_tflops, "peak": tc_peak,
                "unit": "TFLOP/s", "frac": k1_tflops / tc_peak, "traffic": traffic, "traffic_source": tsrc,
                "peak_source": src, "flops_per_launch": k1_flops(B), "launch_us": k1_ms * 1e3}

    # e2e through the public API with host buffers (VLCache.run_from_host):
    # pinned host inputs in, kept counts + last decode output back to the host
    m = c["prompt_len"]
    hp = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).pin_memory()  # noqa: E731
    e_qw, e_qd = hp(qw), hp(qd)
    e_kp, e_vp = hp(ks[:, :, :, :m]), hp(vs[:, :, :, :m])
    e_kd, e_vd = hp(ks[:, :, :, m:m + n_dec]), hp(vs[:, :, :, m:m + n_dec])
    e2e_ms, h2d, d2h = [], 0, 0
    for i in range(max(3, args.warmup)):   # warm-up (untimed, unsampled)
        eng.run_from_host(e_qw, e_kp, e_vp, e_qd, e_kd, e_vd)
    torch.cuda.synchronize()
    with clk:   # the e2e timed region is sampled too
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            h_counts, h_out, copied = eng.run_from_host(e_qw, e_kp, e_vp, e_qd, e_kd, e_vd)
            b.record(st)
            torch.cuda.synchronize()
            h2d = copied + eng.zero_copy_bytes(h_counts)
            d2h = h_counts.numel() * 8 + h_out.numel() * 4
            e2e_ms.append(a.elapsed_time(b))
    t_e2e = torch.tensor([float(np.mean(e2e_ms))], device="cuda")
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = tokens / (float(t_e2e.item()) / 1e3)

    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference trace generator, bf16-rounded; seed = rank*B + b)",
        "config": m7b_config(B, world),
        "compress_ms_per_prompt": (float(np.mean(k1)) + float(np.mean(k234))) / B,
        "k1_ms": k1_ms, "k234_ms": float(np.mean(k234)), "decode_ms_99_steps": dec_ms,
        "decode_tokens_per_s": B * n_dec * world / (dec_ms / 1e3),
        "k1_tensor_tflops": k1_tflops, "k1_tensor_frac": k1_tflops / tc_peak,
        # K1's binding floor is its epilogue: two ex2 per causal entry on the SFU
        # (16 lanes / SM / clock on sm_100); exact mode's fix-ups included in k1_ms
        "k1_mufu": k1_mufu_floor(B, torch),
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "VLCache.run_from_host: pinned host inputs; values pulled zero-copy (kept rows only)"},
        "gpu_launches": args.steps * (9 + n_dec),   # zeroing, K1, 4 exact fix-ups, K2, K3, K4, 99 x K5
        "clocks": clk.summary(),
        "kept_tokens_per_layer_mean": float(counts.mean()),
        # exact mode's counters of the last timed compress and its runtime margin check
        "exact_mode": eng.exact_stats(),
    }
    line["k1_mufu"]["frac"] = line["k1_mufu"]["floor_us"] / (k1_ms * 1e3)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        kind = cpu_kind()
        kk = "reference" if kind == "reference" else "oracle"
        layers_in = _as_layers((qw[:1], qd[:1], ks[:1], vs[:1]))
        runs = [cpu_path(threads, kk, layers_in) for _ in range(max(1, args.cpu_reps))]
        tc = statistics.median(r[0] for r in runs)
        td = statistics.median(r[1] for r in runs)
        ts = statistics.median(r[0] + r[1] for r in runs)
        line["cpu_baseline"] = {"value": n_dec / ts, "unit": "tok/s", **cpu_env(threads, kind),
                                "sample": cpu_sample_desc(threads) + f"; median of {len(runs)} runs",
                                "compress_ms_per_prompt": tc * 1e3, "decode_tokens_per_s": n_dec / td,
                                "same_budgets_as_gpu": bool(np.array_equal(runs[0][2], counts[0]))}
        if not args.no_cpu_extras:
            line["cpu_baseline"].update(cpu_extras(threads, kk, layers_in))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- sharded configurations
SHARDED = {
    # BASELINE.json configs[2]: LLaVA-1.6-34B shapes, batch 4, KV heads sharded across ranks
    "y34b": dict(layers=60, q_heads=56, kv_heads=8, head_dim=128, prompt_len=10320, tau=64, batch=4,
                 shard="heads", workload="llava-1.6-34b shapes: L60 Hq56 Hkv8 d128 m10320 (16+5x2048+64) "
                                           "tau64 alpha0.1 batch4, 99 decode steps"),
    # BASELINE.json configs[3]: 32 frames x 196 tokens on Mistral-7B shapes, batch 8 sharded by prompt
    "vid": dict(layers=32, q_heads=32, kv_heads=8, head_dim=128, prompt_len=6352, tau=64, batch=8,
                shard="batch", workload="video prompt 32 frames x 196 tokens on mistral-7b shapes: L32 Hq32 "
                                        "Hkv8 d128 m6352 (16+6272+64) tau64 alpha0.1 batch8, 99 decode steps"),
}


def run_sharded_arm(args):
    """One BASELINE configuration whose global batch is fixed (strong scaling)
    and sharded over the ranks as SURVEY.md section 8e prescribes:
      y34b -- KV heads split across ranks (parallel.HeadShard); K1, K3-K5 are
              local and K2 needs every head's below counts, so each step
              all-reduces the int64 [B, L, Hq] counts over NCCL inside the
              timed region (engine.compress -> parallel.exchange_head_counts);
      vid  -- prompts split across ranks, no collective.
    Inputs follow the reference generator's recipe, drawn on the device
    (trace.device_synthetic); timing as the default arm (L2 flushed before each
    step, CUDA events on the launching stream, max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2410_23317_b200.engine import Shape, VLCache
    from paper_2410_23317_b200.parallel import HeadShard, shard_batch
    from paper_2410_23317_b200.trace import GenSpec, device_synthetic

    cf = SHARDED[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L, hq, hkv, d, m, tau, B = (cf[k] for k in ("layers", "q_heads", "kv_heads", "head_dim", "prompt_len", "tau",
                                                "batch"))
    g = hq // hkv
    n_dec = CFG["n_out"] - 1
    spec = GenSpec(num_layers=L, num_query_heads=hq, num_kv_heads=hkv, head_dim=d, prompt_len=m, post_vision_len=tau,
                   decode_len=n_dec, seed=0)
    shard = None
    if cf["shard"] == "heads":
        shard = HeadShard(rank, world, hkv, g)
        (klo, khi), (qlo, qhi) = shard.kv_range, shard.q_range
        qw, qd, k, v = device_synthetic(spec, B, tau)
        qw, qd = qw[:, :, qlo:qhi].contiguous(), qd[:, :, qlo:qhi].contiguous()
        k, v = k[:, :, klo:khi].contiguous(), v[:, :, klo:khi].contiguous()
        torch.cuda.empty_cache()
        b_loc, hq_loc, hkv_loc = B, qhi - qlo, khi - klo
        par = f"kv-head-sharded x{world}: {hkv_loc} KV / {hq_loc} query heads per rank, NCCL int64 all-reduce " \
              f"of the [B, L, Hq] below counts in every step" if world > 1 else "1 rank (all heads)"
    else:
        lo, hi = shard_batch(B, rank, world)
        qw, qd, k, v = device_synthetic(spec, hi - lo, tau, seed=1000 + lo)
        b_loc, hq_loc, hkv_loc = hi - lo, hq, hkv
        par = f"batch-sharded x{world}: prompts [{lo}, {hi}) on rank {rank}, no collective"
    eng = VLCache(Shape(b_loc, L, hq_loc, hkv_loc, d, m, tau), alpha=CFG["alpha"], p=CFG["p"],
                  recent_frac=CFG["recent"], decode_steps=n_dec, head_shard=shard)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def step(timers=None):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(st)
        eng.compress(qw, k, v)
        e[1].record(st)
        eng.decode(qd, k, v, graph=True)
        e[2].record(st)
        if timers is not None:
            timers.append(e)

    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    eng.check()
    timers = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            step(timers)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    comp = float(np.mean([t[0].elapsed_time(t[1]) for t in timers]))
    dec = float(np.mean([t[1].elapsed_time(t[2]) for t in timers]))
    t = torch.tensor([comp + dec, comp, dec], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, comp_max, dec_max = (float(x) for x in t.tolist())
    counts = eng.kept_counts.cpu().numpy()
    by = float(np.mean([decode_bytes_per_step(counts, s_, hkv_loc, hq_loc, d) for s_ in range(n_dec)]))
    launch_us = dec * 1e3 / n_dec
    hbm_peak, _, src = peaks()
    ach = by / (launch_us / 1e6) / 1e9
    tokens = B * n_dec
    line = {
        "metric": METRIC, "value": tokens / (step_ms / 1e3), "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: the reference generator's recipe drawn on the device (trace.device_synthetic)",
        "config": {"workload": cf["workload"], "global_batch": B, "seq_len": m, "parallelism": par,
                   "l2": "flushed (512 MB write) before every timed step"},
        "compress_ms_per_prompt": comp_max / B * world if cf["shard"] == "batch" else comp_max / B,
        "compress_ms_step": comp_max, "decode_ms_99_steps": dec_max,
        "decode_tokens_per_s": tokens / (dec_max / 1e3),
        "roofline": {"kernel": "K5 decode_step (rank 0, 99 launches per step, CUDA graph, timed region)",
                     "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": None, "peak_source": src, "bytes_per_launch": by, "launch_us": launch_us,
                     "l2_resident": by < 60e6},
        "gpu_launches": args.steps * (9 + n_dec),
        "clocks": clk.summary(),
        "exact_mode": eng.exact_stats(),
        "kept_tokens_per_layer_mean": float(counts.mean()),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--batch", type=int, default=1, help="prompts per GPU")
    ap.add_argument("--config", choices=("m7b", *SHARDED), default="m7b",
                    help="m7b: BASELINE configs[1], one prompt per GPU (weak scaling, the default line); "
                         "y34b / vid: configs[2] / [3] with their global batch sharded (strong scaling)")
    ap.add_argument("--hbm-batch", type=int, default=8, help="batch of the HBM-resident K5 probe (0: skip)")
    ap.add_argument("--cpu-reps", type=int, default=3, help="runs of the CPU baseline (median)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-extras", action="store_true", help="skip the 1-thread / full-cache CPU legs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.config != "m7b":
        run_sharded_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
