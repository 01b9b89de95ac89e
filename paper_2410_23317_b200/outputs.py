"""The compress step's on-disk outputs: the
allocation.json / kept_sets.json pair the reference CLI writes
(reference cli.py:163-213, payloads budget.py:56-66 and scoring.py:270-288),
produced here from the device path so a pipeline that consumed the CLI's files
can consume these unchanged.  (The CLI itself is out of scope; this is its
compress step as a library call.)
"""

from __future__ import annotations

import json
import os

from .attention import DEFAULT_P, DEFAULT_TILE
from .budget import BudgetConfig, allocate_pyramid, allocate_sparsity_aware, allocate_uniform, measure_gamma_mean
from .errors import ValidationError
from .scoring import EvictionConfig, ScoringConfig, compress_cache, policy_from_name
from .sparsity import SparsityConfig
from .trace import AttentionTrace

DEFAULT_STATS_WINDOW = 50   # reference cli.py / bench.py default stats window


def compress_outputs(trace: AttentionTrace, *, alpha: float = 0.1, p: float = DEFAULT_P, tile: int = DEFAULT_TILE,
                     policy: str = "vlcache", budget: str = "sparsity_aware", pyramid_decay: float = 0.5,
                     sliding_window: int = DEFAULT_STATS_WINDOW, fallback_window: int | None = None,
                     recent_frac: float = 0.10, stats_window: int = DEFAULT_STATS_WINDOW):
    """(allocation payload, kept-sets payload, stdout payload) of
    `vlcache compress` with these arguments (reference cli.py:163-213): gamma
    over the last min(tau, stats_window) rows, the chosen budget, the policy's
    kept sets -- all on the device."""
    h = trace.header
    sparsity_config = SparsityConfig(p=p, tile=tile)
    budget_config = BudgetConfig(alpha=alpha)
    if budget == "sparsity_aware":
        window_rows = min(h.post_vision_len, stats_window) if h.post_vision_len >= 1 else None
        gamma_mean = measure_gamma_mean(trace, sparsity_config, budget_config, window_rows=window_rows)
        allocation = allocate_sparsity_aware(gamma_mean, alpha, h.prompt_len, budget_config)
    elif budget == "uniform":
        allocation = allocate_uniform(alpha, h.num_layers, h.prompt_len, budget_config)
    elif budget == "pyramid":
        allocation = allocate_pyramid(alpha, h.num_layers, h.prompt_len, pyramid_decay, budget_config)
    else:
        raise ValidationError(f"budget: must be sparsity_aware, uniform or pyramid, got {budget!r}")
    if policy == "vlcache" and h.post_vision_len < 1 and fallback_window is None:
        raise ValidationError("--fallback-window: required for the vlcache policy on a trace with tau = 0")
    pol = policy_from_name(policy, sliding_window=sliding_window, fallback_window=fallback_window)
    result = compress_cache(trace, allocation, pol, eviction=EvictionConfig(recent_window_frac=recent_frac),
                            config=ScoringConfig(p=p, tile=tile))
    alloc_payload = {
        "alpha": allocation.alpha,
        "prompt_len": allocation.prompt_len,
        "requested_total": allocation.requested_total,
        "realized_total": allocation.realized_total,
        "layers": allocation.to_rows(),
    }
    stdout = {"requested_total": allocation.requested_total, "realized_total": allocation.realized_total,
              "kept_counts": [int(c) for c in allocation.kept_counts]}
    return alloc_payload, result.to_summary(), stdout


def write_compress_outputs(out_dir, trace: AttentionTrace, **kwargs) -> dict:
    """Write allocation.json and kept_sets.json exactly as the reference CLI
    does (cli.py:195-203: json.dumps(indent=2) + newline); returns the stdout
    payload the CLI prints."""
    alloc, kept, stdout = compress_outputs(trace, **kwargs)
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "allocation.json"), "w") as f:
        f.write(json.dumps(alloc, indent=2) + "\n")
    with open(os.path.join(out_dir, "kept_sets.json"), "w") as f:
        f.write(json.dumps(kept, indent=2) + "\n")
    return stdout
