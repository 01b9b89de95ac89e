"""The C-ABI library: builds, loads without a GPU, exports every symbol of
include/vlc.h, and enforces its argument contracts before touching CUDA."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2410_23317_b200 import _lib
from paper_2410_23317_b200.errors import ValidationError


def header_symbols():
    text = open(os.path.join(ROOT, "include", "vlc.h")).read()
    return sorted(set(re.findall(r"\b(vlc_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == syms
    assert lib.vlc_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_threshold_matches_oracle():
    from oracle import oracle as O

    for p in (0.01, 0.001, 0.05, 0.3, 1e-6):
        assert np.float32(_lib.load().vlc_threshold_logit(p)) == O.threshold_logit(p)


@pytest.mark.parametrize("p", [0.0, 1.0, -0.5, 2.0])
def test_score_stats_rejects_bad_p_before_cuda(p):
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)
    rc = lib.vlc_score_stats(dummy, dummy, 1, 1, 64, 10, 10, 2, 8, p, 0.0, dummy, dummy, dummy, dummy,
                             None, None, 0, None)
    assert rc == _lib.VLC_EINVAL
    assert b"p:" in lib.vlc_last_error()
    with pytest.raises(ValidationError, match="p:"):
        _lib.check(rc)


def test_contract_errors_map_to_reference_types():
    lib = _lib.load()
    d = ctypes.c_void_p(16)
    rc = lib.vlc_allocate(d, 1, 4, 8, 8, 2, 10, 8, 10, 0.0, 0.01, 1.0, 0, d, d, d, d, d, d, d, d, None)
    assert rc == _lib.VLC_EINVAL and b"alpha" in lib.vlc_last_error()
    rc = lib.vlc_select(d, None, 4, 2, 2, 1, 10, 2, d, d, 1.5, d, d, None, None, None)
    assert rc == _lib.VLC_EINVAL and b"recent_window_frac" in lib.vlc_last_error()
    rc = lib.vlc_select_after_allocate(d, d, 4, 2, 2, 1, 10, 2, d, d, 0.1, d, d, None, None, None)
    assert rc == _lib.VLC_EINVAL and b"scores_in" in lib.vlc_last_error()
    rc = lib.vlc_decode_step(d, 64, d, d, 64, d, d, 10, d, d, 0, 1, 1, 1, 9, 64, 0.0, 0, d, None)
    assert rc == _lib.VLC_EUNSUPPORTED
    rc = lib.vlc_score_stats(d, d, 1, 1, 48, 10, 10, 2, 8, 0.01, 0.0, d, d, d, d, None, None, 0, None)
    assert rc == _lib.VLC_EUNSUPPORTED   # head_dim not 64 / 128 (callers zero-pad)
    rc = lib.vlc_score_stats(d, d, 1, 1, 64, 10, 9, 2, 8, 0.01, 0.0, d, d, d, d, None, None, 0, None)
    assert rc == _lib.VLC_EINVAL         # n_keys < q_base + window
    need = lib.vlc_score_exact_bytes(4, 2, 8, 100)
    assert need > 0 and lib.vlc_score_exact_bytes(4, 2, 8, 0) < 0
    ws = ctypes.c_void_p(256)
    rc = lib.vlc_score_stats(d, d, 4, 2, 64, 10, 10, 8, 2, 0.01, 0.0, d, d, d, d, None, ws, 16, None)
    assert rc == _lib.VLC_EINVAL and b"exact_ws" in lib.vlc_last_error()


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_23317_b200 import KernelError, streaming_stats, QueryWindow
    from paper_2410_23317_b200.trace import GenSpec, generate_trace

    tr, _ = generate_trace(GenSpec(1, 1, 1, 16, 32, 4, 1, 0))
    with pytest.raises(KernelError):
        streaming_stats(tr, 0, 0, QueryWindow(28, 32))
