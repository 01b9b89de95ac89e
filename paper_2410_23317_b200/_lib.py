"""ctypes binding of the C-ABI in include/vlc.h (libvlc_b200.so).

The same binding a non-Python host would write.  There is
no fallback: if the library or a CUDA device is missing, every entry point
raises ``KernelError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import KernelError, ValidationError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VLC_LIB_PATH") or os.path.join(_PKG, "libvlc_b200.so")   # override: tuning runs

VLC_OK, VLC_EINVAL, VLC_EUNSUPPORTED, VLC_ECUDA = 0, -1, -2, -3

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F64 = ctypes.c_double

# name -> (restype, argtypes); mirrors include/vlc.h
_SIGNATURES = {
    "vlc_abi_version": (ctypes.c_int, []),
    "vlc_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "vlc_last_error": (ctypes.c_char_p, []),
    "vlc_threshold_logit": (ctypes.c_float, [_F64]),
    "vlc_score_partials": (_I64, [_I64]),
    "vlc_score_exact_bytes": (_I64, [_I32, _I32, _I64, _I64]),
    "vlc_score_stats": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I64, _I64, _I64, _I64, _F64,
                                       _F64, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "vlc_score_stats_given": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I64, _I64, _I64, _I64, _F64, _F64,
                                             _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "vlc_allocate": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _I64, _I64, _I64, _I64, _F64, _F64,
                                    _F64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vlc_allocate_from_gamma": (ctypes.c_int, [_P, _I32, _I32, _I32, _I64, _F64, _F64, _F64, _I64,
                                               _P, _P, _P, _P, _P, _P, _P]),
    "vlc_select": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I32, _I64, _I64, _P, _P, _F64, _P, _P,
                                  _P, _P, _P]),
    "vlc_select_after_allocate": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I32, _I64, _I64, _P, _P, _F64, _P,
                                                 _P, _P, _P, _P]),
    "vlc_gather": (ctypes.c_int, [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "vlc_copy_2d": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "vlc_decode_step": (ctypes.c_int, [_P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _I32,
                                       _I32, _I32, _I32, _I32, _F64, _I32, _P, _P]),
    "vlc_prefill_ws_bytes": (_I64, [_I32, _I32, _I64]),
    "vlc_prefill": (ctypes.c_int, [_P, _I64, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I64, _F64, _P, _I64,
                                   _P, _P, _P, _P]),
    "vlc_attention_rows": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I64, _I64, _I64, _I64, _I64, _P,
                                          _F64, _I64, _I64, _I64, _P, _P]),
    "vlc_stats_f32": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _I64, _F64, _I64, _P, _P, _P, _P, _P, _P]),
    "vlc_decode_f32": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _I32, _P, _P, _P, _P]),
}

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises KernelError if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise KernelError(f"sm_100a extension not built: {LIB_PATH} (run __graft_entry__.build())")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - loader failure
            raise KernelError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's error types."""
    if rc == VLC_OK:
        return
    msg = load().vlc_last_error().decode(errors="replace")
    if rc in (VLC_EINVAL, VLC_EUNSUPPORTED):
        raise ValidationError(msg)
    raise KernelError(msg or f"vlc error {rc}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def require_cuda():
    """The CUDA path is the only path: fail loudly without a device."""
    import torch

    if not torch.cuda.is_available():
        raise KernelError("no CUDA device: the B200 path has no CPU fallback")
    load()
    return torch
