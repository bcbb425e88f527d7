"""ctypes binding of libharmoe.so (C ABI in include/harmoe.h).

The product path has no CPU fallback: if the shared library or a CUDA device is
missing, every entry point raises.  Status codes map to the reference's error
behaviour: HM_EINVAL -> ValueError (the reference raises ValueError for bad
input, e.g. policies.py:168-169), anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

HM_OK, HM_EINVAL, HM_ECUDA, HM_ENCCL, HM_ENOSPC = 0, 1, 2, 3, 4
HM_EPI_STORE, HM_EPI_RELU, HM_EPI_SWIGLU = 0, 1, 2
HM_LAYOUT_LOCAL, HM_LAYOUT_EP, HM_LAYOUT_EP_EXPERT = 0, 1, 2
HM_POLICY_NONE, HM_POLICY_REBALANCE, HM_POLICY_EVEN_SPLIT = 0, 1, 2

# HM_LIB_PATH: load a variant build of the same C ABI (kernel A/B experiments, tools/build_variant.sh)
LIB_PATH = os.environ.get("HM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libharmoe.so")

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64

# name -> argtypes (all return int status unless listed in _RESTYPE)
SIGNATURES = {
    "hm_version": [],
    "hm_last_error": [],
    "hm_num_sms": [],
    "hm_gemm_tile_m": [],
    "hm_gemm_resident_pairs": [_i32, _i32],
    "hm_router_topk": [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
    "hm_hist_scan": [_vp, _i32, _i32, _i32, _vp, _vp, _vp],
    "hm_schedule": [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "hm_rebalance": [_vp, _i32, _i32, _i32, _vp, _vp, _vp],
    "hm_schedule_batched": [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "hm_plan": [_vp, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32] + [_vp] * 11 + [_i32, _vp],
    "hm_dispatch_layout": [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp],
    "hm_permute": [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "hm_grouped_gemm": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _i32, _i32,
                        _vp, _vp, _vp],
    "hm_grouped_gemm_swap": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "hm_grouped_gemm_combine": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp,
                                _vp],
    "hm_fetch_expert": [_vp, _vp, ctypes.c_size_t, _vp, _i32, _vp],
    "hm_combine": [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp],
    "hm_ep_offsets": [_vp, _i32, _i32, _i32, _vp, _vp, _vp],
    "hm_dispatch_push": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "hm_plan_dispatch": [_vp, _vp, _i32, _i32, _i32, _i32, _i32] + [_vp] * 9 + [_i32, _vp, _vp, _vp, _vp],
    "hm_dispatch_push_ordered": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp],
    "hm_grouped_gemm_arrive": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp,
                               _vp, _i32, _vp],
    "hm_grouped_gemm_remote": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _i32,
                               _i32, _vp, _vp, _vp],
    "hm_fetch_experts": [_vp, _vp, _vp, _vp, ctypes.c_size_t, ctypes.c_size_t, _vp, _vp, _i32, _i32, _vp, _vp, _vp,
                         _i32, _i32, _i32, _vp],
    "hm_stream_signal": [ctypes.POINTER(ctypes.c_void_p), _i32, ctypes.c_uint32, _vp],
    "hm_stream_wait": [_vp, _i32, ctypes.c_uint32, _vp],
    "hm_debug_plan_phases": [_vp],
    "hm_ipc_get_handle": [_vp, _vp, ctypes.POINTER(ctypes.c_size_t)],
    "hm_ipc_open": [_vp, ctypes.POINTER(ctypes.c_void_p)],
    "hm_ipc_close": [_vp],
}
_RESTYPE = {"hm_last_error": ctypes.c_char_p}


class FetchPlan(ctypes.Structure):
    """hm_fetch_plan (include/harmoe.h): K6 fetch pairs inside a grouped-GEMM launch."""

    _fields_ = [("fetch", _vp), ("n_fetch", _vp), ("src_in", _vp), ("src_out", _vp), ("dst_in", _vp),
                ("dst_out", _vp), ("in_bytes", ctypes.c_uint64), ("out_bytes", ctypes.c_uint64),
                ("first_slot", _i32), ("n_slots", _i32), ("ready_in", _vp), ("ready_out", _vp), ("counters", _vp),
                ("n_counters", _i32), ("value", _i32), ("pairs", _i32), ("phase", _i32)]

_lib = None


class HarmoeError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and type the library.  Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise HarmoeError(
                f"libharmoe.so not found at {path}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            if os.environ.get("HM_LIB_PATH") and not hasattr(L, name):
                continue  # an older variant build (A/B diagnostics) may lack newer entry points
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == HM_OK:
        return
    msg = load().hm_last_error().decode(errors="replace")
    if rc == HM_EINVAL:
        raise ValueError(msg or what)
    raise HarmoeError(f"{what} failed (status {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
