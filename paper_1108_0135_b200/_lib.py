"""ctypes binding of the C ABI in include/mertens_sm100.h.

The shared library ``libmertens_sm100.so`` (built in-tree by
``paper_1108_0135_b200.build.build()``) is the only compute path: there is no
CPU fallback.  A missing library raises ImportError; a missing GPU raises
DeviceError at the first compute call.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ContractViolationError, DeviceError, ResourceLimitError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MT_LIB") or os.path.join(HERE, "libmertens_sm100.so")

MT_OK, MT_ERR_RESOURCE, MT_ERR_CONTRACT, MT_ERR_CUDA, MT_ERR_VALUE, MT_ERR_OVERFLOW = range(6)

_u64 = ctypes.c_uint64
_pu64 = ctypes.POINTER(ctypes.c_uint64)
_pi64 = ctypes.POINTER(ctypes.c_int64)


class MtJob(ctypes.Structure):
    _fields_ = [
        ("n_targets", ctypes.c_uint32),
        ("n_lo", _pu64),
        ("n_hi", _pu64),
        ("u", _u64),
        ("cap_c_lo", _u64),
        ("cap_c_hi", _u64),
        ("cap_small", _u64),
        ("q_budget_bytes", _u64),
        ("seg_log2_head", ctypes.c_uint32),
        ("seg_log2_tail", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("shard_rank", ctypes.c_uint32),
        ("shard_world", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("stream", ctypes.c_void_p),
    ]


MT_FLAG_FORCE_WIDE, MT_FLAG_FORCE_SLOWDIV, MT_FLAG_TIMING, MT_FLAG_CAP32 = 1, 2, 4, 8
KERNEL_CLASSES = ("sieve_tile", "sieve_large", "counted", "dwin", "dsparse", "qgather", "other", "unused")


class MtStats(ctypes.Structure):
    _fields_ = [(f, _u64) for f in (
        "blocks", "counted_items", "dense_items", "divtable_cap", "divtable_released_at",
        "r4_block_len", "head_end", "n_head_segments", "n_tail_segments", "kernel_launches",
        "max_mcut", "windowed_items", "qgather_items", "q_entries")] + [
        (f, ctypes.c_double) for f in (
            "ms_total", "ms_sieve_head", "ms_update_head", "ms_sieve_tail", "ms_qgather",
            "ms_finalize", "ms_counted_kernel", "ms_dense_kernel")] + [
        ("m_head", ctypes.c_int64), ("tail_total", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double * 8), ("kernel_count", _u64 * 8),
        ("tail_seg_begin", _u64), ("tail_seg_end", _u64), ("ms_setup", ctypes.c_double),
        ("head_cells", _u64), ("tail_cells", _u64)]


class MtResult(ctypes.Structure):
    _fields_ = [
        ("finals", _pi64),
        ("cap_m_out", _pi64),
        ("small_m_out", _pi64),
        ("acc_out", _pu64),
        ("stats", MtStats),
    ]


_lib = None


def lib():
    """Load (once) and return the engine library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.mt_last_error.restype = ctypes.c_char_p
    L.mt_abi_version.restype = ctypes.c_int
    L.mt_device_count.restype = ctypes.c_int
    vp = ctypes.c_void_p
    sigs = {
        "mt_set_device": [ctypes.c_int],
        "mt_sieve_logprime": [_u64, _u64, vp, vp, _u64, vp, vp],
        "mt_logprime_states": [_u64, _u64, vp, vp, _u64, vp, vp],
        "mt_sieve_naive": [_u64, _u64, vp, _u64, vp],
        "mt_apply_block": [_u64, vp, vp, vp, vp, vp, vp, vp, _u64, _u64, vp, _pu64, _pu64],
        "mt_finalize": [_u64, vp, vp, vp],
        "mt_build_divisor_arrays": [_u64, vp, vp, vp],
        "mt_mertens_range": [_u64, _u64, vp],
        "mt_mertens_at": [vp, _u64, vp],
        "mt_sieve_fast": [_u64, _u64, vp, vp],
        "mt_sieve_bench": [_u64, _u64, _u64, vp],
        "mt_sieve_bench2": [_u64, _u64, _u64, ctypes.c_int, vp],
        "mt_sieve_odd": [_u64, _u64, vp],
        "mt_sieve_wheel": [_u64, _u64, ctypes.c_int, vp],
        "mt_udiv128_batch": [vp, vp, vp, _u64, vp, vp],
        "mt_trim_device_memory": [],
        "mt_q_batch": [vp, vp, vp, _u64, ctypes.c_double, ctypes.c_double, _u64, vp],
        "mt_q_points": [vp, vp, vp, _u64, vp, _u64, vp],
        "mt_run": [ctypes.POINTER(MtJob), ctypes.POINTER(MtResult)],
        "mt_plan_create": [ctypes.POINTER(MtJob), ctypes.POINTER(ctypes.c_void_p)],
        "mt_plan_sieve_update": [vp, _pi64, _pi64],
        "mt_plan_sieve_step": [vp, _u64, ctypes.POINTER(ctypes.c_int), _pi64, _pi64],
        "mt_plan_checkpoint": [vp, ctypes.c_char_p],
        "mt_plan_restore": [vp, ctypes.c_char_p],
        "mt_plan_tail_offset": [vp, ctypes.c_int64],
        "mt_plan_q_slice": [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p), _pu64],
        "mt_plan_acc": [vp, ctypes.POINTER(ctypes.c_void_p), _pu64],
        "mt_plan_cap_window": [vp, ctypes.POINTER(ctypes.c_void_p), _pu64],
        "mt_plan_gather": [vp],
        "mt_plan_resolve": [vp, ctypes.POINTER(MtResult)],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.mt_plan_destroy.argtypes = [vp]
    L.mt_plan_destroy.restype = None
    if L.mt_abi_version() != 2:
        raise ImportError(f"{LIB_PATH}: ABI version {L.mt_abi_version()} != 2 (rebuild)")
    _lib = L
    return L


def require_device():
    L = lib()
    if L.mt_device_count() < 1:
        raise DeviceError("no CUDA device visible: the sm_100a engine has no CPU fallback")
    return L


def check(rc: int):
    """Map an ABI return code onto the reference's exception classes."""
    if rc == MT_OK:
        return
    msg = lib().mt_last_error().decode(errors="replace")
    if rc == MT_ERR_RESOURCE:
        raise ResourceLimitError(msg)
    if rc == MT_ERR_CONTRACT:
        raise ContractViolationError(msg)
    if rc == MT_ERR_VALUE:
        raise ValueError(msg)
    if rc == MT_ERR_OVERFLOW:
        raise OverflowError(msg)
    raise DeviceError(msg or f"engine error {rc}")


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


EXPORTED_SYMBOLS = (
    "mt_last_error", "mt_abi_version", "mt_device_count", "mt_set_device",
    "mt_sieve_logprime", "mt_logprime_states", "mt_sieve_naive", "mt_apply_block",
    "mt_finalize", "mt_build_divisor_arrays", "mt_mertens_range", "mt_mertens_at", "mt_sieve_fast", "mt_sieve_odd", "mt_sieve_wheel", "mt_sieve_bench",
    "mt_sieve_bench2", "mt_udiv128_batch", "mt_trim_device_memory", "mt_q_batch", "mt_q_points", "mt_run",
    "mt_plan_create", "mt_plan_sieve_update", "mt_plan_sieve_step", "mt_plan_checkpoint", "mt_plan_restore",
    "mt_plan_tail_offset", "mt_plan_q_slice", "mt_plan_cap_window", "mt_plan_acc",
    "mt_plan_gather", "mt_plan_resolve", "mt_plan_destroy",
)


def stats_dict(st) -> dict:
    """Flatten an MtStats into plain Python values (per-class kernel timings keyed by name)."""
    out = {}
    for f, _ in MtStats._fields_:
        v = getattr(st, f)
        if f in ("kernel_ms", "kernel_count"):
            out[f] = {KERNEL_CLASSES[i]: v[i] for i in range(7)}
        else:
            out[f] = v
    return out
