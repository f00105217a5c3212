"""The sm100 backend module: the reference backend protocol
(NAME, WHEEL_PERIOD, build_divisor_arrays, logprime_states, sieve_logprime,
sieve_naive, apply_block, finalize_recursion — _native.pyx / pure.py) served
by the GPU through the C ABI.  Same argument meaning, same in-place mutation
of acc/dnext/ynext, same return values and error behaviour.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _lib

NAME = "sm100"
WHEEL_PERIOD = 13860


def _load():
    _lib.lib()


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def build_divisor_arrays(cap):
    """Constants for all divisors 1..cap as (magic, shift, scheme) arrays (_native.pyx:32-68)."""
    L = _lib.require_device()
    cap = int(cap)
    magic = np.zeros(cap + 1, np.uint64)
    shift = np.zeros(cap + 1, np.uint8)
    scheme = np.zeros(cap + 1, np.uint8)
    _lib.check(L.mt_build_divisor_arrays(cap, _lib.ptr(magic), _lib.ptr(shift), _lib.ptr(scheme)))
    return magic, shift, scheme


def logprime_states(y1, y2, primes, logs, wheel):
    """Pre-classification 8-bit accumulator states (_native.pyx:113-124)."""
    L = _lib.require_device()
    y1, y2 = int(y1), int(y2)
    p, lg, w = _c(primes, np.uint64), _c(logs, np.uint8), _c(wheel, np.uint8)
    out = np.empty(y2 - y1 + 1, np.uint8)
    _lib.check(L.mt_logprime_states(y1, y2, _lib.ptr(p), _lib.ptr(lg), len(p), _lib.ptr(w), _lib.ptr(out)))
    return out


def sieve_logprime(y1, y2, primes, logs, wheel):
    """Moebius values over [y1, y2] via the 8-bit log-prime sieve; y1 >= 2 (_native.pyx:127-160)."""
    L = _lib.require_device()
    y1, y2 = int(y1), int(y2)
    p, lg, w = _c(primes, np.uint64), _c(logs, np.uint8), _c(wheel, np.uint8)
    out = np.empty(y2 - y1 + 1, np.int8)
    _lib.check(L.mt_sieve_logprime(y1, y2, _lib.ptr(p), _lib.ptr(lg), len(p), _lib.ptr(w), _lib.ptr(out)))
    return out


def sieve_naive(y1, y2, primes):
    """Moebius values over [y1, y2] (_native.pyx:163-206 semantics)."""
    L = _lib.require_device()
    y1, y2 = int(y1), int(y2)
    p = _c(primes, np.uint64)
    out = np.empty(y2 - y1 + 1, np.int8)
    _lib.check(L.mt_sieve_naive(y1, y2, _lib.ptr(p), len(p), _lib.ptr(out)))
    return out


def _inplace(a, dtype, name):
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous and a.flags.writeable):
        raise TypeError(f"{name} must be a writable C-contiguous {np.dtype(dtype).name} array")
    return a


def apply_block(acc, v, lo, xcut, mcut, dnext, ynext, y1, y2, mprefix, divtable=None):
    """Fold one sieved block's M values into every harmonic-array element
    (_native.pyx:227-310).  mprefix[i] must hold M(y1 + i).  acc, dnext and
    ynext are advanced in place.  Returns (counted_items, dense_items).
    `divtable` is accepted for signature compatibility and ignored."""
    L = _lib.require_device()
    acc = _inplace(acc, np.int64, "acc")
    dnext = _inplace(dnext, np.uint64, "dnext")
    ynext = _inplace(ynext, np.uint64, "ynext")
    v, lo, xcut, mcut = (_c(x, np.uint64) for x in (v, lo, xcut, mcut))
    mp = _c(mprefix, np.int64)
    y1, y2 = int(y1), int(y2)
    if len(mp) < y2 - y1 + 1:
        raise ValueError("mprefix shorter than the block")
    c, d = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _lib.check(L.mt_apply_block(len(acc), _lib.ptr(acc), _lib.ptr(v), _lib.ptr(lo), _lib.ptr(xcut),
                                _lib.ptr(mcut), _lib.ptr(dnext), _lib.ptr(ynext), y1, y2, _lib.ptr(mp),
                                ctypes.byref(c), ctypes.byref(d)))
    return c.value, d.value


def finalize_recursion(tails, D):
    """final[k-1] = 1 - tails[k-1] - sum_{d=2..D_k} final[k*d - 1] (_native.pyx:313-334)."""
    L = _lib.require_device()
    t, Dd = _c(tails, np.int64), _c(D, np.uint64)
    out = np.empty(len(t), np.int64)
    _lib.check(L.mt_finalize(len(t), _lib.ptr(t), _lib.ptr(Dd), _lib.ptr(out)))
    return out
