"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference exact-Mertens engine
(/root/reference/pkg/src/mertens/engine.py, sieve.py) driving either

* ``"c"``   — the plain-C restatement of the reference kernels
              (oracle/mertens_oracle.c -> oracle/liboracle_mertens.so), or
* ``"ref"`` — the reference's own compiled kernel module built by
              oracle/build_ref.sh into oracle/_ref/ (Cython -> C, unmodified).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / the timed CPU baseline.  The
product package (paper_1108_0135_b200) never imports anything under oracle/.

Each function cites the reference lines it restates.  The parameter formulas
(choose_u, HarmonicArray) are restated verbatim in semantics so that u, K and
every per-element split match the reference bit for bit.
"""

from __future__ import annotations

import ctypes
import importlib
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from math import isqrt, sqrt

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SENTINEL = np.uint64(2**64 - 1)
WHEEL_PERIOD = 13860
U64_PATH_BOUND = 4 * 10**18  # engine.py:45-47
DIRECT_CUTOFF = 1024  # engine.py:49


def ceil_sqrt(x: int) -> int:  # sieve.py:35-37
    s = isqrt(x)
    return s + (s * s < x)


# ----------------------------------------------------------------------------
# kernel backends
# ----------------------------------------------------------------------------

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_U64 = ctypes.c_uint64


class CKernels:
    """ctypes binding of oracle/liboracle_mertens.so (mirrors the backend
    module protocol of _kernels/__init__.py:15-44)."""

    NAME = "oracle-c"
    WHEEL_PERIOD = WHEEL_PERIOD

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle_mertens.so")
        if not os.path.exists(path):
            raise ImportError(f"oracle library missing: {path} (run `make -C oracle`)")
        L = ctypes.CDLL(path)
        L.o_logprime_states.argtypes = [_U64, _U64, _u64p, _u8p, _U64, _u8p, _u8p]
        L.o_sieve_logprime.argtypes = [_U64, _U64, _u64p, _u8p, _U64, _u8p, _u8p, _i8p]
        L.o_sieve_naive.argtypes = [_U64, _U64, _u64p, _U64, _i64p, _i8p]
        L.o_build_divisor_arrays.argtypes = [_U64, _u64p, _u8p, _u8p]
        L.o_apply_block.argtypes = [_U64, _i64p, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p,
                                    _U64, _U64, _i64p, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
        L.o_apply_block.restype = ctypes.c_int
        L.o_apply_block_wrap.argtypes = [_U64, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p,
                                         _U64, _U64, _i64p, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]
        L.o_finalize.argtypes = [_U64, _i64p, _u64p, _i64p]
        L.o_build_wheel.argtypes = [_u8p]
        self.L = L

    def build_wheel(self):
        w = np.zeros(WHEEL_PERIOD, dtype=np.uint8)
        self.L.o_build_wheel(w)
        return w

    def build_divisor_arrays(self, cap):
        magic = np.zeros(cap + 1, np.uint64)
        shift = np.zeros(cap + 1, np.uint8)
        scheme = np.zeros(cap + 1, np.uint8)
        self.L.o_build_divisor_arrays(cap, magic, shift, scheme)
        return magic, shift, scheme

    def logprime_states(self, y1, y2, primes, logs, wheel):
        out = np.empty(y2 - y1 + 1, np.uint8)
        p = np.ascontiguousarray(primes, np.uint64)
        self.L.o_logprime_states(y1, y2, p, np.ascontiguousarray(logs, np.uint8), len(p),
                                 np.ascontiguousarray(wheel, np.uint8), out)
        return out

    def sieve_logprime(self, y1, y2, primes, logs, wheel):
        n = y2 - y1 + 1
        st = np.empty(n, np.uint8)
        mu = np.empty(n, np.int8)
        p = np.ascontiguousarray(primes, np.uint64)
        self.L.o_sieve_logprime(y1, y2, p, np.ascontiguousarray(logs, np.uint8), len(p),
                                np.ascontiguousarray(wheel, np.uint8), st, mu)
        return mu

    def sieve_naive(self, y1, y2, primes):
        n = y2 - y1 + 1
        acc = np.empty(n, np.int64)
        mu = np.empty(n, np.int8)
        p = np.ascontiguousarray(primes, np.uint64)
        self.L.o_sieve_naive(y1, y2, p, len(p), acc, mu)
        return mu

    def apply_block(self, acc, v, lo, xcut, mcut, dnext, ynext, y1, y2, mprefix, divtable=None):
        c, d = _U64(0), _U64(0)
        ov = self.L.o_apply_block(len(acc), acc, v, lo, xcut, mcut, dnext, ynext, y1, y2,
                                  np.ascontiguousarray(mprefix, np.int64), ctypes.byref(c), ctypes.byref(d))
        if ov:
            raise OverflowError("harmonic accumulator exceeded the signed-64 guard range")
        return c.value, d.value

    def apply_block_wrap(self, acc_u64, v, lo, xcut, mcut, dnext, ynext, y1, y2, mprefix):
        c, d = _U64(0), _U64(0)
        self.L.o_apply_block_wrap(len(acc_u64), acc_u64, v, lo, xcut, mcut, dnext, ynext, y1, y2,
                                  np.ascontiguousarray(mprefix, np.int64), ctypes.byref(c), ctypes.byref(d))
        return c.value, d.value

    def finalize_recursion(self, tails, D):
        out = np.empty(len(tails), np.int64)
        self.L.o_finalize(len(tails), np.ascontiguousarray(tails, np.int64),
                          np.ascontiguousarray(D, np.uint64), out)
        return out


def ref_kernels():
    """The reference's own compiled kernels (oracle/_ref/_native*.so)."""
    d = os.path.join(HERE, "_ref")
    if d not in sys.path:
        sys.path.insert(0, d)
    return importlib.import_module("_native")


_BACKENDS: dict = {}


def get_kernels(name: str = "c"):
    if name not in _BACKENDS:
        _BACKENDS[name] = CKernels() if name == "c" else ref_kernels()
    return _BACKENDS[name]


# ----------------------------------------------------------------------------
# sieve helpers (sieve.py:96-145)
# ----------------------------------------------------------------------------

def generate_primes(limit: int) -> np.ndarray:  # sieve.py:96-108
    flags = np.ones(limit + 1, dtype=bool)
    flags[:2] = False
    for p in range(2, isqrt(limit) + 1):
        if flags[p]:
            flags[p * p :: p] = False
    return np.flatnonzero(flags).astype(np.uint64)


def build_logs(primes: np.ndarray) -> np.ndarray:  # sieve.py:124-131 (ceil(log2 p) | 1)
    shifted = primes - np.uint64(1)
    lengths = np.zeros(len(primes), dtype=np.uint8)
    while shifted.any():
        lengths[shifted > 0] += np.uint8(1)
        shifted >>= np.uint64(1)
    return lengths | np.uint8(1)


def build_wheel() -> np.ndarray:  # sieve.py:134-145
    st = np.zeros(WHEEL_PERIOD, dtype=np.uint8)
    for p in (2, 3, 5, 7):
        st[::p] += np.uint8((p - 1).bit_length() | 1)
    for s in (4, 9):
        st[::s] |= np.uint8(0x80)
    return st


def split_ranges(y1, y2, workers):  # sieve.py:154-165
    length = y2 - y1 + 1
    workers = max(1, min(workers, length))
    step, rem = divmod(length, workers)
    out, start = [], y1
    for i in range(workers):
        span = step + (1 if i < rem else 0)
        if span:
            out.append((start, start + span - 1))
            start += span
    return out


def sieve_block(kern, y1, y2, primes, logs, wheel, workers=1, pool=None):
    """sieve_block_logprime (sieve.py:189-213) incl. the thread split (:168-174)."""
    ranges = split_ranges(y1, y2, workers)
    if len(ranges) == 1:
        return kern.sieve_logprime(y1, y2, primes, logs, wheel)
    if pool is None:
        with ThreadPoolExecutor(max_workers=len(ranges)) as p:
            parts = list(p.map(lambda r: kern.sieve_logprime(r[0], r[1], primes, logs, wheel), ranges))
    else:
        parts = list(pool.map(lambda r: kern.sieve_logprime(r[0], r[1], primes, logs, wheel), ranges))
    return np.concatenate(parts)


def mu_range(kern, y1, y2, primes=None, logs=None, wheel=None):
    """mu over [y1, y2] including the mu(1)=1 special case (engine.py:308-319)."""
    if primes is None:
        primes = generate_primes(max(ceil_sqrt(y2) + 1, 2))
        logs = build_logs(primes)
        wheel = build_wheel()
    if y1 == 1:
        if y2 == 1:
            return np.ones(1, np.int8)
        return np.concatenate([np.ones(1, np.int8), kern.sieve_logprime(2, y2, primes, logs, wheel)])
    return kern.sieve_logprime(y1, y2, primes, logs, wheel)


# ----------------------------------------------------------------------------
# parameters (engine.py:116-185)
# ----------------------------------------------------------------------------

def choose_u(n: int, num_targets: int = 1, mem_budget: int = 2 << 30, alpha: float = 1.0) -> int:
    """engine.py:116-131, restated with identical float semantics."""
    if n < 4:
        raise ValueError("choose_u requires n >= 4")
    base = int(alpha * (n * max(1, num_targets)) ** (2.0 / 3.0))
    u = max(base, ceil_sqrt(n) + 1)
    u = min(u, n)
    max_elements = max(1, mem_budget // 64)
    if n // u > max_elements:
        u = n // max_elements + 1
    if not ceil_sqrt(n) < u <= n:
        raise ValueError(f"no feasible u for n={n} within budget {mem_budget}")
    return u


def _ceil_sqrt_vec(v):  # engine.py:165-174
    s = np.sqrt(v.astype(np.float64)).astype(np.uint64)
    s = np.maximum(s, np.uint64(1))
    for _ in range(2):
        too_big = s * s > v
        s[too_big] -= np.uint64(1)
    grow = (s + np.uint64(1)) * (s + np.uint64(1)) <= v
    s[grow] += np.uint64(1)
    return s + np.uint64(1) * (s * s < v)


def _pow2_at_least(x):  # engine.py:177-185
    e = np.ceil(np.log2(np.maximum(x, np.uint64(1)).astype(np.float64)))
    t = np.uint64(1) << e.astype(np.uint64)
    for _ in range(2):
        low = t < x
        t[low] <<= np.uint64(1)
        high = (t >> np.uint64(1)) >= x
        t[high] >>= np.uint64(1)
    return np.maximum(t, np.uint64(1))


class HarmonicArray:
    """engine.py:134-162 (numpy uint64; n <= 2^64-1)."""

    def __init__(self, n: int, u: int):
        self.n, self.u = n, u
        self.size = n // u
        k = np.arange(1, self.size + 1, dtype=np.uint64)
        self.v = np.uint64(n) // k
        self.D = self.v // np.uint64(u + 1)
        cs = _ceil_sqrt_vec(self.v)
        self.t = _pow2_at_least(np.uint64(2) * cs)
        xcut = np.maximum(self.D, self.v // self.t)
        self.xcut = np.maximum(xcut, np.uint64(1))
        self.mcut = self.v // (self.xcut + np.uint64(1))
        self.lo = np.maximum(np.uint64(2), self.D + np.uint64(1))
        self.dnext = self.xcut.copy()
        active = self.xcut >= self.lo
        self.ynext = np.where(active, self.v // np.maximum(self.xcut, np.uint64(1)), SENTINEL)
        self.acc = np.zeros(self.size, dtype=np.int64)
        self.final = None


def big_params(n: int, u: int):
    """Python-int element parameters (engine.py:475-491; the 128-bit semantics)."""
    K = n // u
    out = []
    for k in range(1, K + 1):
        vk = n // k
        D = vk // (u + 1)
        t = 1 << ((2 * ceil_sqrt(vk) - 1).bit_length())
        xc = max(D, vk // t, 1)
        out.append((vk, D, xc, vk // (xc + 1), max(2, D + 1)))
    return out


def quotient_targets(n: int, K: int, u: int, budget: int) -> np.ndarray:  # engine.py:242-252
    s = isqrt(n)
    if s + K <= budget:
        lo = np.arange(1, s + 1, dtype=np.uint64)
        hi = np.uint64(n) // np.arange(1, s + 1, dtype=np.uint64)
        qs = np.unique(np.concatenate([lo, hi]))
    else:
        c = np.arange(K + 1, K + 1 + budget, dtype=np.uint64)
        qs = np.unique(np.uint64(n) // c)
    return qs[(qs >= 1) & (qs <= np.uint64(u))]


# ----------------------------------------------------------------------------
# the job (engine.py:255-402)
# ----------------------------------------------------------------------------

@dataclass
class Stats:  # engine.py:188-197
    blocks: int = 0
    counted_items: int = 0
    dense_items: int = 0
    divtable_cap: int = 0
    divtable_released_at: int | None = None
    r4_block_len: int | None = None
    sieve_seconds: float = 0.0
    apply_seconds: float = 0.0


@dataclass
class Result:
    n: int
    value: int
    u: int
    final: np.ndarray | None
    cp_q: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint64))
    cp_m: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    stats: Stats | None = None
    elapsed: float = 0.0

    def quotient(self, c: int) -> int:  # engine.py:218-228
        if self.final is not None and c <= len(self.final):
            return int(self.final[c - 1])
        q = self.n // c
        idx = np.searchsorted(self.cp_q, np.uint64(q))
        if idx < len(self.cp_q) and int(self.cp_q[idx]) == q:
            return int(self.cp_m[idx])
        raise KeyError(c)


class Job:
    """_ExactJob restated (engine.py:255-402).  `kern` is a kernel backend;
    `wrap=True` accumulates modulo 2^64 (no 4e18 cap) with the C oracle."""

    def __init__(self, ns, kern="c", u=None, block_len=0, workers=1, capture=True,
                 quotient_budget=4_000_000, c3=2.0, r4_block_factor=4, wrap=False,
                 u_alpha=1.0, mem_budget=2 << 30):
        self.ns = sorted(set(int(x) for x in ns), reverse=True)
        n_max = self.ns[0]
        self.kern = get_kernels(kern) if isinstance(kern, str) else kern
        self.wrap = wrap
        if n_max > U64_PATH_BOUND and not wrap:
            raise ValueError("n exceeds the reference's compiled 64-bit range")
        self.u = u or choose_u(n_max, len(self.ns), mem_budget, u_alpha)
        self.arrays = [HarmonicArray(n, self.u) for n in self.ns]
        if wrap:
            for a in self.arrays:
                a.acc = np.zeros(a.size, dtype=np.uint64)
        self.block_len = block_len or max(ceil_sqrt(self.u), 1 << 22)
        self.workers = workers
        self.next_y1 = 1
        self.m_running = 0
        self.r4 = False
        self.stats = Stats()
        self.r4_factor = r4_block_factor
        self.cp_q = quotient_targets(n_max, self.arrays[0].size, self.u, quotient_budget) if capture \
            else np.empty(0, np.uint64)
        self.cp_m = np.zeros(len(self.cp_q), np.int64)
        self.primes = generate_primes(max(ceil_sqrt(self.u) + 1, 2))
        self.logs = build_logs(self.primes)
        self.wheel = build_wheel()
        self.r4_threshold = max(int(c3 * sqrt(n_max)), max(int(a.mcut.max()) if a.size else 0 for a in self.arrays))

    def _maybe_r4(self, y1):  # engine.py:321-329
        if not self.r4 and y1 > self.r4_threshold:
            self.r4 = True
            bumped = self.r4_factor * ceil_sqrt(self.u)
            if bumped > self.block_len:
                self.block_len = bumped
                self.stats.r4_block_len = bumped
            self.stats.divtable_released_at = y1

    def _sieve(self, y1, y2, pool=None):  # engine.py:308-319
        if y1 == 1:
            if y2 == 1:
                return np.ones(1, np.int8)
            rest = sieve_block(self.kern, 2, y2, self.primes, self.logs, self.wheel, self.workers, pool)
            return np.concatenate([np.ones(1, np.int8), rest])
        return sieve_block(self.kern, y1, y2, self.primes, self.logs, self.wheel, self.workers, pool)

    def run(self, stop_after_blocks=None, on_block=None):
        """engine.py:334-368 — 1-deep sieve prefetch on a helper thread."""
        pre = ThreadPoolExecutor(max_workers=1)
        split = ThreadPoolExecutor(max_workers=max(1, self.workers)) if self.workers > 1 else None
        try:
            pending = None
            while self.next_y1 <= self.u:
                self._maybe_r4(self.next_y1)
                y1, y2 = self.next_y1, min(self.next_y1 + self.block_len - 1, self.u)
                if pending is None or pending[0] != (y1, y2):
                    pending = ((y1, y2), pre.submit(self._sieve, y1, y2, split))
                t0 = time.perf_counter()
                mu = pending[1].result()
                self.stats.sieve_seconds += time.perf_counter() - t0
                pending = None
                if y2 < self.u:
                    ny1 = y2 + 1
                    self._maybe_r4(ny1)
                    nb = (ny1, min(ny1 + self.block_len - 1, self.u))
                    pending = (nb, pre.submit(self._sieve, nb[0], nb[1], split))
                self.apply(y1, y2, mu)
                if on_block is not None:
                    on_block(self, y1, y2)
                if stop_after_blocks is not None and self.stats.blocks >= stop_after_blocks:
                    return False
            return True
        finally:
            pre.shutdown(wait=True)
            if split is not None:
                split.shutdown(wait=True)

    def apply(self, y1, y2, mu):  # engine.py:370-392
        t0 = time.perf_counter()
        mprefix = np.cumsum(mu, dtype=np.int64) + np.int64(self.m_running)
        if len(self.cp_q):
            l = np.searchsorted(self.cp_q, np.uint64(y1), side="left")
            r = np.searchsorted(self.cp_q, np.uint64(y2), side="right")
            if r > l:
                self.cp_m[l:r] = mprefix[(self.cp_q[l:r] - np.uint64(y1)).astype(np.int64)]
        for a in self.arrays:
            if self.wrap:
                c, d = self.kern.apply_block_wrap(a.acc, a.v, a.lo, a.xcut, a.mcut, a.dnext, a.ynext,
                                                  y1, y2, mprefix)
            else:
                c, d = self.kern.apply_block(a.acc, a.v, a.lo, a.xcut, a.mcut, a.dnext, a.ynext,
                                             y1, y2, mprefix, None)
            self.stats.counted_items += int(c)
            self.stats.dense_items += int(d)
        self.m_running = int(mprefix[-1])
        self.next_y1 = y2 + 1
        self.stats.blocks += 1
        self.stats.apply_seconds += time.perf_counter() - t0

    def finalize(self):  # engine.py:394-402
        out = []
        for a in self.arrays:
            acc = a.acc.view(np.int64) if self.wrap else a.acc
            a.final = self.kern.finalize_recursion(acc, a.D)
            out.append(a)
        return out


def mertens_direct(n: int, kern="c") -> Result:  # engine.py:449-458
    k = get_kernels(kern) if isinstance(kern, str) else kern
    plist = generate_primes(max(2, ceil_sqrt(n)))
    mu = k.sieve_naive(1, n, plist)
    prefix = np.cumsum(mu, dtype=np.int64)
    qs = np.unique(np.uint64(n) // np.arange(1, n + 1, dtype=np.uint64))
    return Result(n, int(prefix[-1]), n, None, qs, prefix[(qs - np.uint64(1)).astype(np.int64)], Stats(blocks=1))


def mertens_exact(n: int, kern="c", **kw) -> Result:  # engine.py:405-421
    if n < 1:
        raise ValueError("n must be >= 1")
    if n < DIRECT_CUTOFF:
        return mertens_direct(n, kern)
    t0 = time.perf_counter()
    job = Job([n], kern, **kw)
    job.run()
    a = job.finalize()[0]
    return Result(n, int(a.final[0]), job.u, a.final, job.cp_q, job.cp_m, job.stats, time.perf_counter() - t0)


def mertens_exact_multi(ns, kern="c", **kw) -> dict:  # engine.py:424-446
    ns = sorted(set(int(x) for x in ns))
    out = {n: mertens_exact(n, kern) for n in ns if n < DIRECT_CUTOFF}
    big = [n for n in ns if n >= DIRECT_CUTOFF]
    if big:
        job = Job(big, kern, capture=False, **kw)
        job.run()
        for n, a in zip(job.ns, job.finalize()):
            out[n] = Result(n, int(a.final[0]), job.u, a.final, stats=job.stats)
    return out


def mertens_table(n: int, kern="c") -> np.ndarray:
    """M(1..n) by sieving (the naive oracle, engine.py:553-603)."""
    mu = mu_range(get_kernels(kern) if isinstance(kern, str) else kern, 1, n)
    return np.cumsum(mu, dtype=np.int64)


def mertens_big(n: int, u: int | None = None, block_len: int = 0, kern="c") -> Result:
    """mertens_exact_big restated (engine.py:461-550): Python-int walks, any n
    (the 128-bit semantics).  Slow: tiny n only."""
    k_ = get_kernels(kern) if isinstance(kern, str) else kern
    u = u or choose_u(n)
    params = big_params(n, u)
    K = len(params)
    tails = [0] * K
    dnext = [p[2] for p in params]
    ynext = [p[0] // p[2] if p[2] >= p[4] else None for p in params]
    block_len = block_len or max(ceil_sqrt(u), 1 << 22)
    primes = generate_primes(max(2, ceil_sqrt(u) + 1))
    logs, wheel = build_logs(primes), build_wheel()
    m_running, y1 = 0, 1
    while y1 <= u:
        y2 = min(y1 + block_len - 1, u)
        mu = mu_range(k_, y1, y2, primes, logs, wheel)
        prefix = (np.cumsum(mu, dtype=np.int64) + np.int64(m_running)).tolist()
        for i, (vk, D, xc, mc, lo) in enumerate(params):
            if mc >= y1:
                hi = min(mc, y2)
                qn = vk // (hi + 1)
                if hi == mc:
                    qn = max(qn, xc)
                tot = 0
                for m in range(hi, y1 - 1, -1):
                    q = vk // m
                    tot += (q - qn) * prefix[m - y1]
                    qn = q
                tails[i] += tot
            if ynext[i] is not None and ynext[i] <= y2:
                d = dnext[i]
                d_lo = max(lo, vk // (y2 + 1) + 1)
                tot, q = 0, ynext[i]
                while True:
                    tot += prefix[q - y1]
                    if d == d_lo:
                        break
                    d -= 1
                    q = vk // d
                tails[i] += tot
                if d_lo - 1 >= lo:
                    dnext[i] = d_lo - 1
                    ynext[i] = vk // (d_lo - 1)
                else:
                    ynext[i] = None
        m_running = prefix[-1]
        y1 = y2 + 1
    final = [0] * K
    for idx in range(K - 1, -1, -1):
        k = idx + 1
        s = 1 - tails[idx]
        for d in range(2, params[idx][1] + 1):
            s -= final[k * d - 1]
        final[idx] = s
    return Result(n, final[0], u, np.array(final, dtype=object))
