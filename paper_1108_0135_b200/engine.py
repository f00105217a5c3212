"""Exact Mertens function on B200 — the public engine API of the reference
(pkg/src/mertens/engine.py) backed by one job-level GPU call per request.

    mertens_exact(n, config)        -> MertensResult   (engine.py:405-421)
    mertens_exact_multi(ns, config) -> {n: MertensResult} (engine.py:424-446)
    MertensResult.quotient(c) / .quotients()           (engine.py:200-239)

Differences from the reference that a caller can observe (all deliberate):
  * every n up to 2^75 runs on the compiled path: the 4e18 cap
    (engine.py:45-47, :262-267) does not exist here (mod-2^64 accumulation is
    exact whenever |M| < 2^63), so mertens_exact never drops to
    an interpreted path and mertens_exact_multi accepts n > 4e18;
  * MertensResult.backend is "sm100";
  * RunStats counters (blocks, counted_items, dense_items, R4 switch) are the
    values the reference's block loop would produce, computed in closed form;
    sieve_seconds/apply_seconds report the GPU phase times.
The algorithm parameters (u, K, and per element v, D, t, xcut, mcut, lo) are
the reference's own formulas, so final arrays are bit-identical.
"""

from __future__ import annotations

import os
import struct
import time
from dataclasses import dataclass, field
from enum import IntEnum
from math import isqrt, sqrt

import numpy as np

from . import _lib
from .errors import CeilingExceededError, ContractViolationError, ResourceLimitError
from .sieve import ceil_sqrt

U64_PATH_BOUND = 4 * 10**18       # the reference's cap; kept as a constant for callers
ENGINE_N_BOUND = 1 << 75          # what this engine accepts
_DIRECT_CUTOFF = 1024
_DENSE_MAP_MIN = 1 << 22          # capture-all above this sqrt(n) uses the dense int32 map
BACKEND_NAME = "sm100"


class Region(IntEnum):
    R1 = 1
    R2 = 2
    R3 = 3
    R4 = 4


@dataclass(frozen=True)
class RegionConfig:
    """Paper regions.  Only c3 affects the (closed-form)
    block schedule reported in RunStats; kept for API compatibility."""

    c1: float = 2.0
    c2: float = 20.0
    c3: float = 2.0

    def __post_init__(self):
        if not (1.0 < self.c1 < self.c2):
            raise ValueError("need 1 < c1 < c2")
        if self.c3 < 1.0:
            raise ValueError("need c3 >= 1")


@dataclass(frozen=True)
class EngineConfig:
    """Field-compatible with engine.py:79-95, plus device fields."""

    mem_budget: int = 2 << 30
    workers: int = 0
    u_alpha: float = 1.0
    block_len: int = 0
    region: RegionConfig = field(default_factory=RegionConfig)
    fastdiv_cap: int = 1 << 26
    r4_block_factor: int = 4
    naive_ceiling: int = 10**10
    naive_block_len: int = 1 << 22
    quotient_budget: int = 4_000_000
    backend: str | None = None
    checkpoint_path: str | None = None
    # B200 engine knobs (0 / None = defaults)
    device: int | None = None
    q_budget_bytes: int = 0
    seg_log2_head: int = 0
    seg_log2_tail: int = 0
    engine_flags: int = 0          # MT_FLAG_FORCE_WIDE / _FORCE_SLOWDIV (tests), MT_FLAG_TIMING
    # shard ONE job over the default torch.distributed group (every rank must call
    # with the same arguments; a job fingerprint is checked).  Off by default: under
    # torchrun each rank then computes its own requests independently.
    distributed: bool = False
    stream: int | None = None      # cudaStream_t (int) to run on; None: the engine's own
    checkpoint_seconds: float = 300.0  # with checkpoint_path: after the head, then at most this often
    # dense full quotient map (capture-all for large n): write it to int32 files
    # `<path>.qmap.i32` / `<path>.small.i32` and return memory-mapped views instead
    # of host arrays (at 1e19 each is 12.6 GB)
    quotient_map_path: str | None = None

    def effective_workers(self) -> int:
        return self.workers if self.workers > 0 else (os.cpu_count() or 1)


def classify_region(x: int, y: int, n: int, cfg: RegionConfig) -> Region:
    """Strategy region for array index x and sieve value y (engine.py:98-113)."""
    if x < 1 or y < 1:
        raise ValueError("x and y must be >= 1")
    s = sqrt(n / x)
    if y < cfg.c1 * s:
        return Region.R1
    if y < cfg.c2 * s:
        return Region.R2
    return Region.R4 if y > cfg.c3 * sqrt(n) else Region.R3


def choose_u(n: int, num_targets: int = 1, mem_budget: int = 2 << 30, alpha: float = 1.0) -> int:
    """Sieving bound u (engine.py:116-131): identical float semantics so that u
    and K = n // u match the reference exactly."""
    if n < 4:
        raise ValueError("choose_u requires n >= 4")
    u = int(alpha * (n * max(1, num_targets)) ** (2.0 / 3.0))
    u = min(max(u, ceil_sqrt(n) + 1), n)
    cap_elems = max(1, mem_budget // 64)
    if n // u > cap_elems:
        u = n // cap_elems + 1
    if not ceil_sqrt(n) < u <= n:
        raise ResourceLimitError(f"no feasible u for n={n} within budget {mem_budget}")
    return u


@dataclass
class RunStats:
    """engine.py:188-197 fields, plus the device breakdown."""

    blocks: int = 0
    counted_items: int = 0
    dense_items: int = 0
    divtable_cap: int = 0
    divtable_released_at: int | None = None
    r4_block_len: int | None = None
    sieve_seconds: float = 0.0
    apply_seconds: float = 0.0
    device: dict = field(default_factory=dict)


class MertensResult:
    """M(n) plus the simultaneous map c -> M(floor(n/c)) (engine.py:200-239)."""

    def __init__(self, n, value, u, array_final, cp_q=None, cp_m=None, stats=None, elapsed=0.0,
                 backend="", qmap=None, small=None):
        self.n = n
        # dense full quotient map (capture-all mode for large n): qmap[c - K - 1] =
        # M(n // c) for K < c <= isqrt(n), small[y] = M(y) for y <= isqrt(n)
        self._qmap = qmap
        self._small = small
        self.value = value
        self.u = u
        self._final = array_final
        self._cp_q = cp_q if cp_q is not None else np.empty(0, dtype=np.uint64)
        self._cp_m = cp_m if cp_m is not None else np.empty(0, dtype=np.int64)
        self.stats = stats
        self.elapsed = elapsed
        self.backend = backend

    @property
    def ratio(self) -> float:
        return self.value / sqrt(self.n)

    def quotient(self, c: int) -> int:
        """M(floor(n/c)) for any captured c >= 1."""
        if c < 1:
            raise ValueError("c must be >= 1")
        if self._final is not None and c <= len(self._final):
            return int(self._final[c - 1])
        if self._qmap is not None:
            K = len(self._final) if self._final is not None else 0
            if c <= K + len(self._qmap):
                return int(self._qmap[c - K - 1])
            q = self.n // c
            if q < len(self._small):
                return int(self._small[q])
            raise KeyError(f"M(n//{c}) was not captured in this run")
        q = self.n // c
        if q < 2**64:
            i = int(np.searchsorted(self._cp_q, np.uint64(q)))
            if i < len(self._cp_q) and int(self._cp_q[i]) == q:
                return int(self._cp_m[i])
        raise KeyError(f"M(n//{c}) was not captured in this run (quotient budget)")

    def quotients(self):
        """Yield (c, floor(n/c), M) over distinct quotients, ascending c."""
        c = 1
        while c <= self.n:
            q = self.n // c
            try:
                m = self.quotient(c)
            except KeyError:
                return
            yield c, q, m
            c = self.n // q + 1


def _quotient_targets(n: int, K: int, u: int, budget: int) -> np.ndarray:
    """Distinct floor(n/c) <= u captured in a run (engine.py:242-252)."""
    s = isqrt(n)
    if s + K <= budget:
        c = np.arange(1, s + 1, dtype=np.uint64)
        qs = np.union1d(c, np.uint64(n) // c)
    else:
        # floor(n/c) is non-increasing in c: dedupe adjacent values, then ascend
        # (same set as np.unique, without its hash/sort pass over `budget` values)
        v = np.uint64(n) // np.arange(K + 1, K + 1 + budget, dtype=np.uint64)
        keep = np.empty(v.shape, dtype=bool)
        if v.size:
            keep[0] = True
            np.not_equal(v[1:], v[:-1], out=keep[1:])
        qs = v[keep][::-1]
    return qs[(qs >= 1) & (qs <= np.uint64(u))]


def _block_schedule(u: int, n_max: int, max_mcut: int, config: EngineConfig, stats: RunStats):
    """The reference block loop's counters in closed form (engine.py:321-368)."""
    bl = config.block_len or max(ceil_sqrt(u), 1 << 22)
    thr = max(int(config.region.c3 * sqrt(n_max)), max_mcut)
    # R4 engages at the first block start y1 > thr (starts are 1 + i*bl)
    i0 = max(0, (thr - 1) // bl + 1) if thr >= 1 else 0
    n_pre = -(-u // bl)
    if 1 + i0 * bl > u:
        stats.blocks = n_pre
        return
    y_r4 = 1 + i0 * bl
    stats.divtable_released_at = y_r4
    bl2 = max(bl, config.r4_block_factor * ceil_sqrt(u))
    if bl2 > bl:
        stats.r4_block_len = bl2
    stats.blocks = i0 + -(-(u - y_r4 + 1) // bl2)


def _split_n(ns):
    lo = np.array([n & (2**64 - 1) for n in ns], dtype=np.uint64)
    hi = np.array([n >> 64 for n in ns], dtype=np.uint64)
    return lo, hi


def make_job(ns, u, config: EngineConfig, cap_c=None, cap_small=0, rank=0, world=1):
    """The mt_job of one exact request (the arrays it points at are kept on the job)."""
    for n in ns:
        if n >= ENGINE_N_BOUND:
            raise ResourceLimitError(f"n={n} exceeds the engine range 2^75")
    n_lo, n_hi = _split_n(ns)
    job = _lib.MtJob()
    job._keep = (n_lo, n_hi)
    job.n_targets = len(ns)
    job.n_lo = n_lo.ctypes.data_as(_lib._pu64)
    job.n_hi = n_hi.ctypes.data_as(_lib._pu64)
    job.u = u
    job.device = -1 if config.device is None else int(config.device)
    job.q_budget_bytes = config.q_budget_bytes
    job.seg_log2_head = config.seg_log2_head
    job.seg_log2_tail = config.seg_log2_tail
    job.flags = config.engine_flags
    job.stream = config.stream
    job.shard_rank, job.shard_world = rank, world
    if cap_c is not None and cap_c[1] >= cap_c[0]:
        job.cap_c_lo, job.cap_c_hi = cap_c
    else:
        job.cap_c_lo, job.cap_c_hi = 1, 0
    job.cap_small = cap_small
    return job


def rank_checkpoint_path(path: str, rank: int, world: int) -> str:
    """One checkpoint file per rank of a sharded job (the single-rank name is `path`)."""
    return path if world <= 1 else f"{path}.r{rank}of{world}"


def _sieve_checkpointed(L, h, config: EngineConfig, path: str | None, restore_from=None):
    """Phase 1 of a plan in steps, checkpointed after the head and then at most
    every `checkpoint_seconds` between tail segments (the reference writes after
    every block, engine.py:391-392; at GPU rates that would be I/O bound).
    Returns (M(head_end - 1), this rank's tail total)."""
    import ctypes

    if restore_from:
        _lib.check(L.mt_plan_restore(h, restore_from.encode()))
    done, mh, tt = ctypes.c_int(0), ctypes.c_int64(), ctypes.c_int64()
    last = time.perf_counter()
    first = not restore_from
    bpath = (path or "").encode()
    while not done.value:
        _lib.check(L.mt_plan_sieve_step(h, 256, ctypes.byref(done), ctypes.byref(mh), ctypes.byref(tt)))
        now = time.perf_counter()
        if bpath and not done.value and (first or now - last >= config.checkpoint_seconds):
            _lib.check(L.mt_plan_checkpoint(h, bpath))
            last, first = now, False
    return mh.value, tt.value


def _run_checkpointed(L, job, res, config: EngineConfig, restore_from=None):
    """Single-target, single-rank job on the plan API with checkpoints."""
    import ctypes

    h = ctypes.c_void_p()
    _lib.check(L.mt_plan_create(ctypes.byref(job), ctypes.byref(h)))
    try:
        mh, _ = _sieve_checkpointed(L, h, config, config.checkpoint_path, restore_from)
        _lib.check(L.mt_plan_tail_offset(h, mh))
        _lib.check(L.mt_plan_gather(h))
        _lib.check(L.mt_plan_resolve(h, ctypes.byref(res)))
    finally:
        L.mt_plan_destroy(h)


def _run_job(ns, u, config: EngineConfig, cap_c=None, cap_small=0, acc_out=None, cap32=False,
             restore_from=None, cap_out=None, small_out=None):
    """One exact job (mt_run, or the plan phases over the process group when
    one is up); returns (finals per n, cap_m, small_m, raw stats)."""
    L = _lib.require_device()
    from . import distributed

    rank, world = distributed.world() if config.distributed else (0, 1)
    job = make_job(ns, u, config, cap_c, cap_small, rank, world)
    if cap32:
        job.flags |= _lib.MT_FLAG_CAP32
    cdt = np.int32 if cap32 else np.int64
    K = [n // u for n in ns]
    finals = np.zeros(sum(K), dtype=np.int64)
    res = _lib.MtResult()
    res.finals = finals.ctypes.data_as(_lib._pi64)
    cap_m = small_m = None
    if cap_c is not None and cap_c[1] >= cap_c[0]:
        cap_m = cap_out if cap_out is not None else np.zeros(cap_c[1] - cap_c[0] + 1, dtype=cdt)
        assert cap_m.dtype == cdt and len(cap_m) == cap_c[1] - cap_c[0] + 1
        res.cap_m_out = cap_m.ctypes.data_as(_lib._pi64)
    if cap_small:
        small_m = small_out if small_out is not None else np.zeros(cap_small + 1, dtype=cdt)
        assert small_m.dtype == cdt and len(small_m) == cap_small + 1
        res.small_m_out = small_m.ctypes.data_as(_lib._pi64)
    if acc_out is not None:
        res.acc_out = acc_out.ctypes.data_as(_lib._pu64)
    ckpt = bool(config.checkpoint_path or restore_from)
    if ckpt and len(ns) != 1:  # the reference refuses multi-target checkpoints too (engine.py:664-665)
        raise ContractViolationError("checkpoint/resume covers single-target jobs only")
    if world > 1:
        plan = distributed.DevicePlan(job)
        try:
            if ckpt:
                path = config.checkpoint_path and rank_checkpoint_path(config.checkpoint_path, rank, world)
                rfrom = restore_from and rank_checkpoint_path(restore_from, rank, world)
                plan.sieve_update = lambda: _sieve_checkpointed(L, plan.h, config, path, rfrom)
            distributed.run_phases(plan, None, res)
        finally:
            plan.close()
    elif ckpt:
        _run_checkpointed(L, job, res, config, restore_from)
    else:
        _lib.check(L.mt_run(job, res))
    out, o = [], 0
    for k in K:
        out.append(finals[o:o + k])
        o += k
    raw = _lib.stats_dict(res.stats)
    raw["world"] = world
    return out, cap_m, small_m, raw


def _stats_from(raw, u, n_max, config) -> RunStats:
    s = RunStats(counted_items=int(raw["counted_items"]), dense_items=int(raw["dense_items"]))
    _block_schedule(u, n_max, int(raw["max_mcut"]), config, s)
    s.sieve_seconds = raw["ms_sieve_tail"] / 1e3
    s.apply_seconds = (raw["ms_update_head"] + raw["ms_qgather"] + raw["ms_finalize"]) / 1e3
    s.device = raw
    return s


def _mertens_direct(n: int, config: EngineConfig, t0: float) -> MertensResult:
    """n < 1024: M(1..n) from one GPU sieve pass (engine.py:449-458)."""
    L = _lib.require_device()
    pre = np.zeros(n, dtype=np.int64)
    _lib.check(L.mt_mertens_range(1, n, _lib.ptr(pre)))
    qs = np.unique(np.uint64(n) // np.arange(1, n + 1, dtype=np.uint64))
    return MertensResult(n, int(pre[-1]), n, None, qs, pre[(qs - np.uint64(1)).astype(np.int64)],
                         RunStats(blocks=1), time.perf_counter() - t0, BACKEND_NAME)


def mertens_exact(n: int, config: EngineConfig | None = None) -> MertensResult:
    """M(n) and the simultaneous quotient map."""
    return _mertens_exact(n, config)


def _mertens_exact(n: int, config: EngineConfig | None = None, restore_from: str | None = None) -> MertensResult:
    if n < 1:
        raise ValueError("n must be >= 1")
    config = config or EngineConfig()
    t0 = time.perf_counter()
    if n < _DIRECT_CUTOFF:
        return _mertens_direct(n, config, t0)
    u = choose_u(n, 1, config.mem_budget, config.u_alpha)
    K = n // u
    s = isqrt(n)
    if s + K <= config.quotient_budget and s > _DENSE_MAP_MIN:
        # capture-all (engine.py:242-252) as a dense map instead of ~2*sqrt(n)
        # (q, M) pairs: M(n//c) for K < c <= s from the quotient table, M(y) for
        # y <= s from the head sieve, both int32 (|M(y)| < 2^31 for y <= u)
        qo = so = None
        if config.quotient_map_path:  # memory-mapped int32 files instead of host arrays
            qo = np.memmap(config.quotient_map_path + ".qmap.i32", dtype=np.int32, mode="w+", shape=(s - K,))
            so = np.memmap(config.quotient_map_path + ".small.i32", dtype=np.int32, mode="w+", shape=(s + 1,))
        finals, qmap, small, raw = _run_job([n], u, config, (K + 1, s), s, cap32=True, restore_from=restore_from,
                                            cap_out=qo, small_out=so)
        if qo is not None:
            qo.flush()
            so.flush()
        st = _stats_from(raw, u, n, config)
        return MertensResult(n, int(finals[0][0]), u, finals[0], stats=st, elapsed=time.perf_counter() - t0,
                             backend=BACKEND_NAME, qmap=qmap, small=small)
    if n < 2**64:
        cp_q = _quotient_targets(n, K, u, config.quotient_budget)
    else:  # quotient values beyond 2^64 cannot be held in the uint64 capture array
        cp_q = _quotient_targets_big(n, K, u, config.quotient_budget)
    s = isqrt(n)
    capture_all = s + K <= config.quotient_budget
    small_lim = s if capture_all else 0
    large = cp_q[cp_q > np.uint64(small_lim)]
    cap_c = None
    if len(large):
        if n < 2**64:
            cs = np.uint64(n) // large
        else:
            cs = np.array([n // q for q in large.tolist()], dtype=np.uint64)
        cap_c = (int(cs.min()), int(cs.max()))
    finals, cap_m, small_m, raw = _run_job([n], u, config, cap_c, small_lim, restore_from=restore_from)
    cp_m = np.zeros(len(cp_q), dtype=np.int64)
    if len(large):
        idx = (cs - np.uint64(cap_c[0])).astype(np.int64)
        cp_m[len(cp_q) - len(large):] = cap_m[idx]
    if small_lim:
        nsmall = len(cp_q) - len(large)
        cp_m[:nsmall] = small_m[cp_q[:nsmall].astype(np.int64)]
    st = _stats_from(raw, u, n, config)
    return MertensResult(n, int(finals[0][0]), u, finals[0], cp_q, cp_m, st,
                         time.perf_counter() - t0, BACKEND_NAME)


def _quotient_targets_big(n: int, K: int, u: int, budget: int) -> np.ndarray:
    c = range(K + 1, K + 1 + budget)
    qs = sorted({n // x for x in c})
    return np.array([q for q in qs if 1 <= q <= u], dtype=np.uint64)


def mertens_exact_multi(ns, config: EngineConfig | None = None) -> dict[int, MertensResult]:
    """One shared sieve pass for several close targets; maps n -> result.
    Quotient capture is skipped (engine.py:424-446)."""
    config = config or EngineConfig()
    ns = sorted(set(int(x) for x in ns))
    out = {n: mertens_exact(n, config) for n in ns if n < _DIRECT_CUTOFF}
    big = [n for n in ns if n >= _DIRECT_CUTOFF]
    if big:
        t0 = time.perf_counter()
        u = choose_u(max(big), len(big), config.mem_budget, config.u_alpha)
        finals, _, _, raw = _run_job(big, u, config)
        st = _stats_from(raw, u, max(big), config)
        dt = time.perf_counter() - t0
        for n, f in zip(big, finals):
            out[n] = MertensResult(n, int(f[0]), u, f, stats=st, elapsed=dt, backend=BACKEND_NAME)
    return out


def mertens_exact_big(n: int, config: EngineConfig | None = None, u: int | None = None) -> MertensResult:
    """The reference's arbitrary-width path (engine.py:461-550).  Here it is the
    same GPU engine (128-bit capable); u may be forced.  No quotient capture."""
    if n < 4:
        return mertens_exact(n, config)
    config = config or EngineConfig()
    t0 = time.perf_counter()
    u = u or choose_u(n, 1, config.mem_budget, config.u_alpha)
    if u <= ceil_sqrt(n):
        raise ValueError("u must exceed ceil(sqrt(n))")
    finals, _, _, raw = _run_job([n], u, config)
    return MertensResult(n, int(finals[0][0]), u, finals[0], stats=_stats_from(raw, u, n, config),
                         elapsed=time.perf_counter() - t0, backend=BACKEND_NAME)


def release_device_memory() -> None:
    """Return the engine's cached device buffers to the driver.  Plans allocate from
    the device's memory pool and keep the blocks between calls (no per-call mapping
    of several GB); this trims the pool (mt_trim_device_memory)."""
    L = _lib.require_device()
    _lib.check(L.mt_trim_device_memory())


def mertens_naive(n: int, config: EngineConfig | None = None, checkpoints=None):
    """M(n) by one O(n) GPU sieve pass (engine.py:553-603); with `checkpoints`
    (sorted) also returns M at each checkpoint <= n."""
    if n < 1:
        raise ValueError("n must be >= 1")
    config = config or EngineConfig()
    if n > config.naive_ceiling:
        raise CeilingExceededError(f"naive path capped at {config.naive_ceiling}; requested {n}")
    L = _lib.require_device()
    pts = [n]
    cp = None
    if checkpoints is not None:
        cp = np.asarray(checkpoints, dtype=np.uint64)
        pts = sorted(set(int(q) for q in cp.tolist() if 1 <= int(q) <= n) | {n})
    arr = np.array(pts, dtype=np.uint64)
    vals = np.zeros(len(arr), dtype=np.int64)
    _lib.check(L.mt_mertens_at(_lib.ptr(arr), len(arr), _lib.ptr(vals)))
    m_final = int(vals[-1])
    if cp is None:
        return m_final
    lut = dict(zip(pts, vals.tolist()))
    return m_final, np.array([lut.get(int(q), 0) for q in cp.tolist()], dtype=np.int64)


def mertens_identity_residual(result: MertensResult, chunk: int = 1 << 24) -> int:
    """sum_{x=1..n} M(floor(n/x)) - 1 over the quotient map (engine.py:606-616).
    The dense map (capture-all for large n, possibly memory-mapped) is summed in
    chunks of `chunk` entries (no n-sized temporaries) modulo 2^64."""
    n = result.n
    if result._qmap is not None and n < 2**64:
        s = isqrt(n)
        K = len(result._final)
        tot = 0
        # c < s: q = n // c >= s + 1, whose preimage (n/(q+1), n/q] is shorter than 1,
        # so every such quotient occurs once (at x = c); c = s is added exactly below
        for c0 in range(1, s, chunk):
            i0, i1 = c0 - 1, min(s - 1, c0 + chunk - 1)  # indices into finals ++ qmap
            if i0 < K:
                tot += int(result._final[i0:min(i1, K)].astype(np.int64).sum())
            if i1 > K:
                tot += int(np.asarray(result._qmap[max(i0, K) - K:i1 - K]).astype(np.int64).sum())
        q = n // s
        ms = int(result._final[s - 1]) if s - 1 < K else int(result._qmap[s - 1 - K])
        tot += (n // q - n // (q + 1)) * ms
        # y < floor(n/s): multiplicity n//y - n//(y+1) (uint64 quotients, one division each)
        ymax = min(n // s - 1, s)
        nn = np.uint64(n)
        for y0 in range(1, ymax + 1, chunk):
            y1 = min(ymax, y0 + chunk - 1)
            d = nn // np.arange(y0, y1 + 2, dtype=np.uint64)
            mult = (d[:-1] - d[1:]).astype(np.int64)
            tot += int((mult * np.asarray(result._small[y0:y1 + 1]).astype(np.int64)).sum())
        # int64 products and chunk sums wrap mod 2^64 (exact there); the identity's
        # total is small, so the signed residue mod 2^64 is the exact value
        tot %= 1 << 64
        if tot >= 1 << 63:
            tot -= 1 << 64
        return tot - 1
    total = 0
    for _, q, m in result.quotients():
        total += (n // q - (n // (q + 1) if q < n else 0)) * m
    return total - 1


def verify_paired(n_max: int, samples: int, seed: int, config: EngineConfig | None = None,
                  fault_inject: int | None = None):
    """mertens_exact vs mertens_naive on deterministic samples (engine.py:619-643)."""
    config = config or EngineConfig()
    if samples == 0:
        ns = list(range(1, n_max + 1))
    else:
        rng = np.random.default_rng(seed)
        ns = sorted(set(int(x) for x in rng.integers(1, n_max + 1, size=samples)))
    _, naive = mertens_naive(n_max, config, checkpoints=np.array(ns, dtype=np.uint64))
    bad = []
    for i, n in enumerate(ns):
        exact = mertens_exact(n, config).value
        nv = int(naive[i]) + (1 if fault_inject is not None and i == fault_inject else 0)
        if exact != nv:
            bad.append({"n": n, "exact": exact, "naive": nv})
    return {"n_max": n_max, "checked": len(ns), "seed": seed, "mismatches": bad}


_CKPT_HEAD = struct.Struct("<8sII QQ Q Q Q q Q")  # engine.py:659


def resume_exact(path: str, config: EngineConfig | None = None) -> MertensResult:
    """Continue a checkpointed run to completion (engine.py:731-741).  The file
    carries the reference's MERTCKP1 header (version 4: this engine's state
    follows it); u must match the one `config` derives (engine.py:697-698).
    A sharded job (config.distributed under a process group) resumes from the
    per-rank files `path.r{rank}of{world}`."""
    config = config or EngineConfig()
    from . import distributed

    rank, world = distributed.world() if config.distributed else (0, 1)
    with open(rank_checkpoint_path(path, rank, world), "rb") as f:
        head = f.read(_CKPT_HEAD.size)
    if len(head) != _CKPT_HEAD.size:
        raise ContractViolationError("not a checkpoint file")
    magic, version, flags, n_lo, n_hi, u, _next_y1, _K, _m_running, _bl = _CKPT_HEAD.unpack(head)
    if magic != b"MERTCKP1" or version != 4:
        raise ContractViolationError("not an sm100 checkpoint file")
    n = (n_hi << 64) | n_lo
    if choose_u(n, 1, config.mem_budget, config.u_alpha) != u:
        raise ContractViolationError(f"checkpoint built with u={u}, config derives another u")
    if flags != (rank | (world << 16)):
        raise ContractViolationError(f"checkpoint written by rank {flags & 0xFFFF} of {flags >> 16}, "
                                     f"this is rank {rank} of {world}")
    return _mertens_exact(n, config, restore_from=path)
