"""Benchmark: exact M(n) (default n = 10^19, BASELINE.json's metric) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 1e19] [--impl ours|reference]
                    [--dist-backend nccl|gloo]

One step = one complete exact job: segmented Moebius sieve of y in [1, u],
the harmonic-array update of all K = n // u elements, the quotient-table
gather and the final resolve, giving M(n) and every M(floor(n/c)), c <= K.
`value` is y-values/s = u / device time of the job (plan resident in HBM,
CUDA events on the engine's stream, max over ranks).  `e2e` is the same
metric through the public API `mertens_exact(n)` (host in, host out: M(n),
the K finals and the 4M captured quotients copied back every step).

--gpus N > 1 without a torchrun environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU,
NCCL; --dist-backend gloo lets N ranks share the GPUs of a smaller box, the
ranks then take cuda:(local_rank mod device_count)).  The ranks split the
job as DESIGN.md §5 describes; the world size actually used is asserted.

--impl reference times the reference algorithm on the host cores instead
(oracle/_ref's compiled kernels where they apply, else the oracle's C port),
on a bounded sample of the same job, extrapolated to the whole job, and
measures the reference end to end at the anchor config n = 10^13.
Under torchrun (N > 1) rank 0 alone runs the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASE["metric"]
# Table 1; 10^21 sign corrected (the table prints +3395895277; see
# tests/test_explicit_formula_check.py and profiles/r01_paper_e21_*.json)
PAPER = {10**16: -3195437, 10**17: -21830254, 10**18: -46758740, 10**19: 899990187,
         10**20: 461113106, 10**21: -3395895277, 10**22: -2061910120,
         11609864264058592345: -1995900927}
# reference values measured by running the reference (tests/golden)
ANCHOR_M = {10**13: 599582, 10**12: 62366}


def parse_n(s: str) -> int:
    if "e" in s.lower():
        m, e = s.lower().split("e")
        return int(m) * 10 ** int(e)
    return int(s)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


def ncu_metrics():
    """Per-kernel ncu counters committed under profiles/ (one `--set full` capture each)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_metrics.json")))
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ---------------------------------------------------------------- CPU reference arm
def _walk_state_at(H, y1):
    """The dense-walk cursor of every element at block start y1, in closed form
    (the reference's _replay_walk_state, engine.py:715-728): the next d is the
    largest d <= xcut with floor(v/d) >= y1."""
    from oracle import engine_port as E

    d = np.minimum(H.xcut, H.v // np.uint64(max(1, y1)))
    act = d >= H.lo
    dn = np.where(act, d, H.lo - np.uint64(1))
    yn = np.where(act, H.v // np.maximum(dn, np.uint64(1)), E.SENTINEL)
    return dn, yn


def cpu_reference_sample(n: int, u: int, threads: int):
    """Time the reference algorithm on a bounded sample of the job and
    extrapolate to the whole job (SURVEY.md §8(d) CPU-baseline plan).

    apply : the reference's apply_block, single-threaded as the reference runs it
            (engine.py:380-384), on two y-blocks: [1, 2^22] for every S-th element
            (its counted walks -> t_c per counted pair) and a block at y = 2^30
            inside the dense region for the sampled elements whose counted walk
            ended below it (random M gathers -> t_d per dense pair).  oracle/_ref's
            compiled kernel when n <= 4e18 (where it is defined), else the oracle's C
            port with mod-2^64 wrap (the reference's i128 guard rejects those n).
    sieve : the reference's sieve_logprime on 2^28 y at y = u/2 over `threads`
            threads (its `workers`, sieve.py:168-174).
    job   ~= counted * t_c + dense * t_d + u / sieve rate (the reference overlaps
            one block of sieve with the apply; the head is apply-bound, the tail
            sieve-bound, so the two add)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import engine_port as E

    kern_c = E.get_kernels("c")
    try:
        kern_ref = E.get_kernels("ref")
    except Exception:
        kern_ref = None
    H = E.HarmonicArray(n, u)
    counted = int(H.mcut.sum(dtype=np.uint64))
    dense = int(np.where(H.xcut >= H.lo, H.xcut - H.lo + np.uint64(1), 0).sum(dtype=np.uint64))
    K = n // u
    stride = max(1, K // 256)  # ~1e9 counted pairs at 1e19: ~5 s of one core
    ks = np.arange(0, K, stride)
    primes = E.generate_primes(E.ceil_sqrt(u) + 1)
    logs, wheel = E.build_logs(primes), E.build_wheel()
    use_ref_apply = kern_ref is not None and n <= 4 * 10**18
    L = 1 << 22
    blocks = []
    # block 1: [1, 2^22] -- counted walks of every sampled element (no dense items yet);
    # block 2: [2^30, 2^30 + 2^22) over the elements whose counted walk ended below it
    # (8x denser sample) -- dense items only, the random M gathers
    for y1, ks_b in ((1, ks), (1 << 30, np.arange(0, K, max(1, K // 2048)))):
        y2 = min(y1 + L - 1, u)
        if y1 > 1:
            ks_b = ks_b[H.mcut[ks_b] < np.uint64(y1)]
        mu = E.mu_range(kern_c, y1, y2, primes, logs, wheel)
        mp = np.cumsum(mu, dtype=np.int64)  # the base M(y1 - 1) does not change the work
        dn, yn = _walk_state_at(H, y1)
        a = {f: np.ascontiguousarray(getattr(H, f)[ks_b]) for f in ("v", "lo", "xcut", "mcut")}
        dn, yn = np.ascontiguousarray(dn[ks_b]), np.ascontiguousarray(yn[ks_b])
        acc = np.zeros(len(ks_b), np.int64 if use_ref_apply else np.uint64)
        t0 = time.perf_counter()
        if use_ref_apply:
            c, d = kern_ref.apply_block(acc, a["v"], a["lo"], a["xcut"], a["mcut"], dn, yn, y1, y2, mp, None)
        else:
            c, d = kern_c.apply_block_wrap(acc, a["v"], a["lo"], a["xcut"], a["mcut"], dn, yn, y1, y2, mp)
        blocks.append((int(c), int(d), time.perf_counter() - t0))
    (c1, d1, s1), (c2, d2, s2) = blocks
    tc = s1 / max(1, c1 + d1)
    td = max(0.0, s2 - c2 * tc) / max(1, d2)
    SL = 1 << 28
    y0 = max(2, u // 2)
    sk = kern_ref if kern_ref is not None else kern_c
    rngs = E.split_ranges(y0, y0 + SL - 1, threads)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda r: sk.sieve_logprime(r[0], r[1], primes, logs, wheel), rngs))
    t_sieve = time.perf_counter() - t0
    y_rate = SL / t_sieve
    t_apply = counted * tc + dense * td
    est = t_apply + u / y_rate
    kind = "reference" if (use_ref_apply and kern_ref is not None) else "port"
    sample = (f"apply_block single-threaded (as the reference) on every {stride}-th of K={K} elements over "
              f"[1,2^22] ({c1:.3g} counted + {d1:.3g} dense pairs, {s1:.3g} s) and on the elements of an 8x "
              f"denser sample whose counted walk ended below 2^30 over [2^30,2^30+2^22) "
              f"({c2:.3g} + {d2:.3g} pairs, {s2:.3g} s) -> {tc * 1e9:.3g} ns/counted pair, "
              f"{td * 1e9:.3g} ns/dense pair ({'oracle/_ref compiled kernel' if use_ref_apply else 'oracle C port, mod-2^64 (reference kernel rejects n>4e18)'})"
              f"; sieve_logprime of 2^28 y at y={y0} on {threads} threads ({'oracle/_ref' if kern_ref is not None else 'oracle C port'}); "
              f"job extrapolated as {counted:.4g} counted x t_c + {dense:.4g} dense x t_d + u / {y_rate:.4g} y/s "
              f"= {t_apply:.4g} + {u / y_rate:.4g} = {est:.4g} s")
    return {"value": u / est, "unit": "y-values/s", "cores": threads, "kind": kind, "sample": sample,
            "est_job_s": est, "t_counted_ns": tc * 1e9, "t_dense_ns": td * 1e9, "y_rate": y_rate,
            "sample_s": s1 + s2 + t_sieve, "fits_in_driver_run": False}


def reference_anchor(n: int, threads: int):
    """The reference end to end at a config it finishes in the driver window:
    oracle/engine_port's restated job loop (engine.py:255-402) driving the
    reference's own compiled kernels (oracle/_ref), sieve on `threads` workers,
    apply on one thread -- as the reference runs."""
    from oracle import engine_port as E

    try:
        E.get_kernels("ref")
        kern = "ref"
    except Exception:
        kern = "c"
    t0 = time.perf_counter()
    r = E.mertens_exact(n, kern, workers=threads)
    wall = time.perf_counter() - t0
    return {"n": str(n), "M": r.value, "M_ok": ANCHOR_M.get(n) in (None, r.value), "u": r.u, "wall_s": wall,
            "value": r.u / wall, "unit": "y-values/s", "kernels": "oracle/_ref" if kern == "ref" else "oracle C port",
            "cores": threads, "measured": "end to end, one run", "fits_in_driver_run": True}


def reference_arm(args, n, u, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_sample(n, u, threads)
    vals = [cpu_reference_sample(n, u, threads) for _ in range(args.steps)]
    v = statistics.median(r["value"] for r in vals)
    last = vals[-1]
    anchor = None if args.no_anchor else reference_anchor(parse_n(args.anchor_n), threads)
    line = {
        "metric": METRIC, "value": v, "unit": "y-values/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * u / v, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": f"synthetic: n={n} (deterministic, no dataset)",
        "config": config_block(n, u, world), "impl": "reference",
        "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "y-values/s"},
        "e2e": {"value": v, "unit": "y-values/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "extrapolated": True,
        "anchor": anchor,
    }
    print(json.dumps(line), flush=True)


def config_block(n, u, world):
    return {"workload": f"M({n}) plus all M(floor(n/c)) for c <= K (exact, 1 target)", "n": str(n), "u": u,
            "K": n // u, "parallelism": f"y-shard x{world} (head redundant, tail ranges over the y coprime to 6, 1 int64 allreduce)",
            "l2": "inputs larger than L2: the job streams u sieve cells and a multi-GB quotient table per step"}


# ---------------------------------------------------------------- launch
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relaunch(args) -> int:
    """--gpus N outside torchrun: re-run this script as N ranks (one per GPU)."""
    env = dict(os.environ)
    if args.dist_backend == "nccl":
        env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) for the record
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", default="1e19")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-anchor", action="store_true")
    ap.add_argument("--anchor-n", default="1e13", help="end-to-end config both arms run in full")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps")
    ap.add_argument("--launch-check", action="store_true",
                    help="each rank prints its rank/world and exits (tests the --gpus launcher)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))
    n = parse_n(args.n)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but the launcher started {world} ranks")
    if args.launch_check:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return

    import paper_1108_0135_b200 as P

    u = P.choose_u(n)
    if args.impl == "reference":
        return reference_arm(args, n, u, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1108_0135_b200 import _lib, distributed, engine

    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            # communicator init lines (nranks) for the record, also when launched by torchrun
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    tdev = torch.device("cuda", dev) if args.dist_backend == "nccl" else torch.device("cpu")
    stream = torch.cuda.current_stream()
    # the timed steps run the plain engine: per-kernel CUDA events (MT_FLAG_TIMING)
    # cost ~4 % of a step, so the kernel breakdown and the roofline's per-launch
    # times come from one instrumented step right after the timed region
    cfg = P.EngineConfig(device=dev, stream=stream.cuda_stream)
    cfg_t = P.EngineConfig(device=dev, engine_flags=_lib.MT_FLAG_TIMING, stream=stream.cuda_stream)
    job = engine.make_job([n], u, cfg, rank=rank, world=world)
    job_t = engine.make_job([n], u, cfg_t, rank=rank, world=world)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make_plan(j):
        return distributed.DevicePlan(j) if world > 1 else _SinglePlan(j)

    # ---- device-timed job: plan resident in HBM, phases + collectives per step
    plan = make_plan(job)
    res = _lib.MtResult()
    fin = np.zeros(n // u, np.int64)
    res.finals = fin.ctypes.data_as(_lib._pi64)  # M(n) is read back once per step
    for _ in range(args.warmup):
        _one(plan, world, res)
    barrier()
    times, launches = [], []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _one(plan, world, res)
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1))
            launches.append(int(_lib.stats_dict(res.stats)["kernel_launches"]))
    value_m = int(fin[0])
    plan.close()
    # ---- one instrumented step (same job, per-kernel events on the engine's stream)
    plan = make_plan(job_t)
    _one(plan, world, res)
    barrier()
    stats_last = _lib.stats_dict(res.stats)
    stats_last["_n"], stats_last["_u"] = n, u
    kms = dict(stats_last["kernel_ms"])
    kcnt = dict(stats_last["kernel_count"])
    plan.close()
    if int(fin[0]) != value_m:
        raise RuntimeError("instrumented step disagrees with the timed steps")
    ms = allmax(sum(times) / len(times))  # mean step time over the K timed steps, max over ranks
    clocks = clk.summary()

    # ---- end to end through the public API (host in, host out)
    e2e_steps = args.e2e_steps or args.steps
    e2e_cfg = P.EngineConfig(device=dev, distributed=world > 1)
    r = P.mertens_exact(n, e2e_cfg)  # warm
    wall = []
    for _ in range(e2e_steps):
        barrier()
        t0 = time.perf_counter()
        r = P.mertens_exact(n, e2e_cfg)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall.append(time.perf_counter() - t0)
    e2e_s = allmax(sum(wall) / len(wall))
    K = n // u
    d2h = 8 * K + 8 * len(r._cp_m)
    h2d = 16
    # ---- the anchor config, end to end (the reference arm runs it in full too)
    anchor = None
    if not args.no_anchor:
        na = parse_n(args.anchor_n)
        ra = P.mertens_exact(na, e2e_cfg)  # warm
        aw = []
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            ra = P.mertens_exact(na, e2e_cfg)
            aw.append(time.perf_counter() - t0)
        a_s = allmax(min(aw))
        anchor = {"n": str(na), "M": ra.value, "M_ok": ANCHOR_M.get(na) in (None, ra.value), "u": ra.u,
                  "wall_s": a_s, "value": ra.u / a_s, "unit": "y-values/s",
                  "measured": "end to end through mertens_exact, best of 3"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": u / (ms * 1e-3), "unit": "y-values/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": f"synthetic: n={n} (deterministic, no dataset)", "config": config_block(n, u, world),
        "result": {"M": value_m, "paper": PAPER.get(n), "match": PAPER.get(n) in (None, value_m),
                   "e2e_M": r.value},
    }
    line.update(_rooflines(stats_last, kms, kcnt, torch.cuda.get_device_properties(dev).multi_processor_count))
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(n, u, os.cpu_count() or 1)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "y-values/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {ex!r}"}
    line |= {
        "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": u / e2e_s, "unit": "y-values/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "wall_s": e2e_s, "wall_s_steps": wall},
        "anchor": anchor,
        "gpu_launches": int(statistics.median(launches)) if launches else 0,
        "step_ms": times,
        "clocks": clocks,
        "dist": {"backend": args.dist_backend if world > 1 else None, "world": world},
        "phases_ms": {k: stats_last[k] for k in ("ms_update_head", "ms_sieve_tail", "ms_qgather", "ms_finalize",
                                                  "ms_setup")},
        "kernel_ms_per_step": {k: v for k, v in kms.items() if v},  # the instrumented step (rank 0)
        "work": {"counted_items": stats_last["counted_items"], "dense_items": stats_last["dense_items"],
                 "head_end": stats_last["head_end"], "q_entries": stats_last["q_entries"],
                 "head_cells": stats_last["head_cells"], "tail_cells": stats_last["tail_cells"]},
    }
    if world > 1:
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)


def _rooflines(st, kms, kcnt, nsm):
    """`roofline` of the dominant kernel plus the sieve and counted-walk rooflines.

    sieve tile (k_sieve3): unit = one sieved cell (a y whose mu is computed: every
      y of the head, the odd y of the tail -- the even y follow from mu(2z) =
      -mu(z)); algorithmic bytes = SURVEY.md §8(d)'s 10 B per sieved value (state
      write + read 2 B, M(y) 8 B) against the measured HBM copy bandwidth.  The
      kernel keeps state and prefix on chip, so the ncu DRAM traffic per launch
      (profiles/ncu_metrics.json) is far below that accounting and ncu's
      issue-active is reported beside it.
    counted walk (k_counted): unit = one squarefree m of an element's counted
      range (6/pi^2 of the reference's counted pairs); the implemented
      algorithm needs one fp64-reciprocal DFMA, one IMAD (remainder) and two
      ALU adds (quotient, sign-correction) per unit = 4 issue slots, against the
      measured 4 warp-instructions/clk/SM issue rate -> 32 units/clk/SM."""
    pk = peaks()
    nm = ncu_metrics()
    mhz = pk.get("sm_max_mhz", 1965.0)
    out = {}
    cells = st["head_cells"] + st["tail_cells"]
    tile_ms = kms.get("sieve_tile", 0.0)
    roof_s = None
    if tile_ms > 0:
        n_l = max(1, kcnt.get("sieve_tile", 1))
        avg = tile_ms / n_l
        A = 10 * (cells / n_l) / (avg * 1e-3) / 1e9
        P_ = pk.get("hbm_gbs", 6650.0)
        m = nm.get("k_sieve3", {})
        roof_s = {"kernel": "sieve_tile", "bound": "hbm", "achieved": A, "peak": P_, "unit": "GB/s", "frac": A / P_,
                  "traffic": m.get("dram_bytes_per_launch"),
                  "per_unit": "10 B per sieved value (SURVEY.md §8(d)); a tail cell is a y coprime to 6",
                  "units_per_launch": cells / n_l, "avg_launch_ms": avg, "launches": n_l,
                  "y_covered_per_launch": (st["head_cells"] + 2 * st["tail_cells"]) / n_l,
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in pk else "fallback",
                  "ncu": {k: m.get(k) for k in ("issue_active", "warps_active", "dram_bytes_per_launch",
                                                "shared_bank_conflicts", "source")} if m else None,
                  "timing": "CUDA events around every launch on the engine's stream, one instrumented step "
                            "right after the timed region (events inside the timed steps cost ~4 %)",
                  "note": "state and prefix stay in shared memory: the kernel is bound by shared-memory "
                          "reductions and issue (ncu issue_active), not DRAM; frac compares its cell rate "
                          "with an HBM-bound design of the same algorithmic bytes"}
    roof_u = None
    upd_ms = kms.get("counted", 0.0)
    if upd_ms > 0:
        items = _counted_units(st)
        A = items / (upd_ms * 1e-3) / 1e12
        Pk = 32.0 * nsm * mhz * 1e6 / 1e12
        m = nm.get("k_counted", {})
        roof_u = {"kernel": "counted", "bound": "issue", "achieved": A, "peak": Pk, "unit": "T items/s",
                  "frac": A / Pk,
                  "per_unit": "one squarefree m coprime to 6 of a walk entry (DESIGN.md §2.1: entries walk those "
                              "m up to their largest role limit; 3/pi^2 of the m): DFMA (fp64 reciprocal quotient) + IMAD "
                              "(remainder) + 2 ALU (accumulate, correction) = 4 issue slots",
                  "units_per_step": items,
                  "peak_source": "4 warp-instructions/clk/SM x 32 lanes / 4 slots x SMs x sm_max_mhz; the "
                                 "FP64 and IMAD pipes alone allow 63.8 units/clk/SM (profiles/r01_microbench.txt)",
                  "reference_count_rate": st["counted_items"] / (upd_ms * 1e-3),
                  "ncu": {k: m.get(k) for k in ("issue_active", "warps_active", "pipe_alu", "pipe_fma",
                                                "pipe_fp64", "source")} if m else None}
    dom = max(kms, key=lambda k: kms[k]) if kms else None
    if dom == "counted" and roof_u:
        out["roofline"] = roof_u
    elif roof_s:
        out["roofline"] = roof_s | ({"dominant": dom} if dom != "sieve_tile" else {})
    out["roofline_sieve"] = roof_s
    out["roofline_update"] = roof_u
    return out


def _counted_units(st):
    """Squarefree m coprime to 6 the counted walk processes in one step, in closed form:
    entry j (an element j <= K, or a virtual j = 2k, 3k, 6k > K) walks up to the largest
    of its role limits, mcut_j (own, j <= K) and floor(mcut_{j/d}/d) for d = 2, 3, 6 with
    d | j and j/d <= K; 3/pi^2 of the m are squarefree and coprime to 6.
    mcut follows the engine's counted / dense split (MT_XCUT_ALPHA)."""
    n, u = int(st["_n"]), int(st["_u"])
    K = n // u
    k = np.arange(1, K + 1, dtype=np.uint64)
    v = np.uint64(n) // k
    s = np.sqrt(v.astype(np.float64)).astype(np.uint64)
    s += (s * s < v)  # ceil sqrt (float start, corrected)
    s -= ((s - np.uint64(1)) * (s - np.uint64(1)) >= v) & (s > 0)
    x2 = np.uint64(2) * s
    t = np.uint64(1) << np.ceil(np.log2(x2.astype(np.float64))).astype(np.uint64)
    t = np.where(t < x2, t << np.uint64(1), t)
    t = np.where((t >> np.uint64(1)) >= x2, t >> np.uint64(1), t)
    D = v // np.uint64(u + 1)
    xc = np.maximum(np.maximum(D, v // t), np.uint64(1))
    alpha = float(os.environ.get("MT_XCUT_ALPHA", "0.39"))  # the engine's split
    if alpha > 0:
        xc = np.maximum(np.maximum(D, (alpha * s.astype(np.float64)).astype(np.uint64)), np.uint64(1))
    mc = (v // (xc + np.uint64(1))).astype(np.float64)
    lim = np.zeros(6 * K + 1)
    lim[1:K + 1] = mc
    kk = np.arange(1, K + 1)
    for d in (2, 3, 6):
        lim[d * kk] = np.maximum(lim[d * kk], np.floor(mc / d))
    return 3 / 3.141592653589793 ** 2 * float(lim.sum())


class _SinglePlan:
    """The plan phases at world size 1 (no collectives)."""

    def __init__(self, job):
        import ctypes

        from paper_1108_0135_b200 import _lib

        self.L = _lib.require_device()
        self.h = ctypes.c_void_p()
        _lib.check(self.L.mt_plan_create(ctypes.byref(job), ctypes.byref(self.h)))

    def run(self, res):
        import ctypes

        from paper_1108_0135_b200 import _lib

        mh, tt = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.L.mt_plan_sieve_update(self.h, ctypes.byref(mh), ctypes.byref(tt)))
        _lib.check(self.L.mt_plan_tail_offset(self.h, mh.value))
        _lib.check(self.L.mt_plan_gather(self.h))
        _lib.check(self.L.mt_plan_resolve(self.h, ctypes.byref(res)))

    def close(self):
        if self.h:
            self.L.mt_plan_destroy(self.h)
            self.h = None


def _one(plan, world, res):
    if world > 1:
        from paper_1108_0135_b200 import distributed

        distributed.run_phases(plan, None, res)
    else:
        plan.run(res)


if __name__ == "__main__":
    main()
