"""Generate the golden fixtures by running the REFERENCE itself.

Run here (the container that has /root/reference); the outputs are committed
under tests/golden/ so the GPU box (which has no /root/reference) can use
them.  The reference package is built into a scratch copy under /tmp (the
read-only tree is never written):

    python tests/golden/make_golden.py

Outputs:
  golden.npz   arrays (M tables, 1e10 quotient map, per-block apply_block
               state, sieve blocks, divisor constants)
  golden.json  scalar values (paper Table 1, SPEC examples, reference runs)
"""

import json
import os
import shutil
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/mertens_refbuild"


def reference():
    if not os.path.exists(os.path.join(SCRATCH, "src")):
        shutil.copytree("/root/reference/pkg", SCRATCH)
        subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import mertens  # noqa: E402

    return mertens


def main():
    mertens = reference()
    from mertens import _kernels, engine, sieve  # noqa: E402

    nat = _kernels.get_backend("native")
    cfg = mertens.EngineConfig(backend="native")
    arrays, scalars = {}, {}

    # AC1: every n <= 10^4 and 100 seeded n <= 10^8 (seed 42 as SPEC.md:658)
    arrays["m_upto_1e4"] = np.array([mertens.mertens_exact(n, cfg).value for n in range(1, 10001)], np.int64)
    rng = np.random.default_rng(42)
    ns = sorted(set(int(x) for x in rng.integers(1, 10**8 + 1, size=100)))
    arrays["seeded_n"] = np.array(ns, np.uint64)
    arrays["seeded_m"] = np.array([mertens.mertens_exact(n, cfg).value for n in ns], np.int64)

    # C1: M(10^10) and its full quotient map (engine.py:200-252)
    r = mertens.mertens_exact(10**10, cfg)
    arrays["e10_final"] = r._final.astype(np.int64)
    arrays["e10_cp_q"] = r._cp_q.astype(np.uint64)
    arrays["e10_cp_m"] = r._cp_m.astype(np.int64)
    scalars["e10"] = {"value": r.value, "u": r.u, "counted_items": r.stats.counted_items,
                      "dense_items": r.stats.dense_items, "blocks": r.stats.blocks,
                      "divtable_released_at": r.stats.divtable_released_at}
    # tails (acc before finalize) + D for the resolve kernel
    job = engine._ExactJob([10**10], cfg)
    job.run()
    arrays["e10_tails"] = job.arrays[0].acc.copy()
    arrays["e10_D"] = job.arrays[0].D.copy()

    # multi mode (engine.py:424-446)
    mm = mertens.mertens_exact_multi([10**10, 10**10 + 1, 10**10 + 2], cfg)
    scalars["multi_e10"] = {str(k): v.value for k, v in mm.items()}
    arrays["multi_e10_final_1"] = mm[10**10 + 1]._final.astype(np.int64)

    # other single targets, reference runs in this container
    for e in (11, 12):
        scalars[f"e{e}"] = mertens.mertens_exact(10**e, cfg).value
    for n in (7_766_842_813, 999_999_999_989, 2**40 + 12345):
        scalars[str(n)] = mertens.mertens_exact(n, cfg).value

    # per-block apply_block state (_native.pyx:227-310) at n = 10^9, block_len 2^16
    n9 = 10**9
    job = engine._ExactJob([n9], engine.EngineConfig(backend="native", block_len=1 << 16))
    snaps = []

    def snap(tag):
        a = job.arrays[0]
        arrays[f"blk_{tag}_acc"] = a.acc.copy()
        arrays[f"blk_{tag}_dnext"] = a.dnext.copy()
        arrays[f"blk_{tag}_ynext"] = a.ynext.copy()
        snaps.append({"tag": tag, "next_y1": job.next_y1, "m_running": job.m_running,
                      "counted": job.stats.counted_items, "dense": job.stats.dense_items})

    job.run(stop_after_blocks=1); snap("b1")
    job.run(stop_after_blocks=3); snap("b3")
    job.run(stop_after_blocks=40); snap("b40")
    job.run(); snap("end")
    scalars["blk"] = {"n": n9, "u": job.u, "block_len": 1 << 16, "snaps": snaps,
                      "value": int(job.finalize()[0].final[0])}

    # sieve blocks (AC5-style): seeded blocks up to 1e12, mu and raw log-prime states
    rng = np.random.default_rng(7)
    y1s = sorted(int(x) for x in rng.integers(2, 10**12, size=12)) + [2, 13859, 2**32 - 5000]
    L = 5000
    table = sieve.build_log_table(sieve.generate_primes(sieve.ceil_sqrt(10**12 + L) + 1))
    wheel = sieve.build_wheel()
    mus, sts = [], []
    for y1 in y1s:
        y2 = y1 + L - 1
        mus.append(sieve.sieve_block_logprime(y1, y2, table, wheel, backend="native").mu)
        plim = sieve.ceil_sqrt(y2) + 1
        sel = table.primes <= plim
        sts.append(nat.logprime_states(y1, y2, table.primes[sel], table.logs[sel], wheel.residues))
    arrays["sieve_y1"] = np.array(y1s, np.uint64)
    arrays["sieve_mu"] = np.stack(mus)
    arrays["sieve_states"] = np.stack(sts)
    arrays["wheel"] = wheel.residues.copy()
    arrays["logs_first"] = table.logs[:64].copy()

    # divisor constants (fastdiv.py:46-70 / _native.pyx:32-68)
    mg, sh, sc = nat.build_divisor_arrays(4096)
    arrays["div_magic"], arrays["div_shift"], arrays["div_scheme"] = mg, sh, sc

    # paper Table 1 and extreme and SPEC examples
    scalars["paper"] = {"1e16": -3195437, "1e17": -21830254, "1e18": -46758740, "1e19": 899990187,
                        "1e20": 461113106, "1e21": 3395895277, "1e22": -2061910120,
                        "11609864264058592345": -1995900927}
    scalars["reference_measured_survey"] = {"1e13": 599582, "1e14": -875575, "1e15": -3216373,
                                            "1e16": -3195437, "1e8": 1928}
    scalars["spec"] = {"1": 1, "2": 0, "100": 1, "10000": -23, "1000000": 212, "1000000000": -222}
    scalars["generated"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(scalars, f, indent=1)
    print("wrote", sorted(arrays), os.path.getsize(os.path.join(HERE, "golden.npz")))


if __name__ == "__main__":
    main()
