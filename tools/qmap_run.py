"""Builder run of north_star's "all M(floor(n/c))" at scale: the dense quotient map of
n streamed to memory-mapped int32 files, the reference's identity residual over the
whole map (engine.py:606-616) summed in chunks, and spot checks against the paper.
usage: python tools/qmap_run.py 1e19 /dev/shm/qmap  (a RAM-backed path: the map is 2 x 4 sqrt(n) bytes)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402

m, e = sys.argv[1].lower().split("e")
n = int(m) * 10 ** int(e)
path = sys.argv[2] if len(sys.argv) > 2 else "/tmp/qmap"
t0 = time.time()
r = P.mertens_exact(n, P.EngineConfig(quotient_budget=10**12, quotient_map_path=path))
t1 = time.time()
print(f"mertens_exact {t1 - t0:.1f} s (engine ms_total {r.stats.device['ms_total']:.0f})", file=sys.stderr, flush=True)
res = P.mertens_identity_residual(r)
t2 = time.time()
PAPER = {10**19: 899990187, 10**18: -46758740, 10**17: -21830254, 10**16: -3195437}
out = {"n": sys.argv[1], "M": r.value, "map_entries": len(r._qmap) + len(r._small) + len(r._final),
       "qmap_file_bytes": os.path.getsize(path + ".qmap.i32"), "small_file_bytes": os.path.getsize(path + ".small.i32"),
       "identity_residual": res, "wall_exact_s": round(t1 - t0, 1), "wall_residual_s": round(t2 - t1, 1),
       "quotients": {str(c): r.quotient(c) for c in (10, 100, 1000, 10**6, 10**9)},
       "paper": {str(c): PAPER.get(n // c) for c in (10, 100, 1000)},
       "device_phases_ms": {k: round(r.stats.device[k]) for k in ("ms_update_head", "ms_sieve_tail", "ms_qgather",
                                                                   "ms_finalize", "ms_setup")}}
print(json.dumps(out), flush=True)
for f in (".qmap.i32", ".small.i32"):
    os.remove(path + f)
