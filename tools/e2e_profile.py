"""Where the end-to-end time of mertens_exact(n) goes (host side vs device)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**19
P.mertens_exact(n)  # warm
t = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
r = P.mertens_exact(n)
pr.disable()
print("wall", time.perf_counter() - t, "M", r.value)
d = r.stats.device
print({k: v for k, v in d.items() if k.startswith("ms_")})
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

# ---- the plan phases one by one (host wall per ABI call)
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

from paper_1108_0135_b200 import _lib, engine  # noqa: E402

L = _lib.require_device()
cfg = P.EngineConfig()
u = engine.choose_u(n, 1, cfg.mem_budget, cfg.u_alpha)
job = engine.make_job([n], u, cfg)
res = _lib.MtResult()
fin = np.zeros(n // u, dtype=np.int64)
res.finals = fin.ctypes.data_as(_lib._pi64)
h = ctypes.c_void_p()
T = {}
t = time.perf_counter(); _lib.check(L.mt_plan_create(ctypes.byref(job), ctypes.byref(h))); T["create"] = time.perf_counter() - t
mh, tt = ctypes.c_int64(), ctypes.c_int64()
t = time.perf_counter(); _lib.check(L.mt_plan_sieve_update(h, ctypes.byref(mh), ctypes.byref(tt))); T["sieve_update"] = time.perf_counter() - t
t = time.perf_counter(); _lib.check(L.mt_plan_tail_offset(h, mh.value)); T["tail_offset"] = time.perf_counter() - t
t = time.perf_counter(); _lib.check(L.mt_plan_gather(h)); T["gather"] = time.perf_counter() - t
t = time.perf_counter(); _lib.check(L.mt_plan_resolve(h, ctypes.byref(res))); T["resolve"] = time.perf_counter() - t
t = time.perf_counter(); L.mt_plan_destroy(h); T["destroy"] = time.perf_counter() - t
print({k: round(v, 3) for k, v in T.items()}, "total", round(sum(T.values()), 3))
