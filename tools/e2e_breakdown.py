"""Where the end-to-end time of mertens_exact(n) goes beyond the device phases:
host quotient targets, plan setup, device phases, copies, plan teardown."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402
from paper_1108_0135_b200 import engine as E  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**19
P.mertens_exact(n)  # warm (CUDA context, first allocations)
for _ in range(2):
    t0 = time.perf_counter()
    u = P.choose_u(n)
    K = n // u
    cp_q = E._quotient_targets(n, K, u, 4_000_000)
    t1 = time.perf_counter()
    r = P.mertens_exact(n)
    t2 = time.perf_counter()
    d = r.stats.device
    dev = d["ms_update_head"] + d["ms_sieve_tail"] + d["ms_qgather"] + d["ms_finalize"]
    print(f"targets {1e3*(t1-t0):.0f} ms; mertens_exact {1e3*(t2-t1):.0f} ms = setup {d['ms_setup']:.0f} + device "
          f"{dev:.0f} + mt_run other {d['ms_total'] - dev - d['ms_setup']:.0f} + outside mt_run "
          f"{1e3*(t2-t1) - d['ms_total']:.0f} ms")
