"""Paper-value evidence runs on one GPU: python tools/paper_run.py 1e21 [1e22 ...]
Prints M(n), the paper's value, quotient(10) and (100), wall and device phase times."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402

# Table 1; 10^21 sign corrected (the table prints +3395895277; see
# tests/test_explicit_formula_check.py and profiles/r01_paper_e21_*.json)
PAPER = {10**16: -3195437, 10**17: -21830254, 10**18: -46758740, 10**19: 899990187,
         10**20: 461113106, 10**21: -3395895277, 10**22: -2061910120}
for arg in sys.argv[1:]:
    m, e = arg.lower().split("e")
    n = int(m) * 10 ** int(e)
    t = time.time()
    r = P.mertens_exact(n, P.EngineConfig(engine_flags=4))
    dt = time.time() - t
    d = r.stats.device
    out = {"n": arg, "M": r.value, "paper": PAPER.get(n), "match": r.value == PAPER.get(n),
           "q10": r.quotient(10), "q10_paper": PAPER.get(n // 10), "q100": r.quotient(100),
           "q100_paper": PAPER.get(n // 100), "u": r.u, "K": len(r._final), "wall_s": round(dt, 1),
           "device_ms": {k: round(v) for k, v in d["kernel_ms"].items()},
           "phases_ms": {k: round(d[k]) for k in ("ms_update_head", "ms_sieve_tail", "ms_qgather", "ms_finalize", "ms_setup")}}
    print(json.dumps(out), flush=True)
