#!/usr/bin/env bash
# round-2 check: fast GPU suite, odd-sieve parity, the sieve microbench, and a 1e19 job
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -15
timeout 300 python tools/sieve_bench.py 2.3e12 20 4.64e12 2>&1 | tail -3
timeout 600 python - <<'PY' 2>&1 | tail -20
import time, json
import paper_1108_0135_b200 as P
from paper_1108_0135_b200 import _lib
for n in (10**16, 10**19):
    cfg = P.EngineConfig(engine_flags=_lib.MT_FLAG_TIMING)
    t0 = time.perf_counter(); r = P.mertens_exact(n, cfg); t = time.perf_counter() - t0
    d = r.stats.device
    print(n, r.value, f"{t:.2f} s", {k: round(v, 1) for k, v in d["kernel_ms"].items() if v},
          {k: round(d[k], 1) for k in ("ms_update_head", "ms_sieve_tail", "ms_qgather", "ms_finalize", "ms_setup")},
          "launches", d["kernel_launches"], "tail_cells", d["tail_cells"])
    if n == 10**19:
        print("q10,100,1000", r.quotient(10), r.quotient(100), r.quotient(1000))
PY
