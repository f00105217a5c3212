"""Small jobs for compute-sanitizer (tools/gpu/sanitize.sh): every production
kernel runs at least once -- head sieve + counted/window/sparse walks + Q-gather
+ resolve (mertens_exact), the coprime-to-6 and odd tail sieves with bucket lists
near the 1e19 job's tail, the full-cell production sieve, a 3-target batch, and
the plan API with two ranks' shares computed in one process.
usage: python tools/sanitize_job.py [n=1e9]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402
from paper_1108_0135_b200 import _lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
cfg = P.EngineConfig(seg_log2_head=17, seg_log2_tail=17)
r = P.mertens_exact(n, cfg)
print("mertens_exact", n, r.value)
r = P.mertens_exact(10**12 + 7, P.EngineConfig(seg_log2_head=20, seg_log2_tail=18))
print("mertens_exact 1e12+7", r.value)
mm = P.mertens_exact_multi([n, n + 1, n + 2], cfg)
print("multi", [v.value for v in mm.values()])
L = _lib.lib()
y1 = 4_641_588_833_612 - 10**6
for w in (2, 6):
    keep = np.arange(y1, y1 + 2 * 10**5) % 2 == 1
    if w == 6:
        keep &= np.arange(y1, y1 + 2 * 10**5) % 3 != 0
    mu = np.zeros(int(keep.sum()), np.int8)
    _lib.check(L.mt_sieve_wheel(y1, y1 + 2 * 10**5 - 1, w, _lib.ptr(mu)))
    print("wheel", w, int(mu.sum()))
mu = np.zeros(2 * 10**5, np.int8)
_lib.check(L.mt_sieve_fast(y1, y1 + 2 * 10**5 - 1, _lib.ptr(mu), None))
print("fast", int(mu.sum()))
