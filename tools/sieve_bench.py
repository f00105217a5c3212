"""Time the production sieve alone (tail mode) at a given y: per-kernel ms,
cells/s and y/s, full cells vs the wheel-2 and wheel-6 tail sieves.
usage: python tools/sieve_bench.py [Y0=2.3e12] [nseg=20] [y_last=4.64e12]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_0135_b200 import _lib  # noqa: E402

Y0 = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2_300_000_000_000
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ylast = int(float(sys.argv[3])) if len(sys.argv) > 3 else 4_641_588_833_612
Y0 -= Y0 % (1 << 18)
L = _lib.require_device()
ms = np.zeros(8, np.float64)
Y0 -= Y0 % (9 << 18)
for wheel in (1, 2, 6):
    for rep in range(2):
        _lib.check(L.mt_sieve_bench2(Y0, nseg, ylast, wheel, _lib.ptr(ms)))
    cells = nseg * 148 * 6 * (1 << 17)
    ys = cells * (3 if wheel == 6 else wheel)
    tot = ms[0] + ms[1] + ms[6]
    print(f"{os.environ.get('MT_LIB', 'default')} wheel {wheel}: Y0={Y0:.3e} cells={cells:.3e} "
          f"tile {ms[0]:.2f} ms fill {ms[1]:.2f} ms finish {ms[6]:.2f} ms total {tot:.2f} ms -> "
          f"{cells / tot / 1e6:.3e} cells/ms, {ys / tot / 1e9:.3e} y/s (x1e12); tile-only {cells / ms[0] / 1e6:.3e}")
