"""Fixture for the explicit-formula tests (tests/test_explicit_formula.py): the
reference's bundled zeta-zero constants (pkg/src/mertens/data/zeros_2000.txt,
mpmath dps=45, 30 significant digits) as float64 arrays, plus q_2000 at the
paper's Table 1 arguments evaluated in exact decimal arithmetic (60 digits) as
the golden values.  Run in the container where /root/reference exists:

    python tests/golden/make_zeros.py
"""
import os
from decimal import Decimal, getcontext

import numpy as np

SRC = "/root/reference/pkg/src/mertens/data/zeros_2000.txt"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "zeros_2000.npz")
XS = [10**16, 10**17, 10**18, 10**19, 10**20, 10**21, 10**22, 11609864264058592345, 7766842813]


def main():
    rows = [l.split() for l in open(SRC) if l.strip() and not l.startswith("#")]
    z = np.array([float(r[0]) for r in rows])
    a = np.array([float(r[1]) for r in rows])
    b = np.array([float(r[2]) for r in rows])
    getcontext().prec = 60
    # q at x = 2 sum a cos(z ln x + b) with the phase reduced mod 2 pi in decimal
    pi = Decimal("3.14159265358979323846264338327950288419716939937510582097494")
    q = []
    for x in XS:
        lx = Decimal(x).ln()
        s = 0.0
        for r in rows:
            t = Decimal(r[2]) + Decimal(r[0]) * lx
            t -= 2 * pi * ((t + pi) // (2 * pi))
            s += float(Decimal(r[1])) * np.cos(float(t))
        q.append(2 * s)
    np.savez_compressed(OUT, z=z, a=a, b=b, xs=np.array([str(x) for x in XS]), q=np.array(q))
    print(OUT, len(z), dict(zip(map(str, XS), q)))


if __name__ == "__main__":
    main()
