"""ORACLE — TEST INFRASTRUCTURE ONLY.

fp64 NumPy restatement of the explicit formula (Eq. 2;
SPEC.md:423-497 q_eval / q_batch / q_sigma): q_n(delta) = 2 sum_{i<n} a_i
cos(z_i delta + b'_i), summed in ascending i, one transcendental per term and
point.  The product path is csrc/mt_qsum.cu (GPU); only tests/ use this.
Pinned by tests/golden/zeros_2000.npz (q_2000 at Table 1's x in 60-digit decimal
phase arithmetic, tests/golden/make_zeros.py)."""
import numpy as np


def q_points(z, a, b, n_terms, deltas):
    z, a, b = (np.asarray(x, np.float64)[:n_terms] for x in (z, a, b))
    d = np.asarray(deltas, np.float64)
    out = np.empty(len(d))
    for j, dj in enumerate(d):
        out[j] = 2.0 * float(np.sum(a * np.cos(z * dj + b)))
    return out


def q_batch(z, a, b, n_terms, delta_start, step, count):
    return q_points(z, a, b, n_terms, delta_start + step * np.arange(count, dtype=np.float64))


def q_sigma(a, n_terms):
    a = np.asarray(a, np.float64)[:n_terms]
    return float(np.sqrt(2.0 * np.sum(a * a)))
