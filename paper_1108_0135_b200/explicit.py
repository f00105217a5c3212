"""The paper's approximate algorithm: the explicit formula (Eq. 2)

    M(x) / sqrt(x)  ~  q_n(x) = 2 sum_{i<=n} a_i cos(z_i ln x + b_i),

with z_i = Im rho_i, a_i = 1/|rho_i zeta'(rho_i)|, b_i = -arg(rho_i zeta'(rho_i)) for the
nontrivial zeta zeros rho_i -- the operations of SPEC.md's `zero-table` (:351-422) and
`explicit-formula` (:423-497) modules: load_table, rebase, q_eval, q_batch, q_sigma,
residual_stats.  The cosine sums run on the GPU (mt_q_batch / mt_q_points, csrc/mt_qsum.cu,
fp64); the phase shift b'_i = (b_i + z_i x0) mod 2 pi is done on the host in exact
decimal arithmetic ("decimal fixed-point with 50 digits ... pi to 60
digits"), so evaluating at delta = ln x - x0 keeps the GPU's arguments small.

The zeros are data, not computed here (SPEC.md: "zeta and zeta' are NOT computed by this
artifact"); the format is the reference's `data/zeros_*.txt`: whitespace-separated
decimal triples `z a b`, one per line, `#` comments.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from decimal import Decimal, getcontext

import numpy as np

from . import _lib

# pi to 60 digits (SPEC.md:405 design decision)
_PI60 = Decimal("3.14159265358979323846264338327950288419716939937510582097494")


class ZeroTableError(ValueError):
    """Malformed zero table (parse error, non-monotonic z, b outside [-pi, pi])."""


@dataclass
class ZeroTable:
    """Ordered (z, a, b) records, decimal-string masters plus fp64 copies."""

    z_str: list = field(default_factory=list)
    a_str: list = field(default_factory=list)
    b_str: list = field(default_factory=list)
    source: str = ""

    def __post_init__(self):
        self.z = np.array([float(s) for s in self.z_str], np.float64)
        self.a = np.array([float(s) for s in self.a_str], np.float64)
        self.b = np.array([float(s) for s in self.b_str], np.float64)

    def __len__(self):
        return len(self.z_str)

    @classmethod
    def from_arrays(cls, z, a, b, source="arrays"):
        """From binary floats (their exact decimal expansions become the masters)."""
        return cls([repr(float(x)) for x in z], [repr(float(x)) for x in a], [repr(float(x)) for x in b], source)


@dataclass
class ShiftedTable:
    """(z, a, b') with b'_i = (b_i + z_i x0) mod 2 pi in [-pi, pi)."""

    x0: Decimal
    z: np.ndarray
    a: np.ndarray
    b: np.ndarray

    def __len__(self):
        return len(self.z)


def load_table(source, name: str = "") -> ZeroTable:
    """Parse `z a b` triples; `source` is a path or an iterable of lines."""
    lines = open(source).read().splitlines() if isinstance(source, str) else list(source)
    zs, as_, bs = [], [], []
    prev = None
    for no, raw in enumerate(lines, 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        f = line.split()
        if len(f) != 3:
            raise ZeroTableError(f"line {no}: expected 3 fields, got {len(f)}")
        try:
            z, a, b = (Decimal(x) for x in f)
        except Exception as ex:  # noqa: BLE001 - decimal's InvalidOperation and friends
            raise ZeroTableError(f"line {no}: not a decimal triple ({ex})") from None
        if prev is not None and z <= prev:
            raise ZeroTableError(f"line {no}: z not strictly increasing")
        if a <= 0:
            raise ZeroTableError(f"line {no}: a must be positive")
        if not (-_PI60 <= b < _PI60):
            raise ZeroTableError(f"line {no}: b outside [-pi, pi)")
        prev = z
        zs.append(f[0]); as_.append(f[1]); bs.append(f[2])
    return ZeroTable(zs, as_, bs, name or (source if isinstance(source, str) else "stream"))


def rebase(table: ZeroTable, x0) -> ShiftedTable:
    """b'_i = (b_i + z_i x0) mod 2 pi, reduced into [-pi, pi), at 60-digit working
    precision from the decimal masters, rounded once to fp64."""
    x0 = Decimal(str(x0)) if not isinstance(x0, Decimal) else x0
    if x0 < 0:
        raise ValueError("x0 must be >= 0")
    ctx = getcontext().copy()
    ctx.prec = 60
    two_pi = 2 * _PI60
    b2 = np.empty(len(table), np.float64)
    for i, (zs, bs) in enumerate(zip(table.z_str, table.b_str)):
        t = ctx.add(Decimal(bs), ctx.multiply(Decimal(zs), x0))
        r = ctx.subtract(t, ctx.multiply(two_pi, ctx.divide_int(ctx.add(t, _PI60), two_pi)))
        if r < -_PI60:
            r += two_pi
        if r >= _PI60:
            r -= two_pi
        b2[i] = float(r)
    return ShiftedTable(x0, table.z.copy(), table.a.copy(), b2)


def _check(shifted: ShiftedTable, n_terms: int):
    if n_terms > len(shifted):
        raise ValueError(f"n_terms={n_terms} exceeds the table size {len(shifted)}")


def q_batch(shifted: ShiftedTable, n_terms: int, delta_start: float, step: float, count: int) -> np.ndarray:
    """q_n at delta_j = delta_start + j*step, j < count, on the GPU."""
    _check(shifted, n_terms)
    out = np.zeros(int(count), np.float64)
    if count:
        L = _lib.require_device()
        z, a, b = (np.ascontiguousarray(x[:n_terms]) for x in (shifted.z, shifted.a, shifted.b))
        _lib.check(L.mt_q_batch(_lib.ptr(z), _lib.ptr(a), _lib.ptr(b), n_terms, float(delta_start), float(step),
                                int(count), _lib.ptr(out)))
    return out


def q_points(shifted: ShiftedTable, n_terms: int, deltas) -> np.ndarray:
    """q_n at arbitrary delta = ln x - x0 values, on the GPU."""
    _check(shifted, n_terms)
    d = np.ascontiguousarray(np.asarray(deltas, np.float64))
    out = np.zeros(len(d), np.float64)
    if len(d):
        L = _lib.require_device()
        z, a, b = (np.ascontiguousarray(x[:n_terms]) for x in (shifted.z, shifted.a, shifted.b))
        _lib.check(L.mt_q_points(_lib.ptr(z), _lib.ptr(a), _lib.ptr(b), n_terms, _lib.ptr(d), len(d), _lib.ptr(out)))
    return out


def q_eval(shifted: ShiftedTable, n_terms: int, delta: float = 0.0) -> float:
    """2 sum_{i<=n_terms} a_i cos(z_i delta + b'_i)."""
    return float(q_points(shifted, n_terms, [delta])[0])


def q_at(table: ZeroTable, x: int, n_terms: int | None = None) -> float:
    """q_n(x) for an integer x: rebased at x0 = ln x (exact decimal log), delta = 0."""
    n_terms = len(table) if n_terms is None else n_terms
    ctx = getcontext().copy()
    ctx.prec = 60
    return q_eval(rebase(table, ctx.ln(Decimal(x))), n_terms, 0.0)


def q_sigma(table: ZeroTable, n_terms: int | None = None) -> float:
    """sqrt(2 sum_{i<=n_terms} a_i^2) (PAPER §7: ~0.17 for 10^6 zeros)."""
    n_terms = len(table) if n_terms is None else n_terms
    if n_terms > len(table):
        raise ValueError("n_terms exceeds the table size")
    a = table.a[:n_terms]
    return math.sqrt(2.0 * float(np.dot(a, a)))


def residual_stats(pairs) -> dict:
    """Sample mean and standard deviation (n - 1) of exact - approx."""
    r = np.array([float(e) - float(q) for e, q in pairs], np.float64)
    if len(r) < 2:
        raise ValueError("residual_stats needs at least 2 pairs")
    return {"mean": float(r.mean()), "std": float(r.std(ddof=1)), "n": int(len(r))}
