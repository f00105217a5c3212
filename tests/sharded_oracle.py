"""TEST INFRASTRUCTURE — a CPU stand-in for the engine's plan (mt_plan_*),
computing the same per-rank partial quantities with the oracle, so that the
real multi-rank driver (paper_1108_0135_b200/distributed.run_phases) and the
sharding algebra can be exercised with world_size > 1 over gloo on CPU.

It restates the device plan's decomposition (mt_engine.cu plan_setup /
mt_plan_*):
  acc_k = sum_{m<=mcut} mu(m) floor(v/m) - M(mcut) xcut        counted walk
        + sum_{d=lo_w}^{xcut} M(floor(v/d))                    windowed dense walk (head)
        + sum_{d=lo}^{dq_hi} Q[k d]                            Q-gather (any y)
with Q[j] = M(floor(n/j)).  The head [0, Y_H) is sieved by every rank and
captures Q directly.  The tail [Y_H, E) is split into w ranges [a, b)
balanced by sieve work (tail_partition); rank r sieves only the y coprime to
the wheel W (2 or 6) of the union of [a/d, b/d), d | W, with one running
prefix P, and captures P at floor(n/(d j)) for its own slice j; then
  M(floor(n/j)) = sum_d mu(d) (P(floor(n/(d j))) - P(a/d - 1)) + M(a - 1),
because M(x) = sum_{d | W} mu(d) C_W(floor(x/d)) with C_W the Moebius sum over
the y coprime to W.
The Q-gather of rank r reads only its own slice and every w-th element's
items in the head part.  Work units are dealt to ranks by element index (the
device deals them by work-unit index; either partition yields the same sums).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import engine_port as E


WHEELS = {2: ((1, 2), (1, -1)), 6: ((1, 2, 3, 6), (1, -1, -1, 1))}


def tail_union(a, b, W=6):
    """mt_engine.cu tail_union: the merged y-intervals [a/d, b/d), d | W."""
    if b <= a:
        return []
    iv = sorted((a // d, b // d) for d in WHEELS[W][0])
    out = []
    for x in iv:
        if out and x[0] <= out[-1][1]:
            out[-1][1] = max(out[-1][1], x[1])
        else:
            out.append([x[0], x[1]])
    return out


def tail_cost(a, b, W=6):
    """mt_engine.cu tail_cost: y covered by a rank owning [a, b)."""
    return sum(e - s for s, e in tail_union(a, b, W))


def tail_partition(H, E_, w, align, W=6):
    """mt_engine.cu tail_partition: boundaries on `align` balancing tail_cost."""
    yb = [H] + [E_] * w
    if w <= 1 or E_ <= H:
        return yb

    def cover(c, out=None):
        a = H
        for r in range(w - 1):
            lo, hi = 0, (E_ - a) // align
            while lo < hi:
                mid = (lo + hi + 1) // 2
                if tail_cost(a, a + mid * align, W) <= c:
                    lo = mid
                else:
                    hi = mid - 1
            a += lo * align
            if out is not None:
                out[r + 1] = a
        return tail_cost(a, E_, W) <= c

    lo, hi = 0, tail_cost(H, E_, W)
    while lo < hi:
        mid = (lo + hi) // 2
        if cover(mid):
            hi = mid
        else:
            lo = mid + 1
    cover(lo, yb)
    yb[w] = E_
    return yb


class ShardedOraclePlan:
    device = torch.device("cpu")
    SENTINEL = -(1 << 30)

    def __init__(self, ns, u, rank, world, Rh=1 << 12, align=None, capture=False, W=6):
        self.ns, self.u, self.rank, self.world = list(ns), u, rank, world
        self.W = W
        self.D, self.S = WHEELS[W]
        align = align or (3 << 10 if W == 6 else 1 << 10)  # every a/d an integer
        self.n_targets = len(self.ns)
        self.H = [E.HarmonicArray(n, u) for n in self.ns]
        ymc = max(int(h.mcut.max()) for h in self.H)
        self.J = [n // (ymc + 1) for n in self.ns]
        self.jq0 = [n // (u + 1) + 1 for n in self.ns]
        for t in range(self.n_targets):
            if self.J[t] < self.jq0[t]:
                self.J[t] = 0
        head_end = ymc
        self.low, self.dq = [], []
        for t, h in enumerate(self.H):
            k = np.arange(1, h.size + 1, dtype=np.uint64)
            jk = np.uint64(self.J[t]) // k
            self.dq.append(np.minimum(jk, h.xcut))
            lw = np.maximum(jk + np.uint64(1), h.lo)
            self.low.append(lw)
            act = lw <= h.xcut
            if act.any():
                head_end = max(head_end, int((h.v[act] // lw[act]).max()))
        head_end = min(head_end, u)
        self.head_lim = -(-(head_end + 1) // align) * align
        self.tail_end = -(-(u + 1) // align) * align if u + 1 > self.head_lim else self.head_lim
        self.ybound = tail_partition(self.head_lim, self.tail_end, world, align, W)
        self.a, self.b = self.ybound[rank], self.ybound[rank + 1]
        self.tail_segs = sum(1 for r in range(world) if self.ybound[r + 1] > self.ybound[r])
        self.y_last = max(self.tail_end, self.head_lim) - 1
        self.M = E.mertens_table(self.y_last)  # M[y-1] = M(y)
        mu = np.diff(np.concatenate([[0], self.M]))
        y = np.arange(1, self.y_last + 1)
        keep = (y % 2 == 1) & ((y % 3 != 0) if W == 6 else True)
        self.O = np.cumsum(np.where(keep, mu, 0))  # O[y-1] = sum of mu over the wheel's y' <= y
        self.U = tail_union(self.a, self.b, W)
        self.Q = [np.full(max(0, self.J[t] - self.jq0[t] + 1), self.SENTINEL, np.int64) for t in range(self.n_targets)]
        self.PD = [None] * self.n_targets
        self._acc = [np.zeros(h.size, np.uint64) for h in self.H]
        self.capture = capture

    def Mof(self, y):
        y = np.asarray(y, dtype=np.int64)
        return np.where(y >= 1, self.M[np.maximum(y, 1) - 1], 0)

    def Oof(self, y):
        y = np.asarray(y, dtype=np.int64)
        return np.where(y >= 1, self.O[np.maximum(y, 1) - 1], 0)

    def Pof(self, x):
        """This rank's running wheel prefix P(x) over the union of [a/d, b/d)."""
        x = np.asarray(x, dtype=np.int64)
        p = np.zeros(x.shape, np.int64)
        for lo, hi in self.U:
            p += np.where(x >= lo, self.Oof(np.minimum(x, hi - 1)) - self.Oof(lo - 1), 0)
        return p

    def _slice(self, t, r):
        """j range of target t owned by rank r (mt_plan::q_slice)."""
        a, b = self.ybound[r], self.ybound[r + 1]
        if a >= b or self.J[t] < self.jq0[t]:
            return None
        lo = max(self.ns[t] // b + 1, self.jq0[t])
        hi = min(self.ns[t] // a, self.J[t])
        return (lo, hi) if lo <= hi else None

    def _mine(self, size):
        return np.arange(size) % self.world == self.rank

    def fingerprint(self):
        return [hash(tuple(self.ns)) & ((1 << 62) - 1), self.u, self.n_targets, 0, 0, 0, 0, self.world]

    def sieve_update(self):
        n_ = self.ns
        for t, h in enumerate(self.H):
            acc = np.zeros(h.size, np.uint64)
            for i in np.flatnonzero(self._mine(h.size)):
                v, mc, xc = int(h.v[i]), int(h.mcut[i]), int(h.xcut[i])
                m = np.arange(1, mc + 1, dtype=np.int64)
                mu = np.diff(np.concatenate([[0], self.Mof(m)]))
                s = int((mu * (v // m)).sum())
                d = np.arange(int(self.low[t][i]), xc + 1, dtype=np.int64)
                s += int(self.Mof(v // d).sum()) if len(d) else 0
                acc[i] = np.uint64(s % (1 << 64))
            self._acc[t] = acc
            if len(self.Q[t]):
                j = np.arange(self.jq0[t], self.J[t] + 1, dtype=np.int64)
                y = n_[t] // j
                head = y < self.head_lim
                self.Q[t][head] = self.Mof(y[head])  # head captures: absolute M
                sl = self._slice(t, self.rank)
                if sl:
                    i0, i1 = sl[0] - self.jq0[t], sl[1] - self.jq0[t] + 1
                    self.Q[t][i0:i1] = self.Pof(y[i0:i1])  # P(floor(n/j))
                    self.PD[t] = [self.Pof((n_[t] // d) // j[i0:i1]) for d in self.D[1:]]  # P(floor(n/(dj)))
        m_head = int(self.Mof(self.head_lim - 1))
        if self.b <= self.a:
            self.s_a = 0
            return m_head, 0
        self.s_a = sum(s * int(self.Pof(self.a // d - 1)) for d, s in zip(self.D, self.S))
        return m_head, sum(s * int(self.Pof(self.b // d - 1) - self.Pof(self.a // d - 1)) for d, s in zip(self.D, self.S))

    def tail_offset(self, off):
        for t in range(self.n_targets):
            sl = self._slice(t, self.rank)
            if sl:
                i0, i1 = sl[0] - self.jq0[t], sl[1] - self.jq0[t] + 1
                self.Q[t][i0:i1] += sum(sg * pd for sg, pd in zip(self.S[1:], self.PD[t])) + (int(off) - self.s_a)
        if self.capture and len(self.Q[0]):  # mask the window to the entries this rank owns
            j = np.arange(self.jq0[0], self.J[0] + 1, dtype=np.int64)
            sl = self._slice(0, self.rank)
            mine = np.zeros(len(j), bool)
            if sl:
                mine |= (j >= sl[0]) & (j <= sl[1])
            if self.rank == 0:
                mine |= j >= self.ns[0] // self.head_lim + 1
            self.Q[0][~mine] = 0
            self._win = torch.from_numpy(self.Q[0].astype(np.int32))

    def cap_window(self):
        return self._win if self.capture and len(self.Q[0]) else None

    def q_slice(self, t, r):
        sl = self._slice(t, r)
        if not sl:
            return None
        return torch.from_numpy(self.Q[t][sl[0] - self.jq0[t]:sl[1] - self.jq0[t] + 1])

    def sync(self):
        if self.capture and len(self.Q[0]):
            self.Q[0] = self._win.numpy().astype(np.int64)

    def gather(self):
        for t, h in enumerate(self.H):
            sl = self._slice(t, self.rank)
            jh = self.ns[t] // self.head_lim + 1
            for i in range(h.size):
                k = i + 1
                d = np.arange(int(h.lo[i]), int(self.dq[t][i]) + 1, dtype=np.int64)
                j = k * d
                own = (j >= sl[0]) & (j <= sl[1]) if sl else np.zeros(len(j), bool)
                take = own | ((j >= jh) & (i % self.world == self.rank))
                q = self.Q[t][j[take] - self.jq0[t]]
                assert (q != self.SENTINEL).all(), "read a quotient-table entry this rank does not own"
                s = int(q.sum())
                if self.rank == 0:  # summation-by-parts term, once per element (k_acc_finish)
                    s -= int(self.Mof(int(h.mcut[i]))) * int(h.xcut[i])
                self._acc[t][i] = np.uint64((int(self._acc[t][i]) + s) % (1 << 64))
        self._acc_all = np.concatenate(self._acc)

    def acc(self):
        return torch.from_numpy(self._acc_all.view(np.int64))

    def resolve(self, res):
        out, o = [], 0
        kc = E.get_kernels("c")
        for h in self.H:
            a = self._acc_all[o:o + h.size].view(np.int64)
            out.append(kc.finalize_recursion(np.ascontiguousarray(a), h.D))
            o += h.size
        res["finals"] = out
        if self.capture and len(self.Q[0]):
            res["window"] = self.Q[0].copy()
