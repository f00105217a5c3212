"""TEST INFRASTRUCTURE — a CPU stand-in for the engine's plan (mt_plan_*),
computing the same per-rank partial quantities with the oracle, so that the
real multi-rank driver (paper_1108_0135_b200/distributed.run_phases) and the
sharding algebra can be exercised with world_size > 1 over gloo on CPU.

It restates the device plan's decomposition (mt_engine.cu plan_setup /
mt_plan_*):
  acc_k = sum_{m<=mcut} mu(m) floor(v/m) - M(mcut) xcut        counted walk
        + sum_{d=lo_w}^{xcut} M(floor(v/d))                    windowed dense walk (head)
        + sum_{d=lo}^{dq_hi} Q[k d]                            Q-gather (any y)
with Q[j] = M(floor(n/j)) captured while sieving; the head [0, Y_H) is sieved
by every rank, the tail segments are split contiguously and prefixed locally.
Work units are dealt to ranks by element index (the device deals them by
work-unit index; either partition yields the same sums).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import engine_port as E


class ShardedOraclePlan:
    device = torch.device("cpu")

    def __init__(self, ns, u, rank, world, Rh=1 << 12, Rt=1 << 14):
        self.ns, self.u, self.rank, self.world = list(ns), u, rank, world
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
        self.Rh, self.Rt = Rh, Rt
        self.head_lim = -(-(head_end + 1) // Rh) * Rh
        self.tail_segs = max(0, -(-(u + 1 - self.head_lim) // Rt))
        self.y_last = self.head_lim + self.tail_segs * Rt - 1
        self.M = E.mertens_table(self.y_last)  # M[y-1] = M(y)
        self.Q = [np.full(max(0, self.J[t] - self.jq0[t] + 1), -(1 << 30), np.int32) for t in range(self.n_targets)]
        self._acc = [np.zeros(h.size, np.uint64) for h in self.H]

    def Mof(self, y):
        y = np.asarray(y, dtype=np.int64)
        return np.where(y >= 1, self.M[np.maximum(y, 1) - 1], 0)

    def _tail_y(self, s):
        return self.head_lim + s * self.Rt

    def _slice(self, t, r):
        """j range of target t captured in rank r's tail (mt_plan::q_slice)."""
        s0, s1 = self.tail_segs * r // self.world, self.tail_segs * (r + 1) // self.world
        if s0 >= s1 or self.J[t] < self.jq0[t]:
            return None
        ya, yb = self._tail_y(s0), self._tail_y(s1) - 1
        lo = max(self.ns[t] // (yb + 1) + 1, self.jq0[t])
        hi = min(self.ns[t] // ya, self.J[t])
        return (lo, hi) if lo <= hi else None

    def _mine(self, size):
        return np.arange(size) % self.world == self.rank

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
            # captures: head (absolute) and this rank's tail (local prefix)
            if len(self.Q[t]):
                j = np.arange(self.jq0[t], self.J[t] + 1, dtype=np.int64)
                y = n_[t] // j
                head = y < self.head_lim
                self.Q[t][head] = self.Mof(y[head])
                sl = self._slice(t, self.rank)
                if sl:
                    s0 = self.tail_segs * self.rank // self.world
                    base = int(self.Mof(self._tail_y(s0) - 1))
                    a, b = sl[0] - self.jq0[t], sl[1] - self.jq0[t] + 1
                    self.Q[t][a:b] = self.Mof(y[a:b]) - base
        s0 = self.tail_segs * self.rank // self.world
        s1 = self.tail_segs * (self.rank + 1) // self.world
        m_head = int(self.Mof(self.head_lim - 1))
        t_local = int(self.Mof(self._tail_y(s1) - 1) - self.Mof(self._tail_y(s0) - 1)) if s1 > s0 else 0
        return m_head, t_local

    def tail_offset(self, off):
        for t in range(self.n_targets):
            sl = self._slice(t, self.rank)
            if sl:
                self.Q[t][sl[0] - self.jq0[t]:sl[1] - self.jq0[t] + 1] += np.int32(off)

    def q_slice(self, t, r):
        sl = self._slice(t, r)
        if not sl:
            return None
        return torch.from_numpy(self.Q[t][sl[0] - self.jq0[t]:sl[1] - self.jq0[t] + 1])

    def sync(self):
        pass

    def gather(self):
        for t, h in enumerate(self.H):
            assert (self.Q[t] != -(1 << 30)).all(), "a quotient-table slice was never filled"
            for i in range(h.size):
                s = 0
                if i % self.world == self.rank:
                    k = i + 1
                    d = np.arange(int(h.lo[i]), int(self.dq[t][i]) + 1, dtype=np.int64)
                    s = int(self.Q[t][k * d - self.jq0[t]].astype(np.int64).sum()) if len(d) else 0
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
