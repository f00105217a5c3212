"""Multi-GPU exact job: one process per GPU, collectives over torch.distributed
(NCCL over NVLink/NVSwitch on the box; gloo in the CPU tests).

The reference is single-process; the y-axis split is new work
(SURVEY.md §8(e)).  The engine plan (include/mertens_sm100.h, "plan API") runs
the job in four device phases; this module performs the three exchanges
between them, and nothing else:

  1. sieve_update  every rank sieves the head [0, Y_H) redundantly, takes every
                   w-th work unit of the head update, and sieves its own
                   contiguous share of the tail segments with a LOCAL prefix.
     -> all_gather of the G tail totals T_h (int64, G values):
        offset_r = M(Y_H - 1) + sum_{h<r} T_h          (the deferred M offset)
  2. tail_offset   Q[j] += offset_r on the quotient-table slice whose
                   quotients floor(n/j) fall in rank r's tail.
     -> broadcast of every rank's Q slice (int32, contiguous in j) so that each
        rank holds the complete table M(floor(n/j)).
  3. gather        every w-th chunk of the dense items k*d <= J from Q; rank 0
                   adds the summation-by-parts term -M(mcut)*xcut.
     -> all_reduce(sum) of the K-entry accumulator (int64 two's complement ==
        the engine's mod-2^64 arithmetic).
  4. resolve       level-parallel finalize on every rank; rank 0's outputs are
                   the job's outputs.

Every M value is independent of the rank count: the partition only decides
which rank adds which term of the same mod-2^64 sums.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def world():
    """(rank, world_size) of the default process group, (0, 1) without one."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except ImportError:
        pass
    return 0, 1


class _CudaArray:
    """Zero-copy view of engine-owned device memory for torch (CUDA array interface v3)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None,
        }


def _device_view(ptr: int, count: int, typestr: str, device):
    import torch

    t = torch.as_tensor(_CudaArray(ptr, count, typestr), device=device)
    if count and t.data_ptr() != ptr:
        raise RuntimeError("torch copied an engine buffer instead of aliasing it")
    return t


class DevicePlan:
    """The engine's plan handle (C ABI) with the tensors the collectives need."""

    def __init__(self, job: "_lib.MtJob"):
        import torch

        self.L = _lib.require_device()
        self.h = ctypes.c_void_p()
        _lib.check(self.L.mt_plan_create(ctypes.byref(job), ctypes.byref(self.h)))
        self.device = torch.device("cuda", torch.cuda.current_device() if job.device < 0 else job.device)
        self.n_targets = job.n_targets

    def sieve_update(self):
        mh, tt = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.L.mt_plan_sieve_update(self.h, ctypes.byref(mh), ctypes.byref(tt)))
        return mh.value, tt.value

    def tail_offset(self, off: int):
        _lib.check(self.L.mt_plan_tail_offset(self.h, int(off)))

    def q_slice(self, target: int, rank: int):
        p, c = ctypes.c_void_p(), ctypes.c_uint64()
        _lib.check(self.L.mt_plan_q_slice(self.h, target, rank, ctypes.byref(p), ctypes.byref(c)))
        if not c.value:
            return None
        return _device_view(p.value, c.value, "<i4", self.device)

    def acc(self):
        p, c = ctypes.c_void_p(), ctypes.c_uint64()
        _lib.check(self.L.mt_plan_acc(self.h, ctypes.byref(p), ctypes.byref(c)))
        return _device_view(p.value, c.value, "<i8", self.device) if c.value else None

    def gather(self):
        _lib.check(self.L.mt_plan_gather(self.h))

    def resolve(self, res):
        _lib.check(self.L.mt_plan_resolve(self.h, ctypes.byref(res) if res is not None else None))

    def sync(self):
        import torch

        torch.cuda.synchronize(self.device)

    def close(self):
        if self.h:
            self.L.mt_plan_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tail_offsets(m_head: int, totals) -> list[int]:
    """offset_r = M(Y_H - 1) + sum_{h<r} T_h (SURVEY.md §8(e) collective (i))."""
    out, run = [], int(m_head)
    for t in totals:
        out.append(run)
        run += int(t)
    return out


def _staged(t, fn, group):
    """Run collective `fn` on `t`; gloo (the CPU tests' backend) gets a host copy."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend(group) == "gloo":
        c = t.cpu()
        fn(c)
        t.copy_(c)
    else:
        fn(t)


def run_phases(plan, group=None, res=None):
    """Drive one job through the plan's phases with the three exchanges.
    `plan` is a DevicePlan (or the CPU stand-in of the tests) of THIS rank."""
    import torch
    import torch.distributed as dist

    rank, size = dist.get_rank(group), dist.get_world_size(group)
    gloo = dist.get_backend(group) == "gloo"
    dev = torch.device("cpu") if gloo else getattr(plan, "device", torch.device("cpu"))
    m_head, t_local = plan.sieve_update()
    tot = torch.tensor([t_local], dtype=torch.int64, device=dev)
    allt = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(size)]
    dist.all_gather(allt, tot, group=group)
    offs = tail_offsets(m_head, [int(t.item()) for t in allt])
    plan.tail_offset(offs[rank])
    for t in range(plan.n_targets):
        for r in range(size):
            view = plan.q_slice(t, r)
            if view is not None:
                src = dist.get_global_rank(group, r) if group is not None else r
                _staged(view, lambda x: dist.broadcast(x, src=src, group=group), group)
    plan.sync()
    plan.gather()
    acc = plan.acc()
    if acc is not None:
        _staged(acc, lambda x: dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group), group)
    plan.sync()
    plan.resolve(res)
    return offs
