"""Multi-GPU exact job: one process per GPU, collectives over torch.distributed
(NCCL over NVLink/NVSwitch on the box; gloo in the CPU tests).

The reference is single-process; the y-axis split is new work
(DESIGN.md §5).  The engine plan (include/mertens_sm100.h,
"plan API") runs the job in four device phases; this module performs the
exchanges between them, and nothing else:

  0. fingerprint   all ranks must run the same job: an all_gather of a job
                   fingerprint (targets, u, captures, flags) -> ContractViolationError
                   on any mismatch, before any device work
  1. sieve_update  every rank sieves the head [0, Y_H) redundantly, takes every
                   w-th work unit of the head update, and sieves the odd y of
                   its own tail range [a_r, b_r) and of its half [a_r/2, b_r/2)
                   with a LOCAL prefix (M(x) = O(x) - O(x/2), O = odd-y sum).
     -> all_gather of the G range totals T_h (int64, G values):
        offset_r = M(Y_H - 1) + sum_{h<r} T_h          (the deferred M offset)
  2. tail_offset   Q[j] = M(floor(n/j)) on the quotient-table slice whose
                   quotients fall in rank r's range.
     -> only when quotient captures were requested: sum-reduction of the
        capture window (each rank holds its own entries, zeros elsewhere), so
        the M(floor(n/c)) outputs are complete on every rank
  3. gather        the dense items k*d <= J whose table entry is in rank r's own
                   slice, plus every w-th chunk of those in the replicated head
                   part; rank 0 adds the summation-by-parts term -M(mcut)*xcut.
     -> all_reduce(sum) of the K-entry accumulator (int64 two's complement ==
        the engine's mod-2^64 arithmetic).  This is the
        only bulk collective of the job.
  4. resolve       level-parallel finalize on every rank; rank 0's outputs are
                   the job's outputs.

Every M value is independent of the rank count: the partition only decides
which rank adds which term of the same mod-2^64 sums.
"""

from __future__ import annotations

import ctypes

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
        self._fp = job_fingerprint(job)

    def sieve_update(self):
        mh, tt = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.L.mt_plan_sieve_update(self.h, ctypes.byref(mh), ctypes.byref(tt)))
        return mh.value, tt.value

    def tail_offset(self, off: int):
        _lib.check(self.L.mt_plan_tail_offset(self.h, int(off)))

    def fingerprint(self):
        return self._fp

    def cap_window(self):
        p, c = ctypes.c_void_p(), ctypes.c_uint64()
        _lib.check(self.L.mt_plan_cap_window(self.h, ctypes.byref(p), ctypes.byref(c)))
        return _device_view(p.value, c.value, "<i4", self.device) if c.value else None

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


def job_fingerprint(job) -> list[int]:
    """Eight int64 words that every rank of one sharded job must agree on."""
    import hashlib

    ns = [(int(job.n_hi[i]) << 64) | int(job.n_lo[i]) for i in range(job.n_targets)]
    h = hashlib.sha256(",".join(map(str, ns)).encode()).digest()
    words = [int.from_bytes(h[:7], "little"), int(job.u), int(job.n_targets), int(job.cap_c_lo), int(job.cap_c_hi),
             int(job.cap_small), int(job.flags) & ~_lib.MT_FLAG_TIMING,
             (int(job.seg_log2_head) << 32) | (int(job.seg_log2_tail) << 16) | int(job.shard_world)]
    return [w & ((1 << 63) - 1) for w in words]


def check_same_job(plan, group=None, device=None):
    """All ranks must run the same job; a mismatch (e.g. every rank computing a
    different n under torchrun) raises ContractViolationError on every rank."""
    import torch
    import torch.distributed as dist

    from .errors import ContractViolationError

    size = dist.get_world_size(group)
    fp = torch.tensor(plan.fingerprint(), dtype=torch.int64, device=device)
    allfp = [torch.zeros_like(fp) for _ in range(size)]
    dist.all_gather(allfp, fp, group=group)
    if any(not torch.equal(a, allfp[0]) for a in allfp):
        raise ContractViolationError("ranks of the process group run different exact jobs "
                                     "(set EngineConfig(distributed=False) for independent per-rank jobs)")


def run_phases(plan, group=None, res=None, verify=True):
    """Drive one job through the plan's phases with the exchanges.
    `plan` is a DevicePlan (or the CPU stand-in of the tests) of THIS rank."""
    import torch
    import torch.distributed as dist

    rank, size = dist.get_rank(group), dist.get_world_size(group)
    gloo = dist.get_backend(group) == "gloo"
    dev = torch.device("cpu") if gloo else getattr(plan, "device", torch.device("cpu"))
    if verify:
        check_same_job(plan, group, dev)
    m_head, t_local = plan.sieve_update()
    tot = torch.tensor([t_local], dtype=torch.int64, device=dev)
    allt = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(size)]
    dist.all_gather(allt, tot, group=group)
    offs = tail_offsets(m_head, [int(t.item()) for t in allt])
    plan.tail_offset(offs[rank])
    win = plan.cap_window()
    if win is not None:
        plan.sync()
        _staged(win, lambda x: dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group), group)
    plan.sync()
    plan.gather()
    acc = plan.acc()
    if acc is not None:
        _staged(acc, lambda x: dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group), group)
    plan.sync()
    plan.resolve(res)
    return offs
