"""CPU (gloo, world_size 2 and 3): the multi-rank driver run_phases with the
oracle-backed plan stand-in — tail offsets, Q-slice broadcasts and the int64
all-reduce reproduce the single-process finals bit for bit."""
import os
import socket
import time

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1108_0135_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ns, u, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from sharded_oracle import ShardedOraclePlan

        plan = ShardedOraclePlan(ns, u, rank, world)
        res = {}
        offs = D.run_phases(plan, None, res)
        q.put((rank, [f.tolist() for f in res["finals"]], offs, plan.tail_segs))
    finally:
        dist.destroy_process_group()


def _run(ns, u, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, ns, u, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = []
    deadline = time.time() + 300
    while len(out) < world:
        try:
            out.append(q.get(timeout=2))
        except Exception:
            assert all(p.is_alive() or p.exitcode == 0 for p in ps), "a rank died"
            assert time.time() < deadline, "timeout"
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_tail_offsets():
    assert D.tail_offsets(5, [1, -2, 3]) == [5, 6, 4]
    assert D.tail_offsets(0, []) == []


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_job_matches_single_process(oracle, world):
    ns = [10**8, 10**8 + 7]
    u = oracle.choose_u(max(ns), len(ns))
    ref = oracle.mertens_exact_multi(ns)
    out = _run(ns, u, world)
    for rank, finals, offs, tail_segs in out:
        assert tail_segs >= world  # every rank owns tail segments
        for n, f in zip(ns, finals):
            assert np.array_equal(np.array(f, np.int64), ref[n].final), (rank, n)
    # the offsets are the same on every rank
    assert len({tuple(o[2]) for o in out}) == 1
