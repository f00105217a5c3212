"""CPU (gloo, world_size 2 and 3): the multi-rank driver run_phases with the
oracle-backed plan stand-in — odd-y tail ranges with deferred offsets, the
capture-window reduction and the int64 all-reduce reproduce the
single-process finals bit for bit, no rank reads a quotient-table entry it
does not own, and ranks running different jobs are refused."""
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


def _worker(rank, world, port, ns, u, q, capture, skew, W=6):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from sharded_oracle import ShardedOraclePlan

        my_ns = [n + (rank if skew else 0) for n in ns]
        plan = ShardedOraclePlan(my_ns, u, rank, world, capture=capture, W=W)
        res = {}
        try:
            offs = D.run_phases(plan, None, res)
        except Exception as ex:  # noqa: BLE001 - reported to the parent
            q.put((rank, type(ex).__name__, str(ex), None, None))
            return
        win = res.get("window")
        q.put((rank, [f.tolist() for f in res["finals"]], offs, plan.ybound,
               None if win is None else win.tolist()))
    finally:
        dist.destroy_process_group()


def _run(ns, u, world, capture=False, skew=False, W=6):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, ns, u, q, capture, skew, W)) for r in range(world)]
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


@pytest.mark.parametrize("W", [2, 6])
def test_tail_partition_balanced(W):
    from sharded_oracle import tail_cost, tail_partition

    H, E, al = 6 << 20, 6 << 30, 6 << 12
    for w in (1, 2, 3, 8):
        yb = tail_partition(H, E, w, al, W)
        assert yb[0] == H and yb[-1] == E and all(b >= a for a, b in zip(yb, yb[1:]))
        assert all(y % al == 0 for y in yb)
        costs = [tail_cost(a, b, W) for a, b in zip(yb, yb[1:])]
        assert max(costs) - min(costs) <= 2 * al * w, costs
        assert sum(b - a for a, b in zip(yb, yb[1:])) == E - H
    # one rank: the cells of [H/W, E), i.e. 1/2 (W = 2) or 1/3 (W = 6) of its y
    assert tail_cost(H, E, W) == E - H // W


@pytest.mark.parametrize("world,W", [(2, 6), (3, 6), (3, 2)])
def test_sharded_job_matches_single_process(oracle, world, W):
    ns = [10**8, 10**8 + 7]
    u = oracle.choose_u(max(ns), len(ns))
    ref = oracle.mertens_exact_multi(ns)
    out = _run(ns, u, world, W=W)
    for rank, finals, offs, ybound, _ in out:
        assert sum(1 for a, b in zip(ybound, ybound[1:]) if b > a) == world  # every rank owns a tail range
        for n, f in zip(ns, finals):
            assert np.array_equal(np.array(f, np.int64), ref[n].final), (rank, n)
    # the offsets are the same on every rank
    assert len({tuple(o[2]) for o in out}) == 1


def test_sharded_capture_window(oracle):
    """The capture window (the M(floor(n/c)) outputs) is assembled by one sum-reduction."""
    ns = [10**8 + 3]
    u = oracle.choose_u(ns[0])
    out = _run(ns, u, 2, capture=True)
    from sharded_oracle import ShardedOraclePlan

    p = ShardedOraclePlan(ns, u, 0, 1)
    j = np.arange(p.jq0[0], p.J[0] + 1, dtype=np.int64)
    want = p.Mof(ns[0] // j)
    for rank, finals, _, _, win in out:
        assert np.array_equal(np.array(win, np.int64), want), rank


def test_sharded_job_refuses_mismatched_ranks(oracle):
    ns = [10**7]
    u = oracle.choose_u(ns[0])
    out = _run(ns, u, 2, skew=True)
    assert all(o[1] == "ContractViolationError" for o in out), out
