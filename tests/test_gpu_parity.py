"""GPU parity: the sm100 engine through the C ABI vs the oracle and the
reference's golden vectors.  Bit-exact for every integer output."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tables(oracle, ymax):
    pr = oracle.generate_primes(oracle.ceil_sqrt(ymax) + 1)
    return pr, oracle.build_logs(pr), oracle.build_wheel()


def test_sieve_golden_blocks(engine, golden, oracle):
    from paper_1108_0135_b200._kernels import sm100

    G, _ = golden
    pr, lg, wh = _tables(oracle, 10**12 + 5000)
    for i, y1 in enumerate(G["sieve_y1"].tolist()):
        y2 = y1 + 4999
        assert np.array_equal(sm100.sieve_logprime(y1, y2, pr, lg, wh), G["sieve_mu"][i])
        sel = pr <= oracle.ceil_sqrt(y2) + 1
        assert np.array_equal(sm100.logprime_states(y1, y2, pr[sel], lg[sel], wh), G["sieve_states"][i])


@pytest.mark.parametrize("y1,length", [(2, 3 << 20), (10**9 - 123457, 3 << 20), (2**33 - 70000, 200000),
                                       (4_641_588_833_612 - 10**6, 2 * 10**6)])
def test_sieve_vs_oracle(engine, oracle, y1, length):
    from paper_1108_0135_b200._kernels import sm100

    y2 = y1 + length - 1
    pr, lg, wh = _tables(oracle, y2)
    a = sm100.sieve_logprime(y1, y2, pr, lg, wh)
    b = oracle.get_kernels("c").sieve_logprime(y1, y2, pr, lg, wh)
    assert np.array_equal(a, b)
    assert np.array_equal(sm100.sieve_naive(y1, y2, pr), b)


def test_mertens_range_vs_oracle(engine, oracle):
    from paper_1108_0135_b200 import _lib

    L = _lib.lib()
    n = 3_000_000
    m = np.zeros(n, np.int64)
    _lib.check(L.mt_mertens_range(1, n, _lib.ptr(m)))
    assert np.array_equal(m, oracle.mertens_table(n))


def test_divisor_arrays(engine, golden):
    from paper_1108_0135_b200._kernels import sm100

    G, _ = golden
    m, s, c = sm100.build_divisor_arrays(4096)
    assert np.array_equal(m, G["div_magic"]) and np.array_equal(s, G["div_shift"]) and np.array_equal(c, G["div_scheme"])


def test_finalize_golden(engine, golden):
    from paper_1108_0135_b200._kernels import sm100

    G, _ = golden
    assert np.array_equal(sm100.finalize_recursion(G["e10_tails"], G["e10_D"]), G["e10_final"])


def test_apply_block_chain_golden(engine, golden, oracle):
    """Per-block acc/dnext/ynext and counters of the reference's apply_block."""
    from paper_1108_0135_b200._kernels import sm100

    G, J = golden
    blk = J["blk"]
    H = oracle.HarmonicArray(blk["n"], blk["u"])
    y, m_run, nb, cnt = 1, 0, 0, [0, 0]
    k = oracle.get_kernels("c")
    snaps = {s["tag"]: s for s in blk["snaps"]}
    while y <= blk["u"]:
        y2 = min(y + blk["block_len"] - 1, blk["u"])
        mp = np.cumsum(oracle.mu_range(k, y, y2), dtype=np.int64) + m_run
        c, d = sm100.apply_block(H.acc, H.v, H.lo, H.xcut, H.mcut, H.dnext, H.ynext, y, y2, mp)
        cnt[0] += c
        cnt[1] += d
        m_run, y, nb = int(mp[-1]), y2 + 1, nb + 1
        tag = {1: "b1", 3: "b3"}.get(nb)
        if tag:
            assert np.array_equal(H.acc, G[f"blk_{tag}_acc"])
            assert np.array_equal(H.dnext, G[f"blk_{tag}_dnext"])
            assert np.array_equal(H.ynext, G[f"blk_{tag}_ynext"])
            assert cnt == [snaps[tag]["counted"], snaps[tag]["dense"]]
    assert np.array_equal(H.acc, G["blk_end_acc"])


def test_apply_block_overflow_guard(engine):
    from paper_1108_0135_b200._kernels import sm100

    acc = np.array([2**62 - 5], np.int64)
    v = np.array([10**6], np.uint64)
    one = np.array([1], np.uint64)
    with pytest.raises(OverflowError):
        sm100.apply_block(acc, v, np.array([2], np.uint64), one * 250, one * 3984, one * 250,
                          np.array([4000], np.uint64), 1, 10, np.full(10, 1000, np.int64))


def test_small_n_all(engine, golden):
    G, _ = golden
    ms = G["m_upto_1e4"]
    for n in list(range(1, 60)) + [100, 1000, 1023, 1024, 1025, 2048, 4096, 5000, 9999, 10000]:
        assert engine.mertens_exact(n).value == int(ms[n - 1]), n


def test_seeded_100(engine, golden):
    G, _ = golden
    for n, m in zip(G["seeded_n"].tolist(), G["seeded_m"].tolist()):
        assert engine.mertens_exact(n).value == m, n


def test_e10_full_quotient_map(engine, golden):
    G, J = golden
    r = engine.mertens_exact(10**10)
    assert r.value == -33722 and r.backend == "sm100" and r.u == J["e10"]["u"]
    assert np.array_equal(r._final, G["e10_final"])
    assert np.array_equal(r._cp_q, G["e10_cp_q"]) and np.array_equal(r._cp_m, G["e10_cp_m"])
    assert (r.stats.counted_items, r.stats.dense_items, r.stats.blocks, r.stats.divtable_released_at) == (
        J["e10"]["counted_items"], J["e10"]["dense_items"], J["e10"]["blocks"], J["e10"]["divtable_released_at"])
    assert r.quotient(3) == 14572
    assert engine.mertens_identity_residual(r) == 0
    qs = list(r.quotients())
    assert len(qs) == 2154 + len(G["e10_cp_q"]) - sum(1 for q in G["e10_cp_q"].tolist() if q >= 10**10 // 2154)


@pytest.mark.parametrize("n,key", [(10**11, "e11"), (10**12, "e12"), (7_766_842_813, "7766842813"),
                                   (999_999_999_989, "999999999989"), (2**40 + 12345, "1099511640121")])
def test_reference_values(engine, golden, n, key):
    _, J = golden
    assert engine.mertens_exact(n).value == J[key]


def test_ac2_ratio(engine):
    r = engine.mertens_exact(7_766_842_813)
    assert round(abs(r.ratio), 6) == 0.570591


def test_multi(engine, golden):
    G, J = golden
    mm = engine.mertens_exact_multi([10**10, 10**10 + 1, 10**10 + 2])
    assert {str(k): v.value for k, v in mm.items()} == J["multi_e10"]
    assert np.array_equal(mm[10**10 + 1]._final, G["multi_e10_final_1"])


def test_multi_vs_oracle(engine, oracle):
    ns = [10**9 + 3 * i for i in range(8)]
    got = engine.mertens_exact_multi(ns)
    ref = oracle.mertens_exact_multi(ns)
    for n in ns:
        assert got[n].value == ref[n].value
        assert np.array_equal(got[n]._final, ref[n].final)


def test_u_invariance(engine):
    """M values do not depend on u."""
    n = 3 * 10**11 + 17
    base = engine.mertens_exact(n).value
    for alpha in (0.5, 2.0):
        assert engine.mertens_exact(n, engine.EngineConfig(u_alpha=alpha)).value == base


@pytest.mark.parametrize("n", [10**13, 987654321012345])
def test_counted_dense_split_invariance(engine, monkeypatch, n):
    """The counted / dense split xcut = max(D, alpha ceil(sqrt v)) changes the work
    division, not the result: finals, quotients and the reference-split RunStats
    counters are identical for the reference's split (alpha = 0) and other alphas."""
    runs = {}
    for a in ("0", "0.25", "0.39", "0.5"):
        monkeypatch.setenv("MT_XCUT_ALPHA", a)
        runs[a] = engine.mertens_exact(n)
    ref = runs["0"]
    for a, r in runs.items():
        assert r.value == ref.value, a
        assert np.array_equal(r._final, ref._final), a
        assert (r.stats.counted_items, r.stats.dense_items) == (ref.stats.counted_items, ref.stats.dense_items), a


def test_segment_size_invariance(engine):
    n = 10**13
    a = engine.mertens_exact(n)
    b = engine.mertens_exact(n, engine.EngineConfig(seg_log2_head=20, seg_log2_tail=22))
    c = engine.mertens_exact(n, engine.EngineConfig(q_budget_bytes=1 << 20))
    assert a.value == b.value == c.value == 599582
    assert np.array_equal(a._final, b._final) and np.array_equal(a._final, c._final)


def test_naive_and_verify(engine, golden):
    G, _ = golden
    v, cp = engine.mertens_naive(10**6, checkpoints=np.array([1, 10, 100, 10**4, 10**6], np.uint64))
    assert v == 212 and cp.tolist() == [1, -1, 1, -23, 212]
    rep = engine.verify_paired(10**6, 20, 42)
    assert rep["mismatches"] == [] and rep["checked"] == 20
    rep = engine.verify_paired(10**5, 5, 42, fault_inject=2)
    assert len(rep["mismatches"]) == 1


@pytest.mark.parametrize("e", [13, 14, 15])
def test_survey_reference_values(engine, golden, e):
    _, J = golden
    assert engine.mertens_exact(10**e).value == J["reference_measured_survey"][f"1e{e}"]


@pytest.mark.slow
def test_paper_1e16_and_quotients(engine, golden):
    _, J = golden
    r = engine.mertens_exact(10**16)
    assert r.value == J["paper"]["1e16"] == -3195437
    assert r.quotient(10) == J["reference_measured_survey"]["1e15"]
    assert r.quotient(1000) == J["reference_measured_survey"]["1e13"]


@pytest.mark.parametrize("flags", [1, 2, 3])
def test_forced_wide_paths(engine, golden, flags):
    """The 64-bit remainder / 64-bit quotient-walk / exact-division code paths
    (taken for real only when m or d pass 2^31, i.e. n >~ 1e18) forced on at
    small n: identical finals."""
    G, J = golden
    r = engine.mertens_exact(10**10, engine.EngineConfig(engine_flags=flags))
    assert np.array_equal(r._final, G["e10_final"]) and np.array_equal(r._cp_m, G["e10_cp_m"])
    assert engine.mertens_exact(10**12, engine.EngineConfig(engine_flags=flags)).value == J["e12"]


def test_plan_phases_reexecute(engine, golden):
    """The plan API (mt_plan_*) at world size 1, executed twice on one plan."""
    import ctypes

    from paper_1108_0135_b200 import _lib
    from paper_1108_0135_b200.engine import make_job

    G, _ = golden
    n = 10**10
    job = make_job([n], engine.choose_u(n), engine.EngineConfig(engine_flags=_lib.MT_FLAG_TIMING))
    L = _lib.lib()
    h = ctypes.c_void_p()
    _lib.check(L.mt_plan_create(ctypes.byref(job), ctypes.byref(h)))
    try:
        for _ in range(2):
            res = _lib.MtResult()
            fin = np.zeros(len(G["e10_final"]), np.int64)
            res.finals = fin.ctypes.data_as(_lib._pi64)
            mh, tt = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(L.mt_plan_sieve_update(h, ctypes.byref(mh), ctypes.byref(tt)))
            _lib.check(L.mt_plan_tail_offset(h, mh.value))
            _lib.check(L.mt_plan_gather(h))
            _lib.check(L.mt_plan_resolve(h, ctypes.byref(res)))
            assert np.array_equal(fin, G["e10_final"])
            st = _lib.stats_dict(res.stats)
            assert st["kernel_count"]["sieve_tile"] >= 1 and st["kernel_ms"]["counted"] > 0
    finally:
        L.mt_plan_destroy(h)


@pytest.mark.slow
def test_paper_1e19_and_quotients(engine, golden):
    """C4: M(10^19) and, from the same run, M(10^18), M(10^17),
    M(10^16) as quotients c = 10, 100, 1000."""
    _, J = golden
    r = engine.mertens_exact(10**19)
    assert r.value == 899990187
    assert (r.quotient(10), r.quotient(100), r.quotient(1000)) == (-46758740, -21830254, -3195437)


@pytest.mark.parametrize("y1,length", [(1, 3 << 20), (10**9 - 123457, 3 << 20), (2**32 - 70000, 300000),
                                       (4_641_588_833_612 - 10**6, 2 * 10**6),
                                       (82_036_050_574_571 - 10**6, 10**6), (464_158_883_361_277 - 10**6, 10**6)])
def test_production_sieve_mu(engine, oracle, y1, length):
    """The engine's production sieve (presieve patterns, buckets, look-back)
    gives the reference's mu on ranges up to the 1e22 job's u."""
    from paper_1108_0135_b200 import _lib

    y2 = y1 + length - 1
    mu = np.zeros(length, np.int8)
    _lib.check(_lib.lib().mt_sieve_fast(y1, y2, _lib.ptr(mu), None))
    ref = oracle.mu_range(oracle.get_kernels("c"), y1, y2)
    assert np.array_equal(mu, ref), int((mu != ref).sum())


@pytest.mark.parametrize("env", [{"MT_FILL_BIN": "16"}, {"MT_FILL_BIN": "0"}, {"MT_S2_CAP": "64"}])
def test_production_sieve_stress_paths(engine, oracle, monkeypatch, env):
    """The sieve's rare paths give the same mu: bins too small for a round (entries
    spill to direct global stores), no write-combining at all, and bucket lists far
    over capacity (flagged, and the tile recomputes that producer's hits exactly)."""
    from paper_1108_0135_b200 import _lib

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    y1, length = 4_641_588_833_612 - 10**6, 2 * 10**6
    mu = np.zeros(length, np.int8)
    _lib.check(_lib.lib().mt_sieve_fast(y1, y1 + length - 1, _lib.ptr(mu), None))
    ref = oracle.mu_range(oracle.get_kernels("c"), y1, y1 + length - 1)
    assert np.array_equal(mu, ref), int((mu != ref).sum())


def _coprime(y0, y2, wheel):
    y = np.arange(y0, y2 + 1, dtype=np.int64)
    return (y % 2 == 1) & ((y % 3 != 0) if wheel == 6 else True)


@pytest.mark.parametrize("wheel", [2, 6])
@pytest.mark.parametrize("y1,length", [(1 << 19, 3 << 20), (10**9 - 123457, 3 << 20), (2**32 - 70000, 300001),
                                       (4_641_588_833_612 - 10**6, 2 * 10**6),
                                       (82_036_050_574_571 - 10**6, 10**6), (464_158_883_361_277 - 10**6, 10**6)])
def test_wheel_tail_sieve_mu(engine, oracle, y1, length, wheel):
    """The tail's wheel sieve (W = 2: cells are the odd y; W = 6: the y coprime to
    6, two streams per prime; presieve patterns and every stream re-phased) gives
    the reference's mu at every such y, on ranges up to the 1e22 job's u."""
    from paper_1108_0135_b200 import _lib

    y2 = y1 + length - 1
    keep = _coprime(y1, y2, wheel)
    mu = np.zeros(int(keep.sum()), np.int8)
    _lib.check(_lib.lib().mt_sieve_wheel(y1, y2, wheel, _lib.ptr(mu)))
    ref = oracle.mu_range(oracle.get_kernels("c"), y1, y2)[keep]
    assert np.array_equal(mu, ref), int((mu != ref).sum())


@pytest.mark.parametrize("wheel", [2, 6])
@pytest.mark.parametrize("env", [{"MT_FILL_BIN": "16"}, {"MT_S2_CAP": "64"}])
def test_wheel_tail_sieve_stress_paths(engine, oracle, monkeypatch, env, wheel):
    from paper_1108_0135_b200 import _lib

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    y1, length = 4_641_588_833_612 - 10**6, 2 * 10**6
    keep = _coprime(y1, y1 + length - 1, wheel)
    mu = np.zeros(int(keep.sum()), np.int8)
    _lib.check(_lib.lib().mt_sieve_wheel(y1, y1 + length - 1, wheel, _lib.ptr(mu)))
    ref = oracle.mu_range(oracle.get_kernels("c"), y1, y1 + length - 1)[keep]
    assert np.array_equal(mu, ref), int((mu != ref).sum())


def test_tail_wheel_2_and_6_agree(engine, golden, monkeypatch):
    """The same jobs with the odd-y tail (MT_TAIL_WHEEL=2) and the default
    coprime-to-6 tail: identical finals and quotients."""
    G, J = golden
    for w in ("2", "6"):
        monkeypatch.setenv("MT_TAIL_WHEEL", w)
        r = engine.mertens_exact(10**10)
        assert np.array_equal(r._final, G["e10_final"]) and np.array_equal(r._cp_m, G["e10_cp_m"]), w
        assert engine.mertens_exact(10**13).value == 599582, w


def test_production_sieve_prefix(engine, oracle):
    from paper_1108_0135_b200 import _lib

    n = 5_000_000
    m = np.zeros(n, np.int64)
    _lib.check(_lib.lib().mt_sieve_fast(1, n, None, _lib.ptr(m)))
    assert np.array_equal(m, oracle.mertens_table(n))


def _two_rank_worker(rank, world, port, n, q):
    import os as _os
    import sys as _sys

    _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
    import numpy as _np
    import torch
    import torch.distributed as dist

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1108_0135_b200 as P
        from paper_1108_0135_b200 import _lib, distributed
        from paper_1108_0135_b200.engine import make_job

        u = P.choose_u(n)
        cfg = P.EngineConfig(device=0, seg_log2_head=20, seg_log2_tail=20)
        job = make_job([n], u, cfg, rank=rank, world=world)
        plan = distributed.DevicePlan(job)
        res = _lib.MtResult()
        fin = _np.zeros(n // u, _np.int64)
        res.finals = fin.ctypes.data_as(_lib._pi64)
        distributed.run_phases(plan, None, res)
        st = _lib.stats_dict(res.stats)
        plan.close()
        # the public API over the process group: quotient captures assembled by the
        # capture-window reduction
        r = P.mertens_exact(n, P.EngineConfig(device=0, seg_log2_head=20, seg_log2_tail=20, distributed=True))
        q.put((rank, fin.tolist(), st["tail_seg_begin"], st["tail_seg_end"], r.value, r._final.tolist(),
               r._cp_m.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ranks_on_one_gpu(engine, golden, world):
    """The multi-GPU path (plan API + run_phases: interleaved head units, odd-y
    tail ranges, deferred offsets, rank-local Q-gather, int64 allreduce) with
    `world` ranks sharing cuda:0 over gloo: finals identical to the single-rank
    job; mertens_exact(distributed=True) also assembles the 4M quotient captures."""
    import socket
    import time

    import torch.multiprocessing as mp

    n = 10**12
    ref = engine.mertens_exact(n)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_two_rank_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    out, t0 = [], time.time()
    while len(out) < world:
        try:
            out.append(q.get(timeout=5))
        except Exception:
            assert all(p.is_alive() or p.exitcode == 0 for p in ps), "a rank died"
            assert time.time() - t0 < 600
    for p in ps:
        p.join(timeout=60)
    segs = sorted((o[2], o[3]) for o in out)  # tail ranges [ya, yb) tile [head_end, tail_end)
    assert segs[0][0] > 0 and all(segs[i][1] == segs[i + 1][0] for i in range(world - 1))
    assert all(a < b for a, b in segs) and segs[-1][1] > ref.u
    for rank, fin, _, _, val, fin2, cpm in out:
        assert np.array_equal(np.array(fin, np.int64), ref._final), rank
        assert val == ref.value and np.array_equal(np.array(fin2, np.int64), ref._final), rank
        assert np.array_equal(np.array(cpm, np.int64), ref._cp_m), rank


@pytest.mark.slow
def test_paper_1e20_128bit(engine):
    """n >= 2^64: elements k <= 5 carry 128-bit v.  M(10^20) and,
    from the same run, M(10^19) = quotient(10) and M(10^18) = quotient(100)."""
    r = engine.mertens_exact(10**20)
    assert r.value == 461113106
    assert (r.quotient(10), r.quotient(100)) == (899990187, -46758740)


@pytest.mark.slow
def test_batch_extreme_1161e19(engine):
    """C3 (reduced to 8 targets): one shared sieve for close x around the
    paper's extreme M(11609864264058592345) = -1995900927;
    every target agrees with its own single-target run's value relation."""
    x = 11609864264058592345
    ns = [x + j * 10**10 for j in range(-4, 4)]
    mm = engine.mertens_exact_multi(ns)
    assert mm[x].value == -1995900927
    assert round(mm[x].ratio, 9) == -0.585767684
    # u-invariance: a different shared sieve (4 targets) gives the same values
    sub = engine.mertens_exact_multi(ns[2:6])
    assert all(sub[n].value == mm[n].value for n in ns[2:6])


@pytest.mark.slow
def test_c3_64_targets_1161e19(engine):
    """C3 as specified (BASELINE configs[2]): 64 close targets
    x + j*10^10, j = -32..31, around the paper's extreme, one shared sieve with
    u = choose_u(max, 64).  j = 0 is pinned to the paper; all 64 values agree with
    a second shared-sieve layout (two 32-target jobs, each with its own u) and
    three sampled targets agree with their single-target runs."""
    import json
    import os
    import time

    x = 11609864264058592345
    ns = [x + j * 10**10 for j in range(-32, 32)]
    t0 = time.perf_counter()
    mm = engine.mertens_exact_multi(ns)
    wall = time.perf_counter() - t0
    u = engine.choose_u(max(ns), 64)  # = 82,036,052,034,891 (choose_u of the largest target, engine.py:424-446)
    assert mm[x].u == u and mm[ns[0]].u == u
    assert mm[x].value == -1995900927
    assert round(mm[x].ratio, 9) == -0.585767684
    lo = engine.mertens_exact_multi(ns[:32])
    hi = engine.mertens_exact_multi(ns[32:])
    assert lo[ns[0]].u != u
    for n in ns:
        assert (lo.get(n) or hi.get(n)).value == mm[n].value, n
    for n in (ns[0], ns[40], ns[-1]):  # and three single-target runs (u = choose_u(n))
        assert engine.mertens_exact(n).value == mm[n].value, n
    out = os.environ.get("MT_RESULTS_DIR")
    if out:
        st = mm[x].stats.device
        json.dump({"ns": [str(n) for n in ns], "u": u, "wall_s": wall,
                   "values": {str(n): mm[n].value for n in ns},
                   "kernel_ms": st.get("kernel_ms"), "phases_ms": {k: st[k] for k in (
                       "ms_update_head", "ms_sieve_tail", "ms_qgather", "ms_finalize", "ms_setup")}},
                  open(os.path.join(out, "c3_64.json"), "w"), indent=1)


def test_dense_full_quotient_map(engine, oracle):
    """Capture-all for large n (north_star: M(n) and ALL M(floor(n/c))): the
    dense int32 map covers every c; pinned by the identity sum over the whole
    map (engine.py:606-616), the oracle's M table for y <= sqrt(n), and
    independent runs at sampled c."""
    from math import isqrt

    n = 10**14
    r = engine.mertens_exact(n, engine.EngineConfig(quotient_budget=10**9))
    assert r.value == -875575 and r._qmap is not None
    s = isqrt(n)
    assert np.array_equal(r._small[1:].astype(np.int64), oracle.mertens_table(s))
    assert engine.mertens_identity_residual(r) == 0
    K = len(r._final)
    rng = np.random.default_rng(7)
    for c in [K + 1, s] + [int(x) for x in rng.integers(K + 1, s, size=6)]:
        assert r.quotient(c) == engine.mertens_exact(n // c).value, c
    assert r.quotient(10) == engine.mertens_exact(10**13).value == 599582


@pytest.mark.slow
def test_dense_quotient_map_memmap_1e16(engine, tmp_path):
    """North_star's "all M(floor(n/c))" as a streamed output: the dense map written
    to memory-mapped int32 files (quotient_map_path), the identity over the whole
    map summed in chunks = 0, and sampled quotients against the paper / oracle."""
    from math import isqrt

    n = 10**16
    path = str(tmp_path / "e16")
    r = engine.mertens_exact(n, engine.EngineConfig(quotient_budget=10**12, quotient_map_path=path))
    assert r.value == -3195437 and isinstance(r._qmap, np.memmap) and isinstance(r._small, np.memmap)
    assert len(r._qmap) == isqrt(n) - len(r._final) and len(r._small) == isqrt(n) + 1
    assert engine.mertens_identity_residual(r, chunk=1 << 22) == 0
    assert r.quotient(10) == -3216373 and r.quotient(1000) == 599582  # M(1e15), M(1e13)
    assert r.quotient(10**8) == int(r._small[10**8]) == 1928  # M(1e8)


def test_checkpoint_resume(engine, golden, tmp_path):
    """Checkpoint after the head and between tail segments, then resume
    (engine.py:646-741): identical finals and quotients; the file starts with the
    reference's MERTCKP1 header; wrong u / foreign files are refused."""
    import struct

    from paper_1108_0135_b200 import _lib
    from paper_1108_0135_b200.engine import make_job

    n = 10**13
    path = str(tmp_path / "ck.bin")
    cfg = engine.EngineConfig(checkpoint_path=path, checkpoint_seconds=0.0, seg_log2_tail=18)
    full = engine.mertens_exact(n, cfg)
    assert full.value == 599582
    head = open(path, "rb").read(72)
    magic, version, flags, n_lo, n_hi, u, next_y1, K, m_running, bl = struct.unpack("<8sII QQ Q Q Q q Q", head)
    assert (magic, version, flags, n_lo, u, K) == (b"MERTCKP1", 4, 1 << 16, n, full.u, len(full._final))
    # resume from the last checkpoint of that run (somewhere in the tail)
    r = engine.resume_exact(path, engine.EngineConfig(seg_log2_tail=18))
    assert r.value == full.value and np.array_equal(r._final, full._final)
    assert np.array_equal(r._cp_m, full._cp_m)
    from paper_1108_0135_b200.errors import ContractViolationError

    with pytest.raises(ContractViolationError):
        engine.resume_exact(path, engine.EngineConfig(u_alpha=2.0, seg_log2_tail=18))
    bad = str(tmp_path / "bad.bin")
    open(bad, "wb").write(b"x" * 100)
    with pytest.raises(Exception):
        engine.resume_exact(bad)


def test_udiv128_reciprocal(engine):
    """The exact 128/64 division (reciprocal multiply + correction) that replaces
    the software u128/u64 for v >= 2^64: random v < 2^75 and m of every size,
    plus the edges (m = 1, m = v, q at powers of two, v = q m - 1)."""
    from paper_1108_0135_b200 import _lib

    rng = np.random.default_rng(3)
    vs, ms = [], []
    for _ in range(20000):
        v = int(rng.integers(0, 1 << 63)) << int(rng.integers(0, 13)) | int(rng.integers(0, 1 << 62))
        m = max(1, int(rng.integers(0, 1 << 63)) >> int(rng.integers(0, 63)))
        vs.append(v % (1 << 75)); ms.append(m)
    for m in (1, 2, 3, (1 << 32) - 1, 1 << 32, (1 << 63) - 25, (1 << 64) - 1):
        for q in (1, (1 << 52) + 1, (1 << 64) - 1, 1 << 64, (1 << 74) // m + 1):
            for dv in (-1, 0, 1):
                v = q * m + dv
                if 0 <= v < (1 << 75):
                    vs.append(v); ms.append(m)
    lo = np.array([v & (2**64 - 1) for v in vs], np.uint64)
    hi = np.array([v >> 64 for v in vs], np.uint64)
    mm = np.array(ms, np.uint64)
    qlo, qhi = np.zeros(len(vs), np.uint64), np.zeros(len(vs), np.uint64)
    _lib.check(_lib.lib().mt_udiv128_batch(_lib.ptr(lo), _lib.ptr(hi), _lib.ptr(mm), len(vs), _lib.ptr(qlo), _lib.ptr(qhi)))
    got = [(int(h) << 64) | int(l) for l, h in zip(qlo.tolist(), qhi.tolist())]
    bad = [(v, m) for v, m, g in zip(vs, ms, got) if g != v // m]
    assert not bad, bad[:5]


def test_device_memory_pool_reuse(engine, golden):
    """Plans reuse pooled device buffers across calls (and after a trim) with the same
    results: M(10^16) and its quotients three times around release_device_memory."""
    r1 = engine.mertens_exact(10**16)
    r2 = engine.mertens_exact(10**16)
    engine.release_device_memory()
    r3 = engine.mertens_exact(10**16)
    assert r1.value == r2.value == r3.value == -3195437
    assert np.array_equal(r1._final, r2._final) and np.array_equal(r1._final, r3._final)
