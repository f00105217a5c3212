"""CPU: the oracle (C restatement + engine port) pinned to vectors produced by
running the reference itself (tests/golden/make_golden.py)."""
import numpy as np
import pytest


def test_m_table_upto_1e4(golden, oracle):
    G, _ = golden
    assert np.array_equal(oracle.mertens_table(10000), G["m_upto_1e4"])


def test_seeded_values(golden, oracle):
    G, _ = golden
    ns, ms = G["seeded_n"].tolist(), G["seeded_m"].tolist()
    # the exact engine port on a subsample (each run restates the reference job loop)
    for n, m in list(zip(ns, ms))[::7]:
        assert oracle.mertens_exact(n).value == m


def test_e10_full_map(golden, oracle):
    G, J = golden
    r = oracle.mertens_exact(10**10)
    assert r.value == J["e10"]["value"] == -33722
    assert np.array_equal(r.final, G["e10_final"])
    assert np.array_equal(r.cp_q, G["e10_cp_q"]) and np.array_equal(r.cp_m, G["e10_cp_m"])
    assert (r.stats.counted_items, r.stats.dense_items, r.stats.blocks) == (
        J["e10"]["counted_items"], J["e10"]["dense_items"], J["e10"]["blocks"])


def test_finalize_from_tails(golden, oracle):
    G, _ = golden
    k = oracle.get_kernels("c")
    assert np.array_equal(k.finalize_recursion(G["e10_tails"], G["e10_D"]), G["e10_final"])


def test_per_block_state(golden, oracle):
    G, J = golden
    blk = J["blk"]
    job = oracle.Job([blk["n"]], "c", block_len=blk["block_len"])
    seen = {}

    def snap(j, y1, y2):
        seen[j.stats.blocks] = (j.arrays[0].acc.copy(), j.arrays[0].dnext.copy(), j.arrays[0].ynext.copy(),
                                j.stats.counted_items, j.stats.dense_items)

    job.run(on_block=snap)
    for s in blk["snaps"]:
        nb = {"b1": 1, "b3": 3}.get(s["tag"])
        if nb is None:
            continue
        acc, dn, yn, c, d = seen[nb]
        assert np.array_equal(acc, G[f"blk_{s['tag']}_acc"])
        assert np.array_equal(dn, G[f"blk_{s['tag']}_dnext"])
        assert np.array_equal(yn, G[f"blk_{s['tag']}_ynext"])
        assert (c, d) == (s["counted"], s["dense"])
    assert int(job.finalize()[0].final[0]) == blk["value"]


def test_sieve_blocks(golden, oracle):
    G, _ = golden
    k = oracle.get_kernels("c")
    pr = oracle.generate_primes(oracle.ceil_sqrt(10**12 + 5000) + 1)
    lg, wh = oracle.build_logs(pr), oracle.build_wheel()
    assert np.array_equal(wh, G["wheel"])
    for i, y1 in enumerate(G["sieve_y1"].tolist()):
        y2 = y1 + 4999
        assert np.array_equal(k.sieve_logprime(y1, y2, pr, lg, wh), G["sieve_mu"][i])
        sel = pr <= oracle.ceil_sqrt(y2) + 1
        assert np.array_equal(k.logprime_states(y1, y2, pr[sel], lg[sel], wh), G["sieve_states"][i])
        if y1 < 10**10:
            assert np.array_equal(k.sieve_naive(y1, y2, pr), G["sieve_mu"][i])


def test_divisor_arrays(golden, oracle):
    G, _ = golden
    m, s, c = oracle.get_kernels("c").build_divisor_arrays(4096)
    assert np.array_equal(m, G["div_magic"]) and np.array_equal(s, G["div_shift"]) and np.array_equal(c, G["div_scheme"])


def test_wrap_accumulation_matches_guarded(oracle):
    """mod-2^64 accumulation (the engine's arithmetic) == the reference's i128 path."""
    a = oracle.mertens_exact(10**9).final
    b = oracle.Job([10**9], "c", capture=False, wrap=True)
    b.run()
    assert np.array_equal(b.finalize()[0].final, a)


def test_big_path_small(oracle):
    """Python-int restatement (128-bit semantics) agrees with the compiled port."""
    for n in (10**6 + 7, 3 * 10**6):
        assert oracle.mertens_big(n).value == oracle.mertens_exact(n).value


def test_ref_kernels_match_c_oracle(oracle):
    try:
        ref = oracle.get_kernels("ref")
    except ImportError:
        pytest.skip("oracle/_ref not built")
    c = oracle.get_kernels("c")
    pr = oracle.generate_primes(2000)
    lg, wh = oracle.build_logs(pr), oracle.build_wheel()
    for y1 in (2, 999_983, 3_000_000):
        assert np.array_equal(ref.sieve_logprime(y1, y1 + 20000, pr, lg, wh), c.sieve_logprime(y1, y1 + 20000, pr, lg, wh))
