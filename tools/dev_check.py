"""Developer parity sweep on a GPU box: sm100 engine vs the oracle / golden."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P
from paper_1108_0135_b200._kernels import sm100
from oracle import engine_port as E

G = np.load("tests/golden/golden.npz")
J = json.load(open("tests/golden/golden.json"))
ok = True
def check(name, cond, extra=""):
    global ok
    ok &= bool(cond)
    print(("PASS " if cond else "FAIL ") + name, extra, flush=True)

# sieve blocks vs golden
primes = E.generate_primes(E.ceil_sqrt(10**12 + 5000) + 1); logs = E.build_logs(primes); wheel = E.build_wheel()
for i, y1 in enumerate(G["sieve_y1"].tolist()):
    y2 = y1 + 4999
    mu = sm100.sieve_logprime(y1, y2, primes, logs, wheel)
    check(f"sieve_logprime y1={y1}", np.array_equal(mu, G["sieve_mu"][i]), f"ndiff={(mu != G['sieve_mu'][i]).sum()}")
    st = sm100.logprime_states(y1, y2, primes[primes <= E.ceil_sqrt(y2) + 1], logs[primes <= E.ceil_sqrt(y2) + 1], wheel)
    check(f"states y1={y1}", np.array_equal(st, G["sieve_states"][i]), f"ndiff={(st != G['sieve_states'][i]).sum()}")
# big sieve range vs oracle
y1, y2 = 10**9 - 123457, 10**9 + 3 * 2**20
pr = E.generate_primes(E.ceil_sqrt(y2) + 1)
t = time.time(); a = sm100.sieve_logprime(y1, y2, pr, E.build_logs(pr), wheel); tg = time.time() - t
b = E.get_kernels("c").sieve_logprime(y1, y2, pr, E.build_logs(pr), wheel)
check("sieve 3M block vs oracle", np.array_equal(a, b), f"{tg:.3f}s")
# divisor arrays
m, s, c = sm100.build_divisor_arrays(4096)
check("divisor arrays", np.array_equal(m, G["div_magic"]) and np.array_equal(s, G["div_shift"]) and np.array_equal(c, G["div_scheme"]))
# finalize
f = sm100.finalize_recursion(G["e10_tails"], G["e10_D"])
check("finalize 1e10", np.array_equal(f, G["e10_final"]))
# apply_block chain at n=1e9, block_len 2^16
blk = J["blk"]; n9, u9, bl = blk["n"], blk["u"], blk["block_len"]
H = E.HarmonicArray(n9, u9)
ok_blocks = True; y = 1; m_run = 0; nb = 0; cnt = [0, 0]
while y <= u9:
    y2 = min(y + bl - 1, u9)
    mu = E.mu_range(E.get_kernels("c"), y, y2)
    mp = np.cumsum(mu, dtype=np.int64) + m_run
    c1, d1 = sm100.apply_block(H.acc, H.v, H.lo, H.xcut, H.mcut, H.dnext, H.ynext, y, y2, mp)
    cnt[0] += c1; cnt[1] += d1
    m_run = int(mp[-1]); y = y2 + 1; nb += 1
    for s_ in blk["snaps"]:
        if s_["next_y1"] == y and nb in (1, 3):
            tag = s_["tag"]
            good = np.array_equal(H.acc, G[f"blk_{tag}_acc"]) and np.array_equal(H.dnext, G[f"blk_{tag}_dnext"]) and np.array_equal(H.ynext, G[f"blk_{tag}_ynext"])
            check(f"apply_block state after {tag}", good and cnt == [s_["counted"], s_["dense"]], f"{cnt}")
check("apply_block end state", np.array_equal(H.acc, G["blk_end_acc"]) and np.array_equal(H.ynext, G["blk_end_ynext"]))
# direct path and small n
for n in [1, 2, 3, 10, 100, 1000, 1023]:
    check(f"exact n={n}", P.mertens_exact(n).value == int(G["m_upto_1e4"][n - 1]))
for n in [1024, 1025, 2000, 4096, 9999, 10000]:
    r = P.mertens_exact(n)
    check(f"exact n={n}", r.value == int(G["m_upto_1e4"][n - 1]), f"got {r.value}")
# 1e10
t = time.time(); r = P.mertens_exact(10**10); dt = time.time() - t
check("M(1e10)", r.value == -33722, f"{r.value} {dt:.3f}s")
check("1e10 final array", np.array_equal(r._final, G["e10_final"]), f"ndiff={(r._final != G['e10_final']).sum() if len(r._final)==len(G['e10_final']) else 'len'}")
check("1e10 cp_q", np.array_equal(r._cp_q, G["e10_cp_q"]))
check("1e10 cp_m", np.array_equal(r._cp_m, G["e10_cp_m"]), f"ndiff={(r._cp_m != G['e10_cp_m']).sum()}")
check("1e10 stats", (r.stats.counted_items, r.stats.dense_items, r.stats.blocks) == (J["e10"]["counted_items"], J["e10"]["dense_items"], J["e10"]["blocks"]), str((r.stats.counted_items, r.stats.dense_items, r.stats.blocks, r.stats.divtable_released_at)))
print(r.stats.device)
# seeded
bad = 0
for n, mv in zip(G["seeded_n"].tolist(), G["seeded_m"].tolist()):
    if P.mertens_exact(n).value != mv: bad += 1
check("seeded 100 n <= 1e8", bad == 0, f"bad={bad}")
for e in (11, 12):
    t = time.time(); v = P.mertens_exact(10**e).value
    check(f"M(1e{e})", v == J[f"e{e}"], f"{v} {time.time()-t:.3f}s")
mm = P.mertens_exact_multi([10**10, 10**10 + 1, 10**10 + 2])
check("multi 1e10", {str(k): v.value for k, v in mm.items()} == J["multi_e10"])
for e in (13, 14, 15, 16):
    t = time.time(); r = P.mertens_exact(10**e); dt = time.time() - t
    check(f"M(1e{e})", r.value == J["reference_measured_survey"][f"1e{e}"], f"{r.value} {dt:.3f}s ms={r.stats.device['ms_total']:.1f} head={r.stats.device['ms_update_head']:.1f} tail={r.stats.device['ms_sieve_tail']:.1f} q={r.stats.device['ms_qgather']:.1f}")
print("ALL OK" if ok else "SOME FAILED")
