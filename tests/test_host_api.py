"""CPU: host logic, API surface and the C ABI library (no compute calls)."""
import dataclasses
import math
import os
import re

import numpy as np
import pytest

import paper_1108_0135_b200 as P
from paper_1108_0135_b200 import engine as PE


def test_choose_u_matches_oracle(oracle):
    rng = np.random.default_rng(1)
    ns = [4, 5, 100, 1023, 1024, 10**10, 10**16, 10**19, 10**22, 11609864264058592345] + \
        [int(x) for x in rng.integers(4, 2**62, size=200)]
    for n in ns:
        for N in (1, 3, 64):
            assert P.choose_u(n, N) == oracle.choose_u(n, N)


def test_quotient_targets_match_oracle(oracle):
    for n in (5000, 10**7, 10**10):
        u = P.choose_u(n)
        assert np.array_equal(PE._quotient_targets(n, n // u, u, 4_000_000),
                              oracle.quotient_targets(n, n // u, u, 4_000_000))
    n = 10**13
    u = P.choose_u(n)
    assert np.array_equal(PE._quotient_targets(n, n // u, u, 1000), oracle.quotient_targets(n, n // u, u, 1000))


@pytest.mark.parametrize("n", [10**10, 10**9, 12345678901, 10**8])
def test_block_schedule_matches_reference_loop(n, oracle):
    job = oracle.Job([n], "c")
    job.run()
    st = P.RunStats()
    mc = int(job.arrays[0].mcut.max())
    PE._block_schedule(job.u, n, mc, P.EngineConfig(), st)
    assert st.blocks == job.stats.blocks
    assert st.divtable_released_at == job.stats.divtable_released_at
    assert st.r4_block_len == job.stats.r4_block_len


def test_engine_config_is_field_compatible():
    ref_fields = ["mem_budget", "workers", "u_alpha", "block_len", "region", "fastdiv_cap", "r4_block_factor",
                  "naive_ceiling", "naive_block_len", "quotient_budget", "backend", "checkpoint_path"]
    names = [f.name for f in dataclasses.fields(P.EngineConfig)]
    assert names[:len(ref_fields)] == ref_fields
    assert P.EngineConfig().quotient_budget == 4_000_000


def test_public_names():
    for name in ["EngineConfig", "MertensResult", "RegionConfig", "Region", "choose_u", "classify_region",
                 "mertens_exact", "mertens_exact_big", "mertens_exact_multi", "mertens_naive", "verify_paired",
                 "DivisorConstants", "DivisorTable", "build_table", "fast_div", "precompute_divisor",
                 "LogPrimeTable", "MoebiusBlock", "PrimeList", "WheelTable", "accumulate_mertens",
                 "build_log_table", "build_wheel", "generate_primes", "log_prime", "sieve_block_logprime",
                 "sieve_block_naive"]:
        assert hasattr(P, name), name


def test_classify_region():
    cfg = P.RegionConfig()
    n = 10**12
    assert P.classify_region(1, 10, n, cfg) == P.Region.R1
    assert P.classify_region(1, int(3 * math.sqrt(n)), n, cfg) == P.Region.R2
    assert P.classify_region(10**4, int(3 * math.sqrt(n)), n, cfg) == P.Region.R4
    with pytest.raises(ValueError):
        P.RegionConfig(c1=3, c2=2)


def test_tables_match_oracle(golden, oracle):
    G, _ = golden
    pl = P.generate_primes(10**6)
    assert np.array_equal(pl.primes, oracle.generate_primes(10**6))
    assert np.array_equal(P.build_log_table(pl).logs, oracle.build_logs(pl.primes))
    assert np.array_equal(P.build_wheel().residues, G["wheel"])
    assert [P.log_prime(p) for p in (2, 3, 11, 13, 17)] == [1, 3, 5, 5, 5]


def test_fastdiv_host(golden):
    G, _ = golden
    for d in range(1, 4097):
        c = P.precompute_divisor(d)
        assert (c.m, c.s, c.scheme) == (int(G["div_magic"][d]), int(G["div_shift"][d]), int(G["div_scheme"][d]))
    rng = np.random.default_rng(3)
    for d in [3, 7, 641, 2**40 + 15, 2**63 + 7]:
        c = P.precompute_divisor(d)
        for n in rng.integers(0, 2**63, size=200, dtype=np.uint64).tolist() + [2**64 - 1, 0, d - 1, d]:
            assert P.fast_div(n, c) == n // d


def test_library_exports_every_header_symbol():
    from paper_1108_0135_b200 import _lib, build

    build.build()
    hdr = open(os.path.join(os.path.dirname(build.HERE), "include", "mertens_sm100.h")).read()
    declared = set(re.findall(r"^\s*(?:const char\*|int|void)\s+(mt_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    L = _lib.lib()
    for s in declared:
        assert hasattr(L, s)
    assert L.mt_abi_version() == 2


def test_no_gpu_fails_loudly():
    from paper_1108_0135_b200 import _lib

    if _lib.lib().mt_device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(P.errors.DeviceError if hasattr(P, "errors") else Exception):
        P.mertens_exact(10**6)


def test_errors_hierarchy():
    from paper_1108_0135_b200 import errors as E

    assert issubclass(E.CeilingExceededError, E.ResourceLimitError)
    assert issubclass(E.ResourceLimitError, E.MertensError)
    with pytest.raises(ValueError):
        P.mertens_exact(0)


def test_dense_map_identity_residual(oracle):
    """The vectorised identity sum over a dense quotient map (capture-all mode)
    is 0 on a map built from the oracle, and detects a single wrong value."""
    from math import isqrt

    n = 10**8 + 12345
    r = oracle.mertens_exact(n)
    s, K = isqrt(n), len(r.final)
    small = np.concatenate([[0], oracle.mertens_table(s)]).astype(np.int32)
    qmap = np.array([r.quotient(c) for c in range(K + 1, s + 1)], np.int32)
    R = PE.MertensResult(n, r.value, r.u, r.final, qmap=qmap, small=small)
    assert P.mertens_identity_residual(R) == 0
    assert R.quotient(K + 5) == r.quotient(K + 5) and R.quotient(n // 7) == small[7]
    qmap[3] += 1
    assert P.mertens_identity_residual(R) != 0


def test_bench_gpus_spawns_ranks():
    """`bench.py --gpus 3` outside torchrun launches 3 ranks (torch.distributed.run)
    and every rank sees world size 3 (--gpus was ignored)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3", "--launch-check",
                        "--dist-backend", "gloo"], capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1, 2] and all(d["world"] == 3 for d in lines)


@pytest.mark.parametrize("n", [10**6, 999_983, 1000 * 1001, 1000 * 1001 - 1, 1001**2 - 1, 2 * 10**6 + 7])
@pytest.mark.parametrize("chunk", [1 << 24, 97])
def test_identity_residual_dense_map(n, chunk, oracle):
    """mertens_identity_residual over a dense map built from the oracle's M table:
    zero, including n = s(s+1) - 1, s(s+1) and (s+1)^2 - 1 where c = s is special."""
    M = np.concatenate([[0], oracle.mertens_table(n)])
    s = math.isqrt(n)
    K = max(1, round(n ** (1 / 3)))
    c = np.arange(1, s + 1)
    mq = M[n // c].astype(np.int32)
    r = PE.MertensResult(n, int(M[n]), 0, mq[:K].astype(np.int64), qmap=mq[K:], small=M[: s + 1].astype(np.int32))
    assert PE.mertens_identity_residual(r, chunk=chunk) == 0
    bad = mq[K:].copy()
    bad[-1] += 1
    r2 = PE.MertensResult(n, int(M[n]), 0, mq[:K].astype(np.int64), qmap=bad, small=M[: s + 1].astype(np.int32))
    assert PE.mertens_identity_residual(r2, chunk=chunk) != 0
