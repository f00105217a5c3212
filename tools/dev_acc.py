import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P
from paper_1108_0135_b200 import engine as PE
from oracle import engine_port as E
for n in [4096, 10000, 10**6, 10**8, 10**12]:
    u = PE.choose_u(n)
    K = n // u
    acc = np.zeros(K, np.uint64)
    fin, _, _, raw = PE._run_job([n], u, PE.EngineConfig(), acc_out=acc)
    job = E.Job([n], "c", capture=False, wrap=True)
    job.run()
    ref = job.arrays[0].acc
    bad = np.nonzero(acc != ref)[0]
    print(n, "u", u, "K", K, "bad", len(bad), "head_end", raw["head_end"], "maxmcut", raw["max_mcut"], "q", raw["q_entries"])
    H = job.arrays[0]
    for i in bad[:6]:
        print("  k", i + 1, "gpu", acc[i].astype(np.int64), "ref", ref[i].astype(np.int64), "diff", (acc[i] - ref[i]).astype(np.int64),
              "v", H.v[i], "D", H.D[i], "xcut", H.xcut[i], "mcut", H.mcut[i], "lo", H.lo[i])
