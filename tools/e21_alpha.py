import sys, os, time, json
sys.path.insert(0, os.getcwd())
import paper_1108_0135_b200 as P
n = 10**21
t = time.time()
r = P.mertens_exact(n, P.EngineConfig(u_alpha=0.5, engine_flags=4))
print(json.dumps({"n": "1e21", "u_alpha": 0.5, "u": r.u, "M": r.value, "q10": r.quotient(10), "K": len(r._final),
                  "wall_s": round(time.time() - t, 1)}), flush=True)
