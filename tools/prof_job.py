import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**14
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for _ in range(reps):
    cfg = P.EngineConfig(engine_flags=4 if os.environ.get('MT_TIMING') else 0)
    t = time.time(); r = P.mertens_exact(n, cfg); dt = time.time() - t
    d = r.stats.device
    print(n, r.value, f"{dt:.3f}s", {k: (round(v, 2) if isinstance(v, float) else v) for k, v in d.items()})
