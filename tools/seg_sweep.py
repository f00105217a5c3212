"""Head/tail segment-size sweep: python tools/seg_sweep.py N head_log2[,..] [tail_log2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0135_b200 as P  # noqa: E402

n = int(float(sys.argv[1]))
heads = [int(x) for x in sys.argv[2].split(",")]
tail = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for h in heads:
    cfg = P.EngineConfig(engine_flags=4, seg_log2_head=h, seg_log2_tail=tail)
    t = time.time()
    r = P.mertens_exact(n, cfg)
    dt = time.time() - t
    d = r.stats.device
    km = {k: round(v) for k, v in d["kernel_ms"].items()}
    print(f"n={n:.0e} head=2^{h} tail=2^{tail} M={r.value} wall={dt:.2f}s total={sum(km.values())} {km} "
          f"head_ms={d['ms_update_head']:.0f} tail_ms={d['ms_sieve_tail']:.0f}", flush=True)
