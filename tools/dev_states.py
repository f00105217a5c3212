import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_0135_b200._kernels import sm100
from oracle import engine_port as E
G = np.load("tests/golden/golden.npz")
y1 = 4294962296; y2 = y1 + 4999
pr = E.generate_primes(E.ceil_sqrt(y2) + 1); lg = E.build_logs(pr); w = E.build_wheel()
a = sm100.logprime_states(y1, y2, pr, lg, w)
b = E.get_kernels("c").logprime_states(y1, y2, pr, lg, w)
g = G["sieve_states"][list(G["sieve_y1"]).index(y1)]
print("oracle==golden", np.array_equal(b, g))
idx = np.nonzero(a != b)[0]
for i in idx[:40]:
    y = y1 + i
    f = []; x = y
    for p in pr[:2000].tolist():
        while x % p == 0: f.append(p); x //= p
    if x > 1: f.append(x)
    print(y, "gpu", hex(a[i]), "ref", hex(b[i]), f)
