import sys, time
sys.path.insert(0, '.')
from paper_1806_04211_b200 import gfrref as G
for (p, k) in [(2, 8), (3, 2), (2, 4)]:
    F = G.FieldSpec(p, k)
    A = G.random_matrix(F, 2048, 1024, 1); B = G.random_matrix(F, 1024, 2048, 2)
    G.mul(F, A, B); G.synchronize()
    t = time.perf_counter()
    for _ in range(5): G.mul(F, A, B)
    G.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(F, "mul 2048x1024x2048: %.3f ms, %.1f T GF(q)-MAC/s" % (dt * 1e3, 2048 * 1024 * 2048 / dt / 1e12))
    C = G.random_matrix(F, 1024, 1024, 3)
    G.ech(F, C); G.synchronize()
    t = time.perf_counter(); G.ech(F, C); G.synchronize()
    print(F, "ech 1024^2: %.2f ms" % ((time.perf_counter() - t) * 1e3))
