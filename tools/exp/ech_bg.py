"""Developer experiment: one 8192^2 GF(2) ECH (the cfg5s diagonal block)
alone and next to background load on another stream -- an HBM-bound copy
loop, a compute-bound bf16 GEMM loop, and our own K1f contractions -- to
see which shared resource slows the diagonal ECH inside the step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1806_04211_b200 import gfrref as G  # noqa: E402

G.lib()
f = G.FieldSpec(2)
H = G.random_matrix(f, 8192, 8192, 7)
own = torch.cuda.Stream(priority=-5)
G.set_stream(own.cuda_stream)
G.ech(f, H)
G.synchronize()


def timed_ech(n=3):
    ts = []
    for _ in range(n):
        G.synchronize()
        t0 = time.perf_counter()
        G.ech(f, H)
        G.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return min(ts), sum(ts) / len(ts)


print("alone", timed_ech())
bg = torch.cuda.Stream(priority=0)
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
y = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
A = G.random_matrix(f, 8192, 8192, 1)
B = G.random_matrix(f, 8192, 65536, 2)


def with_bg(name, work, reps):
    torch.cuda.synchronize()
    with torch.cuda.stream(bg):
        for _ in range(reps):
            work()
    r = timed_ech()
    torch.cuda.synchronize()
    print(name, r)


with_bg("hbm_copy", lambda: b.copy_(a), 400)
with_bg("bf16_gemm", lambda: torch.mm(x, y), 800)
bgs = torch.cuda.Stream(priority=0)


def k1f():
    G.set_stream(bgs.cuda_stream)
    G.set_mad_policy(3)
    for _ in range(40):
        G.mul(f, A, B)
    G.set_mad_policy(0)
    G.set_stream(own.cuda_stream)


torch.cuda.synchronize()
k1f()
r = timed_ech()
torch.cuda.synchronize()
print("k1f", r)
