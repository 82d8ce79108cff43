"""Developer micro-benchmarks of the device jobs (not part of the product).

python tools/microbench.py [ech|mad|all]
Times single-block ECH across block sizes / base-case sizes and the K1
contraction across shapes, with CUDA events, and prints JSON lines.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1806_04211_b200 import gfrref as G  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def bench_ech():
    for p in (2, 251):
        f = G.FieldSpec(p)
        for n in (256, 512, 1024, 2048):
            H = G.random_matrix(f, n, n, 7)
            for base in (0, 64, 128):
                G.set_ech_mode(0 if base == 0 else 1)
                G.set_ech_base(max(base, 1))
                G.launch_count(reset=True)
                ms = timed(lambda: G.ech(f, H), reps=2)
                launches = G.launch_count(reset=True) / 3
                print(json.dumps({"job": "ech", "p": p, "n": n, "base": base, "ms": ms, "launches": launches}))
    G.set_ech_base(64)


def bench_mad():
    for p in (2, 251):
        f = G.FieldSpec(p)
        for (m, k, n) in [(1024, 1024, 1024), (1024, 1024, 7168), (4096, 4096, 4096), (8192, 8192, 8192),
                          (1024, 32, 7168), (8192, 1024, 8192)]:
            A = G.random_matrix(f, m, k, 1)
            B = G.random_matrix(f, k, n, 2)
            Cc = G.random_matrix(f, m, n, 3)
            for pol in (2, 1):
                if pol == 1 and m * n * k > 2 ** 33:
                    continue
                G.set_mad_policy(pol)
                ms = timed(lambda: G.mad(f, Cc, A, B))
                tops = 2 * m * n * k / (ms / 1e3) / 1e12
                print(json.dumps({"job": "mad", "p": p, "m": m, "k": k, "n": n,
                                  "path": "tc" if pol == 2 else "simt", "ms": ms, "TOPS": tops}))
        G.set_mad_policy(0)


def bench_mad_shape(p, m, k, n, reps):
    """One K1 shape on the tcgen05 path (for ncu captures of a single launch)."""
    f = G.FieldSpec(p)
    A, B, Cc = G.random_matrix(f, m, k, 1), G.random_matrix(f, k, n, 2), G.random_matrix(f, m, n, 3)
    G.set_mad_policy(2)
    ms = timed(lambda: G.mad(f, Cc, A, B), reps=reps)
    print(json.dumps({"job": "mad", "p": p, "m": m, "k": k, "n": n, "path": "tc", "ms": ms,
                      "TOPS": 2 * m * n * k / (ms / 1e3) / 1e12}))


if __name__ == "__main__":
    G.lib()
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "madshape":
        bench_mad_shape(*(int(x) for x in sys.argv[2:7]))
        sys.exit(0)
    if what in ("mad", "all"):
        bench_mad()
    if what in ("ech", "all"):
        bench_ech()
