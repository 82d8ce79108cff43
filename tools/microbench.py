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


def bench_host_cost(reps=200):
    """Host-side cost of one K1 call (ctypes + dispatch + tensor maps + launch),
    measured without synchronising (the launch queue absorbs the kernels)."""
    f = G.FieldSpec(2)
    for (m, n, k) in [(128, 128, 128), (1024, 1024, 1024)]:
        A, B, D = G.random_matrix(f, m, k, 1), G.random_matrix(f, k, n, 2), G.random_matrix(f, m, n, 3)
        (pa, la), (pb, lb), (pd, ld) = A.device_ptr(), B.device_ptr(), D.device_ptr()
        for pol in (2, 1):
            G.set_mad_policy(pol)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                G.mad_raw(2, m, n, k, pa, la, pb, lb, pd, ld, pd, ld)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(json.dumps({"job": "hostcost", "m": m, "n": n, "k": k, "path": "tc" if pol == 2 else "simt",
                              "host_us_per_call": 1e6 * (t1 - t0) / reps,
                              "total_us_per_call": 1e6 * (t2 - t0) / reps}), flush=True)
    G.set_mad_policy(0)


def bench_mad_graph(p=2, reps=50):
    """K1 launches captured in a CUDA graph (no host cost between kernels):
    device time per launch."""
    f = G.FieldSpec(p)
    shapes = [(1024, 1024, k) for k in (32, 128, 512, 1024, 2048)] + \
             [(128, 1024, 1024), (2048, 2048, 1024), (1024, 7168, 1024), (4096, 4096, 4096)]
    st = torch.cuda.Stream()
    G.set_stream(st.cuda_stream)
    for (m, n, k) in shapes:
        A, B, D = G.random_matrix(f, m, k, 1), G.random_matrix(f, k, n, 2), G.random_matrix(f, m, n, 3)
        (pa, la), (pb, lb), (pd, ld) = A.device_ptr(), B.device_ptr(), D.device_ptr()
        G.synchronize()
        for pol in (2, 1):
            G.set_mad_policy(pol)
            if pol == 1 and m * n * k > 2 ** 32:
                continue
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    G.mad_raw(p, m, n, k, pa, la, pb, lb, pd, ld, pd, ld)
            with torch.cuda.stream(st):
                ms = timed(g.replay, reps=3) / reps
            print(json.dumps({"job": "madgraph", "p": p, "m": m, "n": n, "k": k,
                              "path": "tc" if pol == 2 else "simt", "us": 1e3 * ms,
                              "TOPS": 2 * m * n * k / (ms / 1e3) / 1e12}), flush=True)
    G.set_mad_policy(0)
    G.set_stream(0)


def bench_tc_stamps(p=2):
    """Per-CTA phase timing of single K1 launches (run with GFQ_TC_DEBUG=1)."""
    import ctypes
    import numpy as np
    f = G.FieldSpec(p)
    for (m, n, k) in [(1024, 1024, 32), (1024, 1024, 1024), (4096, 4096, 4096)]:
        A, B, D = G.random_matrix(f, m, k, 1), G.random_matrix(f, k, n, 2), G.random_matrix(f, m, n, 3)
        (pa, la), (pb, lb), (pd, ld) = A.device_ptr(), B.device_ptr(), D.device_ptr()
        G.set_mad_policy(2)
        for rep in range(3):
            G.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            G.mad_raw(p, m, n, k, pa, la, pb, lb, pd, ld, pd, ld)
            e1.record()
            e1.synchronize()
            buf = np.zeros(148 * 8, np.uint64)
            G.lib().gfq_tc_debug_take(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
            st = buf.reshape(148, 8).astype(np.int64)
            used = st[:, 0] > 0
            st = st[used]
            t0 = st[:, 0].min()
            rel = (st - t0) / 1e3
            print(json.dumps({"job": "tcstamps", "m": m, "n": n, "k": k, "rep": rep, "ctas": int(used.sum()),
                              "event_us": 1e3 * e0.elapsed_time(e1),
                              "start_spread_us": float(rel[:, 0].max()),
                              "median_us": [round(float(np.median(rel[:, c])), 2) for c in range(7)],
                              "max_us": [round(float(rel[:, c].max()), 2) for c in range(7)]}), flush=True)
    G.set_mad_policy(0)


def bench_mad_loop(p=2, reps=50):
    """Back-to-back K1 launches on raw pointers (no allocation per call):
    device time per launch across shapes -> fixed cost vs. slope."""
    f = G.FieldSpec(p)
    shapes = [(1024, 1024, k) for k in (32, 128, 256, 512, 1024, 2048, 4096)] + \
             [(1024, 7168, 1024), (128, 1024, 1024), (256, 1024, 1024), (2048, 2048, 1024),
              (8192, 1024, 1024), (1024, 8192, 1024), (4096, 4096, 4096)]
    for (m, n, k) in shapes:
        A, B, D = G.random_matrix(f, m, k, 1), G.random_matrix(f, k, n, 2), G.random_matrix(f, m, n, 3)
        (pa, la), (pb, lb), (pd, ld) = A.device_ptr(), B.device_ptr(), D.device_ptr()
        for pol in (2, 1):
            G.set_mad_policy(pol)
            if pol == 1 and m * n * k > 2 ** 32:
                continue

            def fn():
                for _ in range(reps):
                    G.mad_raw(p, m, n, k, pa, la, pb, lb, pd, ld, pd, ld)
            ms = timed(fn, reps=2) / reps
            print(json.dumps({"job": "madloop", "p": p, "m": m, "n": n, "k": k, "path": "tc" if pol == 2 else "simt",
                              "us": 1e3 * ms, "TOPS": 2 * m * n * k / (ms / 1e3) / 1e12}), flush=True)
    G.set_mad_policy(0)


if __name__ == "__main__":
    G.lib()
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "tcstamps":
        bench_tc_stamps(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
        sys.exit(0)
    if what == "madgraph":
        bench_mad_graph(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
        sys.exit(0)
    if what == "hostcost":
        bench_host_cost()
        sys.exit(0)
    if what == "madloop":
        bench_mad_loop(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
        sys.exit(0)
    if what == "madshape":
        bench_mad_shape(*(int(x) for x in sys.argv[2:7]))
        sys.exit(0)
    if what in ("mad", "all"):
        bench_mad()
    if what in ("ech", "all"):
        bench_ech()
