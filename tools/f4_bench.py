"""K1f (FP4, kind::mxf4) vs K1 (kind::i8) on single contractions, device
resident, CUDA events (includes K1f's two packing passes).

python tools/f4_bench.py [p]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_04211_b200 import gfrref as G  # noqa: E402


def timed(fn, reps=5):
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


p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
f = G.FieldSpec(p)
G.lib()
shapes = [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192),
          (8192, 8192, 57344), (8192, 8192, 65536), (1024, 1024, 7168)]
for (m, k, n) in shapes:
    A = G.random_matrix(f, m, k, 1)
    B = G.random_matrix(f, k, n, 2)
    C = G.random_matrix(f, m, n, 3)
    res = {"p": p, "m": m, "k": k, "n": n}
    outs = {}
    for pol, name in ((2, "i8"), (3, "f4")):
        G.set_mad_policy(pol)
        ms = timed(lambda: G.mad(f, C, A, B))
        outs[name] = G.mad(f, C, A, B).numpy()
        res[name + "_ms"] = round(ms, 4)
        res[name + "_tops"] = round(2.0 * m * n * k / ms / 1e9, 1)
    G.set_mad_policy(3)
    G.profile(True)
    G.profile_take_kinds()
    G.mad(f, C, A, B)
    torch.cuda.synchronize()
    kinds = G.profile_take_kinds()
    G.profile(False)
    res["f4_kernel_ms"] = round(kinds["k1_f4"][2], 4)
    res["f4_pack_ms"] = round(kinds["select"][2], 4)
    res["f4_kernel_tops"] = round(2.0 * m * n * k / kinds["k1_f4"][2] / 1e9, 1) if kinds["k1_f4"][2] else None
    res["equal"] = bool((outs["i8"] == outs["f4"]).all())
    G.set_mad_policy(0)
    print(json.dumps(res), flush=True)
