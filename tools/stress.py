"""Repeat echelonize on cfg2a / cfg2b and check the outputs are identical
run to run (race hunting).  python tools/stress.py [reps] [threads]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04211_b200 import gfrref as G, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 4
G.lib()
if os.environ.get("MADPOL"):
    G.set_mad_policy(int(os.environ["MADPOL"]))
names = (os.environ.get("CFGS") or "cfg2a,cfg2b").split(",")
inputs = {n: workloads.build(G, n) for n in names}
want = {}
bad = 0
for r in range(reps):
    for name, C in inputs.items():
        cfg = workloads.CONFIGS[name]
        out = G.echelonize(C, G.FieldSpec(cfg["p"]), G.EchelonizeOptions(block=cfg["block"], threads=threads,
                                                                   retain_all=bool(os.environ.get("RETAIN"))))
        buf = bytearray(out.block_bytes())
        import numpy as np
        arr = np.frombuffer(buf, np.uint8).copy()
        out.download_blocks(arr)
        h = (out.rank, hashlib.sha1(arr.tobytes()).hexdigest())
        if name not in want:
            want[name] = h
        elif h != want[name]:
            bad += 1
            print("MISMATCH", name, "rep", r, h[0], "want", want[name][0], flush=True)
print(os.environ.get("TAG", ""), "reps", reps, "bad", bad, {k: v[0] for k, v in want.items()}, flush=True)
