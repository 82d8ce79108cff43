"""Repeat echelonize on BASELINE workloads and check every run: identical
outputs run to run (SHA-1 of every output block, downloaded) and the
Freivalds identity T.(C.X) = E.X on the device (race hunting).

  CFGS=cfg5s TAG=x python tools/stress.py [reps] [threads]

Env: CFGS (comma list, default cfg2a,cfg2b), MADPOL, RETAIN, NOVERIFY,
plus any GFQ_* developer switch (GFQ_NO_PDL, GFQ_POISON, ...)."""
import hashlib
import os
import sys
import time

import numpy as np

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
bufs = {}
for r in range(reps):
    for name, C in inputs.items():
        cfg = workloads.CONFIGS[name]
        t0 = time.time()
        out = G.echelonize(C, G.FieldSpec(cfg["p"]), G.EchelonizeOptions(block=cfg["block"], threads=threads,
                                                                   retain_all=bool(os.environ.get("RETAIN"))))
        t1 = time.time()
        ok, diag = True, ""
        if not os.environ.get("NOVERIFY"):
            ok, diag, _ = G.verify(C, out, "freivalds")
        n = out.block_bytes()
        if name not in bufs or bufs[name].nbytes < n:
            bufs[name] = np.empty(n, np.uint8)
        arr = bufs[name][:n]
        out.download_blocks(arr)
        h = (out.rank, hashlib.sha1(arr).hexdigest())
        del out
        status = "ok"
        if name not in want:
            want[name] = h
        elif h != want[name]:
            bad += 1
            status = "MISMATCH"
        if not ok:
            bad += 1
            status += " FREIVALDS-FAIL " + diag
        print(f"{os.environ.get('TAG', '')} {name} rep {r} {t1 - t0:.3f}s rank {h[0]} {h[1][:12]} {status}",
              flush=True)
print(os.environ.get("TAG", ""), "reps", reps, "bad", bad, {k: v[0] for k, v in want.items()}, flush=True)
