"""One e2e (host buffer in, host buffers out) cfg5s call with the
GFQ_E2E_DEBUG timeline (input row arrivals, output block downloads)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1806_04211_b200 import gfrref as G, workloads  # noqa: E402
from paper_1806_04211_b200.workloads import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5s"
cfg = CONFIGS[name]
G.lib()
f = G.FieldSpec(cfg["p"])
C = workloads.build(G, name)
G.reserve_for(cfg["m"], cfg["n"], True)
opts = G.EchelonizeOptions(block=cfg["block"], threads=4)
Ch = torch.empty((cfg["m"], cfg["n"]), dtype=torch.uint8, pin_memory=True)
Ch.numpy()[:] = C.numpy()
probe = G.echelonize(C, f, opts)
nbytes = probe.block_bytes()
del probe
dl = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = opts if rep < 2 else G.EchelonizeOptions(block=cfg["block"], threads=4, collect_trace=True)
    if rep == 2 and "--prof" in sys.argv:
        G.profile(True)
        G.profile_take_kinds()
    out = G.echelonize(Ch.numpy(), f, o, host_out=dl.numpy())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"e2e call {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms (returned at {1e3 * (t1 - t0):.1f})",
          file=sys.stderr, flush=True)
    if rep == 2 and "--prof" in sys.argv:
        G.profile_take_kinds()
        G.profile(False)
    if rep == 2:
        for t in sorted(out.trace(), key=lambda t: t["dev_start_ns"]):
            if t["kind"] in ("ClearDown", "RowLengthen", "PreClearUp") or (t["kind"] == "UpdateRow" and t["i"] == t["j"] + 1):
                print(f"  {t['kind']:12s} {t['i']:3d} {t['j']:3d} {t['k']:3d} dev {t['dev_start_ns'] / 1e6:8.2f}-"
                      f"{t['dev_end_ns'] / 1e6:8.2f} host {t['start_ns'] / 1e6:8.2f}-{t['end_ns'] / 1e6:8.2f}",
                      file=sys.stderr)
    del out
