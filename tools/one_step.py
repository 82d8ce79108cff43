"""One echelonize step of a bench config (for ncu launch lists / traces).

python tools/one_step.py [cfg2a] [threads] [--trace out.csv]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04211_b200 import workloads  # noqa: E402
from paper_1806_04211_b200.workloads import CONFIGS  # noqa: E402
from paper_1806_04211_b200 import gfrref as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2a"
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
G.lib()
f = G.FieldSpec(cfg["p"])
C = workloads.build(G, name)
if "--reserve" in sys.argv:
    G.reserve_for(cfg["m"], cfg["n"], True)
G.synchronize()
if "--warm" in sys.argv:
    G.echelonize(C, f, G.EchelonizeOptions(block=cfg["block"], threads=threads))
    G.synchronize()
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
walls = []
if "--prof" in sys.argv:
    G.profile(True)
    G.profile_take_kinds()
for _ in range(reps):
    t0 = time.time()
    out = G.echelonize(C, f, G.EchelonizeOptions(block=cfg["block"], threads=threads,
                                                 collect_trace="--trace" in sys.argv))
    G.synchronize()
    walls.append(1e3 * (time.time() - t0))
print("rank", out.rank, "wall_ms", " ".join(f"{w:.2f}" for w in walls), "min", f"{min(walls):.2f}")
if "--prof" in sys.argv:
    for k, (l, w, ms, ums) in G.profile_take_kinds(with_union=True).items():
        unit = "TOPS" if k.startswith("k1") else "GB/s"
        rate = (w / (ums / 1e3) / (1e12 if unit == "TOPS" else 1e9)) if ums > 0 else 0
        print(f"prof {k:10s} launches {l / reps:8.1f}/step  event ms {ms / reps:8.2f}/step  busy ms "
              f"{ums / reps:8.2f}/step  {rate:9.1f} {unit} (work / busy)")
    G.profile(False)
print("device_memory", G.device_memory())
if "--trace" in sys.argv:
    import csv
    with open(sys.argv[sys.argv.index("--trace") + 1], "w") as fh:
        w = csv.writer(fh)
        w.writerow(["task_kind", "i", "j", "k", "worker", "start_ns", "end_ns", "detail", "dev_start_ns",
                    "dev_end_ns"])
        for t in out.trace():
            w.writerow([t["kind"], t["i"], t["j"], t["k"], t["worker"], t["start_ns"], t["end_ns"], t["detail"],
                        t["dev_start_ns"], t["dev_end_ns"]])
