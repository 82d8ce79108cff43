"""Run single device jobs once (for ncu launch lists): python tools/one_ech.py [n] [p] [mode]
--reps R: run R times; --time: one untimed warm-up, then print the mean wall ms of R calls;
--prof: launch windows per kernel family (with GFQ_PROF_DUMP=path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04211_b200 import gfrref as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
G.lib()
G.set_ech_mode(mode)
f = G.FieldSpec(p)
H = G.random_matrix(f, n, n, 7)
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
if "--time" in sys.argv:
    G.ech(f, H)
    G.synchronize()
if "--prof" in sys.argv:
    G.profile(True)
    G.profile_take_kinds()
t0 = time.perf_counter()
for _ in range(reps):
    e = G.ech(f, H)
G.synchronize()
if "--prof" in sys.argv:
    G.profile_take_kinds()  # GFQ_PROF_DUMP=path writes the launch windows
    G.profile(False)
dt = (time.perf_counter() - t0) / reps
print("rank", e.rank(), "ms %.3f" % (1e3 * dt) if "--time" in sys.argv else "")
