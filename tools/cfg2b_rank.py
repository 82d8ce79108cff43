import sys, os
sys.path.insert(0, os.getcwd())
from paper_1806_04211_b200 import gfrref as G, workloads
G.lib()
C = workloads.build(G, "cfg2b")
f = G.FieldSpec(2)
for t in (1, 4):
    for rep in range(3):
        out = G.echelonize(C, f, G.EchelonizeOptions(block=1024, threads=t))
        print(os.environ.get("TAG"), "threads", t, "rank", out.rank, flush=True)
