import sys, json, numpy as np
sys.path.insert(0, '.')
from paper_1806_04211_b200 import gfrref as G
import oracle
mode = sys.argv[1]
p, m, n, block = 5, 20, 20, 3
C = oracle.random_matrix(p, m, n, 3)
try:
    if mode == "nofuse":
        out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=1, fuse=False))
    elif mode == "notrans":
        out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=1, with_transform=False))
    else:
        b2 = int(mode)
        out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=b2, threads=1))
    G.synchronize()
    print(mode, "ok", out.rank)
except Exception as e:
    print(mode, "FAIL", str(e)[:100])
