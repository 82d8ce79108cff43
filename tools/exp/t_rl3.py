import sys, json, numpy as np
sys.path.insert(0, '.')
from paper_1806_04211_b200 import gfrref as G
import oracle
p, m, n, block, seed = [int(x) for x in sys.argv[1:6]]
C = oracle.random_matrix(p, m, n, seed)
try:
    out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=1))
    G.synchronize()
    print(p, m, n, block, seed, "ok", out.rank)
except Exception as e:
    print(p, m, n, block, seed, "FAIL", str(e)[:60])
