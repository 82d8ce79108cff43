import sys, json, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1806_04211_b200 import gfrref as G
ref = json.load(open('tests/golden/ref_runs.json'))
for run in ref["echelonize"]:
    C = np.array(run["C"], np.uint8).reshape(run["m"], run["n"])
    print(run["p"], run["m"], run["n"], run["block"], run["with_transform"], flush=True)
    out = G.echelonize(C, G.FieldSpec(run["p"]), G.EchelonizeOptions(block=run["block"], threads=1, with_transform=run["with_transform"]))
    G.synchronize()
print("ok")
