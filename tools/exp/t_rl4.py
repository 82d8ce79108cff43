import sys, json, numpy as np
sys.path.insert(0, '.')
from paper_1806_04211_b200 import gfrref as G
ref = json.load(open('tests/golden/ref_runs.json'))
idx = [int(x) for x in sys.argv[1].split(',')]
for q in idx:
    run = ref["echelonize"][q]
    C = np.array(run["C"], np.uint8).reshape(run["m"], run["n"])
    try:
        out = G.echelonize(C, G.FieldSpec(run["p"]), G.EchelonizeOptions(block=run["block"], threads=1, with_transform=run["with_transform"]))
        G.synchronize()
        print(q, "ok", out.rank, flush=True)
    except Exception as e:
        print(q, "FAIL", str(e)[:80], flush=True)
        break
