#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
( time timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider ) > gpurun_out/r02/gputests.log 2>&1
tail -5 gpurun_out/r02/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02/bench_final1.json 2> gpurun_out/r02/bench_final1.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02/bench_final1.json").read().splitlines()[-1])
r = d["roofline"]
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "cpu", d["cpu_baseline"]["value"])
print("roof", r["family"], r["achieved"], r["frac"], r["share_of_step"], "second", r["second"]["family"], r["second"]["achieved"], r["second"]["frac"])
print("hbm", d["hbm"]["high_water_bytes"], "clocks", d["clocks"])
PY
