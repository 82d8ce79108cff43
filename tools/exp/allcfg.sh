#!/bin/bash
# round-2 bench lines for every config (cfg5s = default headline) + GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
( time timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider ) > gpurun_out/r02/gputests2.log 2>&1
tail -4 gpurun_out/r02/gputests2.log
for c in cfg1 cfg2a cfg2b cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py > gpurun_out/r02/bench_cfg5s.json 2> gpurun_out/r02/bench_cfg5s.err; echo "cfg5s rc=$?"
python - <<'PY'
import json
for c in ["cfg1", "cfg2a", "cfg2b", "cfg3", "cfg4", "cfg5s"]:
    try:
        d = json.loads(open(f"gpurun_out/r02/bench_{c}.json").read().splitlines()[-1])
    except Exception as e:
        print(c, "ERR", e); continue
    r = d["roofline"]
    print(c, "ms %.2f" % d["ms_per_step"], "val %.3e" % d["value"], "e2e_ms %.2f" % d["e2e"]["ms_per_step"],
          "cpu %.3e" % (d["cpu_baseline"]["value"] if d["cpu_baseline"] else 0), r["family"], "%.0f" % r["achieved"], "%.3f" % r["frac"],
          r["second"]["family"] if r.get("second") else None, "hbm %.2f GB" % (d["hbm"]["high_water_bytes"] / 1e9))
PY
