#!/bin/bash
# Step-3 contractions with / without the critical-path SM reserve and K1 lane
cd $GRAFT_REPO_ROOT
run() { python bench.py --config $1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2 $1', round(d['ms_per_step'],2))"; }
for r in 1 2; do
  for c in cfg4 cfg5s; do
    run $c "default"
    GFQ_LATE_LANE=1 run $c "late_lane"
    GFQ_LATE_RESERVE=1 run $c "late_reserve"
    GFQ_LATE_LANE=1 GFQ_LATE_RESERVE=1 run $c "both(old)"
  done
done
