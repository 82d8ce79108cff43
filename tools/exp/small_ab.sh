#!/bin/bash
# the two-half RowLengthen on / off: device-resident and end-to-end step times
cd $GRAFT_REPO_ROOT
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2 $1', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"; }
for r in 1 2 3 4; do for c in ${CFGS:-cfg4 cfg3}; do GFQ_RL_SPLIT=1 run $c split; GFQ_RL_SPLIT=0 run $c nosplit; done; done
