#!/bin/bash
# bulk contractions cut into launches of <= N tile waves (GFQ_K1_MAX_WAVES): the
# critical path's kernels wait for at most one such launch to drain
cd $GRAFT_REPO_ROOT
run() { python bench.py --config cfg5s --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],2))"; }
run default
for w in 64 32 16 8; do GFQ_K1_MAX_WAVES=$w run "waves=$w"; done
for g in 16 32; do GFQ_CRIT_GRID=$g run "crit_grid=$g"; done
run default
