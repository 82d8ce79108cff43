#!/bin/bash
# cfg5s / cfg4 race-hunting matrix: every cell repeats echelonize and checks
# run-to-run identity + Freivalds (tools/stress.py).  Usage on the GPU box:
#   bash tools/exp/race_matrix.sh REPS "cell1 cell2 ..."
cd $GRAFT_REPO_ROOT
REPS=${1:-4}
CELLS=${2:-"base pool nopdl poison pool_poison nocache eager sync"}
declare -A E
E[base]=""
E[pool]="GFQ_POOL_RESERVE_MB=150000"
E[nopdl]="GFQ_NO_PDL=1"
E[poison]="GFQ_POISON=3"
E[pool_poison]="GFQ_POOL_RESERVE_MB=150000 GFQ_POISON=3"
E[nocache]="GFQ_NO_BLOCK_CACHE=1"
E[eager]="GFQ_NO_LAZY_WAITS=1"
E[sync]="GFQ_SYNC_TASKS=1"
E[pool_nopdl]="GFQ_POOL_RESERVE_MB=150000 GFQ_NO_PDL=1"
for c in $CELLS; do
  env ${E[$c]} TAG=$c CFGS=${CFGS:-cfg5s,cfg4} timeout 900 python tools/stress.py $REPS 4 2>&1 | tail -n $((REPS * 2 + 3))
done
