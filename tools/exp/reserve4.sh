#!/bin/bash
# cfg5s step vs the critical-path SM reserve (green partition + K1 cap)
run() { echo "== $1"; shift; env "$@" timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 4 2>&1 | grep -E "rank" ; }
run base GFQ_X=1
run r32 GFQ_GREEN_RESERVE=32 GFQ_K1_SM_RESERVE=32
run r48 GFQ_GREEN_RESERVE=48 GFQ_K1_SM_RESERVE=48
run r64 GFQ_GREEN_RESERVE=64 GFQ_K1_SM_RESERVE=64
run g32k16 GFQ_GREEN_RESERVE=32 GFQ_K1_SM_RESERVE=16
run base2 GFQ_X=1
