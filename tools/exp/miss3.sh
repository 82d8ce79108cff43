#!/bin/bash
cd $GRAFT_REPO_ROOT
echo "== cfg5s fresh"
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 6 2>&1 | grep -E "rank|alloc_miss|sync |device_memory"
echo "== cfg4 fresh"
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg4 4 --reps 6 2>&1 | grep -E "rank|alloc_miss"
echo "== cfg2a fresh"
timeout 300 python tools/one_step.py cfg2a 4 --reps 8 2>&1 | grep -E "rank"
