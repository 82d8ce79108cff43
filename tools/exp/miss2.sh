#!/bin/bash
cd $GRAFT_REPO_ROOT
for mb in 16 4; do
echo "== cache max $mb MB"
GFQ_CACHE_MAX_MB=$mb GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 5 2>&1 | grep -E "rank|alloc_miss|malloc|sync |device_memory"
done
echo "== cfg2a"
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg2a 4 --reps 8 2>&1 | grep -E "rank|alloc_miss|malloc"
echo "== cfg4"
timeout 300 python tools/one_step.py cfg4 4 --reps 4 2>&1 | grep -E "rank"
