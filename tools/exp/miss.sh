#!/bin/bash
cd $GRAFT_REPO_ROOT
echo "== warm reserve 100 GB"
GFQ_POOL_RESERVE_MB=100000 GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 4 2>&1 | grep -E "rank|alloc_miss|sync "
echo "== warm reserve 40 GB"
GFQ_POOL_RESERVE_MB=40000 GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 4 2>&1 | grep -E "rank|alloc_miss|sync "
echo "== no cache"
GFQ_NO_BLOCK_CACHE=1 GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 4 2>&1 | grep -E "rank|alloc_miss|sync "
