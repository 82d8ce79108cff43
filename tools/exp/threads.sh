#!/bin/bash
cd $GRAFT_REPO_ROOT
for t in 4 6 8; do echo "== threads $t"; timeout 300 python tools/one_step.py cfg5s $t --warm --reps 3; done
for t in 4 6; do echo "== cfg4 threads $t"; timeout 300 python tools/one_step.py cfg4 $t --warm --reps 3; done
echo "== first steps (fresh process, 5 reps, hostprof)"
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 5 2>&1 | grep -E "rank|alloc_miss|malloc|sync"
