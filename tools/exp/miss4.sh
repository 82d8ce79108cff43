#!/bin/bash
cd $GRAFT_REPO_ROOT
echo "== cfg5s fresh"
timeout 300 python tools/one_step.py cfg5s 4 --reps 6 2>&1 | grep -E "rank|device_memory"
echo "== cfg5s fresh eager loading"
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/one_step.py cfg5s 4 --reps 6 2>&1 | grep -E "rank|device_memory"
echo "== cfg4 fresh"
timeout 300 python tools/one_step.py cfg4 4 --reps 6 2>&1 | grep -E "rank"
echo "== cfg4 fresh eager"
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/one_step.py cfg4 4 --reps 6 2>&1 | grep -E "rank"
