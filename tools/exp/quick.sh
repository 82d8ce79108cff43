#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_tasks.py tests/test_gpu_chief.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -2
GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 3 --prof
bash tools/exp/madlog.sh cfg5s | head -40
