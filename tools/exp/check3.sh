#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_tasks.py tests/test_gpu_chief.py tests/test_gpu_configs.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "not poison" 2>&1 | tail -3
CFGS=cfg5s,cfg4 TAG=digest timeout 600 python tools/stress.py 1 4 2>&1 | tail -3
timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 --prof
