#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tasks.py tests/test_gpu_chief.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "not cfg3 and not poison" 2>&1 | tail -3
timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 --prof
timeout 300 python tools/one_step.py cfg4 4 --reserve --warm --reps 3
