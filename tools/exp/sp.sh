#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_chief.py tests/test_gpu_dist.py tests/test_gpu_tasks.py -q -x -p no:cacheprovider 2>&1 | tail -2
echo "cfg2a $(timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 12 | head -1)"
echo "cfg1 $(timeout 300 python tools/one_step.py cfg1 4 --reserve --warm --reps 12 | head -1)"
