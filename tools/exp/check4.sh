#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_tasks.py tests/test_gpu_chief.py -q -x -p no:cacheprovider 2>&1 | tail -2
CFGS=cfg5s,cfg4,cfg2b TAG=digest timeout 600 python tools/stress.py 1 4 2>&1 | tail -4
timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 --prof
GFQ_GF2_DEBUG=1 timeout 120 python tools/one_ech.py 1024 2 0 2>&1 | head -12
GFQ_GF2_DEBUG=1 timeout 120 python tools/one_kernel.py ech2 2048 2>&1 | head -12
