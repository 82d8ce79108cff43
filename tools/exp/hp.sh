#!/bin/bash
cd $GRAFT_REPO_ROOT
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 20 2>&1 | grep -v " 0.000 ms"
