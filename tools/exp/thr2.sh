#!/bin/bash
cd $GRAFT_REPO_ROOT
for t in 3 4 5 6 8; do echo "cfg2a threads $t $(timeout 300 python tools/one_step.py cfg2a $t --reserve --warm --reps 10 | head -1)"; done
for t in 4 6; do echo "cfg1 threads $t $(timeout 300 python tools/one_step.py cfg1 $t --reserve --warm --reps 10 | head -1)"; done
for t in 4 6; do echo "cfg3 threads $t $(timeout 300 python tools/one_step.py cfg3 $t --reserve --warm --reps 3 | head -1)"; done
