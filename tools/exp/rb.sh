#!/bin/bash
cd $GRAFT_REPO_ROOT
echo "cfg2a $(timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 10 | head -1)"
echo "ech 8192 GF(2): $(timeout 120 python tools/one_ech.py 8192 2 0 --time --reps 5)"
echo "ech 1024 GF(2): $(timeout 120 python tools/one_ech.py 1024 2 0 --time --reps 20)"
echo "cfg5s $(timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 | head -1)"
