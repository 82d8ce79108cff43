#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_chief.py -q -p no:cacheprovider -k "criterion6 or concurrent" 2>&1 | tail -15
echo "first steps after reserve: $(timeout 300 python tools/one_step.py cfg5s 4 --reserve --reps 4 | head -1)"
