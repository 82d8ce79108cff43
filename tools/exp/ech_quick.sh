#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gf2_split or ech_large or two_level or ech_random" -p no:cacheprovider 2>&1 | tail -2
for n in 1024 2048 4096 8192; do
  echo "ech n=$n $(timeout 300 python tools/one_ech.py $n 2 0 --time --reps 5)"
done
GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 3 --prof
GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg2a 4 --warm --reps 5 --prof
