#!/bin/bash
# GF(2) split ECH: parity tests, single-ECH timings (split vs two-level), cfg5s/cfg2a step
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gf2_split or ech_large or two_level" -p no:cacheprovider 2>&1 | tail -3
for n in 1024 2048 4096 8192; do
  for mode in 0 2; do
    echo "ech n=$n mode=$mode $(timeout 300 python tools/one_ech.py $n 2 $mode --time --reps 3)"
  done
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "cfg5s or poison" -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -2
