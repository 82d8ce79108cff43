#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "ech" 2>&1 | tail -2
for v in 0 1; do
  if [ $v = 1 ]; then export GFQ_CHAIN1=1; else unset GFQ_CHAIN1; fi
  echo "== one-warp=$v"
  for n in 1024 4096; do echo "ech $n GF(251): $(timeout 120 python tools/one_ech.py $n 251 0 --time --reps 5)"; done
  echo "ech 2048 GF(7): $(timeout 120 python tools/one_ech.py 2048 7 0 --time --reps 5)"
  GFQ_STEP_DEBUG=2 timeout 120 python tools/one_ech.py 4096 251 0 2>&1 | grep ech_step | head -2
  for c in cfg4 cfg3 cfg1; do echo "$c $(timeout 300 python tools/one_step.py $c 4 --reserve --warm --reps 3 | head -1)"; done
done
