#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tasks.py tests/test_gpu_chief.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in 0 1; do
  echo "== GFQ_NO_DMA_SELECT=$v"
  if [ $v = 1 ]; then export GFQ_NO_DMA_SELECT=1; else unset GFQ_NO_DMA_SELECT; fi
  timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 3 --prof
done
unset GFQ_NO_DMA_SELECT
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 3 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('cfg4 ms',d['ms_per_step'],'k1 busy frac',r['frac'],r['achieved'],'second',r['second']['family'],r['second']['achieved'])"
