#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_chief.py tests/test_gpu_dist.py tests/test_gpu_tasks.py tests/test_gpu_io.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in 0 1; do
  if [ $v = 1 ]; then export GFQ_NO_WORKER_POOL=1; else unset GFQ_NO_WORKER_POOL; fi
  echo "nowp=$v cfg2a $(timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 20 | head -1)"
  echo "nowp=$v cfg1 $(timeout 300 python tools/one_step.py cfg1 4 --reserve --warm --reps 20 | head -1)"
done
unset GFQ_NO_WORKER_POOL
echo "cfg3 $(timeout 300 python tools/one_step.py cfg3 4 --reserve --warm --reps 3 | head -1)"
echo "cfg4 $(timeout 300 python tools/one_step.py cfg4 4 --reserve --warm --reps 3 | head -1)"
echo "cfg5s $(timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 | head -1)"
