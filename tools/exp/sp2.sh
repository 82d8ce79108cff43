#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export GFQ_NO_STREAM_POOL=1; else unset GFQ_NO_STREAM_POOL; fi
  echo "nopool=$v cfg2a $(timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 20 | head -1)"
  echo "nopool=$v cfg1 $(timeout 300 python tools/one_step.py cfg1 4 --reserve --warm --reps 20 | head -1)"
done
