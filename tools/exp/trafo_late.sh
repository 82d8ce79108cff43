for v in 0 1; do
  echo "== late $v device"; GFQ_TRAFO_LATE=$v timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 5 2>&1 | grep rank
  echo "== late $v e2e"; GFQ_TRAFO_LATE=$v timeout 300 python tools/exp/e2e_dbg.py 2>&1 | grep "e2e call"
  echo "== late $v cfg4"; GFQ_TRAFO_LATE=$v timeout 300 python tools/one_step.py cfg4 4 --reserve --warm --reps 3 2>&1 | grep rank
done
