# cfg5s: K1 lane (serialised non-critical contractions) x SMs reserved for the critical path
for cfgv in "0 0" "1 0" "1 16" "1 24" "1 32" "0 16"; do
  set -- $cfgv
  if [ "$1" = 1 ]; then export GFQ_K1_LANE=1; else unset GFQ_K1_LANE; fi
  echo "== lane $1 reserve $2"; GFQ_K1_SM_RESERVE=$2 timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 4 2>&1 | grep rank
done
