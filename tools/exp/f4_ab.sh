for cfg in cfg5s cfg3 cfg2a; do
  echo "== $cfg i8"; GFQ_NO_F4=1 timeout 300 python tools/one_step.py $cfg 4 --reserve --warm --reps 3 2>&1 | grep rank
  echo "== $cfg f4 1e11"; timeout 300 python tools/one_step.py $cfg 4 --reserve --warm --reps 3 2>&1 | grep rank
  echo "== $cfg f4 2e10"; GFQ_F4_MIN_MACS=2e10 timeout 300 python tools/one_step.py $cfg 4 --reserve --warm --reps 3 2>&1 | grep rank
done
