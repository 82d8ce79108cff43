# the critical-path SM partition (K1 lane + 16 reserved SMs + green-context bulk streams) on/off, every config
for c in cfg5s cfg4 cfg3 cfg2a cfg2b cfg1; do
  echo "== $c on";  timeout 300 python tools/one_step.py $c 4 --reserve --warm --reps 5 2>&1 | grep rank
  echo "== $c off"; GFQ_K1_LANE=0 GFQ_K1_SM_RESERVE=0 GFQ_GREEN_RESERVE=0 timeout 300 python tools/one_step.py $c 4 --reserve --warm --reps 5 2>&1 | grep rank
done
