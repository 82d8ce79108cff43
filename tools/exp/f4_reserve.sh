# cfg5s step time vs SMs kept free of persistent K1 launches and K1 launch pieces
for r in 0 8 16 24; do
  echo "== reserve $r"; GFQ_K1_SM_RESERVE=$r timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 2>&1 | grep rank
done
for w in 1 2 4; do
  echo "== waves $w"; GFQ_K1_MAX_WAVES=$w timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 2>&1 | grep rank
done
