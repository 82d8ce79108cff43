for c in cfg5s cfg4 cfg3 cfg2a; do
  echo "== $c auto";  timeout 300 python tools/one_step.py $c 4 --reserve --warm --reps 5 2>&1 | grep rank
done
