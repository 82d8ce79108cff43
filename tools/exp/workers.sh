for w in 2 3 4 6 8; do echo "== workers $w"; timeout 300 python tools/one_step.py cfg5s $w --reserve --warm --reps 4 2>&1 | grep rank; done
