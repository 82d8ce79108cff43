for v in 0 1; do echo "== GFQ_GF2_OUTER=$v"; GFQ_GF2_OUTER=$v timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 2>&1 | grep rank; done
echo "== ech 8192 outer"; GFQ_GF2_OUTER=1 python tools/one_ech.py 8192 2 0 --time --reps 5
echo "== ech 8192 split"; python tools/one_ech.py 8192 2 0 --time --reps 5
