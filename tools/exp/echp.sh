#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
for n in 1024 2048 4096; do echo "ech $n GF(251): $(timeout 120 python tools/one_ech.py $n 251 0 --time --reps 5)"; done
echo "ech 2048 GF(7): $(timeout 120 python tools/one_ech.py 2048 7 0 --time --reps 5)"
echo "ech 500 GF(3): $(timeout 120 python tools/one_ech.py 500 3 0 --time --reps 5)"
timeout 120 python tools/one_ech.py 4096 251 0 > /dev/null && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/ech4096_251.csv python tools/one_ech.py 4096 251 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02/ech4096_251.csv | head -14
