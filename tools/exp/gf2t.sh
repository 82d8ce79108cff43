#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_chief.py -q -x -p no:cacheprovider -k "ech or gf2 or random_vs or cfg1 or dependency" 2>&1 | tail -2
echo "ech 1024 GF(2): $(timeout 120 python tools/one_ech.py 1024 2 0 --time --reps 20)"
echo "ech 8192 GF(2): $(timeout 120 python tools/one_ech.py 8192 2 0 --time --reps 5)"
echo "cfg2a $(timeout 300 python tools/one_step.py cfg2a 4 --reserve --warm --reps 12 | head -1)"
echo "cfg5s $(timeout 300 python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 | head -1)"
timeout 120 python tools/one_kernel.py ech2 1024 > /dev/null && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ech_gf2_cluster python tools/one_kernel.py ech2 1024 2>&1 | grep duration
