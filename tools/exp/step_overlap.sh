#!/bin/bash
# overlapped two-level ECH steps (chain of step s+1 during the update of s,
# flag handoff chain -> update): parity, single-block timing on/off, timeline
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_chief.py tests/test_gpu_configs.py -x -q > gpurun_out/ov_test.log 2>&1
echo "test exit $?" >> gpurun_out/ov_test.log
for o in 0 1; do
  for a in "4096 251" "2048 7" "1024 3"; do
    set -- $a
    GFQ_STEP_OVERLAP=$o timeout 120 python tools/one_ech.py $1 $2 0 --time --reps 5 >> gpurun_out/ov_time_$o.log 2>&1
  done
done
GFQ_STEP_TL=120 timeout 60 python tools/one_ech.py 4096 251 0 > gpurun_out/tl_1.log 2>&1
for c in cfg4 cfg3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ov_step_${c}_1.log 2>&1
done
