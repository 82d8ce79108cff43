#!/bin/bash
# K1f operand-sharing clusters (GFQ_F4_CLUSTER = 1, 2, 4, 12): parity, then
# kernel throughput, then the cfg5s step.
mkdir -p gpurun_out
for c in 4 12 1; do
  GFQ_F4_CLUSTER=$c timeout 300 python -m pytest tests/test_gpu_f4.py -x -q > gpurun_out/f4cl_test_$c.log 2>&1
  echo "test exit $?" >> gpurun_out/f4cl_test_$c.log
done
for c in 1 2 4 12; do
  GFQ_F4_CLUSTER=$c timeout 300 python tools/f4_bench.py 2 > gpurun_out/f4cl_bench_$c.log 2>&1
done
for c in 2 4; do
  GFQ_F4_CLUSTER=$c timeout 400 python bench.py --no-cpu-baseline > gpurun_out/f4cl_step_$c.log 2>&1
done
