#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "mad or crz or gather" 2>&1 | tail -2
for g in 0 16 32 64; do
  GFQ_K1_GROUP_MB=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gf_mad_tc --launch-skip 2 --launch-count 1 python tools/one_kernel.py mad 2 8192 65536 8192 3 2>&1 | grep -E "duration|dram__bytes" | sed "s/^/group=$g /"
done
GFQ_K1_GROUP_MB=32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gf_mad_tc --launch-skip 2 --launch-count 1 -o gpurun_out/r02/k1_dominant_grouped -f python tools/one_kernel.py mad 2 8192 65536 8192 3 > /dev/null 2>&1; echo "ncu full rc=$?"
for g in 0 32; do
  echo "== group $g"; GFQ_K1_GROUP_MB=$g GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 3 --prof
done
