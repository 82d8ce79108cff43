#!/bin/bash
# round-2 measurement pass: GPU tests subset, bench (cfg5s default + cfg2a),
# ncu --set full of the dominant shapes, launch list of one cfg5s step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider -k "crz or cfg5s or poison or cfg4_vs or dropin" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r02/bench_cfg5s.json 2> gpurun_out/r02/bench_cfg5s.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02/bench_cfg5s.json
timeout 600 python bench.py --config cfg2a --no-cpu-baseline > gpurun_out/r02/bench_cfg2a.json 2>&1; echo "cfg2a rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02/bench_cfg2a.json').read().splitlines()[-1]);print('cfg2a ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gf_mad_tc --launch-skip 2 --launch-count 1 -o gpurun_out/r02/k1_dominant -f python tools/one_kernel.py mad 2 8192 65536 8192 4 > gpurun_out/r02/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select2d_v16 --launch-skip 1 --launch-count 1 -o gpurun_out/r02/sel_dominant -f python tools/one_kernel.py crz 8192 57344 8 > gpurun_out/r02/ncu_sel.log 2>&1; echo "ncu sel rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ech_gf2_cluster --launch-skip 1 --launch-count 1 -o gpurun_out/r02/ech_dominant -f python tools/one_kernel.py ech2 1024 > gpurun_out/r02/ncu_ech.log 2>&1; echo "ncu ech rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/cfg5s_launches.csv python tools/one_step.py cfg5s 4 > gpurun_out/r02/ncu_list.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/r02/cfg5s_launches.csv 2>&1 | head -20
