cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pool_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pool_tests.log
GFQ_HOSTPROF=1 python tools/one_step.py cfg5s 4 --warm --reps 4 > gpurun_out/cfg5_var2.log 2>&1
timeout 900 python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5s.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_final.log 2>&1
