timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gf2_outer.py tests/test_gpu_configs.py -x -q -k "ech or gf2 or cfg2 or cfg5" > gpurun_out/cl_col_tests.log 2>&1; echo EXIT $? >> gpurun_out/cl_col_tests.log
GFQ_GF2_DEBUG=1 python tools/one_ech.py 1024 2 0 > gpurun_out/cl_col_dbg.log 2>&1
python tools/one_ech.py 1024 2 0 --time --reps 20 > gpurun_out/cl_col_time.log 2>&1
python tools/one_ech.py 8192 2 0 --time --reps 5 >> gpurun_out/cl_col_time.log 2>&1
python tools/one_step.py cfg2a 4 --warm --reps 5 >> gpurun_out/cl_col_time.log 2>&1
python tools/one_step.py cfg5s 4 --reserve --warm --reps 3 >> gpurun_out/cl_col_time.log 2>&1
