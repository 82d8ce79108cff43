# full measurement pass: GPU suite, benches, ncu captures (outputs in gpurun_out/meas/)
mkdir -p gpurun_out/meas
python -m pytest tests -m gpu -x -q > gpurun_out/meas/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/meas/gpu_tests.log
python bench.py > gpurun_out/meas/bench_cfg5s.json 2> gpurun_out/meas/bench_cfg5s.err
for c in cfg4 cfg3 cfg2a cfg2b cfg1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/meas/bench_$c.json 2> gpurun_out/meas/bench_$c.err; done
python tools/one_kernel.py mad4 2 8192 65536 8192 2 > gpurun_out/meas/one4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gf_mad_f4 -s 1 -c 1 -o gpurun_out/meas/k1f4_dominant python tools/one_kernel.py mad4 2 8192 65536 8192 2 > gpurun_out/meas/ncu_k1f4.log 2>&1
python tools/one_step.py cfg5s 4 > gpurun_out/meas/step_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/meas/cfg5s_launches.csv python tools/one_step.py cfg5s 4 > gpurun_out/meas/ncu_step.log 2>&1
