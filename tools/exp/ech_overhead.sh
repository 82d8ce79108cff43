cd $GRAFT_REPO_ROOT
for a in "500 3" "1024 7" "4096 251"; do echo "== $a" >> gpurun_out/eo.log; GFQ_HOSTPROF=1 python tools/one_ech.py $a 0 --time --reps 20 >> gpurun_out/eo.log 2>&1; done
n=0; for a in "500 3" "1024 7"; do n=$((n+1)); timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/eo_$n.csv python tools/one_ech.py $a 0 > /dev/null 2>&1; done
