cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 0 1; do
if [ $v = 1 ]; then export GFQ_NO_PDL=1; else unset GFQ_NO_PDL; fi
echo -n "nopdl=$v cfg5s: " >> gpurun_out/pdl5.log; python tools/one_step.py cfg5s 4 --warm --reps 2 >> gpurun_out/pdl5.log 2>&1
python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/pdl5_b.log 2>&1
python -c "
import json
for l in open('gpurun_out/pdl5_b.log'):
    if l.startswith('{'): d=json.loads(l); print('nopdl=$v cfg2a', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))
" >> gpurun_out/pdl5.log
done; done
