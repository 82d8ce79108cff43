#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 2 --prof
GFQ_HOSTPROF=1 timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 1 2>&1 | grep -v "^hostprof .* 0.000 ms"
GFQ_MAD_LOG=1 timeout 300 python tools/one_step.py cfg5s 4 --reps 1 2> gpurun_out/cfg5_madlog.txt
python - <<'PY'
import collections
c = collections.Counter()
for ln in open("gpurun_out/cfg5_madlog.txt"):
    if ln.startswith("mad "):
        f = dict(kv.split("=") for kv in ln.split()[1:])
        k = int(f["k"]); kb = "k0" if k == 0 else "k<32" if k < 32 else "k<256" if k < 256 else "k>=256"
        c[(f["path"], kb)] += 1
for key, v in sorted(c.items()):
    print("madlog", key, v)
PY
timeout 300 python tools/one_ech.py 8192 2 0 --time --reps 3
GFQ_HOSTPROF=1 timeout 300 python tools/one_ech.py 8192 2 0 --time --reps 3 2>&1 | grep -v " 0.000 ms"
timeout 300 python tools/one_ech.py 1024 2 0 --time --reps 20
