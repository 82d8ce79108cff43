#!/bin/bash
cd $GRAFT_REPO_ROOT
for w in 0 4 8 16 32; do
  echo "== waves $w"
  GFQ_K1_MAX_WAVES=$w GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg5s 4 --warm --reps 3 --prof
done
GFQ_MAD_LOG=1 GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py cfg5s 4 --reps 1 2> gpurun_out/cfg5_madlog2.txt
python - <<'PY'
import collections
c = collections.Counter(); b = collections.Counter()
for ln in open("gpurun_out/cfg5_madlog2.txt"):
    if ln.startswith("select "):
        f = dict(kv.split("=") for kv in ln.split()[1:5])
        r, cc = int(f["rows"]), int(f["cols"])
        key = ("inline" if "inline" in ln else "wide", "rmap" if f["rmap"] == "1" else "-", "cmap" if f["cmap"] == "1" else "-",
               "big" if r * cc > 16 << 20 else "mid" if r * cc > 1 << 20 else "small")
        c[key] += 1; b[key] += 2 * r * cc
for k in sorted(c):
    print("selectlog", k, c[k], "%.1f MB" % (b[k] / 1e6))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ech8192_launches.csv python tools/one_ech.py 8192 2 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ech8192_launches.csv 2>&1 | head -30
