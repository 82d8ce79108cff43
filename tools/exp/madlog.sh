#!/bin/bash
# cfg step shape log by task: python-side histogram of selects and SIMT mads
cd $GRAFT_REPO_ROOT
CFG=${1:-cfg5s}
GFQ_MAD_LOG=1 GFQ_POOL_RESERVE_MB=60000 timeout 300 python tools/one_step.py $CFG 4 --reps 1 2> gpurun_out/madlog_$CFG.txt
python - $CFG <<'PY'
import collections, sys
cfg = sys.argv[1]
c = collections.Counter(); b = collections.Counter()
for ln in open(f"gpurun_out/madlog_{cfg}.txt"):
    parts = ln.split()
    if not parts or parts[0] not in ("select", "mad"):
        continue
    f = dict(kv.split("=") for kv in parts[1:] if "=" in kv)
    if parts[0] == "select":
        r, cc = int(f["rows"]), int(f["cols"])
        key = ("sel", f["task"], "r" if f["rmap"] == "1" else "-", "c" if f["cmap"] == "1" else "-")
        c[key] += 1; b[key] += 2 * r * cc
    else:
        m, n, k = int(f["m"]), int(f["n"]), int(f["k"])
        key = ("mad", f["task"], f["path"], "k0" if k == 0 else "k<32" if k < 32 else "k>=32")
        c[key] += 1; b[key] += m * n * max(k, 1)
for k in sorted(c, key=lambda k: -b[k]):
    print("log", k, c[k], "%.1f MB-or-Mmac" % (b[k] / 1e6))
PY
