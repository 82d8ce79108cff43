"""Write profiles/r02_traffic.json from ncu --set full captures of the
bench's dominant shapes (tools/one_kernel.py under ncu, see
tools/exp/bench_r02.sh): per config and kernel family, the launch's DRAM
bytes (dram__bytes_read.sum + dram__bytes_write.sum) next to its
algorithmic bytes.

  python tools/traffic_json.py CONFIG FAMILY REP.ncu-rep SHAPE ALG_BYTES [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02_traffic.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    u = dict(zip(hdr, units))
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[k].replace(",", "")) * SCALE[u[k]]
    return tot, float(d["gpu__time_duration.sum"].replace(",", "")), u["gpu__time_duration.sum"]


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    args = sys.argv[1:]
    while args:
        cfg, fam, rep, shape, alg = args[:5]
        args = args[5:]
        tot, dur, unit = dram_bytes(rep)
        data.setdefault(cfg, {})[fam] = {"shape": shape, "dram_bytes": tot, "algorithmic_bytes": float(alg),
                                         "dram_over_algorithmic": tot / float(alg),
                                         "duration": f"{dur} {unit}", "ncu_rep": os.path.basename(rep)}
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
