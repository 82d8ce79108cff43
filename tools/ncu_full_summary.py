"""Summarise one-kernel `ncu --set full` reports into a JSON dict.

python tools/ncu_full_summary.py name=report.ncu-rep[:m,n,k,p] ... --json out.json
Reads `ncu -i <rep> --page raw --csv`; keeps the duration, DRAM bytes,
tensor-pipe / SM / L2 / DRAM utilisation and launch geometry, and (given the
shape) the algorithmic int8 ops (2 m n k) and achieved TOPS.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def summarise(rep, shape=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    out = {"kernel": v[h.index("Kernel Name")].split("(")[0]}
    for i, name in enumerate(h):
        if name in KEYS:
            val = v[i].replace(",", "")
            try:
                x = float(val) * SCALE.get(u[i], 1.0)
            except ValueError:
                x = val
            out[KEYS[name]] = x
    out["duration_us"] = out.pop("duration")
    out["dram_bytes_per_launch"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    if shape:
        m, n, k, p = shape
        out.update(m=m, n=n, k=k, p=p, int8_ops=2 * m * n * k)
        out["achieved_TOPS"] = 2 * m * n * k / (out["duration_us"] * 1e-6) / 1e12
        out["algorithmic_bytes"] = m * k + k * n + 2 * m * n
    return out


def main():
    res = {}
    args = [a for a in sys.argv[1:] if a != "--json"]
    dst = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    if dst:
        args.remove(dst)
    for a in args:
        name, spec = a.split("=", 1)
        rep, _, shp = spec.partition(":")
        shape = tuple(int(x) for x in shp.split(",")) if shp else None
        res[name] = summarise(rep, shape)
    txt = json.dumps(res, indent=1)
    print(txt)
    if dst:
        open(dst, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
