"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

python tools/ncu_summary.py launches.csv [--json out.json]
Prints per-kernel launch counts, total / mean device time and share.
"""
import csv
import collections
import json
import re
import sys


def short_name(full):
    """`void ns::kern<ns::Cfg<1, 2>, 3>(args)` -> `kern<ns::Cfg<1, 2>, 3>`: cut the
    argument list at the first '(' outside template brackets (not the one in
    `(anonymous namespace)` / `<unnamed>`), then the leading namespaces."""
    # ncu prints names from an anonymous namespace as `unnamed>::kern(...)`
    full = full.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    depth = 0
    end = len(full)
    for i, ch in enumerate(full):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            end = i
            break
    name = re.sub(r"^void\s+", "", full[:end].strip())
    depth = 0
    start = 0
    for i, ch in enumerate(name):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == ":" and depth == 0:
            start = i + 1
    return name[start:]


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = short_name(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def main():
    agg = load(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 2),
                    "share": round(t / tot, 4) if tot else 0})
        print(f"{t:11.1f} us {n:6d} x {t / n:9.2f} us  {100 * t / tot:5.1f}%  {k}")
    print(f"total device time {tot:.1f} us over {sum(n for n, _ in agg.values())} launches")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump({"total_us": tot, "kernels": out}, f, indent=1)


if __name__ == "__main__":
    main()
