"""Summarise a GFQ_PROF_DUMP launch-window dump (one step): per 1 ms bucket
which kernel families ran; K1-idle stretches and what ran during them.

  python tools/timeline.py dump.txt [bucket_ms]"""
import sys
from collections import defaultdict

NAMES = ["k1_tc", "k1_simt", "ech_gf2", "ech_panel", "select", "k1_f4"]
rows = [l.split() for l in open(sys.argv[1]) if l.strip() and not l.startswith("T ")]
iv = defaultdict(list)
for f, a, b in rows:
    iv[int(f)].append((float(a), float(b)))
t0 = min(a for v in iv.values() for a, _ in v)
t1 = max(b for v in iv.values() for _, b in v)
bucket = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
nb = int((t1 - t0) / bucket) + 1
busy = {f: [0.0] * nb for f in iv}
for f, v in iv.items():
    for a, b in v:
        a -= t0
        b -= t0
        q = int(a / bucket)
        while q < nb and q * bucket < b:
            lo, hi = max(a, q * bucket), min(b, (q + 1) * bucket)
            busy[f][q] = min(bucket, busy[f][q] + max(0.0, hi - lo))
            q += 1
print(f"span {t1 - t0:.1f} ms, {nb} buckets of {bucket} ms")
idle = [q for q in range(nb) if busy.get(0, [0] * nb)[q] < 0.05 * bucket]
print(f"K1-idle buckets: {len(idle)} ({len(idle) * bucket:.1f} ms)")
# runs of idle buckets with what else was active
runs, start = [], None
for q in range(nb + 1):
    if q < nb and q in set(idle):
        start = q if start is None else start
    elif start is not None:
        runs.append((start, q))
        start = None
for s, e in runs:
    act = {NAMES[f]: sum(busy[f][s:e]) for f in busy if f != 0 and sum(busy[f][s:e]) > 0}
    print(f"  idle {s * bucket:7.1f}-{e * bucket:7.1f} ms: " + ", ".join(f"{k} {v:.1f}" for k, v in act.items()))
