"""Launch one kernel family on a fixed shape, for ncu captures of the
bench's dominant shapes (profiles/r02_traffic.json):

  python tools/one_kernel.py mad P M N K [reps]     K1: D = D + A.B (in place, like the step)
  python tools/one_kernel.py mad4 P M N K [reps]    the same on K1f (FP4 path, p in {2,3,5,7})
  python tools/one_kernel.py crz ROWS COLS ZEROS    column riffle with zero columns (K4 gather)
  python tools/one_kernel.py ech2 N                 GF(2) cluster ECH of an N x N block

Prints the algorithmic bytes of one launch (the roofline's unit)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04211_b200 import gfrref as G  # noqa: E402

mode = sys.argv[1]
G.lib()
if mode in ("mad", "mad4"):
    import torch
    p, m, n, k = (int(x) for x in sys.argv[2:6])
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    A = torch.randint(0, p, (m, k), dtype=torch.uint8, device="cuda")
    B = torch.randint(0, p, (k, n), dtype=torch.uint8, device="cuda")
    D = torch.randint(0, p, (m, n), dtype=torch.uint8, device="cuda")
    G.set_mad_policy(2 if mode == "mad" else 3)
    G.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(reps):
        G.mad_raw(p, m, n, k, A.data_ptr(), k, B.data_ptr(), n, D.data_ptr(), n, D.data_ptr(), n)
    torch.cuda.synchronize()
    print("algorithmic_bytes", m * k + k * n + 2 * m * n, "ops", 2 * m * n * k)
elif mode == "crz":
    rows, cols, zeros = (int(x) for x in sys.argv[2:5])
    f = G.FieldSpec(2)
    M = G.random_matrix(f, rows, cols, 3)
    rng = np.random.default_rng(1)
    lam = np.ones(cols + zeros, np.uint8)
    lam[rng.choice(cols + zeros, zeros, replace=False)] = 0
    lam = tuple(int(x) for x in lam)
    for _ in range(3):
        out = G.crz(M, lam, len(lam))
    G.synchronize()
    print("algorithmic_bytes", rows * cols + rows * (cols + zeros) + 4 * (cols + zeros))
elif mode == "ech2":
    n = int(sys.argv[2])
    f = G.FieldSpec(2)
    H = G.random_matrix(f, n, n, 7)
    for _ in range(3):
        e = G.ech(f, H)
    G.synchronize()
    r = e.rank()
    print("algorithmic_bytes", n * n + r * (2 * n - r), "rank", r)
else:
    raise SystemExit(__doc__)
