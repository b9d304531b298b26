"""Stage timeline of one tcgen05 GEMM CTA (MPCG_TC2_TRACE=1): where the pipeline waits.

  MPCG_TC2_TRACE=1 python tools/tc2_trace.py [M K N]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import _native as N  # noqa: E402

M, K, N_ = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (131072, 576, 64)
s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
rng = np.random.default_rng(0)
X = s.tensor(rng.integers(0, 2**63, size=(2, M, K), dtype=np.uint64))
Y = s.tensor(rng.integers(0, 2**63, size=(2, K, N_), dtype=np.uint64))
for _ in range(2):
    mp.beaver_matmul(s, X, Y, False, "t")
s.sync()
buf = (C.c_uint64 * (256 * 10))()
N.call("mpcg_debug_tc2_trace", buf, 256 * 10)
t = np.array(buf, dtype=np.int64).reshape(256, 10)
t0 = t[0, 0]
rows = [r for r in t if r[0] or r[3] or r[6]]
print("stage  mma_wait  mma_issue  G_wait  G_work  E_wait  E_work   (cycles)")
for i, r in enumerate(rows[:60]):
    f = lambda a, b: (r[b] - r[a]) if r[a] and r[b] else -1  # noqa: E731
    print(f"{i:5d} {f(0,1):9d} {f(1,2):10d} {f(3,4):7d} {f(4,5):7d} {f(6,7):7d} {f(7,8):7d}  start {r[0]-t0 if r[0] else -1}")
tot = rows[-1][2] - rows[0][0] if rows else 0
print("total", tot, "cycles; mma waiting", int(sum(max(0, r[1] - r[0]) for r in rows if r[0])),
      "issuing", int(sum(max(0, r[2] - r[1]) for r in rows if r[1])))
