"""Stage timeline of one both-slots tcgen05 GEMM CTA (MPCG_TC3_TRACE=1): where the pipeline waits.

  MPCG_TC3_TRACE=1 python tools/tc3_trace.py [cin cout hw batch]   (an executor conv, deferred eps)
"""
import ctypes as C
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

os.environ["MPCG_TC3_TRACE"] = "1"
sys.argv = [sys.argv[0]] + sys.argv[1:]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "conv_probe.py")).read())  # runs the conv
from paper_2209_13643_b200 import _native as N  # noqa: E402

buf = (C.c_uint64 * (256 * 8))()
N.call("mpcg_debug_tc3_trace", buf, 256 * 8)
t = np.array(buf, dtype=np.int64).reshape(256, 8)
rows = [r for r in t[:255] if r[0]]
t0 = rows[0][0]
mma_wait = sum(int(r[1] - r[0]) for r in rows)
mma_issue = sum(int(r[2] - r[1]) for r in rows)
span = int(rows[-1][2] - t0)
epi = int(t[255][1] - t[255][0]) if t[255][0] else -1
print(json.dumps({"stages": len(rows), "mainloop_cycles": span, "mma_wait_cycles": mma_wait, "mma_issue_cycles": mma_issue,
                  "epilogue_cycles": epi, "mma_wait_frac": mma_wait / span}))
print("stage type  mma_wait  mma_issue  gen(start->wait)  empty_wait  store+arrive")
for i, r in enumerate(rows[:40]):
    f = lambda a, b: int(r[b] - r[a]) if r[a] and r[b] else -1  # noqa: E731
    print(f"{i:5d} {'AER'[i % 3]:>4} {f(0, 1):9d} {f(1, 2):10d} {f(3, 4):17d} {f(4, 5):11d} {f(5, 6):13d}")
