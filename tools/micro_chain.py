"""Micro-benchmark: ReLU as a persistent chain vs one kernel per round (device time, CUDA
events on the session stream, graph-captured and eager)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

for n in (7680, 102400, 301056):
    for persistent in (True, False):
        s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
        s.set_persistent(persistent)
        x = s.tensor(np.random.default_rng(n).integers(0, 2**63, size=(2, n), dtype=np.uint64), 16)
        for _ in range(3):
            mp.relu_shares(s, x, "r")
        s.sync()
        api.timer(s, "reset")
        reps = 20
        for _ in range(reps):
            api.timer(s, "start")
            mp.relu_shares(s, x, "r")
            api.timer(s, "stop")
        ms = api.timer(s, "read") / reps
        print(f"n={n:7d} persistent={persistent!s:5s} eager device ms/relu = {ms:.4f}", flush=True)
        s.close()
