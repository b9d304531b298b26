import sys, os, json, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2209_13643_b200 as mp
from paper_2209_13643_b200 import api
s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
rng = np.random.default_rng(0)
M, K, N = 1, 25088, 4096
X = s.tensor(rng.integers(0, 2**63, size=(2, M, K), dtype=np.uint64))
Y = s.tensor(rng.integers(0, 2**63, size=(2, K, N), dtype=np.uint64))
for _ in range(2): mp.beaver_matmul(s, X, Y, False, "w")
s.sync()
for cls in ("gemm", "beaver"):
    pass
api.timer(s, "reset")
api.probe_start("gemm")
for _ in range(5):
    api.timer(s, "start"); mp.beaver_matmul(s, X, Y, False, "t"); api.timer(s, "stop")
s.sync()
ms, n, u = api.probe_stop()
print("total ms/iter", api.timer(s, "read") / 5, "gemm probe ms/iter", ms / 5, "launches", n / 5)
