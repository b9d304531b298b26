"""Beaver-combine GEMM kernel time at the ResNet-18 conv shapes (batch 128): the both-slots
kernel (gemm_tc3.cu, "auto") against one CTA per party slot (gemm_tc2.cu, "tc2").

Probe = CUDA events around the ring-GEMM kernel launches only (pack kernels excluded). Work =
ring MACs of every segment of both parties (party 0: 3 incl. the dealer's A*B, party 1: 2),
72 int8 ops per ring MAC (36 limb-pair MACs).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

SHAPES = [(131072, 576, 64), (32768, 1152, 128), (8192, 2304, 256), (2048, 4608, 512), (131072, 27, 64)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
int8_peak = 2 * peak["bf16_tflops"]
for M, K, N in SHAPES:
    rng = np.random.default_rng(M + K + N)
    s = mp.Session(device=0, n_local=2, seed=5, frac_bits=16)
    X = s.tensor(rng.integers(0, 2**64, size=(2, M, K), dtype=np.uint64))
    Y = s.tensor(rng.integers(0, 2**64, size=(2, K, N), dtype=np.uint64))
    res = {}
    for mode in ("auto", "tc2"):
        api.set_gemm_mode(mode)
        z = mp.beaver_matmul(s, X, Y, False, "warm").numpy()
        s.sync()
        api.probe_start("gemm")
        reps = 5
        for _ in range(reps):
            mp.beaver_matmul(s, X, Y, False, "b")
        s.sync()
        ms, n, macs = api.probe_stop()
        tops = macs * 72 / (ms / 1e3) / 1e12
        res[mode] = {"gemm_us": 1e3 * ms / reps, "int8_tops": tops, "frac_int8_peak": tops / int8_peak, "z": z}
    same = bool(np.array_equal(res["auto"]["z"], res["tc2"]["z"]))
    row = {"M": M, "K": K, "N": N, "identical": same}
    for mode in res:
        row[mode] = {k: round(v, 4) for k, v in res[mode].items() if k != "z"}
    print(json.dumps(row), flush=True)
    api.set_gemm_mode("auto")
    s.close()
