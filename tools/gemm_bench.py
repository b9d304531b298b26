"""Ring-GEMM throughput: tcgen05 int8-limb vs SIMT on Beaver-matmul shapes.

Times only the GEMM kernels (library probe = CUDA events around every ring-GEMM launch)
inside mpcg_beaver_matmul. Work = ring MACs over every segment of both parties
(party 0: 3 segments incl. the dealer's A*B, party 1: 2). One ring MAC = 36 int8 MACs on
the tensor path.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

SHAPES = [(50176, 576, 64), (12544, 1152, 128), (8192, 2048, 64), (1024, 768, 768), (1024, 3072, 768),
          (6400, 150, 16)]
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
int8_peak_tops = 2 * peaks["bf16_tflops"]  # B200 dense int8 = 2x dense bf16 (4.5 vs 2.25 PF nominal)
rows = []
for M, K, N in SHAPES:
    rng = np.random.default_rng(M + K + N)
    s = mp.Session(device=0, n_local=2, seed=5, frac_bits=16)
    X = s.tensor(rng.integers(0, 2**63, size=(2, M, K), dtype=np.uint64))
    Y = s.tensor(rng.integers(0, 2**63, size=(2, K, N), dtype=np.uint64))
    for mode in ("tc", "simt"):
        api.set_gemm_mode(mode)
        mp.beaver_matmul(s, X, Y, False, "warm")
        s.sync()
        api.probe_start("gemm")
        reps = 5
        for _ in range(reps):
            mp.beaver_matmul(s, X, Y, False, "b")
        s.sync()
        ms, n, macs = api.probe_stop()
        rmacs = macs / (ms / 1e3)
        row = {"M": M, "K": K, "N": N, "mode": mode, "gemm_ms": ms / reps, "ring_mac_per_s": rmacs,
               "int8_tops": rmacs * 36 * 2 / 1e12 if mode == "tc" else None,
               "frac_of_int8_peak": rmacs * 36 * 2 / 1e12 / int8_peak_tops if mode == "tc" else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
    api.set_gemm_mode("auto")
    s.close()
