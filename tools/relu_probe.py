"""One relu_shares (ResNet-18 conv1 output: 8.4M elements, batch 128) on cuda:0, both party slots,
chunk lanes 4 as in the bench configuration; for ncu captures of the adder rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 128 * 64 * 32 * 32
s = mp.Session(device=0, n_local=2, seed=3, frac_bits=20)
s.set_pipeline(chunks=4, threshold=2 << 20)
x = s.tensor(np.random.default_rng(0).integers(0, 2**64, size=(2, n), dtype=np.uint64))
for _ in range(2):
    mp.relu_shares(s, x, "relu")
s.sync()

if "--time" in sys.argv[2:] or (len(sys.argv) > 1 and sys.argv[-1] == "--time"):
    import json
    import time
    from paper_2209_13643_b200 import api
    reps = 5
    api.probe_start("adder_round")
    for _ in range(reps):
        mp.relu_shares(s, x, "relu")
    s.sync()
    ms, nl, units = api.probe_stop()
    t0 = time.perf_counter()
    for _ in range(reps):
        mp.relu_shares(s, x, "relu")
    s.sync()
    print(json.dumps({"n": n, "adder_level_us_per_relu": 1e3 * ms / reps, "level_launches": nl / reps,
                      "relu_ms_wall": (time.perf_counter() - t0) / reps * 1e3}))
