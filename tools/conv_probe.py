"""Private 3x3 convolutions through the executor (single-layer graph, default ResNet-18 layer1:
b128 x 64 x 32 x 32 -> 64), pipelined, for ncu captures of the combine GEMM (deferred eps)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13643_b200 as mp  # noqa: E402

_a = [v for v in sys.argv[1:] if not v.startswith("--")]
cin, cout, hw, b = (int(v) for v in (_a[:4] if len(_a) >= 4 else (64, 64, 32, 128)))
cfg = {"name": "conv_probe", "frac_bits": 20, "input": [b, cin, hw, hw],
       "layers": [{"name": "c", "type": "conv2d", "out": cout, "kernel": 3, "stride": 1, "pad": 1}]}
path = os.path.join(tempfile.mkdtemp(), "conv.json")
json.dump(cfg, open(path, "w"))
g = mp.ModelGraph.from_json(path)
s = mp.Session(device=0, n_local=2, seed=1, frac_bits=g.frac_bits)
ex = mp.SecureExecutor(s, g, pipelined=True)
ex.deal_weights(mp.init_weights(g, 12), 1)
x = s.deal_input(mp.demo_input(g, 13), 2)
for _ in range(3):
    ex.run(x)
s.sync()

if "--time" in sys.argv:
    from paper_2209_13643_b200 import api
    reps = 5
    api.probe_start("gemm")
    for _ in range(reps):
        ex.run(x)
    s.sync()
    ms, n, macs = api.probe_stop()
    import time
    t0 = time.perf_counter()
    for _ in range(reps):
        ex.run(x)
    s.sync()
    wall = (time.perf_counter() - t0) / reps * 1e3
    print(json.dumps({"conv": [cin, cout, hw, b], "defer": os.environ.get("MPCG_EPS_DEFER", "1"),
                      "gemm_us": 1e3 * ms / reps, "run_ms": wall}))
