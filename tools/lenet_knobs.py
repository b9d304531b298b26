"""LeNet-5 b64 (the bench workload) under the engine's scheduling knobs: persistent compare
chains (0 = per-round kernels, 1 = always persistent, 2 = auto), PDL, gemm modes.
One CUDA-graph replay per step, CUDA events; prints one JSON line per variant."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

PHI = 0x9E3779B97F4A7C15
name = sys.argv[1] if len(sys.argv) > 1 else "lenet5"
g = mp.ModelGraph.from_json(name)
w = mp.init_weights(g, 12)
xg = mp.demo_input(g, 13)
for persistent in (2, 1, 0):
    for tc in ("auto", "simt"):
        api.set_gemm_mode(tc)
        s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        s.set_persistent(persistent)
        ex = mp.SecureExecutor(s, g, pipelined=True, chunk_threshold=1 << 62)
        ex.deal_weights(w, 1)
        x = s.deal_input(xg, 2)
        ex.run(x)
        ex.time_layers(True)
        ex.capture(x)
        for _ in range(3):
            ex.replay()
        s.sync()
        api.timer(s, "reset")
        for _ in range(20):
            api.timer(s, "start")
            ex.replay()
            api.timer(s, "stop")
        ms = api.timer(s, "read") / 20
        lt = ex.layer_times()
        print(json.dumps({"model": name, "persistent": persistent, "gemm": tc, "ms": round(ms, 4),
                          "layers": {l.name: round(t, 4) for l, t in zip(g.layers, lt)}}), flush=True)
        del ex
        s.close()
api.set_gemm_mode("auto")
