"""Run one model config end to end on cuda:0 (both parties): eager + CUDA-graph latency,
per-layer device times, pipelined vs blocking, optional emulated link and plaintext check.

  python tools/run_model.py vgg16 [--mode both] [--link 10gbps] [--iters 3] [--check]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("model")
ap.add_argument("--mode", default="both", choices=["blocking", "pipelined", "both"])
ap.add_argument("--weights", default="private")
ap.add_argument("--link", default="")
ap.add_argument("--chunks", type=int, default=4)
ap.add_argument("--threshold", type=int, default=2 << 20)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--check", action="store_true", help="decode and compare with the numpy plaintext forward")
ap.add_argument("--no-graph", action="store_true", help="eager runs only (no CUDA-graph capture)")
a = ap.parse_args()

g = mp.ModelGraph.from_json(a.model)
if a.batch:
    g = g.with_batch(a.batch)
t0 = time.time()
w = mp.init_weights(g, 12)
x = mp.demo_input(g, 13)
setup_s = time.time() - t0
link = {"10gbps": (1e-4, 1.25e9, 0.0), "1gbps": (1e-3, 1.25e8, 0.0)}.get(a.link)
out = {"model": g.name, "input": list(g.input), "weights_setup_s": setup_s}
for mode in (["blocking", "pipelined"] if a.mode == "both" else [a.mode]):
    s = mp.Session(device=0, n_local=2, seed=1, frac_bits=g.frac_bits)
    if link:
        s.set_link(*link)
    ex = mp.SecureExecutor(s, g, public_weights=a.weights == "public", pipelined=mode == "pipelined",
                           chunks=a.chunks, chunk_threshold=a.threshold)
    ex.deal_weights(w, 1)
    xin = s.deal_input(x, 2)
    t0 = time.time()
    z = ex.run(xin)
    s.sync()
    first_s = time.time() - t0
    api.timer(s, "reset")
    for _ in range(a.iters):
        api.timer(s, "start")
        z = ex.run(xin)
        api.timer(s, "stop")
    eager_ms = api.timer(s, "read") / a.iters
    ex.time_layers(True)
    if a.no_graph:
        z = ex.run(xin)
        s.sync()
        graph_ms = None
    else:
        ex.capture(xin)
        api.timer(s, "reset")
        for _ in range(a.iters):
            api.timer(s, "start")
            z = ex.replay()
            api.timer(s, "stop")
        graph_ms = api.timer(s, "read") / a.iters
    layers = ex.layer_times()
    st = s.stats(0)
    res = {"first_run_s": first_s, "eager_ms": eager_ms, "graph_ms": graph_ms,
           "bytes_sent_per_party_per_inference": None,
           "per_layer_ms": {l.name: round(t, 4) for l, t in zip(g.layers, layers)}, "stats": st}
    if a.check:
        from oracle import mpc_oracle as O
        import json as _j
        go = O.model_from_json(_j.load(open(os.path.join(ROOT, "configs", a.model + ".json"))))
        if a.batch:
            go = O.Model(go.name, go.frac_bits, tuple(g.input), go.layers)
        ref = O.reference_forward(go, w, x)
        zz = z.numpy()
        dec = (zz[0] + zz[1]).view(np.int64).astype(np.float64) * 2.0 ** -g.frac_bits
        err = np.abs(dec.reshape(-1) - ref.reshape(-1))
        res["max_abs_err_vs_plaintext"] = float(err.max())
        res["frac_within_2^-6"] = float((err <= 2.0 ** -6).mean())
        res["median_abs_err"] = float(np.median(err))
    out[mode] = res
    print(json.dumps({mode: {k: v for k, v in res.items() if k != "per_layer_ms"}}), flush=True)
    del ex
    s.close()
if "blocking" in out and "pipelined" in out:
    key = "eager_ms" if a.no_graph else "graph_ms"
    b, p = out["blocking"][key], out["pipelined"][key]
    out["pipelined_vs_blocking_reduction_pct"] = (b - p) / b * 100
print(json.dumps(out))
