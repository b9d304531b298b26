"""Online-only latency vs the dealer's share.

The engine regenerates every Beaver/mask draw in registers inside the protocol kernels (the
reference's SeededDealer runs inside fetch, H/sharing/triple.hpp:138-151), so there is no
separate offline phase to time. This tool times each config twice on the same GPU: with the
real library and with the measurement build `lib/libmpcg_nodealer.so` (make dealerless), in
which device-side splitmix64 draws are the identity — the protocol's data movement, opens,
GEMMs and kernel launches are unchanged, only the dealer's arithmetic disappears. The
difference is the dealer cost; the second number is the online-only latency an offline
triple pool could at best reach (ignoring the pool's own reads). Values of the measurement
build are NOT the reference's and are never checked.

  python tools/dealer_split.py [--models lenet5,resnet18,...] [--out gpurun_out/dealer_split.json]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, ROOT)
import paper_2209_13643_b200 as mp
from paper_2209_13643_b200 import api
name, graph = sys.argv[1], sys.argv[2] == "1"
g = mp.ModelGraph.from_json(name)
s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ 0x9E3779B97F4A7C15, frac_bits=g.frac_bits)
ex = mp.SecureExecutor(s, g, pipelined=False)
ex.deal_weights(mp.init_weights(g, 12), 1)
x = s.deal_input(mp.demo_input(g, 13), 2)
ex.run(x); ex.run(x); s.sync()
ex.time_layers(True)
if graph:
    ex.capture(x)
    step = ex.replay
else:
    step = lambda: ex.run(x)
step(); s.sync()
api.timer(s, "reset")
for _ in range(5):
    api.timer(s, "start"); step(); api.timer(s, "stop")
print(json.dumps({"ms": api.timer(s, "read") / 5, "layers": {l.name: t for l, t in zip(g.layers, ex.layer_times())}}))
"""


def time_model(name, graph, lib):
    env = dict(os.environ)
    if lib:
        env["MPCG_LIB"] = lib
    out = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT)), name, "1" if graph else "0"],
                         capture_output=True, text=True, env=env, timeout=900)
    if out.returncode:
        raise RuntimeError(out.stderr[-500:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="mlp,lenet5,resnet18,bert_base,vgg16")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "dealer_split.json"))
    a = ap.parse_args()
    nod = os.path.join(ROOT, "paper_2209_13643_b200", "lib", "libmpcg_nodealer.so")
    if not os.path.exists(nod):
        raise SystemExit("build it first: make -C paper_2209_13643_b200/csrc dealerless")
    res = {}
    for m in a.models.split(","):
        graph = True  # whole-inference CUDA graphs fit the capture arena for every config
        full = time_model(m, graph, None)
        online = time_model(m, graph, nod)
        res[m] = {"blocking_ms": full["ms"], "online_only_ms": online["ms"],
                  "dealer_share_pct": (full["ms"] - online["ms"]) / full["ms"] * 100, "exec": "graph" if graph else "eager",
                  "per_layer": {k: {"ms": v, "online_only_ms": online["layers"][k]} for k, v in full["layers"].items()}}
        print(m, json.dumps({k: v for k, v in res[m].items() if k != "per_layer"}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
