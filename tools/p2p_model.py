"""The one-party-per-GPU code path on ONE B200: two n_local=1 sessions (party 0, party 1) on
cuda:0, each driven by its own host thread, linked by the device-flag P2P link (peer stores +
flags, no host events), each party's inference captured as a CUDA graph and replayed
concurrently. Blocking vs pipelined (chunk lanes 4, reference 2 MiB threshold) wall time per
inference — the pipelining effect on a real transport rather than the emulated link.

  python tools/p2p_model.py [model ...]
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13643_b200 as mp  # noqa: E402

PHI = 0x9E3779B97F4A7C15


def run(g, mode, reps=5):
    sess = [mp.Session(device=0, n_local=1, party=p, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
            for p in (0, 1)]
    sess[0].connect_p2p(sess[1])
    w, x = mp.init_weights(g, 12), mp.demo_input(g, 13)
    walls, err = [0.0, 0.0], []
    go = threading.Barrier(2)

    def party(p):
        try:
            s = sess[p]
            ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined", chunks=4, chunk_threshold=2 << 20)
            ex.deal_weights(w, 1)
            xin = s.deal_input(x, 2)
            ex.run(xin)
            ex.capture(xin)
            ex.replay()
            s.sync()
            go.wait()
            t0 = time.perf_counter()
            for _ in range(reps):
                ex.replay()
            s.sync()
            walls[p] = (time.perf_counter() - t0) / reps
            del ex
        except Exception as e:  # noqa: BLE001
            err.append(repr(e))
            go.abort()

    th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    if err:
        raise RuntimeError(err[0])
    return max(walls) * 1e3


models = sys.argv[1:] or ["lenet5", "resnet18"]
for name in models:
    g = mp.ModelGraph.from_json(name)
    b = run(g, "blocking")
    p = run(g, "pipelined")
    print(json.dumps({"model": name, "link": "device-flag P2P, both parties on cuda:0, graph replay",
                      "blocking_ms": b, "pipelined_ms": p, "reduction_pct": (b - p) / b * 100}), flush=True)
