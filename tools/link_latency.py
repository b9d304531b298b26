"""Per-round latency of the party links on one GPU (one JSON line).

A ReLU of n elements is 9 reveals + 1 p2p exchange; its wall time per
round isolates what each transport costs per exchange:
  * two_slot   — both parties in one session (in-device zero-copy opens; persistent chain or
                 one kernel per round, the 1-GPU production path)
  * p2p        — two one-party sessions on two host threads, device-initiated peer stores +
                 acquire/release flags (mpcg_session_connect_p2p), eager and graph-replayed
  * loopback   — two one-party sessions, host-coordinated device copies
Times are wall clock after a stream sync, median of `reps` ReLUs, both parties on cuda:0.
"""
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13643_b200 as mp  # noqa: E402

ROUNDS = 10  # reveals + exchanges of one relu_shares (2PC, merged adder)


def two_slot(n, reps):
    s = mp.Session(device=0, n_local=2, seed=3, mask_seed=4, frac_bits=16)
    x = s.tensor(np.zeros((2, n), dtype=np.uint64), 16)
    ts = []
    for i in range(reps + 2):
        s.sync()
        t0 = time.perf_counter()
        mp.relu_shares(s, x, "r")
        s.sync()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts[2:])


def pair(n, reps, kind, graph=False):
    sess = [mp.Session(device=0, n_local=1, party=p, seed=3, mask_seed=4, frac_bits=16) for p in (0, 1)]
    (sess[0].connect_p2p if kind == "p2p" else sess[0].connect_loopback)(sess[1])
    walls = [[], []]
    bar = threading.Barrier(2)

    def party(p):
        s = sess[p]
        x = s.tensor(np.zeros((1, n), dtype=np.uint64), 16)
        g = mp.ModelGraph.from_json({"name": "relu", "frac_bits": 16, "input": [n],
                                     "layers": [{"name": "r", "type": "relu"}]}) if graph else None
        if graph:
            ex = mp.SecureExecutor(s, g)
            ex.deal_weights({}, 1)
            ex.run(x)
            ex.capture(x)
            step = ex.replay
        else:
            def step():
                return mp.relu_shares(s, x, "r")
        for i in range(reps + 2):
            bar.wait()
            s.sync()
            t0 = time.perf_counter()
            step()
            s.sync()
            walls[p].append(time.perf_counter() - t0)

    th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return statistics.median([max(a, b) for a, b in zip(walls[0][2:], walls[1][2:])])


def main():
    reps = 20
    out = {"note": __doc__.strip().splitlines()[0], "rounds_per_relu": ROUNDS, "sizes": {}}
    for n in (1024, 16384, 262144):
        r = {"two_slot": two_slot(n, reps), "p2p_eager": pair(n, reps, "p2p"),
             "p2p_graph": pair(n, reps, "p2p", graph=True), "loopback_eager": pair(n, reps, "loopback")}
        out["sizes"][str(n)] = {k: {"relu_us": v * 1e6, "per_round_us": v * 1e6 / ROUNDS} for k, v in r.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
