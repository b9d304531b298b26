"""Debug: P2P-link graph replays, two one-party sessions on cuda:0, k replays (MLP by default)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13643_b200 as mp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "pipelined"
g = mp.ModelGraph.from_json(name)
sess = [mp.Session(device=0, n_local=1, party=p, seed=1, mask_seed=1 ^ 0x9E3779B97F4A7C15, frac_bits=g.frac_bits)
        for p in (0, 1)]
sess[0].connect_p2p(sess[1])
w, x = mp.init_weights(g, 12), mp.demo_input(g, 13)


def party(p):
    s = sess[p]
    ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined")
    ex.deal_weights(w, 1)
    xin = s.deal_input(x, 2)
    ex.run(xin)
    ex.capture(xin)
    for i in range(k):
        ex.replay()
        s.sync()
        print(f"party {p} replay {i} done", flush=True)


th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
for t in th:
    t.start()
for t in th:
    t.join()
print("ok")
