import os, sys, threading, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2209_13643_b200 as mp
PHI = 0x9E3779B97F4A7C15
kind = sys.argv[1] if len(sys.argv) > 1 else "loopback"
sess = [mp.Session(device=0, n_local=1, party=p, seed=5, mask_seed=6, frac_bits=16) for p in (0, 1)]
(sess[0].connect_p2p if kind == "p2p" else sess[0].connect_loopback)(sess[1])
def party(p):
    try:
        s = sess[p]
        x = s.tensor(np.arange(16, dtype=np.uint64).reshape(1, 16), 16)
        print(p, "tensor ok", flush=True)
        z = mp.beaver_mul(s, x, x, "m")
        print(p, "mul ok", flush=True)
        s.sync()
        print(p, "sync ok", z.numpy()[0][:3], flush=True)
        z = mp.relu_shares(s, x, "r")
        s.sync()
        print(p, "relu ok", flush=True)
    except Exception:
        traceback.print_exc()
th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
[t.start() for t in th]; [t.join() for t in th]
