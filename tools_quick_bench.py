# scratch timing script (first GPU contact); superseded by bench.py
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import paper_2209_13643_b200 as mp
for name, mode in [("mlp","pipelined"),("mlp","blocking"),("lenet5","pipelined"),("lenet5","blocking"),("toy_transformer","pipelined")]:
    g = mp.ModelGraph.from_json(name)
    s = mp.Session(device=0, n_local=2, seed=1, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, pipelined=mode=="pipelined")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    for i in range(3): ex.run(x); s.sync()
    t=time.time(); K=10
    for i in range(K): out = ex.run(x)
    s.sync(); dt=(time.time()-t)/K
    ex.time_layers(True); ex.run(x); s.sync(); lt = ex.layer_times()
    print(json.dumps({"model":name,"mode":mode,"ms":dt*1e3,"layers":[round(v,3) for v in lt]}))
