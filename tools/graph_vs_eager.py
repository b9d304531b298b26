import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tools'))
import run_configs as R
import paper_2209_13643_b200 as mp
for name in ["bert_base", "resnet18"]:
    g = mp.ModelGraph.from_json(name)
    for graph in (False, True):
        try:
            r = R.run_one(g, "blocking", "private", "device", graph=graph, iters=3)
            print(name, "graph" if graph else "eager", round(r["ms"], 3), flush=True)
        except Exception as e:
            print(name, graph, "ERR", repr(e)[:300], flush=True)
