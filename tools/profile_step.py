"""One eager 2PC inference after one warm-up inference, for ncu captures.

  N=$(python tools/profile_step.py --count)      # kernels per inference
  ncu --set full -s $N -c $N -o prof python tools/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13643_b200 as mp  # noqa: E402
from paper_2209_13643_b200 import api  # noqa: E402

model = os.environ.get("MODEL", "resnet18")
g = mp.ModelGraph.from_json(model)
s = mp.Session(device=0, n_local=2, seed=1, frac_bits=g.frac_bits)
# the bench.py configuration: pipelined, 4 chunk lanes for operands >= the reference's 2 MiB
thr = int(os.environ.get("THR", str(2 << 20)))
ex = mp.SecureExecutor(s, g, pipelined=True, chunks=4, chunk_threshold=thr)
ex.deal_weights(mp.init_weights(g, 12), 1)
x = s.deal_input(mp.demo_input(g, 13), 2)
ex.run(x)            # warm-up (includes the pipelined prologue)
s.sync()
n0 = api.launch_count()
ex.run(x)
s.sync()
if "--count" in sys.argv:
    print(api.launch_count() - n0)
