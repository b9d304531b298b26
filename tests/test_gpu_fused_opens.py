"""The fused in-device opens must leave every output share word-identical to the two-payload
forms: the eps open summed at build time (Open::summed, off with MPCG_EPS_FUSE=0) and the
opened-value wire of pair-evaluated adder rounds (off with MPCG_PAIR_EVAL=0, which evaluates
each party slot separately with its own payload). Runs each form in a subprocess (the knobs
are read once)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import hashlib, json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2209_13643_b200 as mp
PHI = 0x9E3779B97F4A7C15
out = {}
for name in ["mlp", "lenet5", "toy_resnet", "toy_bert"]:
    g = mp.ModelGraph.from_json(name)
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, public_weights=False, pipelined=True, chunks=2)
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    out[name] = [hashlib.sha1(ex.run(x).numpy().tobytes()).hexdigest() for _ in range(2)]
    s.close()
s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
rng = np.random.default_rng(0)
for (M, K, N) in [(1024, 576, 64), (8, 300, 40), (4, 64, 64)]:
    X = s.tensor(rng.integers(0, 2**63, size=(2, M, K), dtype=np.uint64))
    Y = s.tensor(rng.integers(0, 2**63, size=(2, K, N), dtype=np.uint64))
    out[f"mm{M}x{K}x{N}"] = hashlib.sha1(mp.beaver_matmul(s, X, Y, False, "t").numpy().tobytes()).hexdigest()
for n in (1000, 300000):
    X = s.tensor(rng.integers(0, 2**63, size=(2, n), dtype=np.uint64))
    out[f"relu{n}"] = hashlib.sha1(mp.relu_shares(s, X).numpy().tobytes()).hexdigest()
print(json.dumps(out))
''' % ROOT


def run(fuse, pair="1"):
    env = dict(os.environ, MPCG_EPS_FUSE=fuse, MPCG_PAIR_EVAL=pair)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_fused_opens_match_two_payloads():
    a, b, c = run("1"), run("0"), run("0", pair="0")
    assert a == b
    assert a == c
