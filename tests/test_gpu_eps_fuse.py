"""The fused in-device eps open (Open::summed: the eps build writes own0 + own1 once, the
combine GEMM reads it as one operand) must leave every output share word-identical to the
two-payload form (MPCG_EPS_FUSE=0). Runs both forms in subprocesses (the knob is read once)."""
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
for name in ["mlp", "lenet5", "toy_resnet"]:
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
print(json.dumps(out))
''' % ROOT


def run(fuse):
    env = dict(os.environ, MPCG_EPS_FUSE=fuse)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_fused_eps_open_matches_two_payloads():
    a, b = run("1"), run("0")
    assert a == b
