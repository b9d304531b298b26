"""The fused in-device opens must leave every output share word-identical to the two-payload
forms: the eps open summed at build time (Open::summed, off with MPCG_EPS_FUSE=0) and the
opened-value wire of pair-evaluated adder rounds (off with MPCG_PAIR_EVAL=0, which evaluates
each party slot separately with its own payload), and the round-2 fusions (pair GEMV, deferred
delta, fused residual adds, wave-fill split-K) against their unfused forms. Runs each form in a
subprocess (the knobs are read once)."""
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


def run(fuse, pair="1", **extra):
    env = dict(os.environ, MPCG_EPS_FUSE=fuse, MPCG_PAIR_EVAL=pair, **extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_fused_opens_match_two_payloads():
    a, b, c = run("1"), run("0"), run("0", pair="0")
    assert a == b
    assert a == c
    # the pair-evaluated GEMV with the deferred weight-side delta, the residual adds fused into
    # the GEMM epilogues and the wave-fill split-K against their separate / per-slot forms
    d = run("1", MPCG_GEMV_PAIR="0", MPCG_DELTA_DEFER="0", MPCG_FUSE_RESIDUAL="0", MPCG_TC2_WAVESPLIT="0")
    assert a == d


SCRIPT_LANES = r'''
import hashlib, json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2209_13643_b200 as mp
PHI = 0x9E3779B97F4A7C15
out = {}
for name in ["lenet5", "toy_resnet", "toy_bert"]:
    g = mp.ModelGraph.from_json(name)
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, public_weights=False, pipelined=True, chunks=4, chunk_threshold=0)
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    out[name] = [hashlib.sha1(ex.run(x).numpy().tobytes()).hexdigest() for _ in range(2)] + [s.stats(0), s.stats(1)]
    s.close()
s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
s.set_pipeline(chunks=4, threshold=0)
rng = np.random.default_rng(0)
X = s.tensor(rng.integers(0, 2**63, size=(2, 50000), dtype=np.uint64))
Y = s.tensor(rng.integers(0, 2**63, size=(2, 50000), dtype=np.uint64))
out["mul"] = hashlib.sha1(mp.beaver_mul(s, X, Y, "m", 4).numpy().tobytes()).hexdigest()
out["relu"] = hashlib.sha1(mp.relu_shares(s, X).numpy().tobytes()).hexdigest()
out["stats"] = [s.stats(0), s.stats(1)]
print(json.dumps(out))
''' % ROOT


def run_lanes(fuse, defer):
    # tensor cores forced on every eligible GEMM, so the small models' convolutions take the
    # both-slots kernel (and with defer=1 its deferred eps)
    env = dict(os.environ, MPCG_FUSE_LANES=fuse, MPCG_EPS_DEFER=defer, MPCG_TC_GEMM="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT_LANES], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_lane_fusion_and_deferred_eps_keep_shares_and_collectives():
    """Session::fuse_lanes (chunk lanes of a round launched as one kernel, collectives accounted
    per lane) and the deferred eps (E generated in the both-slots GEMM) change neither a share
    word nor the collective log (bytes, counts) of chunked models and ops."""
    ref = run_lanes("0", "0")
    assert run_lanes("1", "0") == ref
    assert run_lanes("1", "1") == ref
