"""GPU parity for the config-enabling extensions (GeLU, LayerNorm, sigmoid, inverse sqrt,
global average pool, residual graphs) — layers the BASELINE configs need (ResNet-18,
BERT-base) and the reference lacks (SURVEY.md §0, §8(a*)).

Parity is UNPINNED by the reference for these: each party's GPU share must equal the oracle
restatement (oracle/mpc_oracle.py) word for word, and decoded values must track the float64
plaintext forward within the reference's model tolerance 2^-6 (P/tools/mpcpipe_bench.cpp:124).
"""
import json
import os

import numpy as np
import pytest

from oracle import mpc_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHI = 0x9E3779B97F4A7C15


@pytest.fixture(scope="module")
def mp():
    import paper_2209_13643_b200 as mp
    return mp


def _shares(seed, shape, f, lo=-2.0, hi=2.0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(lo, hi, size=shape)
    return O.share_additive(O.encode_fixed(x, f), O.CounterRng(seed, 0x55))


def _pair(mp, seed, f, chunks=1, threshold=0, persistent=True):
    s = mp.Session(device=0, n_local=2, seed=seed, mask_seed=seed ^ PHI, frac_bits=f)
    s.set_pipeline(chunks, threshold, True)
    s.set_persistent(persistent)
    ctx = O.make_ctx(seed, f)
    ctx.chunks, ctx.chunk_threshold = chunks, threshold
    return s, ctx


def _eq(Z, ref):
    assert np.array_equal(Z[0].reshape(-1), ref[0].reshape(-1)), "party 0 share differs"
    assert np.array_equal(Z[1].reshape(-1), ref[1].reshape(-1)), "party 1 share differs"


@pytest.mark.parametrize("persistent", [True, False], ids=["persistent", "per-round"])
@pytest.mark.parametrize("chunks", [1, 3])
def test_sigmoid_and_gelu(mp, persistent, chunks):
    f = 20
    X = _shares(5, (7, 33), f, -6, 6)
    s, ctx = _pair(mp, 41, f, chunks, 0, persistent)
    T = s.tensor(np.stack(X), f)
    _eq(mp.sigmoid_shares(s, T, "sg").numpy(), O.sigmoid_shares(X, ctx, "sg"))
    _eq(mp.gelu_shares(s, T, "ge").numpy(), O.gelu_shares(X, ctx, "ge"))
    st = s.stats(0)
    assert [st["bytes_sent"], st["collectives"], st["p2p_sends"]] == \
        [ctx.stats[0].bytes_sent, ctx.stats[0].collectives, ctx.stats[0].p2p_sends]
    x = O.decode_fixed(O.reconstruct(X), f)
    dec = O.decode_fixed(O.reconstruct(O.gelu_shares(X, O.make_ctx(3, f), "g2")), f)
    assert np.abs(dec - x / (1 + np.exp(-1.702 * x))).max() < 2.0 ** -8


def test_inv_sqrt(mp):
    f = 20
    V = _shares(6, (50,), f, 0.1, 50.0)
    s, ctx = _pair(mp, 42, f)
    Y = mp.inv_sqrt_shares(s, s.tensor(np.stack(V), f), "is").numpy()
    ref = O.inv_sqrt_shares(V, ctx, "is")
    _eq(Y, ref)


@pytest.mark.parametrize("public", [False, True], ids=["private", "public"])
def test_layernorm(mp, public):
    f = 20
    d = 24
    X = _shares(7, (5, 6, d), f)
    rng = np.random.default_rng(8)
    gamma = 1 + rng.uniform(-0.1, 0.1, d)
    beta = rng.uniform(-0.1, 0.1, d)
    s, ctx = _pair(mp, 43, f)
    if public:
        G = O.encode_fixed(gamma, f)
        Bt = O.encode_fixed(beta, f)
        gs, bs = np.stack([G, G]), np.stack([Bt, Bt])
        g_o, b_o = G, Bt
    else:
        g_o = O.share_additive(O.encode_fixed(gamma, f), O.CounterRng(9, 1))
        b_o = O.share_additive(O.encode_fixed(beta, f), O.CounterRng(9, 2))
        gs, bs = np.stack(g_o), np.stack(b_o)
    Z = mp.layernorm_shares(s, s.tensor(np.stack(X), f), d, s.tensor(gs, f), s.tensor(bs, f), public, "ln").numpy()
    ref = O.layernorm_shares(X, d, g_o, b_o, ctx, "ln", public)
    _eq(Z, ref)
    x = O.decode_fixed(O.reconstruct(X), f).reshape(-1, d)
    mu = x.mean(1, keepdims=True)
    want = (x - mu) / np.sqrt(((x - mu) ** 2).mean(1, keepdims=True) + 1e-5) * gamma + beta
    assert np.abs(O.decode_fixed(Z[0] + Z[1], f).reshape(-1, d) - want).max() < 2.0 ** -6


def test_global_avg_pool(mp):
    f = 20
    X = _shares(9, (3, 5, 4, 4), f)
    s, _ = _pair(mp, 44, f)
    Z = mp.global_avg_pool(s, s.tensor(np.stack(X), f), 3, 5, 16).numpy()
    _eq(Z, O.global_avg_pool(X, (3, 5, 4, 4), f))


def _oracle_model(name, mode, weights, iters):
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", name + ".json"))))
    out, opened, h, ctx = O.bench_party_values(g, 1, iters, weights == "public")
    return g, out, h, ctx


@pytest.mark.parametrize("persistent", [True, False], ids=["persistent", "per-round"])
@pytest.mark.parametrize("name,mode,weights,iters", [
    ("toy_resnet", "blocking", "private", 1), ("toy_resnet", "pipelined", "private", 2),
    ("toy_resnet", "blocking", "public", 1), ("toy_bert", "blocking", "private", 1),
    ("toy_bert", "pipelined", "private", 2), ("toy_bert", "blocking", "public", 1)])
def test_extension_models_match_oracle(mp, name, mode, weights, iters, persistent):
    go, ref, h, ctx = _oracle_model(name, mode, weights, iters)
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    s.set_persistent(persistent)
    ex = mp.SecureExecutor(s, g, public_weights=weights == "public", pipelined=mode == "pipelined")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    for _ in range(iters):
        z = ex.run(x).numpy()
    _eq(z, ref)
    assert mp.fnv1a_words((z[0] + z[1]).reshape(-1)) == h
    want = O.reference_forward(go, O.init_weights(go, 12), O.demo_input(go, 13))
    dec = O.decode_fixed(z[0] + z[1], g.frac_bits)
    assert np.abs(dec.reshape(-1) - want.reshape(-1)).max() <= 2.0 ** -6


@pytest.mark.parametrize("name", ["toy_resnet", "toy_bert"])
def test_extension_graph_replay(mp, name):
    """CUDA-graph replays of the residual graphs draw the same triples as eager runs."""
    _, ref, _, _ = _oracle_model(name, "pipelined", "private", 3)
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, public_weights=False, pipelined=True)
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    ex.run(x)
    ex.capture(x)
    ex.replay()
    z = ex.replay().numpy()
    _eq(z, ref)
