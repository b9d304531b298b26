"""CPU tests of the oracle's config-enabling extensions (GeLU, LayerNorm, residual graphs,
global average pool). The reference has no such layers, so these pin the
restatement to plaintext float64 math and to the reference's own invariants (chunking and
pipelining change traffic, never values — P/tests/acceptance.cpp AC2)."""
import json
import os

import numpy as np
import pytest

from oracle import mpc_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sh(seed, shape, f, lo, hi):
    x = np.random.default_rng(seed).uniform(lo, hi, shape)
    return x, O.share_additive(O.encode_fixed(x, f), O.CounterRng(seed, 3))


def test_sigmoid_accuracy_over_wide_range():
    f = 20
    x, X = _sh(1, (4000,), f, -30, 30)
    sg = O.decode_fixed(O.reconstruct(O.sigmoid_shares(X, O.make_ctx(2, f), "s")), f)
    assert np.abs(sg - 1 / (1 + np.exp(-x))).max() < 5e-4  # exp_shares: 7 squarings


@pytest.mark.parametrize("f", [16, 20])
def test_gelu_accuracy(f):
    x, X = _sh(2, (3000,), f, -8, 8)
    g = O.decode_fixed(O.reconstruct(O.gelu_shares(X, O.make_ctx(3, f), "g")), f)
    assert np.abs(g - x / (1 + np.exp(-1.702 * x))).max() < (2.0 ** -10 if f == 20 else 2.0 ** -8)


def test_inv_sqrt_accuracy_in_range():
    f = 20
    v, V = _sh(3, (2000,), f, 0.3, 100)
    y = O.decode_fixed(O.reconstruct(O.inv_sqrt_shares(V, O.make_ctx(4, f), "i")), f)
    assert np.abs(y * np.sqrt(v) - 1).max() < 2e-2


@pytest.mark.parametrize("chunks", [1, 4])
def test_layernorm_values_independent_of_chunking(chunks):
    f, d = 20, 32
    x, X = _sh(4, (6, d), f, -2, 2)
    gamma = np.ones(d)
    beta = np.zeros(d)
    G = O.encode_fixed(gamma, f)
    Bt = O.encode_fixed(beta, f)
    c1 = O.make_ctx(5, f)
    cN = O.make_ctx(5, f)
    cN.chunks = chunks
    a = O.layernorm_shares(X, d, G, Bt, c1, "ln", public=True)
    b = O.layernorm_shares(X, d, G, Bt, cN, "ln", public=True)
    assert all(np.array_equal(a[p], b[p]) for p in range(2))
    mu = x.mean(1, keepdims=True)
    want = (x - mu) / np.sqrt(((x - mu) ** 2).mean(1, keepdims=True) + 1e-5)
    assert np.abs(O.decode_fixed(O.reconstruct(a), f) - want).max() < 2.0 ** -7


def test_residual_wiring_and_shapes():
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", "resnet18.json"))))
    shapes = O.infer_shapes(g)
    names = [l.name for l in g.layers]
    assert shapes[names.index("l4b2r2")] == (128, 512, 4, 4)
    assert shapes[-1] == (128, 10)
    src, oth = O.layer_inputs(g)
    assert oth[names.index("l2b1add")] == names.index("l2b1c2")
    assert src[names.index("l2b1sc")] == names.index("l1b2r2")
    b = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", "bert_base.json"))))
    assert O.infer_shapes(b)[-1] == (8, 128, 768)
    assert len(O.model_weight_shapes(b)) == 12 * 12


def test_bad_wiring_rejected():
    j = {"name": "x", "input": [1, 4], "layers": [{"name": "a", "type": "dense", "out": 4},
                                                   {"name": "s", "type": "add", "with": "nope"}]}
    with pytest.raises(ValueError):
        O.model_from_json(j)
    j["layers"][1]["with"] = "input"
    O.model_from_json(j)


@pytest.mark.parametrize("name", ["toy_resnet", "toy_bert"])
@pytest.mark.parametrize("public", [False, True])
def test_extension_models_track_plaintext(name, public):
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", name + ".json"))))
    out, opened, h, ctx = O.bench_party_values(g, 1, 1, public)
    ref = O.reference_forward(g, O.init_weights(g, 12), O.demo_input(g, 13))
    assert np.abs(O.decode_fixed(opened, g.frac_bits).reshape(-1) - ref.reshape(-1)).max() <= 2.0 ** -6


def test_extension_model_pipelined_equals_blocking_values():
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", "toy_bert.json"))))
    a = O.bench_party_values(g, 1, 2, False)
    b = O.bench_party_values(g, 1, 2, False)
    assert a[2] == b[2]
