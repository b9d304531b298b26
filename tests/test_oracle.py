"""CPU tests: the numpy oracle restatement is pinned to the reference's own outputs.

Fixtures come from the UNMODIFIED reference (tests/golden/make_golden.py). Mirrors the
reference's test layout (P/tests/test_sharing.cpp, test_protocols.cpp, test_nonlinear.cpp,
test_engine.cpp) but checks per-party shares word-for-word, not only reconstructions.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import mpc_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_prg_known_answer(golden_ops):
    assert (O.CounterRng(123, 7).take(16) == golden_ops["prg/123_7"]).all()


def test_prg_seekable():
    r = O.CounterRng(9, 2)
    a = r.take(10)
    r2 = O.CounterRng(9, 2)
    r2.counter = 4
    assert (r2.take(6) == a[4:]).all()


def test_additive_share_kat():
    # P/tests/test_sharing.cpp:38-45 pattern: party0 absorbs the randomness.
    r = O.CounterRng(3)
    s = O.share_additive(np.array([5], dtype=np.uint64), r)
    assert int(O.reconstruct(s)[0]) == 5


DEALER = {
    "mul0": (O.TripleSpec.elementwise("arith", (3, 4)), "t.mul"),
    "mul1": (O.TripleSpec.elementwise("arith", (3, 4)), "t.mul"),
    "and": (O.TripleSpec.elementwise("bin", (2, 5)), "t.and"),
    "sq": (O.TripleSpec.square_of((7,)), "t.sq"),
    "mm": (O.TripleSpec.matmul_of((3, 4), (4, 5)), "t.mm"),
    "qk": (O.TripleSpec.matmul_of((2, 3, 4), (2, 5, 4), True), "t.qk"),
    "av": (O.TripleSpec.matmul_of((2, 3, 5), (2, 5, 4)), "t.av"),
    "untag0": (O.TripleSpec.elementwise("arith", (6,)), ""),
    "untag1": (O.TripleSpec.elementwise("arith", (6,)), ""),
}


def test_dealer_matches_reference(golden_ops):
    d = O.SeededDealer(5)
    for name, (spec, tag) in DEALER.items():
        t = d.fetch(spec, tag)
        for p in range(2):
            for j, k in enumerate("abc"):
                assert (t[p][j] == golden_ops[f"dealer/{name}/p{p}/{k}"]).all(), (name, p, k)


def test_spk_constants_and_plain_adder():
    levels, ins, outs, mults, _ = O.SPK64
    assert ins[0] == 0x5555555555555555 and ins[2] == 0x0808080808080808 and ins[5] == 0x80000000
    assert outs[0] == 0xAAAAAAAAAAAAAAAA and outs[3] == 0xFF00FF00FF00FF00 and outs[5] == 0xFFFFFFFF00000000
    assert mults[1] == 6 and mults[4] == 131070 and mults[5] == 8589934590
    assert O.spk_add_plain(3, 1, 8) == 4 and O.spk_add_plain(0xFF, 1, 8) == 0
    assert O.spk_add_plain(0xFFFFFFFFFFFFFFFF, 2) == 1
    rng = np.random.default_rng(1)
    for a, b in rng.integers(0, 2**63, size=(200, 2), dtype=np.uint64):
        assert O.spk_add_plain(int(a), int(b)) == (int(a) + int(b)) % 2**64
    for a in range(256):
        for b in range(0, 256, 7):
            assert O.spk_add_plain(a, b, 8) == (a + b) % 256


OPS = [
    ("mul_c1", 11, 16, 1, lambda c, X, Y: O.beaver_mul(X, Y, c, "mul", 1)),
    ("mul_c3", 11, 16, 3, lambda c, X, Y: O.beaver_mul(X, Y, c, "mul", 3)),
    ("square_c1", 12, 16, 1, lambda c, X, Y: O.beaver_square(X, c, "square", 1)),
    ("square_c3", 12, 16, 3, lambda c, X, Y: O.beaver_square(X, c, "square", 3)),
    ("and_c1", 13, 16, 1, lambda c, X, Y: O.beaver_and(X, Y, c, "and", 1)),
    ("and_c3", 13, 16, 3, lambda c, X, Y: O.beaver_and(X, Y, c, "and", 3)),
    ("badd_c1", 14, 16, 1, lambda c, X, Y: O.binary_add(X, Y, c, "badd", 1)),
    ("badd_c3", 14, 16, 3, lambda c, X, Y: O.binary_add(X, Y, c, "badd", 3)),
    ("a2b", 15, 16, 1, lambda c, X, Y: O.a2b(X, c, "a2b")),
    ("msb", 16, 16, 1, lambda c, X, Y: O.msb(X, c, "msb")),
    ("lt", 17, 16, 1, lambda c, X, Y: O.less_than(X, Y, c, "lt")),
    ("relu", 18, 16, 1, lambda c, X, Y: O.relu_shares(X, c, "relu")),
    ("relu_c4", 18, 16, 4, lambda c, X, Y: O.relu_shares(X, c, "relu")),
    ("trunc", 19, 16, 1, lambda c, X, Y: O.truncate_shares(O.beaver_mul(X, Y, c, "tm"), 16)),
    ("max_L5", 20, 16, 1, lambda c, X, Y: O.max_last_dim(X, 5, c, "max")),
    ("max_L8", 20, 16, 1, lambda c, X, Y: O.max_last_dim(X, 8, c, "max")),
    ("max_L9", 20, 16, 1, lambda c, X, Y: O.max_last_dim(X, 9, c, "max")),
    ("exp", 21, 20, 1, lambda c, X, Y: O.exp_shares(X, c, "exp")),
    ("recip", 22, 20, 1, lambda c, X, Y: O.reciprocal_shares(X, c, "recip")),
    ("softmax", 23, 20, 1, lambda c, X, Y: O.softmax_shares(X, 6, c, "softmax")),
    ("softmax_c2", 23, 20, 2, lambda c, X, Y: O.softmax_shares(X, 6, c, "softmax")),
    ("maxpool", 24, 16, 1, lambda c, X, Y: O.maxpool2d_shares(X, 2, 3, 5, 4, 2, 2, c, "pool")),
    ("matmul", 25, 16, 1, lambda c, X, Y: O.beaver_matmul(X, Y, False, c, "mm")),
    ("matmul_t", 26, 16, 2, lambda c, X, Y: O.beaver_matmul(X, Y, True, c, "qk", 2)),
]


@pytest.mark.parametrize("name,seed,f,chunks,fn", OPS, ids=[o[0] for o in OPS])
def test_op_shares_match_reference(golden_ops, name, seed, f, chunks, fn):
    G = golden_ops
    X = [G[name + "/x0"], G[name + "/x1"]]
    Y = [G[name + "/y0"], G[name + "/y1"]]
    ctx = O.make_ctx(seed + 1, f, mask_key=seed + 2)
    ctx.chunks = chunks
    Z = fn(ctx, X, Y)
    for p in range(2):
        assert (Z[p].reshape(-1) == G[f"{name}/z{p}"].reshape(-1)).all()
    bytes_sent, collectives, p2p = (int(v) for v in G[name + "/stats"])
    s = ctx.stats[0]
    assert (s.bytes_sent, s.collectives, s.p2p_sends) == (bytes_sent, collectives, p2p)


MODEL_FIXTURES = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "model_*.npz")))
# VGG-16 224 through the numpy oracle takes ~8 min on 8 cores: opt-in here (MPCG_SLOW_TESTS=1);
# the GPU suite pins the same fixture (tests/test_gpu_scale.py) in seconds.
SLOW_MODELS = ("vgg16",)


@pytest.mark.parametrize("path", MODEL_FIXTURES, ids=[os.path.basename(p)[6:-4] for p in MODEL_FIXTURES])
def test_model_logit_shares_match_reference(path):
    if os.path.basename(path)[6:].startswith(SLOW_MODELS) and os.environ.get("MPCG_SLOW_TESTS") != "1":
        pytest.skip("numpy oracle on VGG-16 is slow; set MPCG_SLOW_TESTS=1 (GPU suite covers the fixture)")
    name, mode, weights, it = os.path.basename(path)[6:-4].rsplit("_", 3)
    m = np.load(path)
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", name + ".json"))))
    z, opened, h, _ = O.bench_party_values(g, 1, int(it[2:]), weights == "public")
    assert (z[0].reshape(-1) == m["z0"].reshape(-1)).all()
    assert (z[1].reshape(-1) == m["z1"].reshape(-1)).all()
    assert h == int(m["meta"][0])
    ref = m["reference_forward"].view(np.float64).reshape(-1)
    # numpy plaintext forward agrees with the reference's double forward
    w = O.init_weights(g, 12)
    x = O.demo_input(g, 13)
    assert np.allclose(O.reference_forward(g, w, x).reshape(-1), ref, rtol=1e-9, atol=1e-12)
    # decoded MPC logits within the CLI tolerance 2^-6 (P/tools/mpcpipe_bench.cpp:124)
    assert np.abs(O.decode_fixed(opened, g.frac_bits).reshape(-1) - ref).max() <= 2.0 ** -6


def test_mlp_golden_hashes_from_survey():
    # MLP 784-128-128-10 b1 frac16 private s=1.
    g = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", "mlp.json"))))
    assert O.bench_party_values(g, 1, 1)[2] == 0x320997C328457696
    assert O.bench_party_values(g, 1, 2)[2] == 0x6EC2B51E394387CA


def test_encode_fixed_kats():
    # P/tests/test_ring.cpp:132-147: 1.5 -> 3<<15 at scale 16, ties toward +inf.
    assert int(O.encode_fixed(1.5, 16)) == 3 << 15
    assert int(O.encode_fixed(-0.5 / 2**16, 16).view(np.int64)) == 0
    assert int(O.encode_fixed(0.5 / 2**16, 16).view(np.int64)) == 1
