"""GPU parity at BASELINE scale: the CUDA path vs the UNMODIFIED reference at real layer shapes.

The fixtures (tests/golden/scale.npz, made by tests/golden/make_golden.py --scale from
oracle/ref_driver.cpp cmd_scale / model_pin) pin each party's output share by its FNV-1a word
hash (H/engine/report.hpp:18-23) plus the first/last 16 words and the traffic counters, so
shapes too large for word fixtures are still checked word for word:

* ResNet-18 conv1 ReLU (8.4M elements, 4 chunk lanes) and VGG-16 pool1 (3.2M windows of 4);
* BERT-base softmax [12288, 128], Q K^T and P V over [96, 128, 64] heads (4 chunk lanes);
* full-word beaver_matmul at ResNet-18 layer4's im2col shape (2048, 4608, 512): K' = 13,824,
  near the tcgen05 path's exact-accumulation limit of 16,384, through the hybrid left operand;
* full-word beaver_matmul at VGG-16 fc6 (1, 25088, 4096): the split-K GEMV;
* single-layer SecureExecutor runs (im2col eps build + fused combine epilogue) at ResNet-18
  layer1 (131072, 576, 64) and layer4, VGG-16 fc6 and BERT-base ffn1 / ffn2.

Inputs are regenerated here from the same counter streams the driver used (see
oracle/ref_driver.cpp small_shares / draws_t).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
PHI = 0x9E3779B97F4A7C15
THR = 2 << 20  # ExecOptions default chunk threshold (H/engine/executor.hpp:28-36)


@pytest.fixture(scope="module")
def mp():
    import paper_2209_13643_b200 as mp
    return mp


@pytest.fixture(scope="module")
def G():
    d = np.load(os.path.join(GOLD, "scale.npz"))
    return {k.replace("__", "/"): d[k] for k in d.files}


def _draws(seed, stream, shape):
    from paper_2209_13643_b200.model import counter_draws
    return counter_draws(seed, stream, int(np.prod(shape))).reshape(shape)


def _small_shares(shape, seed, bits):
    v = (_draws(seed, 0, shape).view(np.int64) >> np.int64(64 - bits)).view(np.uint64)
    x1 = _draws(seed, 1, shape)
    with np.errstate(over="ignore"):
        x0 = v - x1
    return np.stack([x0, x1])


def _check(mp, G, name, z, stats=None):
    for p in range(2):
        w = np.ascontiguousarray(z[p]).reshape(-1)
        h, n = (int(v) for v in G[f"{name}/z{p}/hash"])
        assert w.size == n, f"{name}: party {p} output size"
        assert np.array_equal(w[:16], G[f"{name}/z{p}/head"]), f"{name}: party {p} head words differ"
        assert np.array_equal(w[-16:], G[f"{name}/z{p}/tail"]), f"{name}: party {p} tail words differ"
        assert mp.fnv1a_words(w) == h, f"{name}: party {p} share hash differs"
    if stats is not None:
        assert [stats["bytes_sent"], stats["collectives"], stats["p2p_sends"]] == [int(v) for v in G[name + "/stats"]]


def _sess(mp, seed, f):
    s = mp.Session(device=0, n_local=2, seed=seed + 1, mask_seed=seed + 2, frac_bits=f)
    s.set_pipeline(4, THR, True)
    return s


OPS = [
    # name, seed, frac, input builder, op
    ("relu_r18", 31, 20, lambda: (_small_shares((128, 64, 32, 32), 31, 24), None),
     lambda mp, s, X, Y: mp.relu_shares(s, X, "relu")),
    ("pool_vgg1", 32, 20, lambda: (_small_shares((1, 64, 224, 224), 32, 24), None),
     lambda mp, s, X, Y: mp.maxpool2d_shares(s, X, 1, 64, 224, 224, 2, 2, "pool1")),
    ("softmax_bert", 33, 16, lambda: (_small_shares((12288, 128), 33, 18), None),
     lambda mp, s, X, Y: mp.softmax_shares(s, X, 128, "softmax")),
    ("qk_bert", 34, 16, lambda: (np.stack([_draws(34, 0, (96, 128, 64)), _draws(34, 1, (96, 128, 64))]),
                                 np.stack([_draws(34, 2, (96, 128, 64)), _draws(34, 3, (96, 128, 64))])),
     lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, True, "attn.qk", 4)),
    ("av_bert", 35, 16, lambda: (np.stack([_draws(35, 0, (96, 128, 128)), _draws(35, 1, (96, 128, 128))]),
                                 np.stack([_draws(35, 2, (96, 128, 64)), _draws(35, 3, (96, 128, 64))])),
     lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, False, "attn.av", 4)),
    ("gemm_r18l4", 36, 20, lambda: (np.stack([_draws(36, 0, (2048, 4608)), _draws(36, 1, (2048, 4608))]),
                                    np.stack([_draws(36, 2, (4608, 512)), _draws(36, 3, (4608, 512))])),
     lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, False, "l4.mm")),
    ("gemm_fc6", 37, 20, lambda: (np.stack([_draws(37, 0, (1, 25088)), _draws(37, 1, (1, 25088))]),
                                  np.stack([_draws(37, 2, (25088, 4096)), _draws(37, 3, (25088, 4096))])),
     lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, False, "fc6.mm")),
]


@pytest.mark.parametrize("name,seed,f,build,fn", OPS, ids=[o[0] for o in OPS])
def test_op_at_baseline_scale(mp, G, name, seed, f, build, fn):
    x, y = build()
    s = _sess(mp, seed, f)
    X = s.tensor(x, f)
    Y = s.tensor(y, f) if y is not None else None
    z = fn(mp, s, X, Y).numpy()
    _check(mp, G, name, z, s.stats(0))


MODELS = ["r18_conv1", "r18_l1conv", "r18_l2sc", "r18_l2conv_s2", "r18_l3conv", "r18_l4conv", "vgg_fc6", "bert_ffn1", "bert_ffn2"]


@pytest.mark.parametrize("mode", ["blocking", "pipelined", "chunked"])
@pytest.mark.parametrize("name", MODELS)
def test_linear_layer_at_baseline_scale(mp, G, name, mode):
    """SecureExecutor::run of one linear layer at a BASELINE shape (private weights, seed 1):
    the reference's per-party output shares, in every mode (AC2: modes are bit-identical;
    "chunked" = pipelined with the inner-layer pipeline on the linear layer, 4 eps row blocks)."""
    g = mp.ModelGraph.from_json(os.path.join(GOLD, "scale", name + ".json"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, pipelined=mode != "blocking", chunks=4, chunk_threshold=THR,
                           linear_chunks=mode == "chunked")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    z = ex.run(x).numpy()
    _check(mp, G, name, z)
    meta = [int(v) for v in G[name + "/meta"]]
    if mode == "blocking":  # pipelined posts the wrap-around delta of the next run as well
        st = s.stats(0)     # the driver's counters include its final "logits.open" reveal
        assert [st["bytes_sent"], st["collectives"], st["p2p_sends"]] == [meta[1] - 8 * z[0].size, meta[2] - 1,
                                                                           meta[3]]


def test_vgg16_whole_model_matches_reference(mp):
    """VGG-16 224 b1, private weights, one inference: per-party logits shares equal the
    reference's (whose CPU run takes ~10 min), opened-logits hash 0x7df935f348a3669e."""
    m = np.load(os.path.join(GOLD, "model_vgg16_blocking_private_it1.npz"))
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", "vgg16.json"))
    for mode in ("blocking", "pipelined"):
        s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined")
        ex.deal_weights(mp.init_weights(g, 12), 1)
        x = s.deal_input(mp.demo_input(g, 13), 2)
        z = ex.run(x).numpy()
        assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1)), mode
        assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1)), mode
        with np.errstate(over="ignore"):
            assert mp.fnv1a_words((z[0] + z[1]).reshape(-1)) == int(m["meta"][0])
