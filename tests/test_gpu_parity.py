"""GPU parity: the CUDA path (through the C ABI) vs the reference's own per-party shares.

Every check is word-for-word on each party's output share (not just reconstructions),
against fixtures dumped by the UNMODIFIED reference (tests/golden/) and, for sizes the
fixtures do not cover, against the oracle restatement (oracle/mpc_oracle.py).
Mirrors P/tests/test_protocols.cpp, test_nonlinear.cpp and test_engine.cpp.
"""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHI = 0x9E3779B97F4A7C15


@pytest.fixture(scope="module")
def mp():
    import paper_2209_13643_b200 as mp
    return mp


def _sess(mp, seed, f, mask_seed, chunks=1, threshold=0, persistent=True):
    s = mp.Session(device=0, n_local=2, seed=seed, mask_seed=mask_seed, frac_bits=f)
    s.set_pipeline(chunks, threshold, True)
    s.set_persistent(persistent)
    return s


GOLDEN_OPS = [
    # name, seed, frac, ctx.chunks, fn(mp, s, X, Y)
    ("mul_c1", 11, 16, 1, lambda mp, s, X, Y: mp.beaver_mul(s, X, Y, "mul", 1)),
    ("mul_c3", 11, 16, 3, lambda mp, s, X, Y: mp.beaver_mul(s, X, Y, "mul", 3)),
    ("square_c1", 12, 16, 1, lambda mp, s, X, Y: mp.beaver_square(s, X, "square", 1)),
    ("square_c3", 12, 16, 3, lambda mp, s, X, Y: mp.beaver_square(s, X, "square", 3)),
    ("and_c1", 13, 16, 1, lambda mp, s, X, Y: mp.beaver_and(s, X, Y, "and", 1)),
    ("and_c3", 13, 16, 3, lambda mp, s, X, Y: mp.beaver_and(s, X, Y, "and", 3)),
    ("badd_c1", 14, 16, 1, lambda mp, s, X, Y: mp.binary_add(s, X, Y, 64, True, 1, "badd")),
    ("badd_c3", 14, 16, 3, lambda mp, s, X, Y: mp.binary_add(s, X, Y, 64, True, 3, "badd")),
    ("a2b", 15, 16, 1, lambda mp, s, X, Y: mp.a2b(s, X, 1, "a2b")),
    ("msb", 16, 16, 1, lambda mp, s, X, Y: mp.msb(s, X, 1, "msb")),
    ("lt", 17, 16, 1, lambda mp, s, X, Y: mp.less_than(s, X, Y, 1, "lt")),
    ("relu", 18, 16, 1, lambda mp, s, X, Y: mp.relu_shares(s, X, "relu")),
    ("relu_c4", 18, 16, 4, lambda mp, s, X, Y: mp.relu_shares(s, X, "relu")),
    ("trunc", 19, 16, 1, lambda mp, s, X, Y: mp.truncate_shares(s, mp.beaver_mul(s, X, Y, "tm"), 16)),
    ("max_L5", 20, 16, 1, lambda mp, s, X, Y: mp.max_last_dim(s, X, 5, "max")),
    ("max_L8", 20, 16, 1, lambda mp, s, X, Y: mp.max_last_dim(s, X, 8, "max")),
    ("max_L9", 20, 16, 1, lambda mp, s, X, Y: mp.max_last_dim(s, X, 9, "max")),
    ("exp", 21, 20, 1, lambda mp, s, X, Y: mp.exp_shares(s, X, "exp")),
    ("recip", 22, 20, 1, lambda mp, s, X, Y: mp.reciprocal_shares(s, X, "recip")),
    ("softmax", 23, 20, 1, lambda mp, s, X, Y: mp.softmax_shares(s, X, 6, "softmax")),
    ("softmax_c2", 23, 20, 2, lambda mp, s, X, Y: mp.softmax_shares(s, X, 6, "softmax")),
    ("maxpool", 24, 16, 1, lambda mp, s, X, Y: mp.maxpool2d_shares(s, X, 2, 3, 5, 4, 2, 2, "pool")),
    ("matmul", 25, 16, 1, lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, False, "mm")),
    ("matmul_t", 26, 16, 2, lambda mp, s, X, Y: mp.beaver_matmul(s, X, Y, True, "qk", 2)),
]


@pytest.mark.parametrize("persistent", [True, False], ids=["persistent", "per-round"])
@pytest.mark.parametrize("name,seed,f,chunks,fn", GOLDEN_OPS, ids=[o[0] for o in GOLDEN_OPS])
def test_op_matches_reference_shares(mp, golden_ops, name, seed, f, chunks, fn, persistent):
    G = golden_ops
    s = _sess(mp, seed + 1, f, seed + 2, chunks, persistent=persistent)
    X = s.tensor(np.stack([G[name + "/x0"], G[name + "/x1"]]), f)
    Y = s.tensor(np.stack([G[name + "/y0"], G[name + "/y1"]]), f)
    Z = fn(mp, s, X, Y).numpy()
    assert np.array_equal(Z[0].reshape(-1), G[name + "/z0"].reshape(-1)), "party 0 share differs"
    assert np.array_equal(Z[1].reshape(-1), G[name + "/z1"].reshape(-1)), "party 1 share differs"
    st = s.stats(0)
    ref = [int(v) for v in G[name + "/stats"]]
    assert [st["bytes_sent"], st["collectives"], st["p2p_sends"]] == ref


MODEL_FIXTURES = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "model_*.npz")))


def _run_model(mp, g, mode, weights, iters, seed=1, persistent=True):
    s = mp.Session(device=0, n_local=2, seed=seed, mask_seed=seed ^ PHI, frac_bits=g.frac_bits)
    s.set_persistent(persistent)
    ex = mp.SecureExecutor(s, g, public_weights=weights == "public", pipelined=mode == "pipelined")
    ex.deal_weights(mp.init_weights(g, seed + 11), seed)
    x = s.deal_input(mp.demo_input(g, seed + 12), seed + 1)
    out = None
    for _ in range(iters):
        out = ex.run(x)
    return s, out.numpy()


@pytest.mark.parametrize("persistent", [True, False], ids=["persistent", "per-round"])
@pytest.mark.parametrize("path", MODEL_FIXTURES, ids=[os.path.basename(p)[6:-4] for p in MODEL_FIXTURES])
def test_model_logit_shares_match_reference(mp, path, persistent):
    name, mode, weights, it = os.path.basename(path)[6:-4].rsplit("_", 3)
    m = np.load(path)
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    s, z = _run_model(mp, g, mode, weights, int(it[2:]), persistent=persistent)
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))
    opened = (z[0] + z[1]).reshape(-1)
    assert mp.fnv1a_words(opened) == int(m["meta"][0])
    ref = m["reference_forward"].view(np.float64).reshape(-1)
    dec = opened.view(np.int64).astype(np.float64) * 2.0 ** -g.frac_bits
    assert np.abs(dec - ref).max() <= 2.0 ** -6  # P/tools/mpcpipe_bench.cpp:124


@pytest.mark.parametrize("name,mode,weights,it", [
    ("mlp", "pipelined", "private", 2), ("toy_cnn", "blocking", "private", 1),
    ("toy_transformer", "blocking", "private", 1), ("toy_transformer", "blocking", "public", 1),
    ("lenet5", "pipelined", "private", 1)])
def test_graph_replay_matches_reference(mp, name, mode, weights, it):
    """CUDA-graph replays draw each iteration's triples exactly like eager runs."""
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    m = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{mode}_{weights}_it{it}.npz"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, public_weights=weights == "public", pipelined=mode == "pipelined")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    eager = 1 if mode == "pipelined" else 0   # pipelined: run once for the delta prologue
    for _ in range(eager):
        z = ex.run(x)
    ex.capture(x)
    for _ in range(it - eager):
        z = ex.replay()
    z = z.numpy()
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))
    # more replays keep tracking eager runs iteration by iteration
    s2 = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex2 = mp.SecureExecutor(s2, g, public_weights=weights == "public", pipelined=mode == "pipelined")
    ex2.deal_weights(mp.init_weights(g, 12), 1)
    x2 = s2.deal_input(mp.demo_input(g, 13), 2)
    for _ in range(it + 2):
        ze = ex2.run(x2)
    for _ in range(2):
        zr = ex.replay()
    assert np.array_equal(zr.numpy(), ze.numpy())
    assert s.stats(0) == s2.stats(0)


@pytest.mark.parametrize("name,pairs", [("lenet5", 2), ("toy_transformer", 2), ("lenet5", 4)])
def test_dp_shards_match_full_batch(mp, name, pairs):
    """Data-parallel pairs: each pair regenerates its slice of the full-batch
    triples and masks, so the concatenated logits equal the single-pair full-batch run."""
    mode = "pipelined" if name == "lenet5" else "blocking"
    m = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{mode}_private_it1.npz"))
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    B = g.input[0]
    local = B // pairs
    gl = g.with_batch(local)
    xg = mp.demo_input(g, 13)
    outs = []
    for p in range(pairs):
        s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        s.set_shard(local, B, p * local)
        ex = mp.SecureExecutor(s, gl, pipelined=mode == "pipelined")
        ex.deal_weights(mp.init_weights(g, 12), 1)
        x = s.deal_input(xg, 2, batch_offset=p * local, local_batch=local)
        outs.append(ex.run(x).numpy())
    z = np.concatenate(outs, axis=1)
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))


@pytest.mark.parametrize("mode", ["blocking", "pipelined"])
def test_emulated_link_keeps_values_and_graphs(mp, mode):
    """An emulated LAN link (comm-stream delay kernels) changes timing only; eager runs and
    graph replays still reproduce the reference's shares iteration by iteration."""
    name = "mlp"
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    m = np.load(os.path.join(ROOT, "tests", "golden", "model_mlp_pipelined_private_it2.npz"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    s.set_link(2e-5, 5e9, 0.0)
    ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined", chunk_threshold=0)
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    ex.run(x)
    ex.capture(x)
    z = ex.replay().numpy()  # iteration 2
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))


def test_blocking_and_pipelined_are_bit_identical(mp):
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", "toy_cnn.json"))
    _, zb = _run_model(mp, g, "blocking", "private", 2)
    _, zp = _run_model(mp, g, "pipelined", "private", 2)
    assert np.array_equal(zb, zp)


@pytest.mark.parametrize("n,chunks", [(1, 1), (1000, 1), (4097, 4), (262144, 1), (300001, 4)])
def test_relu_matches_oracle_at_size(mp, n, chunks):
    from oracle import mpc_oracle as O
    rng = np.random.default_rng(n)
    x = O.encode_fixed(rng.uniform(-100, 100, n), 16)
    sh = O.share_additive(x, O.CounterRng(7))
    ctx = O.make_ctx(5, 16, mask_key=9)
    ref = O.relu_shares(sh, ctx, "r")
    s = _sess(mp, 5, 16, 9, chunks)
    Z = mp.relu_shares(s, s.tensor(np.stack(sh), 16), "r").numpy()
    assert np.array_equal(Z[0], ref[0]) and np.array_equal(Z[1], ref[1])
    v = (Z[0] + Z[1]).view(np.int64)
    assert np.array_equal(v, np.maximum(x.view(np.int64), 0))


@pytest.mark.parametrize("M,K,N", [(1, 784, 128), (67, 25, 6), (130, 150, 16), (64, 400, 120), (33, 70, 300)])
def test_beaver_matmul_matches_oracle(mp, M, K, N):
    from oracle import mpc_oracle as O
    r = O.CounterRng(M * 1000 + N)
    X = [r.take(M * K).reshape(M, K), r.take(M * K).reshape(M, K)]
    Y = [r.take(K * N).reshape(K, N), r.take(K * N).reshape(K, N)]
    ctx = O.make_ctx(3, 16)
    ref = O.beaver_matmul(X, Y, False, ctx, "mm")
    s = _sess(mp, 3, 16, 3 ^ PHI)
    Z = mp.beaver_matmul(s, s.tensor(np.stack(X)), s.tensor(np.stack(Y)), False, "mm").numpy()
    assert np.array_equal(Z[0], ref[0]) and np.array_equal(Z[1], ref[1])
    assert np.array_equal(Z[0] + Z[1], O.matmul(X[0] + X[1], Y[0] + Y[1]))


def test_adversarial_all_ones_matmul(mp):
    # all-0xFF operands stress exact limb accumulation.
    from oracle import mpc_oracle as O
    M, K, N = 40, 600, 24
    X = [np.full((M, K), 2**64 - 1, dtype=np.uint64), np.zeros((M, K), dtype=np.uint64)]
    Y = [np.full((K, N), 2**64 - 1, dtype=np.uint64), np.zeros((K, N), dtype=np.uint64)]
    ctx = O.make_ctx(4, 16)
    ref = O.beaver_matmul(X, Y, False, ctx, "ones")
    s = _sess(mp, 4, 16, 4 ^ PHI)
    Z = mp.beaver_matmul(s, s.tensor(np.stack(X)), s.tensor(np.stack(Y)), False, "ones").numpy()
    assert np.array_equal(Z[0], ref[0]) and np.array_equal(Z[1], ref[1])


def test_shape_mismatch_and_errors(mp):
    s = _sess(mp, 1, 16, 2)
    a = s.tensor(np.zeros((2, 3, 4), dtype=np.uint64))
    b = s.tensor(np.zeros((2, 4, 3), dtype=np.uint64))
    with pytest.raises(mp.ShapeError):
        mp.beaver_mul(s, a, b)
    with pytest.raises(mp.ConfigError):  # the dealer rejects first, as in the reference
        mp.beaver_matmul(s, a, a)  # dealer rejects first, as the reference (triple.hpp:98-100)
    with pytest.raises(mp.ConfigError):
        mp.Session(device=0, n_local=3)


def test_empty_tensor_ops(mp):
    s = _sess(mp, 1, 16, 2)
    e = s.tensor(np.zeros((2, 0), dtype=np.uint64))
    assert mp.beaver_mul(s, e, e).numpy().shape == (2, 0)


def test_graph_owns_dealer_streams_until_released(mp):
    """an eager run between replays would advance the host dealer counters behind
    the graph's back. While a graph is held, run() fails with UsageError; after
    release_graph() the next run continues the iteration sequence (= eager iteration 4)."""
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", "mlp.json"))

    def make():
        s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        ex = mp.SecureExecutor(s, g, pipelined=True)
        ex.deal_weights(mp.init_weights(g, 12), 1)
        return s, ex, s.deal_input(mp.demo_input(g, 13), 2)

    s, ex, x = make()
    ex.run(x)                      # iteration 1
    ex.capture(x)
    ex.replay()                    # iteration 2
    with pytest.raises(mp.UsageError):
        ex.run(x)
    with pytest.raises(mp.UsageError):
        mp.relu_shares(s, x, "stray")
    ex.replay()                    # iteration 3
    ex.release_graph()
    z = ex.run(x).numpy()          # iteration 4
    s2, ex2, x2 = make()
    for _ in range(4):
        ze = ex2.run(x2)
    assert np.array_equal(z, ze.numpy())
    assert s.stats(0) == s2.stats(0)


def test_deal_weights_checks_counts_through_the_abi(mp):
    """the C ABI takes per-tensor element counts and rejects a wrongly shaped
    tensor with ConfigError (the reference's check_weights) instead of over-reading."""
    import ctypes as C
    from paper_2209_13643_b200 import _native as N
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", "mlp.json"))
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g)
    w = mp.init_weights(g, 12)
    names = sorted(w)
    arrs = [np.ascontiguousarray(w[k], dtype=np.float64).reshape(-1) for k in names]
    arrs[0] = arrs[0][:-1]  # one value short
    cn = (C.c_char_p * len(names))(*[n.encode() for n in names])
    cv = (C.POINTER(C.c_double) * len(names))(*[a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs])
    counts = np.array([a.size for a in arrs], dtype=np.uint64)
    with pytest.raises(mp.ConfigError, match="wrong shape"):
        N.call("mpcg_executor_deal_weights", ex._h, len(names), cn, cv,
               counts.ctypes.data_as(C.POINTER(C.c_uint64)), 1)
    with pytest.raises(ValueError):
        w2 = dict(w)
        w2[names[0]] = w2[names[0]].reshape(-1)[:-1]
        ex.deal_weights(w2, 1)


def test_set_link_rejects_latency_only(mp):
    """ADVICE r1 / transport/config.hpp:34-38: bandwidth must be > 0 for an emulated link."""
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1, frac_bits=16)
    with pytest.raises(mp.ConfigError):
        s.set_link(1e-4, 0.0, 0.0)
    with pytest.raises(mp.ConfigError):
        s.set_link(-1.0, 1e9, 0.0)
    s.set_link(1e-4, 1.25e9, 0.0)
    s.set_link(0.0, 0.0, 0.0)  # back to the real transport


@pytest.mark.parametrize("pair_eval", [True, False], ids=["pair", "per-slot"])
@pytest.mark.parametrize("name,golden,chunks", [
    ("lenet5", "model_lenet5_pipelined_private_it1", 4), ("toy_cnn", "model_toy_cnn_blocking_private_it1", 3),
    ("toy_transformer", "model_toy_transformer_blocking_private_it1", 2)])
def test_linear_chunks_keep_reference_shares(mp, name, golden, chunks, pair_eval):
    """Inner-layer pipeline on the linear layers (ExecOptions::linear_chunks): the eps opening
    leaves in row blocks '<tag>.eps.chunk<k>' and each block's combine runs as it lands. The
    triples are keyed by tag, so the per-party shares equal the reference's unchunked run."""
    from paper_2209_13643_b200 import api
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    m = np.load(os.path.join(ROOT, "tests", "golden", golden + ".npz"))
    api.set_pair_eval(pair_eval)
    try:
        s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        ex = mp.SecureExecutor(s, g, pipelined=True, chunks=chunks, chunk_threshold=0, linear_chunks=True)
        ex.deal_weights(mp.init_weights(g, 12), 1)
        x = s.deal_input(mp.demo_input(g, 13), 2)
        s.trace(True)
        z = ex.run(x).numpy()
    finally:
        api.set_pair_eval(True)
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1)), "party 0 share differs"
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1)), "party 1 share differs"
    tags = [r["tag"] for r in s.trace_rows()]
    first = api.linear_tags(g)[0]
    assert first + ".eps.chunk0" in tags and first + ".eps" not in tags
