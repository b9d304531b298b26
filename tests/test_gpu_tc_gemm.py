"""GPU parity of the tcgen05 int8-limb ring GEMM (forced on) against the oracle.

Per-party Beaver-matmul shares must be word-identical to the reference restatement,
including adversarial all-0xFF operands at the exact-accumulation limit (SURVEY §7:
random data does not trip per-diagonal overflow, all-ones operands do).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
PHI = 0x9E3779B97F4A7C15


@pytest.fixture(params=["tc", "tc2"])
def tc(request):
    """Tensor cores forced on for every shape within the exactness budget: "tc" takes the
    both-slots combine kernel (gemm_tc3.cu) wherever its operand pattern applies, "tc2" the
    one-CTA-per-slot kernel only."""
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import api
    api.set_gemm_mode(request.param)
    yield mp
    api.set_gemm_mode("auto")


def _run(mp, X, Y, tb, tag, chunks=1):
    from oracle import mpc_oracle as O
    ctx = O.make_ctx(9, 16)
    ref = O.beaver_matmul(X, Y, tb, ctx, tag, chunks)
    s = mp.Session(device=0, n_local=2, seed=9, mask_seed=9 ^ PHI, frac_bits=16)
    Z = mp.beaver_matmul(s, s.tensor(np.stack(X)), s.tensor(np.stack(Y)), tb, tag, chunks).numpy()
    assert np.array_equal(Z[0], ref[0]), "party 0"
    assert np.array_equal(Z[1], ref[1]), "party 1"
    return Z


@pytest.mark.parametrize("M,K,N", [(128, 32, 32), (256, 64, 64), (300, 100, 48), (128, 576, 64),
                                   (1000, 150, 16), (257, 1000, 130), (300, 25, 6), (129, 33, 7),
                                   (6400, 150, 16), (4000, 25, 6), (640, 96, 256), (512, 1152, 128),
                                   (384, 64, 200), (260, 200, 320), (640, 96, 512),  # N > 256: hybrid pack
                                   (300, 64, 640), (1024, 96, 768)])  # N > 512: fully packed, shared left image
def test_tc_gemm_random(tc, M, K, N):
    from oracle import mpc_oracle as O
    r = O.CounterRng(M * 7 + K * 3 + N)
    X = [r.take(M * K).reshape(M, K), r.take(M * K).reshape(M, K)]
    Y = [r.take(K * N).reshape(K, N), r.take(K * N).reshape(K, N)]
    Z = _run(tc, X, Y, False, "tcmm")
    assert np.array_equal(Z[0] + Z[1], O.matmul(X[0] + X[1], Y[0] + Y[1]))


def test_tc_gemm_batched_transposed(tc):
    from oracle import mpc_oracle as O
    r = O.CounterRng(77)
    B, T, dh = 4, 128, 64
    X = [r.take(B * T * dh).reshape(B, T, dh), r.take(B * T * dh).reshape(B, T, dh)]
    Y = [r.take(B * T * dh).reshape(B, T, dh), r.take(B * T * dh).reshape(B, T, dh)]
    _run(tc, X, Y, True, "attn.qk", chunks=2)


def test_tc_gemm_all_ones_at_budget(tc):
    # K' = 3 segments x 5400 = 16200 <= 16384: the low diagonals must stay exact.
    M, K, N = 128, 5400, 32
    X = [np.full((M, K), 2**64 - 1, dtype=np.uint64), np.zeros((M, K), dtype=np.uint64)]
    Y = [np.full((K, N), 2**64 - 1, dtype=np.uint64), np.zeros((K, N), dtype=np.uint64)]
    _run(tc, X, Y, False, "ones")


def test_tc_gemm_model_parity(tc):
    """A whole model through the tensor-core GEMM (toy transformer: K' up to 768)."""
    import glob
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    m = np.load(os.path.join(root, "tests", "golden", "model_toy_transformer_blocking_private_it1.npz"))
    g = tc.ModelGraph.from_json(os.path.join(root, "configs", "toy_transformer.json"))
    s = tc.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = tc.SecureExecutor(s, g)
    ex.deal_weights(tc.init_weights(g, 12), 1)
    z = ex.run(s.deal_input(tc.demo_input(g, 13), 2)).numpy()
    assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
    assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))


def test_tc_public_gemm_model_path(tc):
    """Public-weight products (one memory segment) through the tensor-core kernels."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for name in ("toy_cnn", "toy_transformer"):
        m = np.load(os.path.join(root, "tests", "golden", f"model_{name}_" +
                                 ("pipelined_public_it1.npz" if name == "toy_cnn" else "blocking_public_it1.npz")))
        g = tc.ModelGraph.from_json(os.path.join(root, "configs", name + ".json"))
        s = tc.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        ex = tc.SecureExecutor(s, g, public_weights=True, pipelined=name == "toy_cnn")
        ex.deal_weights(tc.init_weights(g, 12), 1)
        z = ex.run(s.deal_input(tc.demo_input(g, 13), 2)).numpy()
        assert np.array_equal(z[0].reshape(-1), m["z0"].reshape(-1))
        assert np.array_equal(z[1].reshape(-1), m["z1"].reshape(-1))


@pytest.mark.parametrize("M,K,N", [(16384, 576, 64), (4096, 1152, 128), (2048, 2304, 256), (9000, 27, 64)])
def test_tc3_matches_tc2_at_conv_shapes(M, K, N):
    """Both-slots kernel vs one-CTA-per-slot kernel at ResNet-18 conv shapes (row counts cut):
    word-identical per-party shares (each is pinned to the reference separately)."""
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import api
    rng = np.random.default_rng(M + K + N)
    X = rng.integers(0, 2**64, size=(2, M, K), dtype=np.uint64)
    Y = rng.integers(0, 2**64, size=(2, K, N), dtype=np.uint64)
    out = {}
    try:
        for mode in ("auto", "tc2"):
            api.set_gemm_mode(mode)
            s = mp.Session(device=0, n_local=2, seed=5, mask_seed=5 ^ PHI, frac_bits=16)
            out[mode] = mp.beaver_matmul(s, s.tensor(X), s.tensor(Y), False, "conv").numpy()
    finally:
        api.set_gemm_mode("auto")
    assert np.array_equal(out["auto"], out["tc2"])
    z = out["auto"][0][:64] + out["auto"][1][:64]
    assert np.array_equal(z, (X[0][:64] + X[1][:64]) @ (Y[0] + Y[1]))  # opened product, mod 2^64
