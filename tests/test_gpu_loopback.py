"""GPU: the one-party-per-session path (what each GPU of a 2-GPU pair runs) on ONE device.

Two single-party sessions (party 0, party 1), each driven by its own host thread, linked by
the in-process loopback transport (device copies in place of NCCL send/recv). Every kernel
then runs with one local slot, reads the peer payload from the receive buffer, and the
pipelined wrap-around delta crosses the link — and the per-party output shares must equal
the reference's own (tests/golden) word for word, exactly like the two-slot session's."""
import os
import sys
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHI = 0x9E3779B97F4A7C15


def _run_pair(mp, g, mode, weights, iters, link=None, kind="loopback", graph=False):
    sess = [mp.Session(device=0, n_local=1, party=p, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
            for p in (0, 1)]
    if kind == "p2p":
        sess[0].connect_p2p(sess[1])
    else:
        sess[0].connect_loopback(sess[1])
    if link:
        for s in sess:
            s.set_link(*link)
    out, err = [None, None], []
    w = mp.init_weights(g, 12)
    x = mp.demo_input(g, 13)

    def party(p):
        try:
            s = sess[p]
            ex = mp.SecureExecutor(s, g, public_weights=weights == "public", pipelined=mode == "pipelined")
            ex.deal_weights(w, 1)
            xin = s.deal_input(x, 2)
            z = None
            if graph:  # one eager run (pipelined prologue), capture, then replays = iterations 2..
                z = ex.run(xin)
                ex.capture(xin)
                for _ in range(iters - 1):
                    z = ex.replay()
            else:
                for _ in range(iters):
                    z = ex.run(xin)
            out[p] = z.numpy()[0]
            s.sync()
        except Exception as e:  # noqa: BLE001
            # reported at once: the peer party may now wait on the link until the join timeout
            print(f"party {p} failed: {e!r}", file=sys.stderr, flush=True)
            err.append(e)

    th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    return out, sess


@pytest.mark.parametrize("name,mode,weights,it", [
    ("mlp", "pipelined", "private", 2), ("mlp", "blocking", "public", 1), ("lenet5", "pipelined", "private", 1),
    ("toy_cnn", "blocking", "private", 1), ("toy_transformer", "blocking", "private", 1)])
def test_one_party_sessions_match_reference(name, mode, weights, it):
    import paper_2209_13643_b200 as mp
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    m = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{mode}_{weights}_it{it}.npz"))
    (z0, z1), sess = _run_pair(mp, g, mode, weights, it)
    assert np.array_equal(z0.reshape(-1), m["z0"].reshape(-1)), "party 0 share differs"
    assert np.array_equal(z1.reshape(-1), m["z1"].reshape(-1)), "party 1 share differs"
    st = [s.stats(0) for s in sess]
    assert st[0] == st[1]  # both parties posted the same collectives


def test_one_party_sessions_extension_graph_and_link():
    """Residual graph + GeLU/LayerNorm through the one-party path, over an emulated link."""
    import json
    import paper_2209_13643_b200 as mp
    from oracle import mpc_oracle as O
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", "toy_bert.json"))
    go = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", "toy_bert.json"))))
    ref, _, _, _ = O.bench_party_values(go, 1, 1, False)
    (z0, z1), _ = _run_pair(mp, g, "pipelined", "private", 1, link=(2e-6, 5e9, 0.0))
    assert np.array_equal(z0.reshape(-1), ref[0].reshape(-1))
    assert np.array_equal(z1.reshape(-1), ref[1].reshape(-1))


def _pair_ops(mp, fns):
    """Run fns[p](session_p) for the two loopback-linked one-party sessions on two threads;
    returns the exceptions raised per party."""
    sess = [mp.Session(device=0, n_local=1, party=p, seed=5, mask_seed=6, frac_bits=16) for p in (0, 1)]
    sess[0].connect_loopback(sess[1])
    errs = [None, None]

    def party(p):
        try:
            fns[p](mp, sess[p])
            sess[p].sync()
        except Exception as e:  # noqa: BLE001
            errs[p] = e

    th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a party hung on a desynchronised collective"
    return errs


def _mul(n, tag):
    def f(mp, s):
        x = s.tensor(np.arange(n, dtype=np.uint64).reshape(1, n), 16)
        mp.beaver_mul(s, x, x, tag)
    return f


def test_collective_desync_raises_protocol_error():
    """H/transport/sim.hpp:101-110: parties that issue different collectives at the same
    sequence number fail with ProtocolError (here via the {seq, n, tag} trailer every one-party
    payload carries, checked on the receiving side) instead of computing garbage."""
    import paper_2209_13643_b200 as mp
    errs = _pair_ops(mp, [_mul(16, "same"), _mul(16, "same")])
    assert errs == [None, None]
    errs = _pair_ops(mp, [_mul(16, "alpha"), _mul(16, "beta")])
    assert all(isinstance(e, mp.ProtocolError) for e in errs), errs
    errs = _pair_ops(mp, [_mul(16, "m"), _mul(24, "m")])  # size mismatch: caught at post
    assert all(isinstance(e, mp.ProtocolError) for e in errs), errs


@pytest.mark.parametrize("name,mode,weights,it", [
    ("mlp", "pipelined", "private", 2), ("lenet5", "pipelined", "private", 1),
    ("toy_transformer", "blocking", "private", 1), ("toy_cnn", "pipelined", "public", 1)])
def test_p2p_device_flag_link_matches_reference(name, mode, weights, it):
    """Device-initiated opens (mpcg_session_connect_p2p): the sender's comm stream stores its
    payload into the peer's inbox and releases a flag the peer's stream acquires on device."""
    import paper_2209_13643_b200 as mp
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    m = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{mode}_{weights}_it{it}.npz"))
    (z0, z1), sess = _run_pair(mp, g, mode, weights, it, kind="p2p")
    assert np.array_equal(z0.reshape(-1), m["z0"].reshape(-1)), "party 0 share differs"
    assert np.array_equal(z1.reshape(-1), m["z1"].reshape(-1)), "party 1 share differs"
    assert sess[0].stats(0) == sess[1].stats(0)


@pytest.mark.parametrize("name,mode", [("mlp", "pipelined"), ("lenet5", "pipelined"), ("lenet5", "blocking")])
def test_p2p_link_graph_replays(name, mode):
    """Each party captures its own inference into a CUDA graph (flag slots and values follow the
    replay counter); three concurrent replays of the two graphs reproduce iteration 4 of the
    two-slot session word for word — including the pipelined executor's weight-side opening
    that one replay posts and the next one waits for."""
    import paper_2209_13643_b200 as mp
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    iters = 4
    (z0, z1), _ = _run_pair(mp, g, mode, "private", iters, kind="p2p", graph=True)
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    x = s.deal_input(mp.demo_input(g, 13), 2)
    for _ in range(iters):
        ze = ex.run(x).numpy()
    assert np.array_equal(z0.reshape(-1), ze[0].reshape(-1))
    assert np.array_equal(z1.reshape(-1), ze[1].reshape(-1))
