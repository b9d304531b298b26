"""GPU: the one-party-per-session path (what each GPU of a 2-GPU pair runs) on ONE device.

Two single-party sessions (party 0, party 1), each driven by its own host thread, linked by
the in-process loopback transport (device copies in place of NCCL send/recv). Every kernel
then runs with one local slot, reads the peer payload from the receive buffer, and the
pipelined wrap-around delta crosses the link — and the per-party output shares must equal
the reference's own (tests/golden) word for word, exactly like the two-slot session's."""
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHI = 0x9E3779B97F4A7C15


def _run_pair(mp, g, mode, weights, iters, link=None):
    sess = [mp.Session(device=0, n_local=1, party=p, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
            for p in (0, 1)]
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
            for _ in range(iters):
                z = ex.run(xin)
            out[p] = z.numpy()[0]
            s.sync()
        except Exception as e:  # noqa: BLE001
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
