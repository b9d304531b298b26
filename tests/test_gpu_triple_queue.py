"""GPU: the offline/online split through the TripleSource plugin (H/sharing/triple.hpp:126-307).

* A queue recorded from one session's seeded dealer (offline phase) and consumed by another
  session (online phase, triples read from HBM) reproduces the reference's per-party logits
  shares word for word — the queue holds exactly the triples the dealer would have drawn.
* QueueTripleSource semantics: specs are checked in order ("triple queue spec mismatch at
  record i"), running out is "triple queue exhausted" (ProtocolError), tags are irrelevant.
* The reference's triple-file format round-trips (save_triples / load_triples) and a file
  written by the UNMODIFIED reference (oracle/_ref, fixture tests/golden/triples_ref.bin) loads
  and yields the reference's own triples through dealer_fetch.
"""
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


def _setup(mp, g, mode):
    s = mp.Session(device=0, n_local=2, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex = mp.SecureExecutor(s, g, pipelined=mode == "pipelined")
    ex.deal_weights(mp.init_weights(g, 12), 1)
    return s, ex, s.deal_input(mp.demo_input(g, 13), 2)


@pytest.mark.parametrize("name,mode", [("mlp", "blocking"), ("lenet5", "pipelined"), ("toy_transformer", "blocking")])
def test_recorded_queue_reproduces_reference(mp, name, mode, tmp_path):
    g = mp.ModelGraph.from_json(os.path.join(ROOT, "configs", name + ".json"))
    gold = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{'pipelined' if name == 'lenet5' else 'blocking'}"
                                f"_private_it1.npz"))
    q = mp.TripleQueue()
    s1, ex1, x1 = _setup(mp, g, mode)
    mp.record_triples(s1, q)
    z1 = ex1.run(x1).numpy()  # offline dealer pass (also the seeded online run)
    mp.record_triples(s1, None)
    s1.sync()
    n = q.size()["records"]
    assert n > 0
    # online phase from the queue, in a fresh session whose own dealer would draw nothing useful
    s2 = mp.Session(device=0, n_local=2, seed=777, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
    ex2 = mp.SecureExecutor(s2, g, pipelined=mode == "pipelined")
    w = mp.init_weights(g, 12)
    ex2.deal_weights(w, 1)  # weights/input shares come from the weight owner (seed 1), not the dealer
    x2 = s2.tensor(x1.numpy(), g.frac_bits)
    mp.use_triple_queue(s2, q)
    z2 = ex2.run(x2).numpy()  # pipelined: the same fetch order, wrap-around prefetch included
    assert q.size()["consumed"] == n
    assert np.array_equal(z2, z1)
    assert np.array_equal(z2[0].reshape(-1), gold["z0"].reshape(-1))
    assert np.array_equal(z2[1].reshape(-1), gold["z1"].reshape(-1))
    # exhausted: the next run needs more triples than the queue holds
    with pytest.raises(mp.ProtocolError, match="exhausted"):
        ex2.run(x2)


def test_queue_spec_mismatch_and_file_round_trip(mp, tmp_path):
    s = mp.Session(device=0, n_local=2, seed=5, mask_seed=6, frac_bits=16)
    q = mp.TripleQueue()
    mp.record_triples(s, q)
    a1, b1, c1 = mp.dealer_fetch(s, (3, 4), tag="t.mul")
    am, bm, cm = mp.dealer_fetch(s, (2, 3, 4), (2, 5, 4), matmul=True, transpose_b=True, tag="t.qk")
    ab, bb, cb = mp.dealer_fetch(s, (2, 5), kind="bin", tag="t.and")
    asq, bsq, csq = mp.dealer_fetch(s, (7,), square=True, tag="t.sq")
    mp.record_triples(s, None)
    # the reference's dealer fixtures (tests/golden/ops.npz dealer/*) use seed 5 and these tags
    G = np.load(os.path.join(ROOT, "tests", "golden", "ops.npz"))
    for nm, (a, b, c) in {"mul0": (a1, b1, c1), "qk": (am, bm, cm), "and": (ab, bb, cb), "sq": (asq, bsq, csq)}.items():
        for p in (0, 1):
            assert np.array_equal(a.numpy()[p].reshape(-1), G[f"dealer__{nm}__p{p}__a"].reshape(-1)), nm
            assert np.array_equal(b.numpy()[p].reshape(-1), G[f"dealer__{nm}__p{p}__b"].reshape(-1)), nm
            assert np.array_equal(c.numpy()[p].reshape(-1), G[f"dealer__{nm}__p{p}__c"].reshape(-1)), nm
    path = str(tmp_path / "triples.bin")
    q.save(path)
    q2 = mp.TripleQueue()
    q2.load(path)
    assert q2.size()["records"] == 4
    s2 = mp.Session(device=0, n_local=2, seed=99, mask_seed=6, frac_bits=16)
    mp.use_triple_queue(s2, q2)
    a2, b2, c2 = mp.dealer_fetch(s2, (3, 4), tag="anything")  # tags are irrelevant in a queue
    assert np.array_equal(a2.numpy(), a1.numpy()) and np.array_equal(c2.numpy(), c1.numpy())
    with pytest.raises(mp.ProtocolError, match="spec mismatch at record 1"):
        mp.dealer_fetch(s2, (3, 4), tag="t.mul")  # record 1 is the matmul triple
    # the reference's own triple file (save_triples output) loads and serves its triples
    ref = os.path.join(ROOT, "tests", "golden", "triples_ref.bin")
    q3 = mp.TripleQueue()
    q3.load(ref)
    s3 = mp.Session(device=0, n_local=2, seed=1, mask_seed=6, frac_bits=16)
    mp.use_triple_queue(s3, q3)
    a3, b3, c3 = mp.dealer_fetch(s3, (3, 4), tag="t.mul")
    assert np.array_equal(a3.numpy(), a1.numpy()) and np.array_equal(b3.numpy(), b1.numpy())
    assert np.array_equal(c3.numpy(), c1.numpy())
    a4, b4, c4 = mp.dealer_fetch(s3, (2, 3, 4), (2, 5, 4), matmul=True, transpose_b=True)
    assert np.array_equal(c4.numpy(), cm.numpy()) and np.array_equal(a4.numpy(), am.numpy())
