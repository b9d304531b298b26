"""CPU tests of the executor-level I/O: MPCW weight files byte-identical with
the reference's save_weights (fixture written by the unmodified reference, tests/golden/),
weight checks, and the plaintext replica the CLI's verify uses."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mpcw_matches_reference_bytes(tmp_path):
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import model as M
    g = mp.ModelGraph.from_json("toy_cnn")
    ref = os.path.join(ROOT, "tests", "golden", "toy_cnn_seed12.mpcw")
    w = M.load_weights(ref)
    w0 = mp.init_weights(g, 12)
    assert sorted(w) == sorted(w0) and all(np.array_equal(w[k], w0[k]) for k in w0)
    M.check_weights(g, w)
    out = tmp_path / "w.mpcw"
    M.save_weights(w0, str(out))
    assert out.read_bytes() == open(ref, "rb").read()


def test_mpcw_rejects_bad_files(tmp_path):
    from paper_2209_13643_b200 import model as M
    import paper_2209_13643_b200 as mp
    p = tmp_path / "bad.mpcw"
    p.write_bytes(b"XXXX")
    with pytest.raises(ValueError):
        M.load_weights(str(p))
    g = mp.ModelGraph.from_json("toy_cnn")
    w = mp.init_weights(g, 12)
    w.pop(next(iter(w)))
    with pytest.raises(ValueError):
        M.check_weights(g, w)


@pytest.mark.parametrize("name", ["mlp", "lenet5", "toy_cnn", "toy_transformer", "toy_resnet", "toy_bert"])
def test_plaintext_forward_matches_oracle(name):
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import model as M
    from oracle import mpc_oracle as O
    g = mp.ModelGraph.from_json(name)
    go = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", name + ".json"))))
    w, x = mp.init_weights(g, 12), mp.demo_input(g, 13)
    assert np.allclose(M.plaintext_forward(g, w, x), O.reference_forward(go, w, x), rtol=0, atol=1e-12)


def test_cli_parses_reference_units():
    from paper_2209_13643_b200 import cli
    assert cli.parse_latency("1ms") == pytest.approx(1e-3)
    assert cli.parse_latency("200us") == pytest.approx(2e-4)
    assert cli.parse_latency("0") == 0
    assert cli.parse_bandwidth("1GBps") == pytest.approx(1e9)
    assert cli.parse_bandwidth("100MBps") == pytest.approx(1e8)
    assert cli.parse_bandwidth("10Gbps") == pytest.approx(1e10)  # case-insensitive, bytes/s (reference)
    assert cli.parse_threshold("2MiB") == 2 << 20
    assert cli.parse_threshold("8192") == 8192
