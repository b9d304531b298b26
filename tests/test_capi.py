"""CPU tests of the drop-in boundary: libmpcg.so loads without a GPU and exports every
entry point include/mpcg.h declares; compute calls fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "mpcg.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(mpcg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2209_13643_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2209_13643_b200 import _native
    assert set(_declared()) == set(_native.SIGNATURES)


def test_fnv1a_matches_oracle():
    import numpy as np
    import paper_2209_13643_b200 as mp
    from oracle import mpc_oracle as O
    w = np.arange(100, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    assert mp.fnv1a_words(w) == O.fnv1a_words(w)


def test_model_helpers_match_oracle():
    import numpy as np
    import paper_2209_13643_b200 as mp
    from oracle import mpc_oracle as O
    import json
    for name in ("mlp", "lenet5", "toy_cnn", "toy_transformer", "vgg16", "toy_resnet", "toy_bert", "resnet18",
                 "bert_base"):
        g = mp.ModelGraph.from_json(name)
        go = O.model_from_json(json.load(open(os.path.join(ROOT, "configs", name + ".json"))))
        assert [tuple(s) for s in g.shapes()] == [tuple(s) for s in O.infer_shapes(go)]
        assert g.weight_shapes() == [(k, tuple(v)) for k, v in O.model_weight_shapes(go)]
        if name not in ("vgg16", "resnet18", "bert_base"):
            w1, w2 = mp.init_weights(g, 12), O.init_weights(go, 12)
            assert sorted(w1) == sorted(w2)
            assert all(np.array_equal(w1[k], w2[k]) for k in w1)
            assert np.array_equal(mp.demo_input(g, 13), O.demo_input(go, 13))


def test_compute_without_gpu_fails_loudly():
    import paper_2209_13643_b200 as mp
    n = ctypes.c_int()
    mp.lib().mpcg_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(mp.CudaError):
        mp.Session(device=0, n_local=2)
