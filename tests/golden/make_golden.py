"""Generate golden fixtures from the UNMODIFIED reference (run here, where /root/reference exists).

    make -C oracle && python tests/golden/make_golden.py

Runs oracle/_ref/ref_driver (built from /root/reference/proj/include by oracle/Makefile)
and stores its dumps as compressed .npz fixtures in tests/golden/:

* ops.npz            — per-op inputs and per-party output shares (see oracle/ref_driver.cpp cmd_golden)
* model_<name>_<mode>_<weights>_it<k>.npz — per-party logits shares, opened logits, hash,
                       traffic counters and the double-precision reference_forward output.
* scale.npz          — BASELINE-scale pins (``--scale``): the reference's ops and single-layer
                       models at ResNet-18 / VGG-16 / BERT-base layer shapes, each party's output
                       share pinned by FNV-1a word hash + head/tail words + traffic counters
                       (oracle/ref_driver.cpp cmd_scale / model_pin). About 3 min on 8 cores.

    python tests/golden/make_golden.py --scale [--from DIR]   # DIR: dumps made earlier
"""
import os
import struct
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def read_dump(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    off = 0
    while off < len(data):
        (nl,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + nl].decode()
        off += nl
        (nd,) = struct.unpack_from("<I", data, off)
        off += 4
        dims = struct.unpack_from("<%dQ" % nd, data, off)
        off += 8 * nd
        n = int(np.prod(dims, dtype=np.int64)) if nd else 1
        arr = np.frombuffer(data, dtype="<u8", count=n, offset=off).reshape(dims)
        off += 8 * n
        out[name] = arr.astype(np.uint64)
    return out


MODELS = [
    ("mlp", "blocking", "private", 1),
    ("mlp", "pipelined", "private", 2),
    ("mlp", "blocking", "public", 1),
    ("toy_cnn", "blocking", "private", 1),
    ("toy_cnn", "pipelined", "public", 1),
    ("toy_transformer", "blocking", "private", 1),
    ("toy_transformer", "blocking", "public", 1),
    ("lenet5", "pipelined", "private", 1),
    ("vgg16", "blocking", "private", 1),   # ~10 min: the reference's largest expressible config
]


SCALE_OPS = ["relu_r18", "pool_vgg1", "softmax_bert", "qk_bert", "av_bert", "gemm_fc6", "gemm_r18l4"]
SCALE_MODELS = ["r18_conv1", "r18_l1conv", "r18_l2sc", "r18_l2conv_s2", "r18_l3conv", "r18_l4conv", "vgg_fc6", "bert_ffn1", "bert_ffn2"]


def main_scale(src=None):
    """Pack (or first generate, 4 reference runs at a time) the BASELINE-scale pins."""
    import concurrent.futures as cf
    import tempfile
    tmpd = src or tempfile.mkdtemp(prefix="mpcg_scale_")
    if not src:
        cmds = [[DRIVER, "scale", c, os.path.join(tmpd, c + ".bin")] for c in SCALE_OPS]
        cmds += [[DRIVER, "model_pin", os.path.join(HERE, "scale", m + ".json"), "blocking", "1", "private", "1",
                  os.path.join(tmpd, m + ".bin")] for m in SCALE_MODELS]
        with cf.ThreadPoolExecutor(4) as ex:
            list(ex.map(subprocess.check_call, cmds))
    out = {}
    for c in SCALE_OPS + SCALE_MODELS:
        for k, v in read_dump(os.path.join(tmpd, c + ".bin")).items():
            out[(c + "/" + k if c in SCALE_MODELS else k).replace("/", "__")] = v
    np.savez_compressed(os.path.join(HERE, "scale.npz"), **out)


def main():
    if "--scale" in sys.argv:
        src = sys.argv[sys.argv.index("--from") + 1] if "--from" in sys.argv else None
        return main_scale(src)
    tmp = os.path.join(HERE, "_tmp.bin")
    subprocess.check_call([DRIVER, "golden", tmp])
    d = read_dump(tmp)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **{k.replace("/", "__"): v for k, v in d.items()})
    only = sys.argv[1:]
    for name, mode, weights, iters in MODELS:
        if only and name not in only:
            continue
        cfg = os.path.join(ROOT, "configs", name + ".json")
        subprocess.check_call([DRIVER, "model", cfg, mode, str(iters), weights, "1", tmp])
        d = read_dump(tmp)
        np.savez_compressed(os.path.join(HERE, f"model_{name}_{mode}_{weights}_it{iters}.npz"), **d)
    os.remove(tmp)
    # triple-file pin: two dealer triples written by the reference's save_triples
    subprocess.check_call([DRIVER, "triples", os.path.join(HERE, "triples_ref.bin")])
    # MPCW interchange pin: the reference's init_weights(toy_cnn, 12) written by its save_weights
    subprocess.check_call([DRIVER, "mpcw", os.path.join(ROOT, "configs", "toy_cnn.json"), "12",
                           os.path.join(HERE, "toy_cnn_seed12.mpcw")])


if __name__ == "__main__":
    main()
