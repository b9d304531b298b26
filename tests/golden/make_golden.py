"""Generate golden fixtures from the UNMODIFIED reference (run here, where /root/reference exists).

    make -C oracle && python tests/golden/make_golden.py

Runs oracle/_ref/ref_driver (built from /root/reference/proj/include by oracle/Makefile)
and stores its dumps as compressed .npz fixtures in tests/golden/:

* ops.npz            — per-op inputs and per-party output shares (see oracle/ref_driver.cpp cmd_golden)
* model_<name>_<mode>_<weights>_it<k>.npz — per-party logits shares, opened logits, hash,
                       traffic counters and the double-precision reference_forward output.
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
]


def main():
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
    # MPCW interchange pin: the reference's init_weights(toy_cnn, 12) written by its save_weights
    subprocess.check_call([DRIVER, "mpcw", os.path.join(ROOT, "configs", "toy_cnn.json"), "12",
                           os.path.join(HERE, "toy_cnn_seed12.mpcw")])


if __name__ == "__main__":
    main()
