"""Model configs and deterministic synthetic data (H/engine/model.hpp).

Setup-time host code: JSON model graphs (H/engine/model.hpp:124-191), deterministic
weight init (H/engine/model.hpp:257-275) and demo input (H/engine/model.hpp:417-424),
all drawn from the reference's counter-mode splitmix64 so a model run here sees the
exact weights and inputs the reference sees for the same seed.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

PHI = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1
CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")

LAYER_KINDS = {"dense": 0, "conv2d": 1, "relu": 2, "maxpool2d": 3, "flatten": 4, "attention": 5,
               "softmax": 6, "mean_pool": 7,
               # extensions for the ResNet-18 / BERT-base configs (absent from the reference)
               "add": 8, "global_avg_pool": 9, "gelu": 10, "layernorm": 11}


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z.copy()
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def counter_draws(key: int, stream: int, n: int, first: int = 1) -> np.ndarray:
    """Draws first..first+n-1 of CounterRng(key, stream) (H/sharing/rng.hpp:10-32)."""
    k = np.uint64((key ^ ((stream * PHI) & M64)) & M64)
    with np.errstate(over="ignore"):
        c = np.arange(first, first + n, dtype=np.uint64)
        return _mix(k + c * np.uint64(PHI))


@dataclass
class LayerSpec:
    name: str
    type: str
    out: int = 0
    kernel: int = 0
    stride: int = 1
    pad: int = 0
    heads: int = 0
    bias: bool = True
    src: str = ""     # extension "from": input = this earlier layer's output ("input" = model input)
    other: str = ""   # extension "with": second operand of an "add"


@dataclass
class ModelGraph:
    name: str
    frac_bits: int
    input: tuple
    layers: list = field(default_factory=list)

    @staticmethod
    def from_json(obj) -> "ModelGraph":
        """H/engine/model.hpp:159-179 (same keys and defaults)."""
        if isinstance(obj, str):
            path = obj if os.path.exists(obj) else os.path.join(CONFIG_DIR, obj + ".json")
            with open(path) as f:
                obj = json.load(f)
        fb = int(obj.get("frac_bits", 20))
        layers = []
        for lj in obj["layers"]:
            t = lj["type"]
            if t not in LAYER_KINDS:
                raise ValueError("unknown layer type: " + t)
            layers.append(LayerSpec(lj.get("name", t), t, int(lj.get("out", 0)), int(lj.get("kernel", 0)),
                                    int(lj.get("stride", 1)), int(lj.get("pad", 0)), int(lj.get("heads", 0)),
                                    bool(lj.get("bias", True)), str(lj.get("from", "")), str(lj.get("with", ""))))
        return ModelGraph(obj.get("name", "model"), fb, tuple(int(d) for d in obj["input"]), layers)

    def with_batch(self, batch: int) -> "ModelGraph":
        return ModelGraph(self.name, self.frac_bits, (batch,) + tuple(self.input[1:]), list(self.layers))

    def wiring(self):
        """Producer index of each layer's input (-1 = model input) and of an add's second
        operand (extension; the reference's graphs are chains, H/engine/model.hpp:18-20)."""
        names, src, oth = {}, [], []
        for i, l in enumerate(self.layers):
            def look(n):
                if n == "input":
                    return -1
                if n not in names:
                    raise ValueError(f"{l.name}: unknown or later layer '{n}'")
                return names[n]
            src.append(look(l.src) if l.src else i - 1)
            oth.append(look(l.other) if l.type == "add" else None)
            names[l.name] = i
        return src, oth

    def shapes(self):
        """infer_shapes (H/engine/model.hpp:69-122, + the extension layers)."""
        out = []
        src, oth = self.wiring()
        for i, l in enumerate(self.layers):
            cur = list(self.input if src[i] < 0 else out[src[i]])
            if l.type == "dense":
                cur[-1] = l.out
            elif l.type == "conv2d":
                cur = [cur[0], l.out, (cur[2] + 2 * l.pad - l.kernel) // l.stride + 1,
                       (cur[3] + 2 * l.pad - l.kernel) // l.stride + 1]
            elif l.type == "maxpool2d":
                cur = [cur[0], cur[1], (cur[2] - l.kernel) // l.stride + 1, (cur[3] - l.kernel) // l.stride + 1]
            elif l.type == "flatten":
                cur = [cur[0], int(np.prod(cur[1:]))]
            elif l.type == "mean_pool":
                cur = [cur[0], cur[2]]
            elif l.type == "global_avg_pool":
                cur = [cur[0], cur[1]]
            out.append(tuple(cur))
        return out

    def weight_shapes(self):
        """model_weight_shapes (H/engine/model.hpp:213-252), in layer order."""
        out = []
        shapes = self.shapes()
        src, _ = self.wiring()
        for i, l in enumerate(self.layers):
            cur = self.input if src[i] < 0 else shapes[src[i]]
            if l.type == "dense":
                out.append((l.name + ".W", (cur[-1], l.out)))
                if l.bias:
                    out.append((l.name + ".b", (l.out,)))
            elif l.type == "conv2d":
                out.append((l.name + ".W", (cur[1] * l.kernel * l.kernel, l.out)))
                if l.bias:
                    out.append((l.name + ".b", (l.out,)))
            elif l.type == "attention":
                d = cur[2]
                out.append((l.name + ".Wqkv", (d, 3 * d)))
                if l.bias:
                    out.append((l.name + ".bqkv", (3 * d,)))
                out.append((l.name + ".Wo", (d, d)))
                if l.bias:
                    out.append((l.name + ".bo", (d,)))
            elif l.type == "layernorm":  # extension
                out.append((l.name + ".gamma", (cur[-1],)))
                out.append((l.name + ".beta", (cur[-1],)))
        return out


def _unit(draws: np.ndarray) -> np.ndarray:
    return (draws >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def init_weights(g: ModelGraph, seed: int) -> dict:
    """H/engine/model.hpp:257-275: one CounterRng(seed, 0x77e1 + idx) per tensor."""
    w = {}
    for idx, (key, shape) in enumerate(g.weight_shapes()):
        span = 1.0 / math.sqrt(float(shape[0])) if len(shape) >= 2 else 0.1
        u = _unit(counter_draws(seed, 0x77E1 + idx, int(np.prod(shape))))
        w[key] = ((2.0 * u - 1.0) * span).reshape(shape)
        if key.endswith(".gamma"):  # extension: LayerNorm scale centred on 1
            w[key] = w[key] + 1.0
    return w


def demo_input(g: ModelGraph, seed: int) -> np.ndarray:
    """H/engine/model.hpp:417-424."""
    u = _unit(counter_draws(seed, 0x1D07, int(np.prod(g.input))))
    return (2.0 * u - 1.0).reshape(g.input)


# ---------------------------------------------------------------- MPCW weights file
# H/engine/model.hpp:277-364: magic "MPCW", u32 version 1, u32 count, then per entry
# u32 name length, name, u32 rank, u64 dims, raw little-endian doubles.
def save_weights(w: dict, path: str) -> None:
    import struct
    with open(path, "wb") as f:
        f.write(b"MPCW")
        f.write(struct.pack("<II", 1, len(w)))
        for name in sorted(w):  # std::map order
            t = np.ascontiguousarray(w[name], dtype="<f8")
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)))
            f.write(nb)
            f.write(struct.pack("<I", t.ndim))
            f.write(struct.pack("<%dQ" % t.ndim, *t.shape))
            f.write(t.tobytes())


def load_weights(path: str) -> dict:
    import struct
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"MPCW":
        raise ValueError("not a weights file: " + path)
    off = 4
    version, count = struct.unpack_from("<II", data, off)
    off += 8
    if version != 1:
        raise ValueError("unsupported weights version")
    w = {}
    for _ in range(count):
        (nl,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + nl].decode()
        off += nl
        (rank,) = struct.unpack_from("<I", data, off)
        off += 4
        shape = struct.unpack_from("<%dQ" % rank, data, off)
        off += 8 * rank
        n = int(np.prod(shape)) if rank else 1
        if off + 8 * n > len(data):
            raise ValueError("weights file truncated")
        w[name] = np.frombuffer(data, dtype="<f8", count=n, offset=off).reshape(shape).copy()
        off += 8 * n
    return w


def check_weights(g: ModelGraph, w: dict) -> None:
    """H/engine/model.hpp:366-376: exactly the declared tensors, with their shapes."""
    expected = g.weight_shapes()
    if len(expected) != len(w):
        raise ValueError("weights entry count mismatch for model " + g.name)
    for key, shape in expected:
        if key not in w:
            raise ValueError("missing weight tensor: " + key)
        if tuple(w[key].shape) != tuple(shape):
            raise ValueError("wrong shape for weight tensor: " + key)


# ---------------------------------------------------------------- plaintext forward
# H/engine/reference.hpp:128-200: the double-precision replica the CLI's verify/replica
# check compares the decoded MPC logits against (+ the extension layers, with the same
# definitions as the secure ones: GeLU = x sigmoid(1.702 x), LayerNorm eps 1e-5).
def _im2col(x, k, stride, pad):
    N, C, H, W = x.shape
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad), dtype=x.dtype)
    xp[:, :, pad:pad + H, pad:pad + W] = x
    cols = np.empty((N, OH, OW, C, k, k), dtype=x.dtype)
    for ki in range(k):
        for kj in range(k):
            cols[:, :, :, :, ki, kj] = xp[:, :, ki:ki + stride * (OH - 1) + 1:stride,
                                          kj:kj + stride * (OW - 1) + 1:stride].transpose(0, 2, 3, 1)
    return cols.reshape(N * OH * OW, C * k * k)


def plaintext_forward(g: ModelGraph, w: dict, x: np.ndarray) -> np.ndarray:
    shapes = g.shapes()
    src, oth = g.wiring()
    x0 = np.asarray(x, dtype=np.float64)
    outs = []
    for i, l in enumerate(g.layers):
        cur = x0 if src[i] < 0 else outs[src[i]]
        shape = g.input if src[i] < 0 else shapes[src[i]]
        if l.type == "add":
            cur = cur + (x0 if oth[i] < 0 else outs[oth[i]])
        elif l.type == "dense":
            cur = cur.reshape(-1, shape[-1]) @ w[l.name + ".W"]
            if l.bias:
                cur = cur + w[l.name + ".b"]
        elif l.type == "conv2d":
            y = _im2col(cur.reshape(shape), l.kernel, l.stride, l.pad) @ w[l.name + ".W"]
            if l.bias:
                y = y + w[l.name + ".b"]
            N, _, OH, OW = shapes[i]
            cur = y.reshape(N, OH, OW, l.out).transpose(0, 3, 1, 2)
        elif l.type == "relu":
            cur = np.maximum(cur, 0.0)
        elif l.type == "maxpool2d":
            N, C, H, W = shape
            v = cur.reshape(shape)
            OH, OW = (H - l.kernel) // l.stride + 1, (W - l.kernel) // l.stride + 1
            m = np.full((N, C, OH, OW), -np.inf)
            for ki in range(l.kernel):
                for kj in range(l.kernel):
                    m = np.maximum(m, v[:, :, ki:ki + l.stride * (OH - 1) + 1:l.stride,
                                        kj:kj + l.stride * (OW - 1) + 1:l.stride])
            cur = m
        elif l.type in ("softmax",):
            v = cur.reshape(-1, shape[-1])
            e = np.exp(v - v.max(axis=1, keepdims=True))
            cur = e / e.sum(axis=1, keepdims=True)
        elif l.type == "mean_pool":
            cur = cur.reshape(shape).mean(axis=1)
        elif l.type == "global_avg_pool":
            cur = cur.reshape(shape).mean(axis=(2, 3))
        elif l.type == "gelu":
            cur = cur / (1.0 + np.exp(-1.702 * cur))
        elif l.type == "layernorm":
            v = cur.reshape(-1, shape[-1])
            mu = v.mean(axis=1, keepdims=True)
            var = ((v - mu) ** 2).mean(axis=1, keepdims=True)
            cur = (v - mu) / np.sqrt(var + 1e-5) * w[l.name + ".gamma"] + w[l.name + ".beta"]
        elif l.type == "attention":
            B, T, d = shape
            H = l.heads
            dh = d // H
            qkv = cur.reshape(B * T, d) @ w[l.name + ".Wqkv"]
            if l.bias:
                qkv = qkv + w[l.name + ".bqkv"]
            q, k, v = (qkv.reshape(B, T, 3, H, dh)[:, :, j].transpose(0, 2, 1, 3) for j in range(3))
            s = np.matmul(q, np.swapaxes(k, -1, -2)) / np.sqrt(dh)
            e = np.exp(s - s.max(axis=-1, keepdims=True))
            o = np.matmul(e / e.sum(axis=-1, keepdims=True), v)
            o = o.transpose(0, 2, 1, 3).reshape(B * T, d) @ w[l.name + ".Wo"]
            if l.bias:
                o = o + w[l.name + ".bo"]
            cur = o
        elif l.type == "flatten":
            pass
        cur = cur.reshape(shapes[i])
        outs.append(cur)
    return outs[-1]
