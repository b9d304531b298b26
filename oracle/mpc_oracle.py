"""CPU restatement of the MPC-Pipe reference's 2PC online path.

TEST INFRASTRUCTURE ONLY. This module is the parity checker: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline`/reference legs may
import it. The product path (paper_2209_13643_b200 + libmpcg.so) never calls
it and fails loudly when the CUDA library is missing.

Both parties are simulated jointly: every share-valued quantity is a list
`[share_party0, share_party1]` of numpy uint64 arrays, and an "open" is the
wrapping sum (or XOR) of the two payloads. Values do not depend on chunking
or pipelining (the reference proves this with AC2), so the oracle computes the
blocking schedule only; chunk counts enter only the traffic accounting.

Pinning: the restatement is checked against golden vectors dumped by the real
reference (oracle/ref_driver.cpp compiled into oracle/_ref/ by
oracle/Makefile, fixtures in tests/golden/, generator tests/golden/make_golden.py).

Citations are `path:line` into /root/reference/proj/include/mpcpipe (H/).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

U64 = np.uint64
PHI = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1
N_PARTIES = 2

np.seterr(over="ignore")


def _u(x) -> np.ndarray:
    return np.asarray(x, dtype=U64)


# ---------------------------------------------------------------- ring ops
# H/ring/ring_ops.hpp:13-25 — wrapping Z_2^64 arithmetic, arithmetic shift.

def sar(x: np.ndarray, k: int) -> np.ndarray:
    """H/ring/ring_ops.hpp:23-25 (sar under the signed view)."""
    return (_u(x).view(np.int64) >> np.int64(k)).view(U64)


def to_signed(x) -> np.ndarray:
    return _u(x).view(np.int64)


# ---------------------------------------------------------------- PRG
# H/sharing/rng.hpp:10-32 — counter-mode splitmix64.

def mix(z: np.ndarray) -> np.ndarray:
    z = _u(z).copy()
    z ^= z >> U64(30)
    z *= U64(0xBF58476D1CE4E5B9)
    z ^= z >> U64(27)
    z *= U64(0x94D049BB133111EB)
    z ^= z >> U64(31)
    return z


def draws(key: int, first_ctr: int, n: int) -> np.ndarray:
    """Block `first_ctr .. first_ctr+n-1` of key's stream: mix(key + c*phi)."""
    c = np.arange(first_ctr, first_ctr + n, dtype=U64)
    return mix(U64(key) + c * U64(PHI))


class CounterRng:
    """H/sharing/rng.hpp:10-32: key = key ^ (stream*phi); draw = mix(key + (++ctr)*phi)."""

    def __init__(self, key: int, stream: int = 0):
        self.key = (key ^ ((stream * PHI) & M64)) & M64
        self.counter = 0

    def take(self, n: int) -> np.ndarray:
        out = draws(self.key, self.counter + 1, n)
        self.counter += n
        return out

    def __call__(self) -> int:
        return int(self.take(1)[0])


def fnv1a(data: bytes) -> int:
    """Tag hash of H/sharing/triple.hpp:138-151 (FNV-1a 64)."""
    h = 0xCBF29CE484222325
    for c in data:
        h = ((h ^ c) * 0x100000001B3) & M64
    return h


def fnv1a_words(words: np.ndarray) -> int:
    """H/engine/report.hpp:18-23: FNV-1a over the LE bytes of the ring words."""
    return fnv1a(_u(words).astype("<u8").tobytes())


def mix_int(z: int) -> int:
    return int(mix(np.array([z], dtype=U64))[0])


# ---------------------------------------------------------------- fixed point
# H/ring/fixed.hpp:16-52.

def encode_fixed(x, scale_bits: int) -> np.ndarray:
    """round(x*2^s), ties toward +inf, computed exactly (H/ring/fixed.hpp:16-22)."""
    t = np.asarray(x, dtype=np.float64) * float(2 ** scale_bits)  # exact power-of-two scale
    f = np.floor(t)
    r = f + ((t - f) >= 0.5)  # t - f is exact for |t| < 2^52
    return r.astype(np.int64).view(U64)


def decode_fixed(v, scale_bits: int) -> np.ndarray:
    return to_signed(v).astype(np.float64) * (2.0 ** -scale_bits)


# ---------------------------------------------------------------- ring matmul
# H/ring/tensor.hpp:242-281 — batched wrapping GEMM, optional transpose_b.

def matmul(a: np.ndarray, b: np.ndarray, transpose_b: bool = False) -> np.ndarray:
    a = _u(a)
    b = _u(b)
    if transpose_b:
        b = np.swapaxes(b, -1, -2)
    M, K = a.shape[-2], a.shape[-1]
    if b.shape[-2] != K:
        raise ValueError("matmul: inner dim mismatch")
    if b.ndim > 2:
        batch = a.size // (M * K)
        out = np.matmul(a.reshape(batch, M, K), b.reshape(batch, K, b.shape[-1]))
    else:
        out = np.matmul(a.reshape(-1, K), b)
    return out.reshape(a.shape[:-1] + (b.shape[-1],))


# ---------------------------------------------------------------- comm stats
@dataclass
class CommStats:
    """H/transport/transport.hpp:39-45 (bytes_sent/collectives/p2p per party)."""
    bytes_sent: int = 0
    collectives: int = 0
    p2p_sends: int = 0
    trace: list = field(default_factory=list)  # (kind, tag, bytes)

    def reveal(self, numel: int, kind: str, tag: str):
        b = 8 * numel * (N_PARTIES - 1)
        self.bytes_sent += b
        self.collectives += 1
        self.trace.append((kind, tag, 8 * numel))

    def p2p(self, numel: int):
        self.bytes_sent += 8 * numel
        self.p2p_sends += 1


# ---------------------------------------------------------------- dealer
# H/sharing/triple.hpp:22-151.

@dataclass(frozen=True)
class TripleSpec:
    kind: str = "arith"          # "arith" | "bin"
    op: str = "elem"             # "elem" | "matmul"
    square: bool = False
    transpose_b: bool = False
    shape_a: tuple = ()
    shape_b: tuple = ()

    @staticmethod
    def elementwise(kind, shape):
        return TripleSpec(kind, "elem", False, False, tuple(shape), tuple(shape))

    @staticmethod
    def square_of(shape):
        return TripleSpec("arith", "elem", True, False, tuple(shape), tuple(shape))

    @staticmethod
    def matmul_of(a, b, transpose_b=False):
        return TripleSpec("arith", "matmul", False, transpose_b, tuple(a), tuple(b))


def dealer_gen_triple(spec: TripleSpec, rng: CounterRng):
    """H/sharing/triple.hpp:85-120 for n=2. Returns [(a,b,c) party0, (a,b,c) party1]."""
    na = int(np.prod(spec.shape_a, dtype=np.int64))
    A = rng.take(na).reshape(spec.shape_a)
    B = A if spec.square else rng.take(int(np.prod(spec.shape_b, dtype=np.int64))).reshape(spec.shape_b)
    if spec.op == "matmul":
        C = matmul(A, B, spec.transpose_b)
    elif spec.kind == "bin":
        C = A & B
    else:
        C = A * B
    out = [[], []]
    for T in (A, B, C):  # deal(A), deal(B), deal(C): H/sharing/share.hpp:22-50
        r = rng.take(T.size).reshape(T.shape)
        out[1].append(r)
        out[0].append((T ^ r) if spec.kind == "bin" else (T - r))
    return [tuple(out[0]), tuple(out[1])]


class SeededDealer:
    """H/sharing/triple.hpp:138-151, both parties at once (they agree by construction)."""

    def __init__(self, seed: int):
        self.seed = seed
        self.index = 0
        self.tag_counts: dict[int, int] = {}

    def stream_for(self, tag: str) -> int:
        if not tag:
            s = 0x7452 ^ self.index
            self.index += 1
            return s
        h = fnv1a(tag.encode())
        c = self.tag_counts.get(h, 0)
        self.tag_counts[h] = c + 1
        return mix_int((h + 0x51ED270B * c) & M64)

    def fetch(self, spec: TripleSpec, tag: str = ""):
        return dealer_gen_triple(spec, CounterRng(self.seed, self.stream_for(tag)))


# ---------------------------------------------------------------- sharing
def share_additive(x: np.ndarray, rng: CounterRng):
    """H/sharing/share.hpp:22-35 (n=2): party1 = r, party0 = x - r."""
    r = rng.take(x.size).reshape(x.shape)
    return [_u(x) - r, r]


def reconstruct(sh):
    return sh[0] + sh[1]


def reconstruct_bin(sh):
    return sh[0] ^ sh[1]


# ---------------------------------------------------------------- protocol context
@dataclass
class Ctx:
    """H/protocols/context.hpp:17-35 (ProtoCtx) for the joint 2-party simulation."""
    dealer: SeededDealer
    masks: list                   # [CounterRng party0, CounterRng party1]
    frac_bits: int = 16
    chunks: int = 1
    chunk_threshold: int = 0
    stats: list = field(default_factory=lambda: [CommStats(), CommStats()])

    def chunks_for(self, numel: int) -> int:
        if self.chunks <= 1:
            return 1
        if self.chunk_threshold and numel * 8 < self.chunk_threshold:
            return 1
        return self.chunks

    def reveal(self, numel: int, kind: str, tag: str, chunks: int = 1):
        chunks = max(1, min(chunks, numel if numel else 1))
        for s in self.stats:
            if chunks == 1:
                s.reveal(numel, kind, tag)
            else:
                for k in range(chunks):
                    lo, hi = numel * k // chunks, numel * (k + 1) // chunks
                    s.reveal(hi - lo, kind, f"{tag}.chunk{k}")


def make_ctx(seed: int, frac_bits: int, mask_key: int | None = None) -> Ctx:
    mk = (seed ^ PHI) if mask_key is None else mask_key
    return Ctx(SeededDealer(seed), [CounterRng(mk, 0), CounterRng(mk, 1)], frac_bits)


# ---------------------------------------------------------------- Beaver ops
# H/protocols/beaver.hpp:43-250.

def beaver_mul(X, Y, ctx: Ctx, tag="mul", chunks=1):
    """H/protocols/beaver.hpp:43-84."""
    t = ctx.dealer.fetch(TripleSpec.elementwise("arith", X[0].shape), tag)
    eps = (X[0] - t[0][0]) + (X[1] - t[1][0])
    dlt = (Y[0] - t[0][1]) + (Y[1] - t[1][1])
    ctx.reveal(2 * X[0].size, "sum", tag, _clamp(chunks, X[0].size))
    out = []
    for p in range(2):
        a, b, c = t[p]
        z = c + (eps * b + dlt * a)
        if p == 0:
            z = z + eps * dlt
        out.append(z)
    return out


def _clamp(chunks, numel):
    return max(1, min(chunks, numel if numel else 1))


def beaver_square(X, ctx: Ctx, tag="square", chunks=1):
    """H/protocols/beaver.hpp:88-125: z = c + 2*eps*a (+eps^2 on party 0)."""
    t = ctx.dealer.fetch(TripleSpec.square_of(X[0].shape), tag)
    eps = (X[0] - t[0][0]) + (X[1] - t[1][0])
    ctx.reveal(X[0].size, "sum", tag, _clamp(chunks, X[0].size))
    out = []
    for p in range(2):
        a, _, c = t[p]
        z = c + (eps * a) * U64(2)
        if p == 0:
            z = z + eps * eps
        out.append(z)
    return out


def beaver_and(X, Y, ctx: Ctx, tag="and", chunks=1):
    """H/protocols/beaver.hpp:129-169."""
    t = ctx.dealer.fetch(TripleSpec.elementwise("bin", X[0].shape), tag)
    eps = (X[0] ^ t[0][0]) ^ (X[1] ^ t[1][0])
    dlt = (Y[0] ^ t[0][1]) ^ (Y[1] ^ t[1][1])
    ctx.reveal(2 * X[0].size, "xor", tag, _clamp(chunks, X[0].size))
    out = []
    for p in range(2):
        a, b, c = t[p]
        z = c ^ ((eps & b) ^ (dlt & a))
        if p == 0:
            z = z ^ (eps & dlt)
        out.append(z)
    return out


def matmul_combine(t, eps, dlt, transpose_b, p):
    """H/protocols/beaver.hpp:175-180."""
    a, b, c = t
    z = c + (matmul(eps, b, transpose_b) + matmul(a, dlt, transpose_b))
    if p == 0:
        z = z + matmul(eps, dlt, transpose_b)
    return z


def beaver_matmul(X, Y, transpose_b, ctx: Ctx, tag="matmul", chunks=1):
    """H/protocols/beaver.hpp:186-250 (values; chunking only changes traffic)."""
    t = ctx.dealer.fetch(TripleSpec.matmul_of(X[0].shape, Y[0].shape, transpose_b), tag)
    dlt = (Y[0] - t[0][1]) + (Y[1] - t[1][1])
    eps = (X[0] - t[0][0]) + (X[1] - t[1][0])
    M, K = X[0].shape[-2], X[0].shape[-1]
    batched = Y[0].ndim > 2
    rows = X[0].size // (M * K) if batched else X[0].size // K
    ch = _clamp(chunks, rows)
    ctx.reveal(Y[0].size, "sum", tag + ".delta")
    if ch == 1:
        ctx.reveal(X[0].size, "sum", tag + ".eps")
    else:
        row_w = M * K if batched else K
        for k in range(ch):
            lo, hi = rows * k // ch, rows * (k + 1) // ch
            for s in ctx.stats:
                s.reveal((hi - lo) * row_w, "sum", f"{tag}.eps.chunk{k}")
    return [matmul_combine(t[p], eps, dlt, transpose_b, p) for p in range(2)]


# ---------------------------------------------------------------- SPK adder
# H/protocols/adder.hpp:25-327.

def make_spk_constants(width=64):
    """H/protocols/adder.hpp:37-57."""
    m = 0
    while (1 << m) < width:
        m += 1
    ins, outs, mults = [], [], []
    for i in range(m):
        half = 1 << i
        inn = out = 0
        for p in range(width):
            r = p & (2 * half - 1)
            if r == half - 1:
                inn |= 1 << p
            if r >= half:
                out |= 1 << p
        ins.append(inn)
        outs.append(out)
        mults.append((((1 << half) - 1) << 1) & M64)
    word_mask = M64 if width == 64 else (1 << width) - 1
    return m, ins, outs, mults, word_mask


SPK64 = make_spk_constants(64)


def spk_add_plain(a: int, b: int, width=64) -> int:
    """H/protocols/adder.hpp:74-89."""
    levels, ins, outs, mults, wm = make_spk_constants(width)
    s = a & b
    p = a ^ b
    p_orig = p
    for i in range(levels):
        p0 = p & outs[i]
        upd_s = p0 & (((s & ins[i]) * mults[i]) & M64)
        upd_p = p0 & (((p & ins[i]) * mults[i]) & M64)
        p = (p & ~outs[i] & M64) ^ upd_p
        s ^= upd_s
    return (p_orig ^ ((s << 1) & M64)) & wm


def binary_add(X, Y, ctx: Ctx, tag="badd", chunks=1, width=64):
    """H/protocols/adder.hpp:237-327 (merged/plain/chunked are bit-identical)."""
    levels, ins, outs, mults, wm = make_spk_constants(width)
    n = X[0].size
    ch = _clamp(chunks, n)
    S = beaver_and(X, Y, ctx, tag + ".g", ch)
    P = [X[0] ^ Y[0], X[1] ^ Y[1]]
    P_orig = [P[0].copy(), P[1].copy()]
    stacked = (2,) + tuple(X[0].shape)
    for i in range(levels):
        ltag = f"{tag}.l{i}"
        t = ctx.dealer.fetch(TripleSpec.elementwise("bin", stacked), ltag)
        inn, out, mult = U64(ins[i]), U64(outs[i]), U64(mults[i])
        pay = []
        for p in range(2):
            a, b, _ = t[p]
            p0 = P[p] & out
            pay.append((p0 ^ a[0], p0 ^ a[1], ((S[p] & inn) * mult) ^ b[0], ((P[p] & inn) * mult) ^ b[1]))
        e0, e1, d0, d1 = (pay[0][j] ^ pay[1][j] for j in range(4))
        ctx.reveal(4 * n, "xor", ltag, ch)
        for p in range(2):
            a, b, c = t[p]
            z0 = c[0] ^ (e0 & b[0]) ^ (d0 & a[0])
            z1 = c[1] ^ (e1 & b[1]) ^ (d1 & a[1])
            if p == 0:
                z0 = z0 ^ (e0 & d0)
                z1 = z1 ^ (e1 & d1)
            S[p] = S[p] ^ z0
            P[p] = (P[p] & ~out) ^ z1
    out_sh = [P_orig[p] ^ (S[p] << U64(1)) for p in range(2)]
    if width < 64:
        out_sh = [o & U64(wm) for o in out_sh]
    return out_sh


# ---------------------------------------------------------------- conversions
# H/protocols/compare.hpp:24-93.

def a2b(X, ctx: Ctx, tag="a2b", chunks=1):
    """2PC a2b: mask, p2p, one adder (H/protocols/compare.hpp:24-54)."""
    shape = X[0].shape
    r = [ctx.masks[p].take(X[p].size).reshape(shape) for p in range(2)]
    keep = [X[p] ^ r[p] for p in range(2)]
    for s in ctx.stats:
        s.p2p(X[0].size)
    # party0: parts = [keep0, r1]; party1: parts = [r0, keep1]
    return binary_add([keep[0], r[0]], [r[1], keep[1]], ctx, tag + ".add1", chunks)


def msb(X, ctx: Ctx, tag="msb", chunks=1):
    """H/protocols/compare.hpp:57-62."""
    b = a2b(X, ctx, tag, chunks)
    return [x >> U64(63) for x in b]


def b2a_bit(B, ctx: Ctx, tag="b2a", chunks=1):
    """H/protocols/compare.hpp:67-83 (n=2: one Beaver multiply)."""
    mine = [b & U64(1) for b in B]
    zero = np.zeros_like(mine[0])
    acc = [mine[0], zero]
    bq = [zero, mine[1]]
    prod = beaver_mul(acc, bq, ctx, tag + ".m1", chunks)
    return [(acc[p] + bq[p]) - (prod[p] + prod[p]) for p in range(2)]


def less_than(X, Y, ctx: Ctx, tag="lt", chunks=1):
    """H/protocols/compare.hpp:87-93."""
    d = [X[p] - Y[p] for p in range(2)]
    m = msb(d, ctx, tag + ".msb", chunks)
    return b2a_bit(m, ctx, tag + ".b2a", chunks)


def truncate_shares(X, bits):
    """2PC branch of H/protocols/trunc.hpp:25-42: local arithmetic shift."""
    return [sar(x, bits) for x in X]


def add_public(X, v):
    return [X[0] + U64(v & M64), X[1]]


# ---------------------------------------------------------------- nonlinear
# H/nonlinear/*.hpp.

def relu_shares(X, ctx: Ctx, tag="relu"):
    """H/nonlinear/activations.hpp:39-47."""
    ch = ctx.chunks_for(X[0].size)
    s = msb(X, ctx, tag + ".msb", ch)
    c = b2a_bit(s, ctx, tag + ".b2a", ch)
    xc = beaver_mul(X, c, ctx, tag + ".gate", ch)
    return [X[p] - xc[p] for p in range(2)]


def max_last_dim(X, L, ctx: Ctx, tag="max"):
    """H/nonlinear/activations.hpp:51-89: first-half vs second-half tournament."""
    outer = X[0].size // L
    cur = [x.reshape(outer, L) for x in X]
    ln = L
    rnd = 0
    while ln > 1:
        h = ln // 2
        odd = ln & 1
        a = [c[:, :h].copy() for c in cur]
        b = [c[:, h:2 * h].copy() for c in cur]
        rt = f"{tag}.r{rnd}"
        rnd += 1
        gate = less_than(a, b, ctx, rt, ctx.chunks_for(a[0].size))
        diff = [b[p] - a[p] for p in range(2)]
        step = beaver_mul(diff, gate, ctx, rt + ".pick", ctx.chunks_for(a[0].size))
        m = [a[p] + step[p] for p in range(2)]
        if odd:
            cur = [np.concatenate([m[p], cur[p][:, ln - 1:ln]], axis=1) for p in range(2)]
            ln = h + 1
        else:
            cur = m
            ln = h
    return [c.reshape(outer, 1) for c in cur]


def exp_shares(X, ctx: Ctx, tag="exp", square_iters=7):
    """H/nonlinear/approx.hpp:22-39."""
    f = ctx.frac_bits
    ch = ctx.chunks_for(X[0].size)
    w = truncate_shares(X, square_iters)
    w2 = beaver_square(w, ctx, tag + ".w2", ch)
    w2 = truncate_shares(w2, f + 1)
    y = add_public([w[p] + w2[p] for p in range(2)], 1 << f)
    for i in range(square_iters):
        y = beaver_square(y, ctx, f"{tag}.sq{i}", ch)
        y = truncate_shares(y, f)
    return y


def reciprocal_shares(X, ctx: Ctx, tag="recip", newton_iters=10):
    """H/nonlinear/approx.hpp:43-62."""
    f = ctx.frac_bits
    ch = ctx.chunks_for(X[0].size)
    t = add_public([U64(0) - X[0], U64(0) - X[1]], int(encode_fixed(0.5, f)))
    y = exp_shares(t, ctx, tag + ".seed")
    y = add_public([y[0] * U64(3), y[1] * U64(3)], int(encode_fixed(0.003, f)))
    for i in range(newton_iters):
        xy = beaver_mul(X, y, ctx, f"{tag}.xy{i}", ch)
        xy = truncate_shares(xy, f)
        u = add_public([U64(0) - xy[0], U64(0) - xy[1]], 2 << f)
        y = beaver_mul(y, u, ctx, f"{tag}.yu{i}", ch)
        y = truncate_shares(y, f)
    return y


def softmax_shares(X, L, ctx: Ctx, tag="softmax"):
    """H/nonlinear/activations.hpp:93-110."""
    shape = X[0].shape
    outer = X[0].size // L
    ch = ctx.chunks_for(X[0].size)
    mx = max_last_dim(X, L, ctx, tag + ".max")
    centered = [X[p].reshape(outer, L) - mx[p] for p in range(2)]
    e = exp_shares(centered, ctx, tag + ".exp")
    rowsum = [x.sum(axis=1, keepdims=True, dtype=U64) for x in e]
    r = reciprocal_shares(rowsum, ctx, tag + ".recip")
    rb = [np.broadcast_to(r[p], (outer, L)).copy() for p in range(2)]
    prod = beaver_mul(e, rb, ctx, tag + ".scale", ch)
    prod = truncate_shares(prod, ctx.frac_bits)
    return [x.reshape(shape) for x in prod]


def maxpool2d_windows(x, N, C, H, W, k, s):
    OH, OW = (H - k) // s + 1, (W - k) // s + 1
    xv = x.reshape(N, C, H, W)
    cols = []
    for i in range(k):
        for j in range(k):
            cols.append(xv[:, :, i:i + s * (OH - 1) + 1:s, j:j + s * (OW - 1) + 1:s])
    return np.stack(cols, axis=-1).reshape(N * C * OH * OW, k * k), OH, OW


def maxpool2d_shares(X, N, C, H, W, k, s, ctx: Ctx, tag="maxpool"):
    """H/nonlinear/activations.hpp:114-137."""
    win = []
    for p in range(2):
        w_, OH, OW = maxpool2d_windows(X[p], N, C, H, W, k, s)
        win.append(w_)
    mx = max_last_dim(win, k * k, ctx, tag)
    return [m.reshape(N, C, OH, OW) for m in mx]


# ---------------------------------------------------------------- extensions (NOT in the reference)
# Layers the BASELINE configs need that the reference lacks (SURVEY §0, §8(a*), §8f row 1):
# GeLU and LayerNorm (BERT-base), residual add and global average pooling (ResNet-18; BatchNorm
# is folded into the conv weights/bias by the weight owner). They are composed only from the
# reference's own building blocks — beaver_mul/square, msb/b2a_bit (compare.hpp), exp_shares /
# reciprocal_shares (approx.hpp), local truncation — with tags "<layer>.<step>" in the style of
# relu_shares/softmax_shares. PARITY UNPINNED by the reference (it has no such layers): the GPU
# path is held bit-exact to THIS restatement, and decoded values to the float64 forward below.

GELU_K = 1.702        # GeLU(x) ~= x * sigmoid(1.702 x)  (the sigmoid form of Hendrycks & Gimpel)
LN_EPS = 1e-5
ISQRT_ITERS = 3


def scale_rescale(X, c, f):
    """H/engine/executor.hpp:326-330 (scale_and_rescale) as a free function."""
    k = encode_fixed(c, f)
    return truncate_shares([x * k for x in X], f)


def recip_unit_iters(f: int) -> int:
    """Newton steps for 1/d on [1, 2] from the 1/17-accurate linear seed: the relative error
    after k steps is (1/17)^(2^k), below 2^-f once 2^k * log2(17) > f (f=16: 2, f=20: 3)."""
    k = 1
    while (2 ** k) * math.log2(17.0) <= f:
        k += 1
    return k


def recip_unit_shares(D, ctx: Ctx, tag="recip", iters=None):
    """1/d for d in [1, 2]: linear seed y0 = 24/17 - 8/17 d (relative error <= 1/17), then the
    reference's Newton step y <- trunc(y (2 - trunc(d y))) (H/nonlinear/approx.hpp:52-60);
    recip_unit_iters(f) steps take the error below the fixed-point resolution, so the
    reference's exp seed and ten steps are not needed on this interval."""
    f = ctx.frac_bits
    if iters is None:
        iters = recip_unit_iters(f)
    ch = ctx.chunks_for(D[0].size)
    y = add_public([U64(0) - v for v in scale_rescale(D, 8.0 / 17.0, f)], int(encode_fixed(24.0 / 17.0, f)))
    for i in range(iters):
        xy = truncate_shares(beaver_mul(D, y, ctx, f"{tag}.xy{i}", ch), f)
        u = add_public([U64(0) - xy[0], U64(0) - xy[1]], 2 << f)
        y = truncate_shares(beaver_mul(y, u, ctx, f"{tag}.yu{i}", ch), f)
    return y


def sigmoid_shares(X, ctx: Ctx, tag="sigmoid"):
    """sigma(x) = b ? 1 - sigma(|x|) : sigma(|x|), b = [x < 0], sigma(|x|) = 1/(1 + exp(-|x|)).
    exp only ever sees -|x| <= 0 (exp_shares' accurate side, H/nonlinear/approx.hpp:22-39) and the
    reciprocal only (1, 2] (recip_unit_shares)."""
    f = ctx.frac_bits
    ch = ctx.chunks_for(X[0].size)
    s = msb(X, ctx, tag + ".msb", ch)
    b = b2a_bit(s, ctx, tag + ".b2a", ch)
    xb = beaver_mul(X, b, ctx, tag + ".abs", ch)
    nabs = [(xb[p] + xb[p]) - X[p] for p in range(2)]                 # -|x|
    e = exp_shares(nabs, ctx, tag + ".exp")
    r = recip_unit_shares(add_public(e, 1 << f), ctx, tag + ".recip")  # sigma(|x|)
    t = add_public([U64(0) - (r[p] + r[p]) for p in range(2)], 1 << f)  # 1 - 2 sigma(|x|)
    sel = beaver_mul(b, t, ctx, tag + ".sel", ch)                      # b has scale 0: no truncation
    return [r[p] + sel[p] for p in range(2)]


def gelu_shares(X, ctx: Ctx, tag="gelu"):
    f = ctx.frac_bits
    ch = ctx.chunks_for(X[0].size)
    z = scale_rescale(X, GELU_K, f)
    sg = sigmoid_shares(z, ctx, tag + ".sig")
    return truncate_shares(beaver_mul(X, sg, ctx, tag + ".out", ch), f)


def inv_sqrt_shares(V, ctx: Ctx, tag="isqrt", newton_iters=ISQRT_ITERS):
    """1/sqrt(v): seed y0 = 2.2 exp(-(v/2 + 0.2)) + 0.2 - v/1024, then Newton
    y <- y (3 - v y^2) / 2 (CrypTen's inv_sqrt recipe; accurate for v in ~[0.1, 200])."""
    f = ctx.frac_bits
    ch = ctx.chunks_for(V[0].size)
    t = add_public([U64(0) - sar(V[p], 1) for p in range(2)], -int(encode_fixed(0.2, f)))
    e = exp_shares(t, ctx, tag + ".seed")
    y = scale_rescale(e, 2.2, f)
    y = add_public([y[p] - sar(V[p], 10) for p in range(2)], int(encode_fixed(0.2, f)))
    three = int(encode_fixed(3.0, f))
    for i in range(newton_iters):
        y2 = truncate_shares(beaver_square(y, ctx, f"{tag}.y2{i}", ch), f)
        vy2 = truncate_shares(beaver_mul(V, y2, ctx, f"{tag}.vy{i}", ch), f)
        u = add_public([U64(0) - vy2[p] for p in range(2)], three)
        y = truncate_shares(beaver_mul(y, u, ctx, f"{tag}.yu{i}", ch), f + 1)   # /2 folded in
    return y


def layernorm_shares(X, d, gamma, beta, ctx: Ctx, tag="ln", public=False):
    """LayerNorm over the last dim: (x - mean) * inv_sqrt(var + eps) * gamma + beta.
    gamma/beta: [share0, share1] of [d] (private) or encoded plaintext [d] (public)."""
    f = ctx.frac_bits
    shape = X[0].shape
    rows = X[0].size // d
    ch = ctx.chunks_for(X[0].size)
    x = [v.reshape(rows, d) for v in X]
    mu = scale_rescale([v.sum(axis=1, keepdims=True, dtype=U64) for v in x], 1.0 / d, f)
    c = [x[p] - mu[p] for p in range(2)]
    sq = truncate_shares(beaver_square(c, ctx, tag + ".sq", ch), f)
    var = scale_rescale([v.sum(axis=1, keepdims=True, dtype=U64) for v in sq], 1.0 / d, f)
    var = add_public(var, int(encode_fixed(LN_EPS, f)))
    y = inv_sqrt_shares(var, ctx, tag + ".isqrt")
    yb = [np.broadcast_to(y[p], (rows, d)).copy() for p in range(2)]
    n = truncate_shares(beaver_mul(c, yb, ctx, tag + ".norm", ch), f)
    if public:
        out = truncate_shares([v * gamma[None, :] for v in n], f)
        out = [out[0] + beta[None, :], out[1]]
    else:
        gb = [np.broadcast_to(gamma[p][None, :], (rows, d)).copy() for p in range(2)]
        out = truncate_shares(beaver_mul(n, gb, ctx, tag + ".gamma", ch), f)
        out = [out[p] + beta[p][None, :] for p in range(2)]
    return [o.reshape(shape) for o in out]


def global_avg_pool(X, in_shape, f):
    """NCHW -> [N, C]: sum over H*W then scale_and_rescale(1/(H*W)) (as MeanPool,
    H/engine/executor.hpp:399-410)."""
    N, C, H, W = in_shape
    s = [x.reshape(N, C, H * W).sum(axis=2, dtype=U64) for x in X]
    return scale_rescale(s, 1.0 / (H * W), f)


# ---------------------------------------------------------------- engine
# H/engine/model.hpp, H/engine/executor.hpp.

LAYER_KINDS = ("dense", "conv2d", "relu", "maxpool2d", "flatten", "attention", "softmax", "mean_pool",
               # extensions for the ResNet-18 / BERT-base configs (absent from the reference)
               "add", "global_avg_pool", "gelu", "layernorm")


@dataclass
class Layer:
    name: str
    type: str
    out: int = 0
    kernel: int = 0
    stride: int = 1
    pad: int = 0
    heads: int = 0
    bias: bool = True
    src: str = ""      # extension: "from" — input is this earlier layer's output ("input" = model input)
    other: str = ""    # extension: "with" — second operand of an "add"


@dataclass
class Model:
    name: str
    frac_bits: int
    input: tuple
    layers: list


def model_from_json(j: dict) -> Model:
    """H/engine/model.hpp:159-179."""
    fb = int(j.get("frac_bits", 20))
    layers = []
    for lj in j["layers"]:
        t = lj["type"]
        if t not in LAYER_KINDS:
            raise ValueError("unknown layer type: " + t)
        layers.append(Layer(lj.get("name", t), t, int(lj.get("out", 0)), int(lj.get("kernel", 0)),
                            int(lj.get("stride", 1)), int(lj.get("pad", 0)), int(lj.get("heads", 0)),
                            bool(lj.get("bias", True)), str(lj.get("from", "")), str(lj.get("with", ""))))
    m = Model(j.get("name", "model"), fb, tuple(int(d) for d in j["input"]), layers)
    infer_shapes(m)
    return m


def layer_inputs(g: Model):
    """Extension (non-chain graphs): index of each layer's input producer (-1 = model input)
    and of an "add"'s second operand. The reference only has chains (H/engine/model.hpp:18-20)."""
    names = {}
    src, oth = [], []
    for i, l in enumerate(g.layers):
        def look(n):
            if n == "input":
                return -1
            if n not in names:
                raise ValueError(f"{l.name}: unknown or later layer '{n}'")
            return names[n]
        src.append(look(l.src) if l.src else i - 1)
        if l.type == "add":
            if not l.other:
                raise ValueError(f"{l.name}: add needs 'with'")
            oth.append(look(l.other))
        else:
            oth.append(None)
        if l.name in names:
            raise ValueError("duplicate layer name: " + l.name)
        names[l.name] = i
    return src, oth


def infer_shapes(g: Model):
    """H/engine/model.hpp:69-122 (+ the extension layers)."""
    out = []
    src, oth = layer_inputs(g)
    for i, l in enumerate(g.layers):
        cur = list(g.input if src[i] < 0 else out[src[i]])
        if l.type == "add":
            other = list(g.input if oth[i] < 0 else out[oth[i]])
            if other != cur:
                raise ValueError(f"{l.name}: add operand shapes differ {cur} vs {other}")
        elif l.type == "global_avg_pool":
            cur = [cur[0], cur[1]]
        elif l.type == "dense":
            cur[-1] = l.out
        elif l.type == "conv2d":
            h, w = cur[2], cur[3]
            cur = [cur[0], l.out, (h + 2 * l.pad - l.kernel) // l.stride + 1,
                   (w + 2 * l.pad - l.kernel) // l.stride + 1]
        elif l.type == "maxpool2d":
            cur = [cur[0], cur[1], (cur[2] - l.kernel) // l.stride + 1, (cur[3] - l.kernel) // l.stride + 1]
        elif l.type == "flatten":
            cur = [cur[0], int(np.prod(cur[1:]))]
        elif l.type == "mean_pool":
            cur = [cur[0], cur[2]]
        out.append(tuple(cur))
    return out


def layer_weight_shapes(l: Layer, in_shape):
    """H/engine/model.hpp:213-241."""
    if l.type == "dense":
        r = [(l.name + ".W", (in_shape[-1], l.out))]
        if l.bias:
            r.append((l.name + ".b", (l.out,)))
        return r
    if l.type == "conv2d":
        r = [(l.name + ".W", (in_shape[1] * l.kernel * l.kernel, l.out))]
        if l.bias:
            r.append((l.name + ".b", (l.out,)))
        return r
    if l.type == "attention":
        d = in_shape[2]
        r = [(l.name + ".Wqkv", (d, 3 * d))]
        if l.bias:
            r.append((l.name + ".bqkv", (3 * d,)))
        r.append((l.name + ".Wo", (d, d)))
        if l.bias:
            r.append((l.name + ".bo", (d,)))
        return r
    if l.type == "layernorm":  # extension: affine LayerNorm over the last dim
        return [(l.name + ".gamma", (in_shape[-1],)), (l.name + ".beta", (in_shape[-1],))]
    return []


def model_weight_shapes(g: Model):
    shapes = infer_shapes(g)
    src, _ = layer_inputs(g)
    out = []
    for i, l in enumerate(g.layers):
        out += layer_weight_shapes(l, g.input if src[i] < 0 else shapes[src[i]])
    return out


def _unit_doubles(rng: CounterRng, n: int) -> np.ndarray:
    return (rng.take(n) >> U64(11)).astype(np.float64) * (2.0 ** -53)


def init_weights(g: Model, seed: int) -> dict:
    """H/engine/model.hpp:257-275."""
    w = {}
    for idx, (key, shape) in enumerate(model_weight_shapes(g)):
        rng = CounterRng(seed, 0x77E1 + idx)
        span = 1.0 / math.sqrt(float(shape[0])) if len(shape) >= 2 else 0.1
        u = _unit_doubles(rng, int(np.prod(shape)))
        w[key] = ((2.0 * u - 1.0) * span).reshape(shape)
        if key.endswith(".gamma"):  # extension: LayerNorm scale centred on 1
            w[key] = w[key] + 1.0
    return w


def demo_input(g: Model, seed: int) -> np.ndarray:
    """H/engine/model.hpp:417-424."""
    rng = CounterRng(seed, 0x1D07)
    u = _unit_doubles(rng, int(np.prod(g.input)))
    return (2.0 * u - 1.0).reshape(g.input)


def deal_weight_shares(g: Model, w: dict, seed: int):
    """H/engine/executor.hpp:49-59: one CounterRng(seed, 0x3e1f) over sorted names."""
    rng = CounterRng(seed, 0x3E1F)
    out = {}
    for key in sorted(w):
        enc = encode_fixed(w[key], g.frac_bits)
        out[key] = share_additive(enc, rng)
    return out


def deal_input_share(x: np.ndarray, frac_bits: int, seed: int):
    """H/engine/executor.hpp:70-75."""
    return share_additive(encode_fixed(x, frac_bits), CounterRng(seed, 0x11A9))


def im2col(x, k, stride, pad):
    """H/engine/executor.hpp:82-108: row=(n,oh,ow), col=(ci,ki,kj), zero taps."""
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


def col2im(y, N, Cout, OH, OW):
    """H/engine/executor.hpp:110-123."""
    return y.reshape(N, OH, OW, Cout).transpose(0, 3, 1, 2).copy()


def split_heads(qkv, B, T, d, heads, part):
    dh = d // heads
    v = qkv.reshape(B, T, 3, heads, dh)[:, :, part]          # [B,T,H,dh]
    return v.transpose(0, 2, 1, 3).reshape(B * heads, T, dh).copy()


def merge_heads(x, B, T, d, heads):
    dh = d // heads
    return x.reshape(B, heads, T, dh).transpose(0, 2, 1, 3).reshape(B * T, d).copy()


class SecureExecutor:
    """Values of H/engine/executor.hpp:173-413 for both parties jointly."""

    def __init__(self, g: Model, wshares: dict, ctx: Ctx, public: bool = False):
        self.g = g
        self.shapes = infer_shapes(g)
        self.w = wshares      # name -> [share0, share1] (private) or name -> encoded (public)
        self.public = public
        self.ctx = ctx
        ctx.frac_bits = g.frac_bits

    def weight_matmul(self, tag, wkey, x2d):
        f = self.g.frac_bits
        if self.public:
            return [matmul(x2d[p], self.w[wkey]) for p in range(2)]
        W = self.w[wkey]
        t = self.ctx.dealer.fetch(TripleSpec.matmul_of(x2d[0].shape, W[0].shape), tag)
        dlt = (W[0] - t[0][1]) + (W[1] - t[1][1])
        self.ctx.reveal(W[0].size, "sum", tag + ".delta")
        eps = (x2d[0] - t[0][0]) + (x2d[1] - t[1][0])
        self.ctx.reveal(x2d[0].size, "sum", tag + ".eps")
        return [matmul_combine(t[p], eps, dlt, False, p) for p in range(2)]

    def finish_linear(self, z, bkey):
        z = truncate_shares(z, self.g.frac_bits)
        if bkey:
            if self.public:
                z = [z[0] + self.w[bkey], z[1]]
            else:
                z = [z[p] + self.w[bkey][p] for p in range(2)]
        return z

    def scale_and_rescale(self, X, c):
        k = encode_fixed(c, self.g.frac_bits)
        return truncate_shares([x * k for x in X], self.g.frac_bits)

    def attention(self, l, X, in_shape):
        B, T, d = in_shape
        heads = l.heads
        dh = d // heads
        x2 = [x.reshape(B * T, d) for x in X]
        qkv = self.finish_linear(self.weight_matmul(l.name + ".qkv", l.name + ".Wqkv", x2),
                                 l.name + ".bqkv" if l.bias else "")
        q = [split_heads(qkv[p], B, T, d, heads, 0) for p in range(2)]
        k = [split_heads(qkv[p], B, T, d, heads, 1) for p in range(2)]
        v = [split_heads(qkv[p], B, T, d, heads, 2) for p in range(2)]
        sc = beaver_matmul(q, k, True, self.ctx, l.name + ".qk", self.ctx.chunks_for(B * heads * T * T))
        sc = truncate_shares(sc, self.g.frac_bits)
        sc = self.scale_and_rescale(sc, 1.0 / math.sqrt(dh))
        probs = softmax_shares(sc, T, self.ctx, l.name + ".softmax")
        mixed = beaver_matmul(probs, v, False, self.ctx, l.name + ".av", self.ctx.chunks_for(B * heads * T * dh))
        mixed = truncate_shares(mixed, self.g.frac_bits)
        merged = [merge_heads(mixed[p], B, T, d, heads) for p in range(2)]
        out = self.finish_linear(self.weight_matmul(l.name + ".proj", l.name + ".Wo", merged),
                                 l.name + ".bo" if l.bias else "")
        return [o.reshape(B, T, d) for o in out]

    def run_layer(self, l, X, in_shape):
        if l.type == "dense":
            x2 = [x.reshape(-1, in_shape[-1]) for x in X]
            z = self.finish_linear(self.weight_matmul(l.name + ".mm", l.name + ".W", x2),
                                   l.name + ".b" if l.bias else "")
            return [zz.reshape(tuple(in_shape[:-1]) + (l.out,)) for zz in z]
        if l.type == "conv2d":
            N, C, H, W = in_shape
            OH = (H + 2 * l.pad - l.kernel) // l.stride + 1
            OW = (W + 2 * l.pad - l.kernel) // l.stride + 1
            cols = [im2col(x.reshape(in_shape), l.kernel, l.stride, l.pad) for x in X]
            z = self.finish_linear(self.weight_matmul(l.name + ".mm", l.name + ".W", cols),
                                   l.name + ".b" if l.bias else "")
            return [col2im(zz, N, l.out, OH, OW) for zz in z]
        if l.type == "relu":
            return relu_shares(X, self.ctx, l.name)
        if l.type == "maxpool2d":
            N, C, H, W = in_shape
            return maxpool2d_shares(X, N, C, H, W, l.kernel, l.stride, self.ctx, l.name)
        if l.type == "flatten":
            return [x.reshape(in_shape[0], -1) for x in X]
        if l.type == "attention":
            return self.attention(l, X, in_shape)
        if l.type == "softmax":
            return softmax_shares(X, in_shape[-1], self.ctx, l.name)
        if l.type == "mean_pool":
            B, T, d = in_shape
            s = [x.reshape(B, T, d).sum(axis=1, dtype=U64) for x in X]
            return self.scale_and_rescale(s, 1.0 / T)
        if l.type == "global_avg_pool":
            return global_avg_pool(X, in_shape, self.g.frac_bits)
        if l.type == "gelu":
            return gelu_shares(X, self.ctx, l.name)
        if l.type == "layernorm":
            return layernorm_shares(X, in_shape[-1], self.w[l.name + ".gamma"], self.w[l.name + ".beta"],
                                    self.ctx, l.name, self.public)
        raise ValueError(l.type)

    def run(self, X):
        """Chain order as the reference (H/engine/executor.hpp:193-205); the extension's
        "from"/"with" read earlier outputs (an "add" is a local share addition)."""
        src, oth = layer_inputs(self.g)
        outs = []
        for i, l in enumerate(self.g.layers):
            x = X if src[i] < 0 else outs[src[i]]
            shape = self.g.input if src[i] < 0 else self.shapes[src[i]]
            if l.type == "add":
                y = X if oth[i] < 0 else outs[oth[i]]
                cur = [x[p] + y[p] for p in range(2)]
            else:
                cur = self.run_layer(l, x, shape)
            outs.append(cur)
        return outs[-1]


def bench_party_values(g: Model, seed: int = 1, iterations: int = 1, public: bool = False,
                       weights: dict | None = None, x: np.ndarray | None = None):
    """Values of H/engine/bench.hpp:36-63 for both parties: returns (logit shares, opened logits, hash, ctx)."""
    weights = init_weights(g, seed + 11) if weights is None else weights
    x = demo_input(g, seed + 12) if x is None else x
    ctx = make_ctx(seed, g.frac_bits)
    if public:
        wsh = {k: encode_fixed(v, g.frac_bits) for k, v in weights.items()}
    else:
        wsh = deal_weight_shares(g, weights, seed)
    ex = SecureExecutor(g, wsh, ctx, public)
    xin = deal_input_share(x, g.frac_bits, seed + 1)
    out = None
    for _ in range(iterations):
        out = ex.run(xin)
    opened = reconstruct(out)
    return out, opened, fnv1a_words(opened.reshape(-1)), ctx


# ---------------------------------------------------------------- plaintext reference
def reference_forward(g: Model, w: dict, x: np.ndarray) -> np.ndarray:
    """Double-precision forward of H/engine/reference.hpp:128-200."""
    x0 = np.asarray(x, dtype=np.float64)
    shapes = infer_shapes(g)
    src, oth = layer_inputs(g)
    outs = []
    for i, l in enumerate(g.layers):
        cur = x0 if src[i] < 0 else outs[src[i]]
        shape = g.input if src[i] < 0 else shapes[src[i]]
        if l.type == "add":
            cur = cur + (x0 if oth[i] < 0 else outs[oth[i]])
        elif l.type == "global_avg_pool":
            cur = cur.reshape(shape).mean(axis=(2, 3))
        elif l.type == "gelu":
            cur = cur / (1.0 + np.exp(-GELU_K * cur))
        elif l.type == "layernorm":
            v = cur.reshape(-1, shape[-1])
            mu = v.mean(axis=1, keepdims=True)
            var = ((v - mu) ** 2).mean(axis=1, keepdims=True)
            cur = (v - mu) / np.sqrt(var + LN_EPS) * w[l.name + ".gamma"] + w[l.name + ".beta"]
        elif l.type == "dense":
            cur = cur.reshape(-1, shape[-1]) @ w[l.name + ".W"]
            if l.bias:
                cur = cur + w[l.name + ".b"]
        elif l.type == "conv2d":
            N = shape[0]
            cols = im2col(cur.reshape(shape), l.kernel, l.stride, l.pad)
            y = cols @ w[l.name + ".W"]
            if l.bias:
                y = y + w[l.name + ".b"]
            cur = col2im(y, N, l.out, shapes[i][2], shapes[i][3])
        elif l.type == "relu":
            cur = np.maximum(cur, 0.0)
        elif l.type == "maxpool2d":
            N, C, H, W = shape
            win, OH, OW = maxpool2d_windows(cur.reshape(shape), N, C, H, W, l.kernel, l.stride)
            cur = win.max(axis=1)
        elif l.type == "softmax":
            v = cur.reshape(-1, shape[-1])
            e = np.exp(v - v.max(axis=1, keepdims=True))
            cur = e / e.sum(axis=1, keepdims=True)
        elif l.type == "mean_pool":
            cur = cur.reshape(shape).mean(axis=1)
        elif l.type == "attention":
            B, T, d = shape
            H = l.heads
            dh = d // H
            qkv = cur.reshape(B * T, d) @ w[l.name + ".Wqkv"]
            if l.bias:
                qkv = qkv + w[l.name + ".bqkv"]
            q, k, v = (split_heads(qkv, B, T, d, H, j) for j in range(3))
            s = np.matmul(q, np.swapaxes(k, 1, 2)) / math.sqrt(dh)
            e = np.exp(s - s.max(axis=2, keepdims=True))
            pr = e / e.sum(axis=2, keepdims=True)
            o = merge_heads(np.matmul(pr, v), B, T, d, H) @ w[l.name + ".Wo"]
            if l.bias:
                o = o + w[l.name + ".bo"]
            cur = o
        cur = cur.reshape(shapes[i])
        outs.append(cur)
    return outs[-1]
