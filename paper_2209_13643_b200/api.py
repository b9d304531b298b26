"""Python mirror of the reference operator API over the C ABI (include/mpcg.h).

Names and argument meaning follow the reference free functions
(H/protocols/*.hpp, H/nonlinear/*.hpp, H/engine/executor.hpp); each `Tensor` holds the
shares of every party slot that lives in this process (2 in 1-GPU mode, 1 otherwise),
so one call runs the op for all local parties. Exceptions mirror H/errors.hpp.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .model import LAYER_KINDS, ModelGraph

PHI = 0x9E3779B97F4A7C15


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(N.U64P)


def _tag(t: str):
    return t.encode() if t is not None else None


class Session:
    """Local party slots on one GPU: Communicator + SeededDealer + mask rng + ProtoCtx knobs.

    n_local=2 runs both parties of a pair on `device`; n_local=1 runs `party` only and
    needs `connect_nccl`. mask_seed defaults to the CLI's seed ^ phi (H/engine/bench.hpp:40).
    """

    def __init__(self, device=0, n_local=2, party=0, seed=1, mask_seed=None, frac_bits=16):
        if mask_seed is None:
            mask_seed = seed ^ PHI
        h = C.c_void_p()
        N.call("mpcg_session_create", device, n_local, party, seed, mask_seed & ((1 << 64) - 1), frac_bits,
               C.byref(h))
        self._h = h
        self.n_local = n_local
        self.party = party
        self.frac_bits = frac_bits

    def close(self):
        if getattr(self, "_h", None):
            N.lib().mpcg_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_pipeline(self, chunks=1, threshold=0, merged=True):
        N.call("mpcg_session_set_pipeline", self._h, chunks, threshold, int(merged))

    def set_link(self, latency_s=0.0, bandwidth_Bps=0.0, sec_per_message=0.0):
        N.call("mpcg_session_set_link", self._h, latency_s, bandwidth_Bps, sec_per_message)

    def set_shard(self, local_batch, global_batch, batch_offset):
        N.call("mpcg_session_set_shard", self._h, local_batch, global_batch, batch_offset)

    def connect_loopback(self, peer: "Session"):
        """Link this single-party session with `peer` (the other party) on the same GPU: the
        2-GPU code path with device copies instead of NCCL (each party on its own thread)."""
        N.call("mpcg_session_connect_loopback", self._h, peer._h)

    def connect_p2p(self, peer: "Session"):
        """Device-initiated peer-store link with `peer` (the other party's single-party session in
        this process, same GPU or a peer-accessible one): flags, no host events; graph-capturable."""
        N.call("mpcg_session_connect_p2p", self._h, peer._h)

    def connect_socket(self, host: str, port: int, timeout_s: float = 60.0):
        """TCP link to the other party's process (party 0 listens, party 1 connects): the
        reference's SocketComm for one-party sessions in different processes / hosts."""
        N.call("mpcg_session_connect_socket", self._h, host.encode(), int(port), float(timeout_s))

    def connect_nccl(self, unique_id: bytes, rank: int):
        N.call("mpcg_session_connect_nccl", self._h, unique_id, rank)

    def sync(self):
        N.call("mpcg_session_sync", self._h)

    def set_persistent(self, mode=True):
        """1-GPU mode: persistent compare chains (True/1), one kernel per round (False/0) or
        auto by size (2, the session default)."""
        N.call("mpcg_session_set_persistent", self._h, int(mode))

    def trace(self, enable=True):
        """Record one row per collective (Communicator::trace, H/transport/transport.hpp:25-37)
        with device timestamps; see trace_rows()."""
        N.call("mpcg_session_trace", self._h, int(enable))

    def trace_rows(self):
        """Synchronise and return the trace: dicts with seq, kind, tag, bytes, t_issue, t_sent,
        t_wait_begin, t_wait_end (seconds since trace start), occupancy, stall."""
        n = C.c_uint64()
        N.call("mpcg_session_trace_count", self._h, C.byref(n))
        rows = []
        seq, kind, nb = C.c_uint32(), C.c_int32(), C.c_uint64()
        t = (C.c_double * 4)()
        buf = C.create_string_buffer(256)
        for i in range(n.value):
            N.call("mpcg_session_trace_get", self._h, i, C.byref(seq), C.byref(kind), C.byref(nb), t, buf, 256)
            rows.append({"seq": seq.value, "kind": "xor" if kind.value else "sum", "tag": buf.value.decode(),
                         "bytes": nb.value, "t_issue": t[0], "t_sent": t[1], "t_wait_begin": t[2],
                         "t_wait_end": t[3], "occupancy": t[1] - t[0], "stall": t[3] - t[2]})
        return rows

    def clear_trace(self):
        N.call("mpcg_session_clear_trace", self._h)

    def now(self) -> float:
        """Host wall seconds since the session was created (Communicator::now)."""
        v = C.c_double()
        N.call("mpcg_session_now", self._h, C.byref(v))
        return v.value

    def add_delay(self, seconds: float):
        """Fault injection (Communicator::add_delay): this session's stream idles `seconds`."""
        N.call("mpcg_session_add_delay", self._h, float(seconds))

    def stats(self, slot=0):
        out = (C.c_uint64 * 3)()
        N.call("mpcg_session_stats", self._h, slot, out)
        return {"bytes_sent": out[0], "collectives": out[1], "p2p_sends": out[2]}

    def tensor(self, shares: np.ndarray, scale=0) -> "Tensor":
        """shares: array [n_local, *shape] of uint64 (slot-major)."""
        a = np.ascontiguousarray(shares, dtype=np.uint64)
        if a.shape[0] != self.n_local:
            raise N.ShapeError(f"expected {self.n_local} share slots, got {a.shape[0]}")
        shape = a.shape[1:]
        dims = np.array(shape, dtype=np.uint64)
        h = C.c_void_p()
        N.call("mpcg_tensor_create", self._h, len(shape), _u64p(dims), scale, _u64p(a), C.byref(h))
        return Tensor(self, h)

    def deal_input(self, x_global: np.ndarray, seed: int, batch_offset=0, local_batch=None) -> "Tensor":
        """deal_input_share (H/engine/executor.hpp:70-75) of rows [off, off+local)."""
        x = np.ascontiguousarray(x_global, dtype=np.float64)
        local_batch = x.shape[0] if local_batch is None else local_batch
        dims = np.array(x.shape, dtype=np.uint64)
        h = C.c_void_p()
        N.call("mpcg_deal_input", self._h, x.ctypes.data_as(C.POINTER(C.c_double)), x.ndim, _u64p(dims),
               batch_offset, local_batch, seed, C.byref(h))
        return Tensor(self, h)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.call("mpcg_nccl_unique_id", buf)
    return buf.raw


class Tensor:
    """Device shares of every local slot (RingTensor layout, H/ring/tensor.hpp:36-76)."""

    def __init__(self, sess: Session, h):
        self.sess = sess
        self._h = h

    def __del__(self):
        try:
            if self._h:
                N.lib().mpcg_tensor_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def meta(self):
        nd = C.c_int()
        dims = (C.c_uint64 * 8)()
        sc = C.c_int()
        N.call("mpcg_tensor_shape", self._h, C.byref(nd), dims, C.byref(sc))
        return tuple(dims[i] for i in range(nd.value)), sc.value

    @property
    def shape(self):
        return self.meta()[0]

    @property
    def scale_bits(self):
        return self.meta()[1]

    def numpy(self) -> np.ndarray:
        shape = self.shape
        out = np.empty((self.sess.n_local,) + tuple(shape), dtype=np.uint64)
        N.call("mpcg_tensor_download", self._h, _u64p(out))
        return out


def _op(name, sess, *args):
    h = C.c_void_p()
    N.call(name, sess.handle, *args, C.byref(h))
    return Tensor(sess, h)


# ---- protocol ops (reference names) -----------------------------------------------
def open_(s, x, kind="sum", tag=""):
    return _op("mpcg_open", s, x.handle, 1 if kind == "xor" else 0, _tag(tag))


def beaver_mul(s, x, y, tag="mul", chunks=1):
    return _op("mpcg_beaver_mul", s, x.handle, y.handle, _tag(tag), chunks)


def beaver_square(s, x, tag="square", chunks=1):
    return _op("mpcg_beaver_square", s, x.handle, _tag(tag), chunks)


def beaver_and(s, x, y, tag="and", chunks=1):
    return _op("mpcg_beaver_and", s, x.handle, y.handle, _tag(tag), chunks)


def beaver_matmul(s, x, y, transpose_b=False, tag="matmul", chunks=1):
    return _op("mpcg_beaver_matmul", s, x.handle, y.handle, int(transpose_b), _tag(tag), chunks)


def binary_add(s, x, y, width=64, merged=True, chunks=1, tag="badd"):
    return _op("mpcg_binary_add", s, x.handle, y.handle, width, int(merged), chunks, _tag(tag))


def a2b(s, x, chunks=1, tag="a2b"):
    return _op("mpcg_a2b", s, x.handle, chunks, _tag(tag))


def msb(s, x, chunks=1, tag="msb"):
    return _op("mpcg_msb", s, x.handle, chunks, _tag(tag))


def b2a_bit(s, b, tag="b2a", chunks=1):
    return _op("mpcg_b2a_bit", s, b.handle, _tag(tag), chunks)


def less_than(s, x, y, chunks=1, tag="lt"):
    return _op("mpcg_less_than", s, x.handle, y.handle, chunks, _tag(tag))


def truncate_shares(s, x, bits):
    return _op("mpcg_truncate", s, x.handle, bits)


def relu_shares(s, x, tag="relu"):
    return _op("mpcg_relu", s, x.handle, _tag(tag))


def max_last_dim(s, x, L, tag="max"):
    return _op("mpcg_max_last_dim", s, x.handle, L, _tag(tag))


def exp_shares(s, x, tag="exp"):
    return _op("mpcg_exp", s, x.handle, _tag(tag))


def reciprocal_shares(s, x, tag="recip"):
    return _op("mpcg_reciprocal", s, x.handle, _tag(tag))


def softmax_shares(s, x, L, tag="softmax"):
    return _op("mpcg_softmax", s, x.handle, L, _tag(tag))


def maxpool2d_shares(s, x, N_, C_, H, W, k, stride, tag="maxpool"):
    return _op("mpcg_maxpool2d", s, x.handle, N_, C_, H, W, k, stride, _tag(tag))


# ---- extensions (not in the reference; restated in oracle/mpc_oracle.py) ----
def sigmoid_shares(s, x, tag="sigmoid"):
    return _op("mpcg_sigmoid", s, x.handle, _tag(tag))


def gelu_shares(s, x, tag="gelu"):
    return _op("mpcg_gelu", s, x.handle, _tag(tag))


def inv_sqrt_shares(s, v, tag="isqrt", newton_iters=3):
    return _op("mpcg_inv_sqrt", s, v.handle, _tag(tag), newton_iters)


def layernorm_shares(s, x, d, gamma, beta, public=False, tag="ln"):
    return _op("mpcg_layernorm", s, x.handle, d, gamma.handle, beta.handle, int(public), _tag(tag))


def global_avg_pool(s, x, N_, C_, HW):
    return _op("mpcg_global_avg_pool", s, x.handle, N_, C_, HW)


def set_pair_eval(on: bool = True):
    """1-GPU mode: one thread evaluates both co-located party slots and writes each open's
    opened value once (True, default), or per-slot kernels with two payloads per open, as two
    separate parties compute (False). Values are identical; set before building executors."""
    N.call("mpcg_set_pair_eval", int(on))


def set_gemv(on: bool = True):
    """Small-M combines: fused-segment streaming kernel (True) or the tiled GEMM paths."""
    N.call("mpcg_set_gemv", int(on))


def set_gemm_mode(mode: str = "auto"):
    """Ring-GEMM engine: "simt", "tc" (tcgen05 int8 limbs wherever exact), "tc2" (as "tc" with
    one CTA per party slot only: the both-slots combine kernel off) or "auto"."""
    N.call("mpcg_set_gemm_mode", {"simt": 0, "tc": 1, "auto": 2, "tc2": 3}[mode])


def launch_count() -> int:
    """Kernels launched by libmpcg.so since load."""
    return int(N.lib().mpcg_launch_count())


KERNEL_CLASS = {"adder_round": 1, "gemm": 2, "beaver": 3, "chain": 4, "chain_reg": 5}


def draw_peak(device=0):
    """Measured dealer draw rate (splitmix64 draws / s) on `device` (mpcg_debug_draw_peak)."""
    v = C.c_double()
    N.call("mpcg_debug_draw_peak", int(device), C.byref(v))
    return v.value


def probe_start(kernel_class="adder_round"):
    N.call("mpcg_probe_start", KERNEL_CLASS[kernel_class])


def probe_stop():
    """-> (total device ms, launches, algorithmic units) of the probed kernel class."""
    ms, n, u = C.c_double(), C.c_uint64(), C.c_double()
    N.call("mpcg_probe_stop", C.byref(ms), C.byref(n), C.byref(u))
    return ms.value, n.value, u.value


class PinnedBuffer:
    """Page-locked host buffer of uint64 words (e2e host<->device copies)."""

    def __init__(self, nwords):
        p = C.c_void_p()
        N.call("mpcg_pinned_alloc", nwords * 8, C.byref(p))
        self._p = p
        self.array = np.ctypeslib.as_array(C.cast(p, N.U64P), shape=(max(nwords, 1),))[:nwords]

    def __del__(self):
        try:
            N.lib().mpcg_pinned_free(self._p)
        except Exception:
            pass


def copy_from_host(t: "Tensor", buf: PinnedBuffer):
    N.call("mpcg_tensor_copy_from_host", t.handle, buf.array.ctypes.data_as(N.U64P))


def download_into(t: "Tensor", buf: PinnedBuffer):
    N.call("mpcg_tensor_download", t.handle, buf.array.ctypes.data_as(N.U64P))


def flush_l2(s: Session):
    N.call("mpcg_session_flush_l2", s.handle)


def timer(s: Session, op: str) -> float:
    """op in start|stop|reset|read; returns accumulated device ms of completed pairs."""
    ms = C.c_double()
    code = {"start": 0, "stop": 1, "reset": 2, "read": 3}[op]
    N.call("mpcg_session_timer", s.handle, code, C.byref(ms) if op == "read" else None)
    return ms.value


# ---- TripleSource plugin (H/sharing/triple.hpp:126-307) ---------------------------
class TripleQueue:
    """Materialised 2PC triples consumed in fetch order (QueueTripleSource): recorded by a
    session's seeded dealer (offline phase) or loaded from a reference triple file."""

    def __init__(self):
        h = C.c_void_p()
        N.call("mpcg_triple_queue_create", C.byref(h))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                N.lib().mpcg_triple_queue_destroy(self._h)
        except Exception:
            pass

    def size(self):
        r, c = C.c_uint64(), C.c_uint64()
        N.call("mpcg_triple_queue_size", self._h, C.byref(r), C.byref(c))
        return {"records": r.value, "consumed": c.value}

    def rewind(self):
        N.call("mpcg_triple_queue_rewind", self._h)

    def save(self, path):
        N.call("mpcg_triple_queue_save", self._h, path.encode())

    def load(self, path):
        N.call("mpcg_triple_queue_load", self._h, path.encode())


def record_triples(s: Session, q):
    """Offline dealer: every triple `s` fetches is also materialised into `q` (None stops)."""
    N.call("mpcg_session_record_triples", s.handle, q._h if q is not None else None)


def use_triple_queue(s: Session, q):
    """Online phase: `s` consumes triples from `q` in order (None = back to the seeded dealer)."""
    N.call("mpcg_session_use_triple_queue", s.handle, q._h if q is not None else None)


def dealer_fetch(s: Session, shape_a, shape_b=None, kind="arith", matmul=False, square=False, transpose_b=False,
                 tag=""):
    """TripleSource::fetch: (a, b, c) tensors holding this session's party shares."""
    sa = np.array(shape_a, dtype=np.uint64)
    sb = np.array(shape_b if shape_b is not None else shape_a, dtype=np.uint64)
    ha, hb, hc = C.c_void_p(), C.c_void_p(), C.c_void_p()
    N.call("mpcg_dealer_fetch", s.handle, int(kind == "bin"), int(matmul), int(square), int(transpose_b), sa.size,
           _u64p(sa), sb.size, _u64p(sb), _tag(tag), C.byref(ha), C.byref(hb), C.byref(hc))
    return Tensor(s, ha), Tensor(s, hb), Tensor(s, hc)


# ---- run report (H/engine/report.hpp:25-81) --------------------------------------
def linear_tags(g: ModelGraph):
    """SecureExecutor::linear_tags (H/engine/executor.hpp:208-218): one per weight op, in
    build order; attention packs Wqkv and Wo as two ops."""
    tags = []
    for l in g.layers:
        if l.type in ("dense", "conv2d"):
            tags.append(l.name + ".mm")
        elif l.type == "attention":
            tags += [l.name + ".qkv", l.name + ".proj"]
    return tags


def _belongs(tag, prefixes):
    return any(len(tag) > len(t) and tag.startswith(t) and tag[len(t)] == "." for t in prefixes)


def party_report_fields(rows, g: ModelGraph):
    """stall_s, occupancy_s, delta_wait_s, first_delta_wait_s, linear_comm_s, linear_bytes of
    a PartyReport (H/engine/report.hpp:42-81, H/engine/bench.hpp:61-78) from trace rows."""
    tags = linear_tags(g)
    first = tags[0] if tags else ""
    hideable = [t for t in tags if t != first]
    return {"stall_s": sum(r["stall"] for r in rows),
            "occupancy_s": sum(r["occupancy"] for r in rows),
            "delta_wait_s": sum(r["stall"] for r in rows if r["tag"].endswith(".delta") and _belongs(r["tag"], hideable)),
            "first_delta_wait_s": sum(r["stall"] for r in rows if r["tag"].endswith(".delta")
                                      and _belongs(r["tag"], [first])) if first else 0.0,
            "linear_comm_s": sum(r["occupancy"] for r in rows if _belongs(r["tag"], tags)),
            "linear_bytes": sum(r["bytes"] for r in rows if _belongs(r["tag"], tags))}


def fnv1a_words(words: np.ndarray) -> int:
    a = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
    return int(N.lib().mpcg_fnv1a_words(_u64p(a), a.size))


# ---- executor ---------------------------------------------------------------------
class SecureExecutor:
    """H/engine/executor.hpp:173-205 on the GPU. ExecOptions: pipelined, chunks, threshold."""

    def __init__(self, sess: Session, g: ModelGraph, public_weights=False, pipelined=False, chunks=4,
                 chunk_threshold=2 << 20, merged_adder=True, linear_chunks=False):
        mh = C.c_void_p()
        dims = np.array(g.input, dtype=np.uint64)
        N.call("mpcg_model_create", g.name.encode(), g.frac_bits, len(g.input), _u64p(dims), C.byref(mh))
        try:
            for l in g.layers:
                N.call("mpcg_model_add_layer_ex", mh, l.name.encode(), LAYER_KINDS[l.type], l.out, l.kernel,
                       l.stride, l.pad, l.heads, int(l.bias), l.src.encode(), l.other.encode())
            eh = C.c_void_p()
            N.call("mpcg_executor_create", sess.handle, mh, int(public_weights), int(pipelined), chunks,
                   chunk_threshold, int(merged_adder), C.byref(eh))
        finally:
            N.lib().mpcg_model_destroy(mh)
        self._h = eh
        self.sess = sess
        self.graph = g
        if linear_chunks:
            # extension: the inner-layer pipeline also on conv / dense eps openings
            N.call("mpcg_executor_set_linear_chunks", eh, 1)

    def __del__(self):
        try:
            if self._h:
                N.lib().mpcg_executor_destroy(self._h)
        except Exception:
            pass

    def deal_weights(self, weights: dict, seed: int):
        """deal_weight_shares / public_weight_set (H/engine/executor.hpp:49-68), after the
        reference's check_weights (H/engine/model.hpp:366-376); the C ABI re-checks every
        tensor's element count before reading it."""
        from .model import check_weights
        check_weights(self.graph, weights)
        names = sorted(weights)
        arrs = [np.ascontiguousarray(weights[k], dtype=np.float64).reshape(-1) for k in names]
        cn = (C.c_char_p * len(names))(*[n.encode() for n in names])
        cv = (C.POINTER(C.c_double) * len(names))(*[a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs])
        counts = np.array([a.size for a in arrs], dtype=np.uint64)
        N.call("mpcg_executor_deal_weights", self._h, len(names), cn, cv, _u64p(counts), seed)

    def release_graph(self):
        """Drop the captured graph so run() and other session ops may fetch triples again."""
        N.call("mpcg_executor_release_graph", self._h)

    def run(self, x: Tensor) -> Tensor:
        h = C.c_void_p()
        N.call("mpcg_executor_run", self._h, x.handle, C.byref(h))
        return Tensor(self.sess, h)

    def capture(self, x: Tensor):
        """CUDA-graph capture of one inference reading `x` in place (run() once first)."""
        N.call("mpcg_executor_capture", self._h, x.handle)

    def replay(self) -> Tensor:
        """Next inference as one graph launch; output valid until the next replay."""
        h = C.c_void_p()
        N.call("mpcg_executor_replay", self._h, C.byref(h))
        return Tensor(self.sess, h)

    def time_layers(self, enable=True):
        N.call("mpcg_executor_time_layers", self._h, int(enable))

    def layer_times(self):
        buf = (C.c_float * 256)()
        n = C.c_int()
        N.call("mpcg_executor_layer_times", self._h, 256, buf, C.byref(n))
        return [buf[i] for i in range(min(n.value, 256))]
