"""CPU, world_size 2 over gloo: the one-party-per-process path (what an n_local=1 session
does on each GPU of a pair) reproduces the reference's per-party shares.

Each rank holds ONE party's shares, builds its own payloads, exchanges them over a real
2-process transport (torch.distributed gloo, standing in for NCCL send/recv) and combines
locally — the exact dataflow of Session::post/wait with n_local=1. Results are compared
word for word with the reference's golden fixtures. Also checks the data-parallel
rank -> (pair, party, batch offset) layout used by bench.py for 4/8 GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Wire:
    """Open/reveal over gloo: every party contributes its payload, reduction local."""

    def __init__(self):
        self.bytes = 0
        self.collectives = 0
        self.p2p = 0

    def _gather(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64).copy())
        out = [torch.empty_like(t) for _ in range(2)]
        dist.all_gather(out, t)
        return [o.numpy().view(np.uint64) for o in out]

    def reveal(self, a, kind):
        self.bytes += a.size * 8
        self.collectives += 1
        g = self._gather(a)
        return (g[0] + g[1]) if kind == "sum" else (g[0] ^ g[1])

    def exchange(self, a):  # p2p send_to/recv_from of the peer
        self.bytes += a.size * 8
        self.p2p += 1
        g = self._gather(a)
        return g[1 - dist.get_rank()]


def party_mul(p, x, y, t, w):
    a, b, c = t[p]
    ed = w.reveal(np.concatenate([x.reshape(-1) - a.reshape(-1), y.reshape(-1) - b.reshape(-1)]), "sum")
    n = x.size
    e, d = ed[:n].reshape(x.shape), ed[n:].reshape(x.shape)
    z = c + (e * b + d * a)
    return z + e * d if p == 0 else z


def party_adder(p, x, y, O, dealer, tag, w):
    levels, ins, outs, mults, _ = O.SPK64
    n = x.size
    t = dealer.fetch(O.TripleSpec.elementwise("bin", x.shape), tag + ".g")
    a, b, c = t[p]
    ed = w.reveal(np.concatenate([(x ^ a).reshape(-1), (y ^ b).reshape(-1)]), "xor")
    e, d = ed[:n].reshape(x.shape), ed[n:].reshape(x.shape)
    s = c ^ (e & b) ^ (d & a)
    if p == 0:
        s = s ^ (e & d)
    pp = x ^ y
    p_orig = pp.copy()
    U = np.uint64
    for i in range(levels):
        t = dealer.fetch(O.TripleSpec.elementwise("bin", (2,) + x.shape), f"{tag}.l{i}")
        a, b, c = t[p]
        inn, out, mult = U(ins[i]), U(outs[i]), U(mults[i])
        p0 = pp & out
        pay = np.concatenate([(p0 ^ a[0]).reshape(-1), (p0 ^ a[1]).reshape(-1),
                              (((s & inn) * mult) ^ b[0]).reshape(-1), (((pp & inn) * mult) ^ b[1]).reshape(-1)])
        r = w.reveal(pay, "xor")
        e0, e1, d0, d1 = (r[k * n:(k + 1) * n].reshape(x.shape) for k in range(4))
        z0 = c[0] ^ (e0 & b[0]) ^ (d0 & a[0])
        z1 = c[1] ^ (e1 & b[1]) ^ (d1 & a[1])
        if p == 0:
            z0, z1 = z0 ^ (e0 & d0), z1 ^ (e1 & d1)
        s = s ^ z0
        pp = (pp & ~out) ^ z1
    return p_orig ^ (s << U(1))


def party_relu(p, x, O, dealer, mask_rng, tag, w):
    r = mask_rng.take(x.size).reshape(x.shape)
    keep = x ^ r
    peer_r = w.exchange(r)
    xs, ys = (keep, peer_r) if p == 0 else (peer_r, keep)
    bits = party_adder(p, xs, ys, O, dealer, tag + ".msb.add1", w) >> np.uint64(63)
    mine = bits & np.uint64(1)
    zero = np.zeros_like(mine)
    acc, bq = (mine, zero) if p == 0 else (zero, mine)
    prod = party_mul(p, acc, bq, dealer.fetch(O.TripleSpec.elementwise("arith", x.shape), tag + ".b2a.m1"), w)
    cbit = (acc + bq) - (prod + prod)
    xc = party_mul(p, x, cbit, dealer.fetch(O.TripleSpec.elementwise("arith", x.shape), tag + ".gate"), w)
    return x - xc


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from oracle import mpc_oracle as O
        g = np.load(os.path.join(ROOT, "tests", "golden", "ops.npz"))
        G = {k.replace("__", "/"): g[k] for k in g.files}
        res = {}
        # beaver_mul (seed 11 -> dealer 12)
        w = Wire()
        d = O.SeededDealer(12)
        x, y = G[f"mul_c1/x{rank}"], G[f"mul_c1/y{rank}"]
        z = party_mul(rank, x, y, d.fetch(O.TripleSpec.elementwise("arith", x.shape), "mul"), w)
        res["mul"] = bool(np.array_equal(z.reshape(-1), G[f"mul_c1/z{rank}"].reshape(-1)))
        # relu (seed 18 -> dealer 19, mask CounterRng(20, party))
        w = Wire()
        d = O.SeededDealer(19)
        x = G[f"relu/x{rank}"]
        z = party_relu(rank, x, O, d, O.CounterRng(20, rank), "relu", w)
        res["relu"] = bool(np.array_equal(z.reshape(-1), G[f"relu/z{rank}"].reshape(-1)))
        st = [int(v) for v in G["relu/stats"]]
        res["relu_traffic"] = [w.bytes, w.collectives, w.p2p] == st
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_process_parties_reproduce_reference_shares():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert out[r] == {"mul": True, "relu": True, "relu_traffic": True}, out


def test_dp_pair_layout():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    # 8 GPUs = 4 pairs; rank 2k <-> 2k+1; each pair a 64-row shard of a 256-row batch
    layout = [bench.pair_layout(r, 8, 64) for r in range(8)]
    assert [l["pair"] for l in layout] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert [l["party"] for l in layout] == [0, 1] * 4
    assert [l["batch_offset"] for l in layout] == [0, 0, 64, 64, 128, 128, 192, 192]
    assert all(l["global_batch"] == 256 and l["peer"] == (r ^ 1) for r, l in enumerate(layout))
    assert bench.pair_layout(0, 1, 64) == {"pair": 0, "party": 0, "pairs": 1, "batch_offset": 0,
                                           "global_batch": 64, "peer": None}
    with pytest.raises(ValueError):
        bench.pair_layout(0, 3, 64)
