"""GPU: the two parties in two PROCESSES, one single-party session each (what a 2-GPU pair
or two hosts run), linked by the TCP socket link (the reference's SocketComm,
H/transport/socket.hpp) — here both processes share cuda:0.

Every kernel runs with one local slot and reads the peer's payload from its own inbox; the
pipelined wrap-around delta crosses processes. The per-party output shares must equal the
reference's own (tests/golden) word for word, and a desynchronised collective must fail in
both processes with ProtocolError.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PARTY = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2209_13643_b200 as mp
party, port, model, mode, weights, iters, out, case = (sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5],
                                                       sys.argv[6], sys.argv[7], sys.argv[8], sys.argv[9])
party, port, iters = int(party), int(port), int(iters)
PHI = 0x9E3779B97F4A7C15
res = {"party": party}
try:
    if case == "model":
        g = mp.ModelGraph.from_json(model)
        s = mp.Session(device=0, n_local=1, party=party, seed=1, mask_seed=1 ^ PHI, frac_bits=g.frac_bits)
        s.connect_socket("127.0.0.1", port, 120.0)
        ex = mp.SecureExecutor(s, g, public_weights=weights == "public", pipelined=mode == "pipelined")
        ex.deal_weights(mp.init_weights(g, 12), 1)
        x = s.deal_input(mp.demo_input(g, 13), 2)
        for _ in range(iters):
            z = ex.run(x)
        np.save(out, z.numpy()[0])
        res["stats"] = s.stats(0)
    else:  # desync: party 1 issues a different collective at the same sequence number
        s = mp.Session(device=0, n_local=1, party=party, seed=5, mask_seed=6, frac_bits=16)
        s.connect_socket("127.0.0.1", port, 120.0)
        x = s.tensor(np.arange(16, dtype=np.uint64).reshape(1, 16), 16)
        mp.beaver_mul(s, x, x, "mul" if party == 0 else "other")
        s.sync()
    res["ok"] = True
except mp.Error as e:
    res["error"] = type(e).__name__
    res["message"] = str(e)
print("RESULT " + json.dumps(res), flush=True)
"""


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run_two(tmp_path, case, model="", mode="blocking", weights="private", iters=1):
    port = _free_port()
    procs = []
    for p in (0, 1):
        out = str(tmp_path / f"z{p}.npy")
        procs.append(subprocess.Popen([sys.executable, "-c", PARTY, ROOT, str(p), str(port), model, mode, weights,
                                       str(iters), out, case], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    res = []
    for pr in procs:
        try:
            so, se = pr.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("a party process hung")
        lines = [l for l in so.splitlines() if l.startswith("RESULT ")]
        assert lines, se[-2000:]
        res.append(json.loads(lines[-1][7:]))
    return res


@pytest.mark.parametrize("name,mode,weights,it", [
    ("mlp", "pipelined", "private", 2), ("lenet5", "pipelined", "private", 1),
    ("toy_transformer", "blocking", "public", 1)])
def test_two_processes_match_reference(tmp_path, name, mode, weights, it):
    m = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}_{mode}_{weights}_it{it}.npz"))
    res = _run_two(tmp_path, "model", os.path.join(ROOT, "configs", name + ".json"), mode, weights, it)
    assert all(r.get("ok") for r in res), res
    z0, z1 = np.load(tmp_path / "z0.npy"), np.load(tmp_path / "z1.npy")
    assert np.array_equal(z0.reshape(-1), m["z0"].reshape(-1)), "party 0 share differs"
    assert np.array_equal(z1.reshape(-1), m["z1"].reshape(-1)), "party 1 share differs"
    assert res[0]["stats"] == res[1]["stats"]


def test_two_processes_desync_raises_protocol_error(tmp_path):
    res = _run_two(tmp_path, "desync")
    assert [r.get("error") for r in res] == ["ProtocolError", "ProtocolError"], res
