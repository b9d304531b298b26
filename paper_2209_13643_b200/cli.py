"""mpcpipe_bench on the GPU: `python -m paper_2209_13643_b200.cli run|verify|sweep_threshold`.

Mirrors the reference CLI (P/tools/mpcpipe_bench.cpp:508-579) — the same subcommands, flags,
defaults, unit parsing and report.json schema 1 (H/engine/report.hpp:104-140) — with the
secure inference running on a B200 through libmpcg.so. Both parties of the 2PC pair run on
one GPU (in-device opens); `--latency/--bandwidth` emulate the link (the reference's sim
backend link model, H/transport/config.hpp:41-43) with the comm-stream token bucket, and
`--backend device` ignores them. Per-iteration times are CUDA-event device times; the report
adds per-layer rows. 3PC is out of scope (BASELINE is 2PC).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import _native as N, api, tuning
from .model import CONFIG_DIR, ModelGraph, check_weights, demo_input, init_weights, load_weights, plaintext_forward

PHI = 0x9E3779B97F4A7C15


def _unit(text, what, units):
    t = text.strip()
    i = 0
    while i < len(t) and (t[i].isdigit() or t[i] in ".+-eE"):
        # stop at an 'e' that starts a unit rather than an exponent
        if t[i] in "eE" and (i + 1 >= len(t) or not (t[i + 1].isdigit() or t[i + 1] in "+-")):
            break
        i += 1
    try:
        v = float(t[:i])
    except ValueError:
        raise N.ConfigError(f"bad {what}: {text}") from None
    unit = t[i:].lower()
    if not unit:
        return v
    if unit not in units:
        raise N.ConfigError(f"bad {what} unit in: {text}")
    return v * units[unit]


def parse_latency(text):
    v = _unit(text, "latency", {"s": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9})
    if v < 0:
        raise N.ConfigError("latency must be >= 0")
    return v


def parse_bandwidth(text):
    v = _unit(text, "bandwidth", {"bps": 1.0, "b/s": 1.0, "kbps": 1e3, "kb/s": 1e3, "mbps": 1e6, "mb/s": 1e6,
                                  "gbps": 1e9, "gb/s": 1e9})
    if v <= 0:
        raise N.ConfigError("bandwidth must be > 0")
    return v


def parse_threshold(text):
    v = _unit(text, "threshold", {"b": 1.0, "k": 1024.0, "kb": 1024.0, "kib": 1024.0, "m": 1 << 20, "mb": 1 << 20,
                                  "mib": 1 << 20})
    if v < 0:
        raise N.ConfigError("threshold must be >= 0")
    return int(v)


def resolve_model(name):
    aliases = {"transformer-toy": "toy_transformer", "toy-transformer": "toy_transformer", "cnn-toy": "toy_cnn",
               "toy-cnn": "toy_cnn"}
    name = aliases.get(name, name)
    if "/" in name or name.endswith(".json"):
        return ModelGraph.from_json(name)
    if not os.path.exists(os.path.join(CONFIG_DIR, name + ".json")):
        raise N.ConfigError("unknown builtin model: " + name)
    return ModelGraph.from_json(name)


def _link(a):
    if a.backend == "device":
        return None
    return (parse_latency(a.latency), parse_bandwidth(a.bandwidth), 0.0)


def _spec(a):
    if a.parties != 2:
        raise N.ConfigError("only 2 parties are supported on the GPU path (3PC is out of scope)")
    g = resolve_model(a.model)
    w = load_weights(a.weights_file) if a.weights_file else init_weights(g, a.seed + 11)
    check_weights(g, w)
    x = demo_input(g, a.seed + 12)
    return g, w, x


def run_one_mode(g, w, x, a, mode, threshold):
    """H/engine/bench.hpp:36-79 for both parties: deal shares, `iterations` timed inferences,
    open the logits; per-iteration CUDA-event device seconds per party."""
    s = api.Session(device=a.device, n_local=2, seed=a.seed, mask_seed=a.seed ^ PHI, frac_bits=g.frac_bits)
    link = _link(a)
    if link:
        s.set_link(*link)
    ex = api.SecureExecutor(s, g, public_weights=a.weights == "public", pipelined=mode == "pipelined",
                            chunks=a.chunks, chunk_threshold=threshold)
    ex.deal_weights(w, a.seed)
    xin = s.deal_input(x, a.seed + 1)
    ex.time_layers(True)
    iters, layer_ms = [], np.zeros(len(g.layers))
    out = None
    st0 = s.stats(0)
    s.trace(True)
    for _ in range(a.iterations):
        api.timer(s, "reset")
        api.timer(s, "start")
        out = ex.run(xin)
        api.timer(s, "stop")
        iters.append(api.timer(s, "read") / 1e3)
        layer_ms += np.array(ex.layer_times())
    st1 = s.stats(0)
    z = out.numpy()
    opened = (z[0] + z[1]).reshape(-1)
    logits = opened.view(np.int64).astype(np.float64) * 2.0 ** -g.frac_bits
    rows = s.trace_rows()
    fields = api.party_report_fields(rows, g)
    parties = []
    for p in (0, 1):  # both parties' collectives are the session's rows (same order, same bytes)
        st = s.stats(p)
        parties.append(dict({"party": p, "iter_wall_s": iters, "wall_s": float(sum(iters)),
                             "bytes_sent": st["bytes_sent"] - st0["bytes_sent"],
                             "collectives": st["collectives"] - st0["collectives"],
                             "p2p_sends": st["p2p_sends"] - st0["p2p_sends"]}, **fields))
    rep = {"schema": 1, "model": g.name, "mode": mode, "weights": a.weights,
           "session": {"n_parties": 2, "backend": a.backend, "latency_s": link[0] if link else 0.0,
                       "bandwidth_bps": link[1] if link else None, "seed": a.seed, "device": a.device},
           "chunks": a.chunks if mode == "pipelined" else 1,
           "chunk_threshold": threshold if mode == "pipelined" else 0, "iterations": a.iterations,
           "wall_s": float(sum(iters)), "logit_shape": list(g.shapes()[-1]), "logits": logits.tolist(),
           "logits_hash": "0x%016x" % api.fnv1a_words(opened),
           "bytes_sent_per_iteration": (st1["bytes_sent"] - st0["bytes_sent"]) / a.iterations,
           "layers": [{"name": l.name, "type": l.type, "mean_ms": float(t / a.iterations)}
                      for l, t in zip(g.layers, layer_ms)],
           "parties": parties}
    del ex
    s.close()
    return rep


def check_oracle(g, w, x, rep, tol):
    ref = plaintext_forward(g, w, x).reshape(-1)
    err = np.abs(np.asarray(rep["logits"]) - ref)
    return {"mode": rep["mode"], "max_abs_err": float(err.max()), "argmax": int(err.argmax()), "tolerance": tol,
            "pass": bool(err.max() <= tol)}


def cmd_run(a):
    g, w, x = _spec(a)
    os.makedirs(a.out, exist_ok=True)
    thr = 2 << 20  # library default (H/engine/executor.hpp:28-36)
    if a.threshold == "auto":
        t = tuning.calibrate_threshold(a.chunks, _link(a), device=a.device)
        if t is None:
            print("calibrated threshold: chunking never wins at this latency; inner pipeline stays off")
            thr = 1 << 62
        else:
            print(f"calibrated threshold: {t} bytes")
            thr = t
    elif a.threshold:
        thr = parse_threshold(a.threshold)
    modes = ["blocking", "pipelined"] if a.mode == "both" else [a.mode]
    reps = [run_one_mode(g, w, x, a, m, thr) for m in modes]
    checks = [check_oracle(g, w, x, r, a.tolerance) for r in reps]
    out = {"schema": 1, "runs": reps, "oracle": checks}
    text = []
    for r, c in zip(reps, checks):
        text.append(f"model {r['model']}  mode {r['mode']}  weights {r['weights']}  iterations {r['iterations']}\n"
                    f"  wall_s {r['wall_s']:.6f}  per-iteration {r['wall_s'] / r['iterations'] * 1e3:.3f} ms  "
                    f"bytes/iter {r['bytes_sent_per_iteration']:.0f}  hash {r['logits_hash']}\n"
                    f"replica check: max |err| = {c['max_abs_err']:.3e} at logit {c['argmax']} "
                    f"(tolerance {c['tolerance']}) -> {'pass' if c['pass'] else 'FAIL'}\n")
    if len(reps) == 2:
        b, p = reps
        cmp = {"wall_s": {"blocking": b["wall_s"], "pipelined": p["wall_s"],
                          "reduction_pct": (b["wall_s"] - p["wall_s"]) / b["wall_s"] * 100},
               "bytes_sent": {"blocking": b["parties"][0]["bytes_sent"], "pipelined": p["parties"][0]["bytes_sent"]},
               "hashes_equal": b["logits_hash"] == p["logits_hash"],
               "per_layer": [{"name": lb["name"], "blocking_ms": lb["mean_ms"], "pipelined_ms": lp["mean_ms"],
                              "reduction_pct": (lb["mean_ms"] - lp["mean_ms"]) / lb["mean_ms"] * 100
                              if lb["mean_ms"] > 0 else 0.0} for lb, lp in zip(b["layers"], p["layers"])]}
        out["comparison"] = cmp
        text.append(f"pipelined vs blocking: {cmp['wall_s']['reduction_pct']:.2f}% "
                    f"({'hashes equal' if cmp['hashes_equal'] else 'OUTPUT HASH MISMATCH'})\n")
    with open(os.path.join(a.out, "report.json"), "w") as f:
        json.dump(out, f, indent=2)
    with open(os.path.join(a.out, "report.txt"), "w") as f:
        f.write("\n".join(text))
    print("\n".join(text))
    if len(reps) == 2 and not out["comparison"]["hashes_equal"]:
        print("FAIL: blocking and pipelined output hashes differ", file=sys.stderr)
        return 1
    if not all(c["pass"] for c in checks):
        print("FAIL: MPC output deviates from the plaintext replica beyond tolerance", file=sys.stderr)
        return 1
    return 0


def cmd_verify(a):
    a.backend, a.mode, a.iterations = "device", "blocking", 1
    g, w, x = _spec(a)
    r = run_one_mode(g, w, x, a, "blocking", 0)
    c = check_oracle(g, w, x, r, a.tolerance)
    print(f"model {g.name}  parties {a.parties}  weights {a.weights}")
    print(f"max |MPC - replica| = {c['max_abs_err']:.6e} at logit {c['argmax']} (tolerance {a.tolerance})")
    print("verify PASS" if c["pass"] else "verify FAIL")
    return 0 if c["pass"] else 1


def cmd_sweep(a):
    sizes = [int(v) for v in a.sizes.split(",") if v]
    r = tuning.sweep_threshold(a.op, sizes, a.chunks, _link(a), seed=a.seed, device=a.device)
    print(f"op {r['op']}  chunks {r['chunks']}  parties 2  backend {a.backend}")
    print("  elems      bytes        blocking_ms  chunked_ms   winner")
    for p in r["points"]:
        print(f"  {p['elems']:<10d} {p['bytes']:<12d} {p['blocking_ms']:<12.4f} {p['chunked_ms']:<12.4f} "
              f"{'chunked' if p['chunked_wins'] else 'blocking'}")
    if r["threshold_bytes"] is not None:
        print(f"recommended threshold: {r['threshold_bytes']} bytes")
    else:
        print("chunking never won; threshold = inf (keep the inner pipeline off)")
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "sweep.json"), "w") as f:
        json.dump(r, f, indent=2)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="mpcpipe_bench", description="MPC pipeline inference benchmark (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def net(c):
        c.add_argument("--parties", type=int, default=2, choices=[2, 3])
        c.add_argument("--latency", default="1ms")
        c.add_argument("--bandwidth", default="1GBps")
        c.add_argument("--seed", type=int, default=1)
        c.add_argument("--chunks", type=int, default=4)
        c.add_argument("--out", default=".")
        c.add_argument("--backend", default="sim", choices=["sim", "device"],
                       help="sim: emulate --latency/--bandwidth between the parties; device: in-device opens")
        c.add_argument("--device", type=int, default=0)

    r = sub.add_parser("run", help="run blocking/pipelined inference and report")
    net(r)
    r.add_argument("--model", default="toy_transformer")
    r.add_argument("--mode", default="both", choices=["blocking", "pipelined", "both"])
    r.add_argument("--weights", default="private", choices=["private", "public"])
    r.add_argument("--weights-file", default="", help="MPCW weights (H/engine/model.hpp:277-364)")
    r.add_argument("--threshold", default="")
    r.add_argument("--iterations", type=int, default=50)
    r.add_argument("--tolerance", type=float, default=2.0 ** -6)
    v = sub.add_parser("verify", help="check MPC output against the plaintext replica")
    net(v)
    v.add_argument("--model", default="toy_transformer")
    v.add_argument("--weights", default="private", choices=["private", "public"])
    v.add_argument("--weights-file", default="")
    v.add_argument("--tolerance", type=float, default=2.0 ** -6)
    sw = sub.add_parser("sweep_threshold", aliases=["sweep-threshold"], help="blocking vs chunked across sizes")
    net(sw)
    sw.add_argument("--op", default="relu", choices=["relu", "and"])
    sw.add_argument("--sizes", default="1024,4096,16384,65536,262144")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            if a.iterations < 1:
                raise N.ConfigError("iterations must be >= 1")
            return cmd_run(a)
        if a.cmd == "verify":
            return cmd_verify(a)
        return cmd_sweep(a)
    except (N.Error, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
