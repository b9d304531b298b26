"""Inner-pipeline threshold sweep / calibration on the GPU (H/engine/bench.hpp:118-205).

`sweep_threshold` times one op (ReLU or AND) blocking vs chunked across operand sizes on
the session's own link (in-device zero-copy opens, an emulated LAN/WAN link, or NCCL),
with CUDA events on the session stream, and reports the smallest operand size where
chunking wins — the reference's calibration step ("Steps to apply").
`calibrate_threshold` returns that size in bytes, or None when chunking never wins (the
reference's SIZE_MAX), which is the expected answer for in-device opens: there is no
transfer for chunking to overlap.
"""
from __future__ import annotations

import numpy as np

from . import api

DEFAULT_SIZES = (1 << 10, 1 << 12, 1 << 14, 1 << 16, 1 << 18)


def _time_op(op, elems, chunks, link, seed, reps, device=0):
    s = api.Session(device=device, n_local=2, seed=seed, mask_seed=seed ^ 0x5309, frac_bits=16)
    if link:
        s.set_link(*link)
    s.set_pipeline(chunks, 0, True)
    rng = np.random.default_rng(seed)
    x = s.tensor(rng.integers(0, 2**63, size=(2, elems), dtype=np.uint64), 16)
    y = s.tensor(rng.integers(0, 2**63, size=(2, elems), dtype=np.uint64), 16)
    run = (lambda: api.beaver_and(s, x, y, "sweep.and", chunks)) if op == "and" else \
        (lambda: api.relu_shares(s, x, "sweep.relu"))
    run()  # warm-up (module load, pool growth)
    s.sync()
    api.timer(s, "reset")
    for _ in range(reps):
        api.timer(s, "start")
        run()
        api.timer(s, "stop")
    ms = api.timer(s, "read") / reps
    s.close()
    return ms


def sweep_threshold(op="relu", sizes=DEFAULT_SIZES, chunks=4, link=None, seed=7, reps=5, device=0,
                    margin=0.05):
    """Blocking vs chunked per operand size (bench.hpp:175-193). link=(latency_s, bytes/s, msg_s).

    The reference compares deterministic simulated clocks with a strict `<`; measured device
    times carry run-to-run noise, so chunking must win by `margin` (default 5%) to count."""
    if len(sizes) < 2:
        raise ValueError("insufficient sweep: need at least two operand sizes")
    if chunks < 2:
        raise ValueError("sweep needs chunks >= 2")
    points = []
    for elems in sizes:
        b = _time_op(op, elems, 1, link, seed, reps, device)
        c = _time_op(op, elems, chunks, link, seed, reps, device)
        wins = c < b * (1.0 - margin)
        points.append({"elems": elems, "bytes": elems * 8, "blocking_ms": b, "chunked_ms": c,
                       "chunked_wins": wins})
    # A crossover: chunking wins at this size and at every larger swept size (an isolated
    # noisy "win" below a loss does not gate chunking on).
    thr = None
    for i in range(len(points) - 1, -1, -1):
        if not points[i]["chunked_wins"]:
            break
        thr = points[i]["bytes"]
    return {"op": op, "chunks": chunks, "points": points, "threshold_bytes": thr}


def calibrate_threshold(chunks=4, link=None, seed=7, device=0):
    """bench.hpp:200-205: ReLU probe; None = chunking never won (gate it off)."""
    return sweep_threshold("relu", DEFAULT_SIZES, chunks, link, seed, 3, device)["threshold_bytes"]
