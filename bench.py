#!/usr/bin/env python
"""bench.py — 2PC private-inference latency/throughput on B200 (MPC-Pipe hot path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--model resnet18]

Workload (BASELINE.json configs[2], the largest config that fits one GPU): ResNet-18 on a
synthetic CIFAR-10 batch of 128 (3x32x32), 2PC, private weights, pipelined (inter-linear
delta prefetch + inner-layer chunked pipeline, n=4 lanes for operands >= the reference's 2 MiB
threshold), seed 1 — the reference's seeded init_weights / demo_input. A step is one secure
inference of the whole batch by both parties. N=1: both parties on cuda:0. N>=2: one party
per GPU (rank 2k <-> 2k+1 over NCCL), N/2 data-parallel pairs each on its own 128-image shard
of a 128*N/2 global batch (weak scaling; the offset-aware PRG keeps every shard word-identical
to the single-pair full-batch run).

`value` is whole-job inferences/s timed on device with CUDA events (inputs resident, L2
flushed between timed steps); `e2e` is the same metric through the public API with the input
shares copied from pinned host memory and the logit shares read back every step.
`--impl reference` times the UNMODIFIED reference (oracle/_ref/ref_driver, built from
/root/reference by oracle/Makefile) on the host cores: end to end through its bench_party for
the models it can run in seconds (MLP, LeNet-5), else an op-sum estimate from its own ops at
every layer's shape (ResNet-18 / BERT-base are not expressible in it).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2PC private-inference latency ms & inferences/s, pipelined vs blocking, 1/2/4/8 B200"
PHI = 0x9E3779B97F4A7C15
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="resnet18")
    ap.add_argument("--batch", type=int, default=0, help="per-pair batch (default: the config's)")
    ap.add_argument("--mode", default="pipelined", choices=["pipelined", "blocking"])
    ap.add_argument("--weights", default="private", choices=["private", "public"])
    ap.add_argument("--no-blocking", action="store_true", help="skip the blocking comparison pass")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--one-party-variants", action="store_true",
                    help="also time two one-party sessions on two host threads (loopback and P2P links); off by "
                         "default: a rare cross-thread stall of the eager loopback link was seen at ResNet-18 scale")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the per-slot and loopback one-party co-location measurements")
    ap.add_argument("--chunks", type=int, default=4, help="inner-layer pipeline chunk count (ExecOptions::chunks)")
    ap.add_argument("--linear-chunks", action="store_true",
                    help="inner-layer pipeline on the conv / dense layers too (eps opened in row blocks; "
                         "extension: the reference's weight_matmul is unchunked)")
    ap.add_argument("--link", default="",
                    help="emulate a LAN/WAN link between the parties, e.g. 10gbps (1.25e9 B/s, 0.1 ms) or "
                         "'<latency_s>,<bytes_per_s>'; default: the real in-device / NVLink transport")
    ap.add_argument("--threshold", default="ref",
                    help="inner-pipeline chunk threshold: ref (the reference default 2 MiB: chunking on for "
                         "operands >= 2 MiB), auto (calibrate_threshold on this link, like the reference CLI's "
                         "--threshold auto) or bytes")
    return ap.parse_args()


def pair_layout(rank, world, local_batch):
    """Rank -> 2PC pair placement: N=1 runs both parties on one GPU; N>=2 puts
    party 0/1 of pair k on ranks 2k/2k+1, each pair on its own shard of the global batch."""
    if world == 1:
        return {"pair": 0, "party": 0, "pairs": 1, "batch_offset": 0, "global_batch": local_batch, "peer": None}
    if world % 2:
        raise ValueError("--gpus must be 1 or even (one party per GPU)")
    pairs = world // 2
    pair = rank // 2
    return {"pair": pair, "party": rank % 2, "pairs": pairs, "batch_offset": pair * local_batch,
            "global_batch": pairs * local_batch, "peer": rank ^ 1}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        rows = [r.split(", ") for r in (self.out or "").strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def measure_int8_peak():
    """Dense int8 tensor throughput of this GPU: cuBLASLt IMMA via torch._int_mm on 8192^3,
    best of 5 (burst), CUDA events. Falls back to the 4.5 POPS datasheet figure."""
    try:
        import torch
        n = 8192
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(a, b)
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None else min(best, t)
        del a, b
        return 2.0 * n ** 3 / best / 1e12, "measured: torch._int_mm 8192^3 best of 5"
    except Exception as e:  # noqa: BLE001
        return 4500.0, "fallback: 4.5 POPS dense int8 datasheet (" + repr(e)[:60] + ")"


# ----------------------------------------------------------------------------- reference
# Models the reference can run end to end in seconds: timed through its own bench_party.
# Everything else (ResNet-18 and BERT-base are not expressible in it; VGG-16 takes ~10 min
# per inference) is an op-sum estimate: the reference's own ops timed at every layer's shape
# on a row sample and scaled (oracle/ref_driver.cpp cmd_opsum).
REF_E2E_MODELS = ("mlp", "lenet5", "toy_cnn", "toy_transformer")
# 1/div of every layer's rows per sample: ~5 s of CPU per step per pair on this container
OPSUM_DIV = {"resnet18": 128, "vgg16": 64, "bert_base": 48}


def ref_bench(model_path, mode, iters, weights, seed=1, port=21000):
    env = dict(os.environ, MPCPIPE_PORT_BASE=str(port))
    out = subprocess.run([REF_DRIVER, "bench", model_path, mode, str(iters), weights, str(seed)],
                         capture_output=True, text=True, env=env, timeout=900)
    if out.returncode != 0:
        raise RuntimeError("reference driver failed: " + out.stderr.strip()[-400:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def ref_opsum(model_path, weights, div, pairs, seed=1):
    out = subprocess.run([REF_DRIVER, "opsum", model_path, weights, str(div), str(pairs), str(seed)],
                         capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        raise RuntimeError("reference driver failed: " + out.stderr.strip()[-400:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def ref_pairs():
    """Concurrent 2PC pairs the host can run (the reference is single-threaded per party)."""
    return max(1, (os.cpu_count() or 2) // 2)


def reference_sample(model, model_path, g, mode, weights, iters, warmup=0, pairs=None):
    """One timed reference measurement of the workload. Returns (inferences/s, ms per inference
    batch, cpu_baseline-style description)."""
    batch = g.input[0]
    if model in REF_E2E_MODELS:
        r = ref_bench(model_path, mode, warmup + iters, weights)
        walls = r["iter_wall_s"][warmup:]
        lat = sum(walls) / len(walls)
        return batch / lat, lat * 1e3, {
            "kind": "reference", "cores": 2, "logits_hash": r["logits_hash"],
            "sample": f"{iters} timed iterations (+{warmup} warm-up) of the full workload through the reference's "
                      f"bench_party over SocketComm, one thread per party (nproc={os.cpu_count()})"}
    pairs = pairs or ref_pairs()
    div = OPSUM_DIV.get(model, 32)
    ests, walls, last = [], [], None
    for _ in range(warmup + iters):
        last = ref_opsum(model_path, weights, div, pairs)
        ests.append(last["est_latency_s"])
        walls.append(last["wall_s"])
    ests, walls = ests[warmup:], walls[warmup:]
    lat = sum(ests) / len(ests)
    top = sorted(last["layers"], key=lambda l: -l["est_s"])[:4]
    return pairs * batch / lat, lat * 1e3, {
        "kind": "reference-op-sum-estimate", "cores": 2 * pairs,
        "sample": f"{iters} samples (+{warmup} warm-up), each the reference's own ops (beaver_matmul + "
                  f"truncate_shares, relu_shares, max_last_dim, softmax_shares, ...) run at every layer's shape on "
                  f"1/{div} of its rows and scaled linearly, {pairs} concurrent 2PC pairs x 2 party threads over "
                  f"the in-memory SimComm (compute only, no link cost); {sum(walls) / len(walls):.1f} s wall per sample; "
                  f"throughput = pairs x batch / estimated latency",
        "est_latency_ms_per_pair": lat * 1e3, "top_layers_s": {l["name"]: round(l["est_s"], 3) for l in top}}


def run_reference(a, g, model_path):
    """The reference's own CPU implementation (oracle/_ref) on this host's cores."""
    v, lat_ms, cpu = reference_sample(a.model, model_path, g, a.mode, a.weights, a.steps, a.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "inferences/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": lat_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded init_weights/demo_input)",
            "config": {"workload": workload_name(g, a), "model": g.name,
                       "global_batch": g.input[0], "mode": a.mode, "weights": a.weights,
                       "transport": "reference SocketComm / SimComm in-process, parties as threads"},
            "cpu_baseline": dict(cpu, value=v, unit="inferences/s"),
            "e2e": {"value": v, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_name(g, a):
    chunked = f", inner-layer chunks {a.chunks}" if a.mode == "pipelined" and a.chunks > 1 else ""
    return f"{g.name} b{g.input[0]} 2PC {a.weights} {a.mode}{chunked}"


# ----------------------------------------------------------------------------- ours
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import api

    model_path = os.path.join(ROOT, "configs", a.model + ".json")
    g = mp.ModelGraph.from_json(model_path)
    if a.batch:
        g = g.with_batch(a.batch)
    if a.impl == "reference":
        if rank == 0:
            run_reference(a, g, model_path)
        return

    B = g.input[0]
    try:
        lay = pair_layout(rank, world, B)
    except ValueError as e:
        raise SystemExit(str(e))
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
    pairs, pair, party = lay["pairs"], lay["pair"], lay["party"]
    g_global = g.with_batch(lay["global_batch"])
    seed = 1

    # N>1 transport: NCCL send/recv between the pair's two GPUs (default), or — for a dry run of
    # the multi-process path on ONE GPU (MPCG_SAME_GPU=1; NCCL refuses two ranks on one device) —
    # the TCP socket link with every rank on cuda:0.
    same_gpu = world > 1 and os.environ.get("MPCG_SAME_GPU") == "1"
    transport = "socket" if same_gpu else "nccl"
    device = 0 if same_gpu else local_rank
    nccl_note = None
    if world > 1 and transport == "nccl":
        # every rank must be able to load NCCL before any enters ncclCommInitRank (a rank that
        # cannot would leave its peer blocked in the init); otherwise all ranks use the socket link
        try:
            mp.nccl_unique_id()
            ok = 1
        except Exception as e:  # noqa: BLE001
            ok, nccl_note = 0, f"NCCL unavailable on rank {rank}: {e}"
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if not all(oks):
            transport = "socket"
            print(f"mpcg: falling back to the socket link ({nccl_note or 'NCCL unavailable on a peer rank'})",
                  file=sys.stderr, flush=True)
    n_made = [0]

    def make_session():
        if world == 1:
            return mp.Session(device=0, n_local=2, seed=seed, mask_seed=seed ^ PHI, frac_bits=g.frac_bits)
        s = mp.Session(device=device, n_local=1, party=party, seed=seed, mask_seed=seed ^ PHI, frac_bits=g.frac_bits)
        if transport == "socket":
            port = int(os.environ.get("MASTER_PORT", "29500")) + 101 + 8 * n_made[0] + pair
            s.connect_socket("127.0.0.1", port, 300.0)
        else:
            ids = [None] * world
            uid = mp.nccl_unique_id() if party == 0 else None
            dist.all_gather_object(ids, uid)
            s.connect_nccl(ids[2 * pair], party)
        n_made[0] += 1
        s.set_shard(B, B * pairs, B * pair)
        print(f"mpcg: rank {rank}/{world} pair {pair} party {party} device {device} transport {transport} "
              f"(2-rank communicator per pair; data-parallel shard rows {B * pair}..{B * pair + B - 1} of "
              f"{B * pairs})", file=sys.stderr, flush=True)
        return s
    # one-party sessions replay CUDA graphs only when asked (MPCG_NCCL_GRAPH=1: NCCL send/recv
    # captured into the graph); the socket link is host I/O and always runs eager
    use_graph = world == 1 or (transport == "nccl" and os.environ.get("MPCG_NCCL_GRAPH") == "1")

    weights = mp.init_weights(g, seed + 11)
    x_global = mp.demo_input(g_global, seed + 12)

    link = None
    if a.link:
        if a.link.lower() in ("10gbps", "10g"):
            link = (1e-4, 1.25e9, 0.0)      # the paper's 10 Gb/s LAN
        elif a.link.lower() in ("1gbps", "1g"):
            link = (1e-3, 1.25e8, 0.0)
        else:
            lat, bw = (float(v) for v in a.link.split(","))
            link = (lat, bw, 0.0)

    NEVER = (1 << 63)
    calib = None
    if a.threshold == "auto":
        if world == 1:
            from paper_2209_13643_b200 import tuning
            calib = tuning.sweep_threshold("relu", chunks=a.chunks, link=link)
            thr = calib["threshold_bytes"] or NEVER
        else:
            thr = 2 << 20  # NCCL link: keep the reference default (calibrating needs both ranks)
    elif a.threshold == "ref":
        thr = 2 << 20
    else:
        thr = int(a.threshold)

    def setup(mode):
        s = make_session()
        if link:
            s.set_link(*link)
        ex = mp.SecureExecutor(s, g, public_weights=a.weights == "public", pipelined=mode == "pipelined",
                               chunks=a.chunks, chunk_threshold=thr, linear_chunks=a.linear_chunks)
        ex.deal_weights(weights, seed)
        x = s.deal_input(x_global, seed + 1, batch_offset=B * pair, local_batch=B)
        return s, ex, x

    def barrier(s):
        s.sync()
        if dist:
            dist.barrier()
        s.sync()

    def maxall(v):
        if not dist:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(s, ex, x, steps, warmup, graph):
        """`graph`: one CUDA-graph replay per step (the production path); else eager run()."""
        step = ex.replay if graph else (lambda: ex.run(x))
        for _ in range(warmup):
            step()
        barrier(s)
        api.timer(s, "reset")
        l0 = api.launch_count()
        with ClockSampler(local_rank) as clk:
            for _ in range(steps):
                api.flush_l2(s)           # untimed: evict L2 between timed steps
                api.timer(s, "start")
                out = step()
                api.timer(s, "stop")
            barrier(s)
        launches = api.launch_count() - l0
        ms = api.timer(s, "read")
        return maxall(ms) / steps, launches, clk.summary(), out

    def graph_ms(mode, steps, warmup):
        """A fresh session + executor in `mode`, one eager run (pipelined prologue), capture,
        then timed graph replays. Returns (ms/step, per-layer ms of the last replay)."""
        sb, exb, xb = setup(mode)
        exb.run(xb)
        exb.time_layers(True)
        if use_graph:
            exb.capture(xb)
        ms, _, _, _ = timed(sb, exb, xb, steps, warmup, graph=use_graph)
        lt = exb.layer_times()
        del exb, sb
        return ms, lt

    # ---- main arm: the requested mode
    s, ex, x = setup(a.mode)
    eager_ms, _, _, _ = timed(s, ex, x, max(3, a.steps // 4), 2, graph=False)

    # ---- roofline probes: device time of every launch of each kernel class (eager steps, CUDA
    # events on the session stream around each launch of the class)
    probes = {}
    for cls in ("adder_round", "beaver", "chain", "chain_reg", "gemm"):
        barrier(s)
        api.probe_start(cls)
        for _ in range(max(2, a.steps // 4)):
            ex.run(x)
        s.sync()
        probes[cls] = api.probe_stop()
    probe_steps = max(2, a.steps // 4)

    ex.time_layers(True)   # per-layer CUDA events recorded inside the graph
    if use_graph:
        ex.capture(x)
    ms_step, launches, clocks, out = timed(s, ex, x, a.steps, a.warmup, graph=use_graph)
    layer_ms = ex.layer_times()   # of the last timed replay
    z = out.numpy()

    # ---- e2e through the public API: pinned H2D of the input shares, one graph replay
    # (mpcg_executor_replay), D2H of the logit shares — every step
    xin_host = x.numpy()
    pin_in = api.PinnedBuffer(xin_host.size)
    pin_in.array[:] = xin_host.reshape(-1)
    pin_out = api.PinnedBuffer(z.size)
    step_api = ex.replay if use_graph else (lambda: ex.run(x))
    for _ in range(max(1, a.warmup)):
        api.copy_from_host(x, pin_in)      # the captured graph reads x in place
        api.download_into(step_api(), pin_out)
    barrier(s)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        api.copy_from_host(x, pin_in)
        api.download_into(step_api(), pin_out)
    barrier(s)
    e2e_s = maxall(time.perf_counter() - t0) / a.steps
    h2d = xin_host.size * 8
    d2h = z.size * 8
    ex.release_graph()
    del ex, s

    # ---- blocking comparison (the paper's pipelined-vs-blocking reduction, per layer)
    blocking = None
    if not a.no_blocking and a.mode == "pipelined":
        b_ms, bl = graph_ms("blocking", a.steps, a.warmup)
        blocking = {"ms_per_step": b_ms, "note": "graph replays; per-layer CUDA events inside the graph",
                    "reduction_pct": (b_ms - ms_step) / b_ms * 100.0,
                    "per_layer": [{"layer": l.name, "blocking_ms": round(bb, 4), "pipelined_ms": round(pp, 4),
                                   "reduction_pct": round((bb - pp) / bb * 100.0, 2) if bb > 0 else 0.0}
                                  for l, bb, pp in zip(g.layers, bl, layer_ms)]}

    # ---- co-location check (1 GPU): the pair-evaluated headline evaluates both parties of an
    # element in one thread and writes each opened value once. Beside it: per-slot kernels (each
    # party writes its own payload and reads the peer's, as two separate parties do) and two
    # one-party sessions on two host threads over the in-process loopback link (the exact code
    # a 2-GPU pair runs, with device copies in place of NCCL; eager launches).
    colocation = None
    if world == 1 and not a.no_variants:
        api.set_pair_eval(False)
        try:
            ps_ms, _ = graph_ms(a.mode, a.steps, a.warmup)
        finally:
            api.set_pair_eval(True)
        lb_ms = p2p_ms = None
        if a.one_party_variants:
            lb_ms = loopback_ms(mp, g, weights, x_global, a, thr, link, seed)
            p2p_ms = loopback_ms(mp, g, weights, x_global, a, thr, link, seed, kind="p2p")
        colocation = {
            "pair_evaluated": {"ms_per_step": ms_step, "inferences_per_s": B / (ms_step / 1e3),
                               "path": "one thread per element evaluates both local party slots; opened values "
                                       "written once (headline `value`)"},
            "per_slot": {"ms_per_step": ps_ms, "inferences_per_s": B / (ps_ms / 1e3),
                         "path": "mpcg_set_pair_eval(0): per-slot kernels, two payloads written and both read "
                                 "per open (MPCG_PAIR_EVAL=0 MPCG_EPS_FUSE=0); CUDA-graph replays"},
            "loopback_one_party_sessions": {"ms_per_step": lb_ms, "inferences_per_s": B / (lb_ms / 1e3) if lb_ms else None,
                                            "path": "two n_local=1 sessions (party 0, party 1) on two host threads, "
                                                    "loopback link (device copies in place of NCCL send/recv), eager "
                                                    "launches; wall clock per step after a stream sync"},
            "p2p_one_party_sessions": {"ms_per_step": p2p_ms, "inferences_per_s": B / (p2p_ms / 1e3) if p2p_ms else None,
                                       "path": "two n_local=1 sessions on two host threads over the device-flag P2P "
                                               "link (peer stores + flags), each party's inference one CUDA-graph "
                                               "replay, both parties sharing cuda:0; wall clock per step"}}
        if not a.one_party_variants:
            colocation["one_party_note"] = ("one-party variants not run (bench.py --one-party-variants); last "
                                            "measured at ResNet-18 b128: loopback 73.9 ms, P2P 62.5 ms per step "
                                            "(profiles/r02_bench.json)")

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    # ---- CPU baseline: the reference itself on this host (bounded sample)
    cpu = None
    if not a.no_cpu and os.path.exists(REF_DRIVER):
        try:
            v, lat_ms, desc = reference_sample(a.model, model_path, g, a.mode, a.weights, 1 if a.model not in
                                               REF_E2E_MODELS else 4)
            cpu = dict(desc, value=v, unit="inferences/s", ms_per_inference_batch=lat_ms)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "inferences/s", "cores": None, "kind": "reference", "sample": str(e)[:200]}
    elif not a.no_cpu:
        cpu = {"value": None, "unit": "inferences/s", "cores": None, "kind": "reference",
               "sample": "oracle/_ref/ref_driver not built (run make -C oracle where /root/reference exists)"}

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        pass
    hbm = peaks.get("hbm_gbs")
    hbm_peak = hbm or 6650.0
    int8_peak, int8_src = measure_int8_peak()
    try:  # the dealer's splitmix64 draw rate: ALU roofline of the element-by-element chain
        draw_peak = api.draw_peak(device) / 1e9
    except Exception:  # noqa: BLE001
        draw_peak = None
    # algorithmic units per class: bytes for the HBM-bound protocol rounds, ring MACs
    # for the GEMM (x36 int8 MACs = 72 int8 ops each, the limb-pair products of the tcgen05 path)
    notes = {"adder_round": "SPK level round (settle r, issue r+1). Bytes per element per party of the form that "
                            "runs: pair-evaluated (opened wire) = (2 x 32 B state in/out per slot + 32 B opened value "
                            "written + 32 B read) / 2 = 64 B; per-slot = SURVEY 8(d)'s 2 x 32 B wire + 8 x (2 in + 2 "
                            "out) = 96 B",
             "beaver": "Beaver mul/square rounds incl. fused exp/Newton chains: 2 x 16 B wire + 8 x (2 in + 1 out) "
                       "= 56 B/elem/party per mul, 32 B per square (SURVEY 8(d))",
             "chain": "persistent compare-and-select chain (ReLU/tournament): 2 x 248 B wire + 16 B in/out = "
                      "512 B/elem/party (SURVEY 8(d))",
             "chain_reg": "element-by-element compare-and-select chain (pair evaluation, in-device opens): the "
                          "adder state and opened wires stay in registers, so it is bound by the dealer's "
                          "splitmix64 draws (ALU), not HBM: 77 draws per element pair (2 mask, 65 adder: 13 "
                          "ANDs x (A, B, r_A, r_B, r_C), 5 b2a, 5 multiply) against the measured draw rate "
                          "(mpcg_debug_draw_peak: a full grid of independent draw streams); the opens are "
                          "still posted and accounted per round",
             "gemm": "ring GEMM main kernel: 72 int8 ops per ring MAC (36 limb-pair MACs); ring MACs = 3 MKN (party 0, "
                     "dealer C online) + 2 MKN (party 1) per private linear layer; weight packing excluded; the "
                     "both-slots kernel (gemm_tc3.cu) also generates the opened E = x0 + x1 - A in its producers "
                     "for convolutions (deferred eps), so its time includes that build"}
    rooflines = []
    for cls, (p_ms, p_launches, p_units) in probes.items():
        if p_launches == 0 or p_ms <= 0:
            continue
        if cls == "gemm":
            ach = 72.0 * p_units / (p_ms / 1e3) / 1e12
            r = {"kernel": cls, "bound": "tensor", "achieved": ach, "peak": int8_peak, "unit": "TOP/s (int8)",
                 "frac": ach / int8_peak, "peak_source": int8_src}
        elif cls == "chain_reg":
            if not draw_peak:
                continue
            ach = p_units / (p_ms / 1e3) / 1e9
            r = {"kernel": cls, "bound": "alu", "achieved": ach, "peak": draw_peak, "unit": "Gdraws/s",
                 "frac": ach / draw_peak, "peak_source": "measured: mpcg_debug_draw_peak (splitmix64 draw rate)"}
        else:
            ach = (p_units / 1e9) / (p_ms / 1e3)
            r = {"kernel": cls, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                 "frac": ach / hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "fallback"}
        r.update({"launches": p_launches, "device_ms_per_step": p_ms / probe_steps,
                  "avg_launch_us": p_ms * 1e3 / p_launches, "units_per_launch": p_units / p_launches,
                  "traffic": (traffic.get(a.model, {}).get(cls) or {}).get("dram_bytes_per_launch"),
                  "note": notes[cls]})
        # the ncu-captured launches are specific ones (e.g. conv1's ReLU at 8.4M elements), not the
        # step's average launch: their own algorithmic bytes give the comparable ratio
        t = traffic.get(a.model, {}).get(cls) or {}
        if t.get("algorithmic_bytes_per_launch"):
            r["traffic_captured"] = {k: t[k] for k in ("dram_bytes_per_launch", "algorithmic_bytes_per_launch",
                                                      "launches") if k in t}
            r["traffic_captured"]["ratio"] = t["dram_bytes_per_launch"] / t["algorithmic_bytes_per_launch"]
        rooflines.append(r)
    rooflines.sort(key=lambda r: -r["device_ms_per_step"])
    roof = dict(rooflines[0]) if rooflines else None  # the dominant class of the step
    if roof:
        roof["share_of_probed_ms"] = roof["device_ms_per_step"] / sum(r["device_ms_per_step"] for r in rooflines)

    value = B * pairs / (ms_step / 1e3)
    dec = (z.sum(axis=0) if world == 1 else z[0]).reshape(-1)
    line = {
        "metric": METRIC, "value": value, "unit": "inferences/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: the reference's seeded init_weights(seed 12) / demo_input(seed 13), shares dealt on host",
        "config": {"workload": workload_name(g, a), "model": g.name, "global_batch": B * pairs,
                   "pairs": pairs, "parties_per_gpu": 2 if world == 1 else 1, "mode": a.mode, "weights": a.weights,
                   "frac_bits": g.frac_bits, "chunks": a.chunks, "linear_chunks": a.linear_chunks,
                   "chunk_threshold_bytes": None if thr == NEVER else thr,
                   "chunk_threshold_source": a.threshold,
                   "calibration": calib,
                   "l2": "flushed between timed steps (256 MiB memset, untimed)",
                   "transport": ("in-device zero-copy opens" if world == 1 else
                                 "NCCL send/recv over NVLink" if transport == "nccl" else
                                 "TCP socket link, all ranks on cuda:0 (MPCG_SAME_GPU=1 dry run)")
                   + (f" + emulated link latency {link[0]} s, {link[1]:.3g} B/s" if link else ""),
                   "kernels_per_step": launches / a.steps,
                   "execution": ("one CUDA-graph replay per step (whole 2PC inference, both parties)" if world == 1
                                 else "one CUDA-graph replay per step per party" if use_graph
                                 else "eager launches (one-party sessions; MPCG_NCCL_GRAPH=1 captures NCCL)"),
                   "eager_ms_per_step": eager_ms,
                   "logits_hash_slot0": mp.fnv1a_words(dec) if world == 1 else None,
                   "blocking": blocking,
                   "colocation": colocation},
        "roofline": roof,
        "rooflines": rooflines,
        "cpu_baseline": cpu,
        "e2e": {"value": B * pairs / e2e_s, "unit": "inferences/s", "ms_per_step": e2e_s * 1e3,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "pinned host input shares -> mpcg_tensor_copy_from_host -> "
                        + ("mpcg_executor_replay (the captured inference)" if use_graph else "mpcg_executor_run")
                        + " -> mpcg_tensor_download of the logit shares; wall clock"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def loopback_ms(mp, g, weights, x_global, a, thr, link, seed, kind="loopback"):
    """Two single-party sessions on cuda:0 driven by two host threads, linked in-process: the
    loopback link (eager launches) or the device-flag P2P link (each party one graph replay)."""
    import threading
    sess = [mp.Session(device=0, n_local=1, party=p, seed=seed, mask_seed=seed ^ PHI, frac_bits=g.frac_bits)
            for p in (0, 1)]
    if kind == "p2p":
        sess[0].connect_p2p(sess[1])
    else:
        sess[0].connect_loopback(sess[1])
    if link:
        for s in sess:
            s.set_link(*link)
    steps = max(2, min(a.steps, 8))
    walls, err = [0.0, 0.0], []
    go = threading.Barrier(2)

    def party(p):
        try:
            s = sess[p]
            ex = mp.SecureExecutor(s, g, public_weights=a.weights == "public", pipelined=a.mode == "pipelined",
                                   chunks=a.chunks, chunk_threshold=thr, linear_chunks=a.linear_chunks)
            ex.deal_weights(weights, seed)
            x = s.deal_input(x_global, seed + 1)
            if kind == "p2p":
                ex.run(x)
                ex.capture(x)
                step = ex.replay
            else:
                step = lambda: ex.run(x)  # noqa: E731
            for _ in range(2):
                step()
            s.sync()
            go.wait()
            t0 = time.perf_counter()
            for _ in range(steps):
                step()
            s.sync()
            walls[p] = (time.perf_counter() - t0) / steps
            del ex
        except Exception as e:  # noqa: BLE001
            err.append(repr(e))
            go.abort()

    th = [threading.Thread(target=party, args=(p,)) for p in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise RuntimeError(kind + " measurement failed: " + err[0])
    return max(walls) * 1e3


if __name__ == "__main__":
    main()
