#!/usr/bin/env python
"""bench.py — 2PC private-inference latency/throughput on B200 (MPC-Pipe hot path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--model lenet5]

Workload (BASELINE.json configs[1]): LeNet-5 on a synthetic 28x28 batch of 64, 2PC,
private weights, inter-linear-layer pipeline on (pipelined mode), seed 1 — the
reference's seeded init_weights / demo_input. A step is one secure inference of the
whole batch by both parties. N=1: both parties on cuda:0. N>=2: one party per GPU
(rank 2k <-> 2k+1 over NCCL), N/2 data-parallel pairs each on its own 64-row shard
of a 64*N/2 global batch (weak scaling; offset-aware PRG keeps every shard
word-identical to the single-pair full-batch run).

`value` is whole-job inferences/s timed on device with CUDA events (inputs resident,
L2 flushed between timed steps); `e2e` is the same metric through the public API with
the input shares copied from pinned host memory and the logit shares read back every
step. `--impl reference` times the UNMODIFIED reference (oracle/_ref/ref_driver, built
from /root/reference by oracle/Makefile) on the host cores on the same workload.
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
    ap.add_argument("--model", default="lenet5")
    ap.add_argument("--batch", type=int, default=0, help="per-pair batch (default: the config's)")
    ap.add_argument("--mode", default="pipelined", choices=["pipelined", "blocking"])
    ap.add_argument("--weights", default="private", choices=["private", "public"])
    ap.add_argument("--no-blocking", action="store_true", help="skip the blocking comparison pass")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--link", default="",
                    help="emulate a LAN/WAN link between the parties, e.g. 10gbps (1.25e9 B/s, 0.1 ms) or "
                         "'<latency_s>,<bytes_per_s>'; default: the real in-device / NVLink transport")
    ap.add_argument("--threshold", default="auto",
                    help="inner-pipeline chunk threshold: auto (calibrate_threshold on this link, like the "
                         "reference CLI's --threshold auto), ref (the reference default 2 MiB) or bytes")
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
def ref_bench(model_path, mode, iters, weights, seed=1, port=21000):
    env = dict(os.environ, MPCPIPE_PORT_BASE=str(port))
    out = subprocess.run([REF_DRIVER, "bench", model_path, mode, str(iters), weights, str(seed)],
                         capture_output=True, text=True, env=env, timeout=900)
    if out.returncode != 0:
        raise RuntimeError("reference driver failed: " + out.stderr.strip()[-400:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(a, g, model_path):
    """The reference's own CPU implementation (oracle/_ref) on this host's cores."""
    batch = g.input[0]
    r = ref_bench(model_path, a.mode, a.warmup + a.steps, a.weights)
    walls = r["iter_wall_s"][a.warmup:]
    lat = sum(walls) / len(walls)
    v = batch / lat
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "inferences/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": lat * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded init_weights/demo_input)",
            "config": {"workload": f"{g.name} b{batch} 2PC {a.weights} {a.mode}", "model": g.name,
                       "global_batch": batch, "mode": a.mode, "weights": a.weights,
                       "transport": "reference SocketComm over loopback, parties as threads",
                       "logits_hash": r["logits_hash"], "bytes_sent_per_party": r["bytes_sent"]},
            "cpu_baseline": {"value": v, "unit": "inferences/s", "cores": 2, "kind": "reference",
                             "sample": f"{a.steps} timed iterations (+{a.warmup} warm-up) of the full workload, "
                                       "one thread per party"},
            "e2e": {"value": v, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
        dist.init_process_group("gloo")
    pairs, pair, party = lay["pairs"], lay["pair"], lay["party"]
    g_global = g.with_batch(lay["global_batch"])
    seed = 1

    def make_session():
        if world == 1:
            s = mp.Session(device=0, n_local=2, seed=seed, mask_seed=seed ^ PHI, frac_bits=g.frac_bits)
        else:
            s = mp.Session(device=local_rank, n_local=1, party=party, seed=seed, mask_seed=seed ^ PHI,
                           frac_bits=g.frac_bits)
            ids = [None] * world
            uid = mp.nccl_unique_id() if party == 0 else None
            dist.all_gather_object(ids, uid)
            s.connect_nccl(ids[2 * pair], party)
            s.set_shard(B, B * pairs, B * pair)
        return s

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
            calib = tuning.sweep_threshold("relu", chunks=4, link=link)
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
                               chunk_threshold=thr)
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

    # ---- main arm: the requested mode
    s, ex, x = setup(a.mode)
    eager_ms, _, _, _ = timed(s, ex, x, max(3, a.steps // 4), 2, graph=False)

    # ---- roofline probes: device time of every launch of each kernel class (eager steps, CUDA
    # events on the session stream around each launch of the class)
    probes = {}
    for cls in ("adder_round", "beaver", "chain", "gemm"):
        barrier(s)
        api.probe_start(cls)
        for _ in range(a.steps):
            ex.run(x)
        s.sync()
        probes[cls] = api.probe_stop()

    ex.time_layers(True)   # per-layer CUDA events recorded inside the graph
    ex.capture(x)
    ms_step, launches, clocks, out = timed(s, ex, x, a.steps, a.warmup, graph=True)
    layer_ms = ex.layer_times()   # of the last timed replay
    z = out.numpy()

    # ---- e2e through the public API: pinned H2D of the input shares, run, D2H of the logits
    nloc = 2 if world == 1 else 1
    xin_host = x.numpy()
    pin_in = api.PinnedBuffer(xin_host.size)
    pin_in.array[:] = xin_host.reshape(-1)
    pin_out = api.PinnedBuffer(z.size)
    for _ in range(max(1, a.warmup)):
        api.copy_from_host(x, pin_in)      # the captured graph reads x in place
        api.download_into(ex.replay(), pin_out)
    barrier(s)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        api.copy_from_host(x, pin_in)
        api.download_into(ex.replay(), pin_out)
    barrier(s)
    e2e_s = maxall(time.perf_counter() - t0) / a.steps
    h2d = xin_host.size * 8
    d2h = z.size * 8

    # ---- blocking comparison (the paper's pipelined-vs-blocking reduction, per layer)
    blocking = None
    if not a.no_blocking and a.mode == "pipelined":
        sb, exb, xb = setup("blocking")
        exb.run(xb)
        exb.time_layers(True)
        exb.capture(xb)
        b_ms, _, _, _ = timed(sb, exb, xb, a.steps, a.warmup, graph=True)
        bl = exb.layer_times()
        blocking = {"ms_per_step": b_ms, "note": "graph replays; per-layer CUDA events inside the graph",
                    "reduction_pct": (b_ms - ms_step) / b_ms * 100.0,
                    "per_layer": [{"layer": l.name, "blocking_ms": round(bb, 4), "pipelined_ms": round(pp, 4),
                                   "reduction_pct": round((bb - pp) / bb * 100.0, 2) if bb > 0 else 0.0}
                                  for l, bb, pp in zip(g.layers, bl, layer_ms)]}
        del exb, sb

    if rank != 0:
        return
    # ---- CPU baseline: the reference itself on this host (bounded sample)
    cpu = None
    if not a.no_cpu and os.path.exists(REF_DRIVER):
        try:
            iters = 6 if a.model == "lenet5" else 3
            r = ref_bench(model_path, a.mode, iters, a.weights)
            lat = sum(r["iter_wall_s"]) / len(r["iter_wall_s"])
            cpu = {"value": g.input[0] / lat, "unit": "inferences/s", "cores": 2, "kind": "reference",
                   "sample": f"{iters} iterations of {g.name} b{g.input[0]} 2PC {a.weights} {a.mode} "
                             f"(reference bench_party over SocketComm, 1 thread/party; nproc={os.cpu_count()})",
                   "ms_per_inference_batch": lat * 1e3, "logits_hash": r["logits_hash"]}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "inferences/s", "cores": 2, "kind": "reference", "sample": str(e)[:200]}
    elif not a.no_cpu:
        cpu = {"value": None, "unit": "inferences/s", "cores": 2, "kind": "reference",
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
    # algorithmic units per class: bytes for the HBM-bound protocol rounds, ring MACs
    # for the GEMM (x36 int8 MACs = 72 int8 ops each, the limb-pair products of the tcgen05 path)
    notes = {"adder_round": "SPK level round (settle r, issue r+1), opened wire (pair evaluation): 64 B/elem/party = "
                            "32 B opened value written + read once per element pair + 8x(2 in + 2 out) state "
                            "(per-slot form: 96 B = 2x32 B wire + state)",
             "beaver": "Beaver mul/square rounds incl. fused exp/Newton chains: 40 (opened wire) or 56 / 32 B/elem/party "
                       "per op",
             "chain": "persistent compare-and-select chain (ReLU/tournament): 512 B/elem/party",
             "gemm": "ring GEMM main kernel: 72 int8 ops per ring MAC (36 limb-pair MACs), packing excluded"}
    rooflines = []
    for cls, (p_ms, p_launches, p_units) in probes.items():
        if p_launches == 0 or p_ms <= 0:
            continue
        if cls == "gemm":
            ach = 72.0 * p_units / (p_ms / 1e3) / 1e12
            r = {"kernel": cls, "bound": "tensor", "achieved": ach, "peak": int8_peak, "unit": "TOP/s (int8)",
                 "frac": ach / int8_peak, "peak_source": int8_src}
        else:
            ach = (p_units / 1e9) / (p_ms / 1e3)
            r = {"kernel": cls, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                 "frac": ach / hbm_peak, "peak_source": "measured" if hbm else "fallback"}
        r.update({"launches": p_launches, "device_ms_per_step": p_ms / a.steps,
                  "avg_launch_us": p_ms * 1e3 / p_launches, "units_per_launch": p_units / p_launches,
                  "traffic": (traffic.get(cls) or {}).get("dram_bytes_per_launch"), "note": notes[cls]})
        rooflines.append(r)
    rooflines.sort(key=lambda r: -r["device_ms_per_step"])
    roof = dict(rooflines[0]) if rooflines else None  # the dominant class of the step
    if roof:
        roof["share_of_probed_ms"] = roof["device_ms_per_step"] / sum(r["device_ms_per_step"] for r in rooflines)

    pipelined_ms = ms_step
    value = B * pairs / (ms_step / 1e3)
    dec = (z.sum(axis=0) if world == 1 else z[0]).reshape(-1)
    line = {
        "metric": METRIC, "value": value, "unit": "inferences/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": pipelined_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: the reference's seeded init_weights(seed 12) / demo_input(seed 13), shares dealt on host",
        "config": {"workload": f"{g.name} b{B} 2PC {a.weights} {a.mode}", "model": g.name, "global_batch": B * pairs,
                   "pairs": pairs, "parties_per_gpu": 2 if world == 1 else 1, "mode": a.mode, "weights": a.weights,
                   "frac_bits": g.frac_bits, "chunks": 4,
                   "chunk_threshold_bytes": None if thr == NEVER else thr,
                   "chunk_threshold_source": a.threshold,
                   "calibration": calib,
                   "l2": "flushed between timed steps (256 MiB memset, untimed)",
                   "transport": ("in-device zero-copy opens" if world == 1 else "NCCL send/recv over NVLink")
                   + (f" + emulated link latency {link[0]} s, {link[1]:.3g} B/s" if link else ""),
                   "kernels_per_step": launches / a.steps,
                   "execution": "one CUDA-graph replay per step (whole 2PC inference, both parties)",
                   "eager_ms_per_step": eager_ms,
                   "logits_hash_slot0": mp.fnv1a_words(dec) if world == 1 else None,
                   "blocking": blocking},
        "roofline": roof,
        "rooflines": rooflines,
        "cpu_baseline": cpu,
        "e2e": {"value": B * pairs / e2e_s, "unit": "inferences/s", "ms_per_step": e2e_s * 1e3,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "pinned host shares -> mpcg_tensor_copy_from_host -> mpcg_executor_run -> mpcg_tensor_download"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
