"""Copy the judged measurement artefacts from gpurun_out/ (scratch) into profiles/ (tracked).

  python tools/save_profiles.py r01
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_raw_summary import load  # noqa: E402
from ncu_summary import launches  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def last_json_line(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


if os.path.exists(os.path.join(G, "bench.log")):
    json.dump(last_json_line(os.path.join(G, "bench.log")), open(os.path.join(P, f"{tag}_bench.json"), "w"), indent=1)
if os.path.exists(os.path.join(G, "bench_ref.log")):
    json.dump(last_json_line(os.path.join(G, "bench_ref.log")), open(os.path.join(P, f"{tag}_bench_reference.json"), "w"),
              indent=1)
if os.path.exists(os.path.join(G, "configs.json")):
    shutil.copy(os.path.join(G, "configs.json"), os.path.join(P, f"{tag}_configs.json"))
for m in ("lenet5", "resnet18", "vgg16", "bert_base"):
    f = os.path.join(G, f"{m}_launches.csv")
    if os.path.exists(f):
        json.dump(launches(f), open(os.path.join(P, f"{tag}_{m}_launches.json"), "w"), indent=1)
classes = {"adder_round": "AdderRound", "gemm": "ring_gemm_tc2", "chain": "chain_kernel", "gemm_simt": "ring_gemm_simt"}
summary = {"note": "ncu --set full --clock-control none on the bench workload (lenet5 b64), mean over the captured "
                   "launches of each class; cold caches (ncu flushes between replays). tools/gpu_profile.sh"}
traffic = {"note": summary["note"] + "; traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch",
           "model": "lenet5"}
for cls, f in classes.items():
    path = os.path.join(G, f"prof_lenet5_{f}_raw.csv")
    if not os.path.exists(path):
        continue
    rows = load(path)
    if not rows:
        continue
    n = len(rows)
    keys = ["time_us", "dram_read_B", "dram_write_B", "dram_pct", "sm_pct", "issue_active_pct", "tensor_imma_pct",
            "tc_pipe_pct", "warps_active_pct", "regs", "inst"]
    summary[cls] = {"launches_captured": n, "kernel": rows[0]["kernel"],
                    **{k: round(sum(r.get(k, 0) for r in rows) / n, 3) for k in keys}}
    traffic[cls] = {"dram_bytes_per_launch": sum(r.get("dram_read_B", 0) + r.get("dram_write_B", 0) for r in rows) / n,
                    "launches_captured": n}
json.dump(summary, open(os.path.join(P, f"{tag}_lenet5_ncu_classes.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(sorted(os.listdir(P)))
