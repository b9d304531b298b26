"""Summarise ncu outputs into committable profile files.

  python tools/ncu_summary.py launches <launches.csv> [out.json]   # per-kernel-class shares
  python tools/ncu_summary.py raw <report.ncu-rep> [out.json]       # key metrics per launch
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

CLASSES = [
    ("chain_reg", r"chain_reg_kernel"),
    ("chain_fused", r"chain_pair_kernel|beaver_chain_pair_kernel|MulFused"),
    ("adder_round", r"AdderRound"),
    ("beaver_mul_build", r"MulBuild"),
    ("beaver_mul_combine", r"MulCombine"),
    ("beaver_square", r"Sq(Build|Combine)"),
    ("beaver_and", r"And(Build|Combine)"),
    ("ring_gemm_tc", r"ring_gemm_tc|tc_gemm|limb"),
    ("ring_gemm_simt", r"ring_gemm_simt|ring_gemm_splitk|gemm_splitk_epilogue"),
    ("link_delay", r"link_delay"),
    ("memset", r"memset|Memset"),
    ("ew_lambda", r"lambda"),
]


def classify(name):
    for k, pat in CLASSES:
        if re.search(pat, name):
            return k
    return name[:60]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(unit, v)


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or not r[vi]:
            continue
        c = classify(r[ki])
        agg[c][0] += 1
        agg[c][1] += to_us(r[vi], r[ui])
    tot = sum(v[1] for v in agg.values())
    return {"total_launches": sum(v[0] for v in agg.values()), "total_us": tot,
            "note": "ncu gpu__time_duration, --clock-control none, serialized cold-cache launches: compare shares",
            "classes": [{"class": k, "launches": n, "us": round(us, 2), "share_pct": round(100 * us / tot, 2),
                         "avg_us": round(us / n, 3)} for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])]}


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for m in RAW:
            if m in hdr:
                d[m] = r[hdr.index(m)] + " " + units[hdr.index(m)]
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = launches(path) if kind == "launches" else raw(path)
    s = json.dumps(res, indent=1)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(s + "\n")
    print(s)
