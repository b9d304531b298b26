"""Per-class summary of an ncu launch list (`--metrics gpu__time_duration.sum --csv`).

  python tools/launch_classes.py <launches.csv> [--json out.json]

Launch times from ncu are cold-cache and serialised, so only the SHARE of each class in the
profiled command is comparable with the bench line's live probes (bench.py `rooflines`).
"""
import csv
import json
import re
import sys
from collections import defaultdict

CLASSES = [
    ("chain_fused", r"chain_reg_kernel|chain_pair_kernel|beaver_chain_pair_kernel|MulFused"),
    ("adder_round", r"AdderRound"),
    ("gemm", r"ring_gemm_tc2|ring_gemm_tc3|ring_gemm_simt|ring_gemv|ring_gemm_rows"),
    ("gemm_aux", r"tc2_pack|pack_|gemm_splitk_epilogue"),
    ("eps_delta_build", r"eps_|delta_build|EpsIm2col"),
    ("chain", r"chain_kernel|ChainStep"),
    ("beaver", r"MulBuild|MulCombine|SqBuild|SqCombine|AndBuild|AndCombine|square_chain|mul_chain"),
    ("a2b_b2a_gate", r"A2b|B2a|Gate|Pick|a2b|b2a|Tail"),
    ("link", r"trailer|p2p_|link_delay|delay_kernel"),
    ("rekey", r"rekey"),
]


def classify(name):
    for c, rx in CLASSES:
        if re.search(rx, name):
            return c
    return "other"


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        rows.append((r["Kernel Name"], ns))
    return rows


def summarise(rows):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for name, ns in rows:
        c = classify(name)
        tot[c] += ns
        cnt[c] += 1
    all_ns = sum(tot.values())
    return {"launches": len(rows), "total_ms": all_ns / 1e6,
            "classes": {c: {"launches": cnt[c], "total_ms": tot[c] / 1e6, "share": tot[c] / all_ns,
                            "avg_us": tot[c] / cnt[c] / 1e3}
                        for c in sorted(tot, key=lambda k: -tot[k])}}


if __name__ == "__main__":
    s = summarise(load(sys.argv[1]))
    print(json.dumps(s, indent=1))
    if "--json" in sys.argv:
        json.dump(s, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
