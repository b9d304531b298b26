"""Summarise an `ncu --page raw --csv` export: per-launch key metrics + class average.

  python tools/ncu_raw_summary.py <raw.csv> [--json out.json]
"""
import csv
import json
import sys

KEYS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_B": ("dram__bytes_read.sum", 1),
    "dram_write_B": ("dram__bytes_write.sum", 1),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_imma_pct": ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "tc_pipe_pct": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "inst": ("smsp__inst_executed.sum", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
        "ns": 1, "us": 1e3, "ms": 1e6,
        "%": 1, "register/thread": 1, "inst": 1, "": 1}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:100]}
        for k, (m, scale) in KEYS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    d[k] = float(v) * UNIT.get(units[hdr.index(m)], 1) * scale
                except ValueError:
                    pass
        out.append(d)
    return out


if __name__ == "__main__":
    rows = load(sys.argv[1])
    avg = {k: sum(r.get(k, 0) for r in rows) / len(rows) for k in KEYS} if rows else {}
    for r in rows:
        print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()})
    print("AVG", {k: round(v, 2) for k, v in avg.items()})
    if "--json" in sys.argv:
        json.dump({"launches": rows, "avg": avg}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
