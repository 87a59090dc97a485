"""Summarise ncu CSV exports (launch list, --page raw) into profiles/*.md/json.

  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py raw <raw.csv> [--algo-bytes B] [--json out.json]
"""
import csv
import json
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (warps active %)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("lts__t_sectors_evict_last_lookup_hit.sum", "L2 evict_last sector hits"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        t = float(r[vi].replace(",", "")) / 1e6  # ns -> ms
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")


def raw(path, algo_bytes=None, out_json=None):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        print(f"### `{d['kernel'][:110]}`\n\n| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in h:
                v, unit = r[h.index(key)], u[h.index(key)]
                d[key] = (v, unit)
                print(f"| {label} (`{key}`) | {v} {unit} |")
        if "dram__bytes_read.sum" in d:
            rb = float(d["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
            wb = float(d["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
            d["dram_bytes"] = rb + wb
            print(f"| DRAM read+write | {(rb + wb) / 1e9:.3f} GB |")
            if algo_bytes:
                print(f"| traffic / algorithmic bytes | {(rb + wb) / algo_bytes:.3f} |")
        print()
        res.append(d)
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        algo = None
        js = None
        if "--algo-bytes" in sys.argv:
            algo = float(sys.argv[sys.argv.index("--algo-bytes") + 1])
        if "--json" in sys.argv:
            js = sys.argv[sys.argv.index("--json") + 1]
        raw(sys.argv[2], algo, js)
