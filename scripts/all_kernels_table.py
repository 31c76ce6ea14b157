"""Per-kernel table of one steady superstep from the all-kernel ncu capture
(profiles/rNN_all_raw.csv, the raw page of `ncu --set full`):
    python scripts/all_kernels_table.py profiles/r02_all_raw.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, name, scale=None):
    v = r[ix[name]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return 0.0
    u = units[ix[name]]
    if scale == "us":
        x *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(u, 1.0)
    if scale == "MB":
        x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
    return x


agg = defaultdict(lambda: defaultdict(float))
for r in rows[2:]:
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "").replace("unnamed>::", "").strip()
    a = agg[name]
    t = val(r, "gpu__time_duration.sum", "us")
    a["n"] += 1
    a["us"] += t
    a["mb"] += val(r, "dram__bytes_read.sum", "MB") + val(r, "dram__bytes_write.sum", "MB")
    for k, m in (("warps", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                 ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 ("fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                 ("dram", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")):
        a[k] += t * val(r, m)
tot = sum(a["us"] for a in agg.values())
print("| kernel | launches | µs per step (ncu) | share | DRAM MB per launch | warps active | issue active | FP64 pipe | DRAM % of peak |")
print("|---|---|---|---|---|---|---|---|---|")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    t = a["us"]
    print(f"| `{name}` | {int(a['n'])} | {t:.0f} | {100 * t / tot:.1f}% | {a['mb'] / a['n']:.0f} | {a['warps'] / t:.0f}% | "
          f"{a['issue'] / t:.0f}% | {a['fp64'] / t:.0f}% | {a['dram'] / t:.0f}% |")
print(f"\ntotal {tot:.0f} µs over {int(sum(a['n'] for a in agg.values()))} launches")
