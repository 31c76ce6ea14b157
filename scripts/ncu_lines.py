"""Warp-stall samples per CUDA source line of an ncu report (needs -lineinfo):
python scripts/ncu_lines.py rep.ncu-rep [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
fname = None
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    if r[0]:
        cur = (fname, r[0], r[1].strip())
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if cur:
        agg.setdefault(cur, [0.0, {}])
        agg[cur][0] += v
        for k, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    agg[cur][1][h] = agg[cur][1].get(h, 0.0) + float(r[k] or 0)
                except ValueError:
                    pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot:.0f}")
for (f, ln, src), (v, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    best = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    bs = ", ".join(f"{k[6:]} {x / max(v, 1) * 100:.0f}%" for k, x in best if x > 0)
    print(f"{v / tot * 100:5.1f}%  {f}:{ln}  {src[:70]:70s} [{bs}]")
