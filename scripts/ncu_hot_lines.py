"""Hottest source lines of an ncu report (stall samples per CUDA source line,
aggregated over the SASS it compiled to):
    python scripts/ncu_hot_lines.py rep.ncu-rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
extra = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *extra, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))

        def num(k):
            v = d.get(k, "0")
            try:
                return int(float(v))
            except ValueError:
                return 0

        s = num("Warp Stall Sampling (All Samples)")
        if s:
            rows.append((s, num("Warp Stall Sampling (Not-issued Samples)"), num("Instructions Executed"), fname,
                         int(r[0]), r[1].strip()))
tot = sum(r[0] for r in rows)
print(f"total samples {tot}")
for s, ni, ie, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% (not issued {100 * ni / max(s, 1):3.0f}%) inst {ie:>10d}  {f}:{ln}  {src[:90]}")
