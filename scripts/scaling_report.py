"""E^s / E^w table (the reference's scaling_csv) from bench.py JSON lines:
    python scripts/scaling_report.py weak_N1.json weak_N2.json ... [--csv out.csv]
Each file holds the JSON line(s) bench.py printed (e.g. --gpus N --scaling
weak|strong). The driver computes its own efficiency from the per-N values;
this is the reference's metric for the same runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import scaling as S  # noqa: E402

args = [a for a in sys.argv[1:] if a != "--csv"]
out = None
if "--csv" in sys.argv:
    out = sys.argv[sys.argv.index("--csv") + 1]
    args.remove(out)
lines = []
for f in args:
    with open(f) as fh:
        lines += [ln for ln in fh if ln.strip().startswith("{")]
csv = S.scaling_csv(S.scaling_metrics(S.records_from_bench(lines)))
print(csv, end="")
if out:
    with open(out, "w") as fh:
        fh.write(csv)
