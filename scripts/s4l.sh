# filter passes with 4 instead of 8 lines per CTA: configs 2, 3, 4 per-step times
cat > /tmp/cfg.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2506_19370_b200 import _native as N
ctx = N.Context(0)
for f in (bench.config2_rate, bench.config3_rate, bench.config4_rate):
    d = f(ctx)
    print(d["config"][:8], round(d["ms_per_step"], 4), d.get("kernel_groups_ms", {}).get("filter"), flush=True)
PY
echo "== default"; python /tmp/cfg.py 2>&1 | tail -3
for v in paper_2506_19370_b200/lib/variants/libfcsg_*.so; do echo "== $v"; FCSG_LIB=$PWD/$v python /tmp/cfg.py 2>&1 | tail -3; done
