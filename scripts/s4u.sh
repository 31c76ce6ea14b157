cat > /tmp/cfg.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2506_19370_b200 import _native as N
ctx = N.Context(0)
for f in (bench.config3_rate, bench.config4_rate):
    d = f(ctx)
    print(d["config"][:8], round(d["ms_per_step"], 4), flush=True)
PY
for c in 0 3 2; do echo "== FCSG_WPASS_CAP=$c"; FCSG_WPASS_CAP=$c python /tmp/cfg.py 2>&1 | tail -2; done
