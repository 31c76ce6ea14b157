cat > /tmp/cfg.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2506_19370_b200 import _native as N
ctx = N.Context(0)
for rep in range(2):
    for f in (bench.config2_rate, bench.config4_rate):
        d = f(ctx)
        print(d["config"][:8], round(d["ms_per_step"], 4), flush=True)
PY
python /tmp/cfg.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_kernels.py -m gpu -q -x -k "small_compile or superstep" 2>&1 | tail -2
