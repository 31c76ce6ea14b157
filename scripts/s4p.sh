cat > /tmp/cfg.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2506_19370_b200 import _native as N
ctx = N.Context(0)
for f in (bench.config2_rate, bench.config3_rate, bench.config4_rate):
    d = f(ctx)
    print(d["config"][:8], round(d["ms_per_step"], 4), flush=True)
g, ms = bench.fc_derivative_gbs(ctx, n_cont=27, degree=4)
print("fc degree 4:", round(g, 1), "GB/s", round(ms * 1e3, 2), "us")
PY
python /tmp/cfg.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_kernels.py tests/test_multipatch.py tests/test_geometries.py tests/test_horizon.py -m gpu -q -x 2>&1 | tail -2
