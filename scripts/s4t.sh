cat > /tmp/fc4.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_2506_19370_b200 import _native as N
ctx = N.Context(0)
g, ms = bench.fc_derivative_gbs(ctx, n_cont=27, degree=4)
print("fc degree 4:", round(g, 1), "GB/s", round(ms * 1e3, 2), "us")
PY
for lb in 0 4 5 6 8; do echo "== FCSG_FC_LB=$lb"; FCSG_FC_LB=$lb python /tmp/fc4.py 2>&1 | tail -1; done
