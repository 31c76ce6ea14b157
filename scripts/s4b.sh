# session 4 debug: the ct passes on one 256 x 256 subpatch
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import os, sys
print("start", flush=True)
sys.path.insert(0, os.getcwd())
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P
print("imported", flush=True)
ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=1, s=1)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
print("engine", flush=True)
try:
    print("run", E.run(2, use_graph=False), flush=True)
except BaseException as ex:
    print("EXC", repr(ex), flush=True)
    raise
PY
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -X faulthandler -u /tmp/one.py > gpurun_out/s4b_plain.log 2>&1; echo "plain rc=$?"; tail -30 gpurun_out/s4b_plain.log
dmesg 2>/dev/null | tail -5
