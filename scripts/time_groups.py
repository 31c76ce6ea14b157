"""Per-group device times of the config-5 superstep (bench workload) and the
config-1 FC derivative, quick: python scripts/time_groups.py [r s]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402
import bench  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = N.Context(0)
gbs, ms = bench.fc_derivative_gbs(ctx)
print(f"fc_derivative config1: {ms * 1e3:.2f} us/call {gbs:.0f} GB/s", flush=True)
gbs, ms = bench.fc_derivative_gbs(ctx, n_cont=27, degree=4)
print(f"fc_derivative degree4: {ms * 1e3:.2f} us/call {gbs:.0f} GB/s", flush=True)
dec, ic, meta = P.vortex_tiles(r=r, s=s)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(3)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(E.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 20
e0.record(st)
E.enqueue(steps)
e1.record(st)
torch.cuda.synchronize()
E.check_error()
ms = e0.elapsed_time(e1) / steps
npts = E.total_points()
print(f"config5 {r}x{s}x256^2: {ms:.3f} ms/step  {5 * npts / (ms * 1e-3):.3e} pt-stage/s", flush=True)
for g in ("viscosity", "blend", "filter", "pass_a", "pass_b", "bc", "exchange"):
    t = E.time_group(g, reps=5)
    extra = ""
    if g in bench.ALG_BYTES_CART:
        extra = f"  {bench.ALG_BYTES_CART[g] * npts / (t * 1e-3) / 1e9:.0f} GB/s alg"
    print(f"  {g}: {t:.4f} ms{extra}", flush=True)
