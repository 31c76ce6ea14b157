"""Run a few supersteps of the bench workload (for ncu launch lists and
single-kernel captures). Usage: python scripts/profile_step.py [tiles] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=tiles, s=tiles)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(1)  # step 0 (smear) outside the profiled window
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures only the steady steps
E.run(steps, use_graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
torch.cuda.synchronize()
print("ok", E.time())
