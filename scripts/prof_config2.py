"""A few supersteps of BASELINE config 2 (one 512 x 512 subpatch) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

ctx = N.Context(0)
dec, ic, _ = P.riemann_quadrants(n=512, seed=2)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
E.run(1, use_graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
