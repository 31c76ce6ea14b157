"""Run supersteps of BASELINE config 3 or 4 for an ncu launch list.
Usage: python scripts/profile_config.py 3|4 [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = N.Context(0)
dec, ic, meta = P.step_flow(2) if which == 4 else P.cylinder_flow(True)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(1)  # step 0 (smear)
E.run(steps, use_graph=False)
torch.cuda.synchronize()
print("ok", E.time())
