"""Pass timings without the error check (for timing-only experiments whose
arithmetic is deliberately wrong): python scripts/time_passes_raw.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=8, s=8)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.enqueue(3)
torch.cuda.synchronize()
for g in ("pass_a", "pass_b", "filter"):
    print(f"  {g}: {E.time_group(g, reps=10):.4f} ms", flush=True)
