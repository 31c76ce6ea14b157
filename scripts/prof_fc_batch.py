"""The FC derivative on 262144 lines in one call, for ncu (development script)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, fc, problems as P  # noqa: E402

ctx = N.Context(0)
op = fc.FcOperator(ctx, 256)
_, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
t = torch.from_numpy(f).cuda().repeat(64, 1).contiguous()
o = torch.empty_like(t)
for _ in range(3):
    op.apply(t, 1, out=o)
torch.cuda.synchronize()
print("ok")
