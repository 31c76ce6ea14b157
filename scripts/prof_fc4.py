"""config-1 FC derivative with BASELINE's degree-4 / C = 27 operator (n_ext = 282), for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, fc, problems as P  # noqa: E402

ctx = N.Context(0)
op = fc.FcOperator(ctx, 256, n_cont=27, degree=4)
_, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
t = torch.from_numpy(f).cuda()
o = torch.empty_like(t)
for _ in range(5):
    op.apply(t, 1, out=o)
torch.cuda.synchronize()
print("ok")
