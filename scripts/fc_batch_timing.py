"""FC derivative (reference operator, N = 256 rows) against the batch size:
one call per measurement, CUDA-event timed, rotating buffers beyond L2.
    python scripts/fc_batch_timing.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, fc, problems as P  # noqa: E402

ctx = N.Context(0)
op = fc.FcOperator(ctx, 256)
_, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
base = torch.from_numpy(f).cuda()
for n_lines in (4096, 16384, 65536, 262144):
    src = base.repeat(n_lines // 4096, 1).contiguous()
    nbuf = max(2, min(16, (1 << 30) // (src.numel() * 8)))
    ins = [src.clone() for _ in range(nbuf)]
    outs = [torch.empty_like(src) for _ in range(nbuf)]
    for k in range(nbuf):
        op.apply(ins[k], 1, out=outs[k])
    torch.cuda.synchronize()
    reps = 4 * nbuf
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        op.apply(ins[k % nbuf], 1, out=outs[k % nbuf])
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    print(f"n_lines {n_lines}: {us:.1f} us/call -> {16 * src.numel() / (us * 1e-6) / 1e9:.0f} GB/s", flush=True)
