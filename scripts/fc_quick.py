"""Quick GPU check of the batched FC line kernel (development script)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fcs_oracle as O  # noqa: E402  (checker only)
from paper_2506_19370_b200 import _native as N, fc  # noqa: E402

ctx = N.Context(0)
for n, L in [(256, 4096), (512, 4096), (147, 2048), (101, 2048)]:
    op = fc.FcOperator(ctx, n)
    o = O.get_op(n)
    rng = np.random.default_rng(0)
    x = np.linspace(0, 1, n)
    a = rng.uniform(-1, 1, (L, 4, 1))
    w = rng.uniform(1, 20, (L, 4, 1))
    ph = rng.uniform(0, 2 * np.pi, (L, 4, 1))
    f = (a * np.sin(w * x + ph)).sum(1)
    ref = o.derivative(f, 1)
    t = torch.from_numpy(f).cuda()
    out = op.apply(t, 1)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    tc = t.T.contiguous()
    outc = op.apply(tc, 1, axis=0)
    gotc = outc.T.cpu().numpy()
    relc = np.linalg.norm(gotc - ref, axis=1) / np.linalg.norm(ref, axis=1)
    # timing, rotating buffers > L2
    nbuf = max(2, int(np.ceil(400e6 / (2 * t.numel() * 8))))
    bufs = [torch.randn_like(t) for _ in range(nbuf)]
    outs = [torch.empty_like(t) for _ in range(nbuf)]
    for k in range(3):
        op.apply(bufs[k % nbuf], 1, out=outs[k % nbuf])
    torch.cuda.synchronize()
    iters = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(iters):
        op.apply(bufs[k % nbuf], 1, out=outs[k % nbuf])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    gbs = 16 * t.numel() / (ms * 1e-3) / 1e9
    print(f"n={n} lines={L} rows rel={rel.max():.2e} cols rel={relc.max():.2e}  {ms*1e3:.1f} us/call  {gbs:.0f} GB/s",
          flush=True)
