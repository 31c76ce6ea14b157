"""Config-1 FC derivative: kernel time under a CUDA graph of 64 launches
(no host launch overhead in the loop) against the plain Python loop."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, fc, problems as P  # noqa: E402

ctx = N.Context(0)
op = fc.FcOperator(ctx, 256)
_, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
src = torch.from_numpy(f).cuda()
nbuf = 16
ins = [src.clone() for _ in range(nbuf)]
outs = [torch.empty_like(src) for _ in range(nbuf)]
for k in range(4):
    op.apply(ins[k], 1, out=outs[k])
torch.cuda.synchronize()
reps = 64
t0 = time.perf_counter()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(reps):
    op.apply(ins[k % nbuf], 1, out=outs[k % nbuf])
b.record()
host = (time.perf_counter() - t0) / reps
torch.cuda.synchronize()
print(f"python loop: {a.elapsed_time(b) / reps * 1e3:.2f} us/call (host {host * 1e6:.1f} us/call)")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    op.apply(ins[0], 1, out=outs[0])
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for k in range(reps):
            op.apply(ins[k % nbuf], 1, out=outs[k % nbuf])
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a.record()
g.replay()
b.record()
torch.cuda.synchronize()
print(f"graph: {a.elapsed_time(b) / reps * 1e3:.2f} us/call -> {16 * f.size / (a.elapsed_time(b) / reps * 1e-3) / 1e9:.0f} GB/s")
