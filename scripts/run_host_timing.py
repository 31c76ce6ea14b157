"""Marginal per-step time of fcsg_engine_run_host against the device-only
step on the bench workload (is the host-I/O pipeline overlapped?)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P
ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=8, s=8)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(3)
n = E.total_points()
hi = torch.empty((4, n), dtype=torch.float64, pin_memory=True); E.get_state_bulk(hi)
ho = torch.empty((4, n), dtype=torch.float64, pin_memory=True)
for steps in (5, 10, 20, 40):
    torch.cuda.synchronize(); a = time.perf_counter()
    E.run_host(hi, ho, steps=steps)
    dt = time.perf_counter() - a
    print(f"run_host {steps:3d} steps: {dt*1e3:8.1f} ms  ({dt/steps*1e3:.2f} ms/step)")
for steps in (10, 40):
    torch.cuda.synchronize(); a = time.perf_counter()
    E.run(steps)
    dt = time.perf_counter() - a
    print(f"run      {steps:3d} steps: {dt*1e3:8.1f} ms  ({dt/steps*1e3:.2f} ms/step)")
for rep in range(2):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(10):
        E.set_state_bulk(hi)
    dt = (time.perf_counter() - a) / 10
    torch.cuda.synchronize(); b = time.perf_counter()
    for _ in range(10):
        E.get_state_bulk(ho)
    dt2 = (time.perf_counter() - b) / 10
    print(f"set_state_bulk {dt*1e3:.2f} ms ({hi.numel()*8/dt/1e9:.1f} GB/s), get_state_bulk {dt2*1e3:.2f} ms")
for steps in (20, 40):
    torch.cuda.synchronize(); a = time.perf_counter()
    E.run_host(hi, ho, steps=steps)
    dt = time.perf_counter() - a
    print(f"run_host again {steps:3d} steps: {dt/steps*1e3:.2f} ms/step")
