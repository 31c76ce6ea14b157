"""The Python API end to end on the GPU: config 2
with pipelined host I/O, then the config-4 layout with the fallback
classifier, its mesh file, integrals, |grad rho| raster, Schlieren PGM and
CSV output (written under /tmp). Usage: python scripts/api_demo.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P, diagnostics as DG, multipatch as M
ctx = N.Context(0)
dec, ic, _ = P.riemann_quadrants(n=512, seed=2)
eng = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
eng.run(20)
n = eng.total_points()
st_in = torch.empty((4, n), dtype=torch.float64, pin_memory=True); eng.get_state_bulk(st_in)
st_out = torch.empty_like(st_in)
print("run_host", eng.run_host(st_in, st_out, steps=10))
dec4, ic4, _ = P.step_flow(1)
M.save_mesh("/tmp/step.json", dec4.patches, nv=9, n0=0)
eng4 = EN.Engine(ctx, dec4, ic4, EN.EngineConfig(cfl=0.5, classifier="fallback"))
eng4.run(10)
DG.set_quadrature(eng4, dec4)
print("energy", DG.energy_integral(eng4), "area", DG.area_integral(eng4), "exact area", 3.0 - 2.4 * 0.2)
t = time.time()
g = DG.density_gradient_raster(eng4, dec4, 600, 200)
print("raster", g.v.shape, float(g.v.max()), time.time() - t)
DG.write_pgm(DG.schlieren(g), "/tmp/step.pgm")
DG.write_subpatch_csv(eng4, dec4, "/tmp/step_csv")
print("ok")
