"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck): one
superstep of each stage-pass family on 2 x 2 tiles of 48 x 48 (generic
plan), one superstep on a 256 x 256 subpatch (compile-time n_ext = 280 plan,
Cartesian flux passes), the fallback classifier, and one FC line batch per
mode. Exits non-zero on any error the library reports."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, fc, problems as P  # noqa: E402

ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=30)
for general in (False, True):
    for refo in (False, True):
        E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, force_general=general, reference_order=refo))
        assert E.run(2, use_graph=False) == 2
        E.close()
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, classifier="fallback"))
assert E.run(2, use_graph=False) == 2
E.close()
dec, ic, _ = P.vortex_tiles(r=1, s=1)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
assert E.run(2, use_graph=False) == 2
E.close()
_, f, _ = P.fc_lines_config1(n_lines=32, n=256, seed=3)
for n_cont, deg in ((25, 2), (27, 4)):
    op = fc.FcOperator(ctx, 256, n_cont=n_cont, degree=deg)
    for mode in (1, 2, 3, 4):
        op.apply(f, mode)
        op.apply(np.ascontiguousarray(f.T), mode, axis=0)
print("sanitize_small ok")
