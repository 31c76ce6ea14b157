"""Race / synchronisation discipline (compute-sanitizer is
closed on the GPU pool, so the evidence is built from the engine itself):

* donor purity, which the reference's barriers rely on (src/runtime.cpp:
  140-144, 239-247, 482-512): the engine refuses at finalize a plan whose
  copy donor is a fringe point (a point the same exchange writes) --
  DecompositionError, as the reference's build_plan;
* launch-shape invariance on the B200: the same superstep with the RK-stage
  chunks on 1 or 2 streams per group, 2 or 8 streams in the pool, eager
  launches or CUDA-graph replays, and run twice, is bitwise identical.
  Kernels whose threads read what other threads of the same launch write
  without ordering (a missing __syncwarp / __syncthreads, a stage reading a
  chunk another stream still writes) give schedule-dependent results, which
  these schedules would expose;
* the kernel bodies' index logic under AddressSanitizer + UBSan:
  scripts/asan_emu.sh (the emulation build, CPU parity tests).
"""
import copy
import os

import numpy as np
import pytest

from paper_2506_19370_b200 import _native as N, engine as EN, problems as P


def test_impure_plan_is_rejected(emu_ctx):
    dec, ic, _ = P.vortex_tiles(r=2, s=1, n0=30)
    bad = copy.deepcopy(dec)
    pl = bad.plan
    # point the first copy at a fringe point of its donor subpatch
    s = int(pl.sol_src_sub[0])
    fringe = np.flatnonzero(bad.subs[s].mask.ravel() == 2)
    pl.sol_src = pl.sol_src.copy()
    pl.sol_src[0] = fringe[0]
    with pytest.raises(N.DecompositionError, match="donor-pure"):
        EN.Engine(emu_ctx, bad, ic, EN.EngineConfig(cfl=0.5))


def _run(ctx, steps, chunks, streams, graph):
    os.environ["FCSG_STAGE_CHUNKS"] = str(chunks)
    os.environ["FCSG_STAGE_STREAMS"] = str(streams)
    try:
        dec, ic, _ = P.vortex_tiles(r=8, s=8)  # 4.19M points: two stage chunks per group
        E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
        assert E.run(steps, use_graph=graph) == steps
        out = [E.get_state(k) for k in range(len(dec.subs))] + [E.get(k, "mu") for k in range(len(dec.subs))]
        E.close()
        return out
    finally:
        os.environ.pop("FCSG_STAGE_CHUNKS", None)
        os.environ.pop("FCSG_STAGE_STREAMS", None)


@pytest.mark.gpu
def test_superstep_is_schedule_invariant(gpu_ctx):
    steps = 4
    base = _run(gpu_ctx, steps, 2, 8, True)
    for chunks, streams, graph in ((2, 8, True), (1, 2, True), (2, 2, False), (1, 8, False)):
        got = _run(gpu_ctx, steps, chunks, streams, graph)
        for a, b in zip(got, base):
            assert np.array_equal(a, b), (chunks, streams, graph)
