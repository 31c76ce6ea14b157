"""Parity at the stated horizons (north_star), on the B200
against the compiled reference's own ``Engine::run`` (oracle/_ref, all host
threads; src/runtime.cpp:460-530):

* config 5 (smooth: isentropic vortex + 1e-3 seeded noise), a 4 x 2 tiling
  of the bench's 256 x 256 subpatches, the stated 100 supersteps: every field
  of every subpatch within 1e-8 relative L2; tau equal wherever the logit
  margin (top1 - top2, recomputed by the numpy oracle from the reference's
  own state at the start of the last step) exceeds 1e-9, and at least 99.9%
  of the points clear that margin;
* config 4 at the benched size (problems.step_flow(2), 3.22M points, CFL 0.25
  as the reference runs every problem with C1 patches, D7), 20 supersteps of
  Mach 3 flow from the impulsive start, against the reference on the same
  patches (ref_engine_testgeom 6).
"""
import os

import numpy as np
import pytest

from oracle import fcs_oracle as O, ref
from paper_2506_19370_b200 import engine as EN, problems as PR

from .helpers import RefDecomposition, engine_from_reference, rel_err

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

THREADS = os.cpu_count() or 1


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def tau_margins(mlp, e):
    """oracle classifier margins of the state e (phase 0, src/viscosity.cpp:211-238)"""
    proxy, _ = O.proxy_mwsb(e)
    return O.classify_field(mlp, proxy)


@pytest.mark.gpu
def test_config5_100_steps_against_reference(gpu_ctx):
    tiles = (4, 2)
    dec, ic, meta = PR.vortex_tiles(r=tiles[0], s=tiles[1])
    p = dec.patches[0]
    R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], tiles[0], tiles[1], 238, p.nv, [5, 5, 5, 5],
                      cfl=meta["cfl"], workers=THREADS, weight_path=EN.DEFAULT_WEIGHTS)
    states = [PR.initial_state(dec, ic, k) for k in range(len(dec.subs))]
    for k, e in enumerate(states):
        R.set_state(k, e)
    R.finish_ic()
    E = EN.Engine(gpu_ctx, dec, cfg=EN.EngineConfig(cfl=meta["cfl"]), initial_states=states)
    for k in range(len(dec.subs)):
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-15
    R.run(99)
    assert E.run(99) == 99
    mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)
    margins = [tau_margins(mlp, R.get_state(k))[1] for k in range(len(dec.subs))]
    R.run(100)
    assert E.run(1) == 1
    assert R.time()[1] == 100 and E.time()[1] == 100
    assert E.time()[0] == pytest.approx(R.time()[0], rel=1e-12)
    worst = 0.0
    npts = sure_pts = low_tau = 0
    for k in range(len(dec.subs)):
        got, want = E.get_state(k), R.get_state(k)
        for c in range(4):
            err = rel_l2(got[c], want[c])
            worst = max(worst, err)
            assert err <= 1e-8, (k, c, err)
        tau, tau_ref = E.get(k, "tau"), R.get(k, "tau")
        sure = margins[k] > 1e-9
        assert np.array_equal(tau[sure], tau_ref[sure]), k
        npts += tau.size
        sure_pts += int(sure.sum())
        low_tau += int((tau_ref < 4).sum())
    frac = sure_pts / npts
    print(f"config5 100 steps: worst per-field rel L2 {worst:.3e}; tau<4 at {low_tau} of {npts} points; "
          f"{npts - sure_pts} points with margin <= 1e-9 (sure fraction {frac:.6f})")
    assert frac >= 0.999


@pytest.mark.gpu
def test_config4_benched_size_20_steps_against_reference(gpu_ctx):
    dec, ic, meta = PR.step_flow(2)
    assert meta["cfl"] == 0.25
    R = ref.RefEngine.testgeom(6, 0, cfl=meta["cfl"], workers=THREADS, weight_path=EN.DEFAULT_WEIGHTS)
    RD = RefDecomposition(R)
    assert len(RD.subs) == len(dec.subs)
    for d, r in zip(dec.subs, RD.subs):
        assert (d.cut_i, d.cut_j, d.ni, d.nj) == (r.cut_i, r.cut_j, r.ni, r.nj)
        assert np.array_equal(d.mask, r.mask)
    # the product steps the reference's own geometry and plan (the builder's
    # equality with it is tested in test_multipatch.py; a few viscosity-blend
    # donor stencils tie at round-off there). The L-shaped corner subpatch is
    # Cartesian (axis-aligned arms): its group runs the Cartesian passes on
    # the compile-time 163 / 94 plans.
    E, _ = engine_from_reference(gpu_ctx, R, EN.EngineConfig(cfl=meta["cfl"]))
    assert E.shapes == [tuple(d.mask.shape) for d in RD.subs]
    R.run(20)
    assert E.run(20) == 20
    # relative L2 per field over the whole domain: in the Mach 3 free stream
    # rho v is zero up to round-off on most subpatches, so a per-subpatch
    # relative norm of it would compare round-off with round-off
    dn, wn = np.zeros(4), np.zeros(4)
    for k in range(R.nsubs):
        got, want = E.get_state(k), R.get_state(k)
        dn += ((got - want) ** 2).sum(axis=(1, 2))
        wn += (want ** 2).sum(axis=(1, 2))
        assert np.array_equal(E.get(k, "tau"), R.get(k, "tau")), k
    err = np.sqrt(dn / wn)
    print(f"config4 step_flow(2), 20 steps at CFL 0.25: rel L2 per field over the domain {err}")
    assert err.max() <= 1e-8, err


@pytest.mark.gpu
def test_config3_positivity_loss_matches_reference(gpu_ctx):
    """The config-3 cylinder layout (0.70M points, ref_engine_testgeom 3) at
    the reference's CFL 0.5 from the impulsive Mach 3 start: the reference's
    own Engine::run loses positivity at the body wall after a few steps
    (InvalidStateError, src/euler.cpp:37-39 / src/viscosity.cpp:13-29); the
    product must fail at the same superstep and the same point, with the
    states equal to round-off until then."""
    from paper_2506_19370_b200 import _native as N

    from .helpers import engine_from_reference

    R = ref.RefEngine.testgeom(3, 0, cfl=0.5, workers=THREADS, weight_path=EN.DEFAULT_WEIGHTS)
    E, _ = engine_from_reference(gpu_ctx, R, EN.EngineConfig(cfl=0.5))
    ours, last = None, None
    for k in range(1, 40):
        last = [E.get_state(s) for s in range(R.nsubs)]  # the state after step k - 1
        try:
            E.run(1)
        except N.InvalidStateError as ex:
            ours = (k, ex.patch, ex.subpatch, ex.i, ex.j)
            break
    assert ours is not None, "the product did not lose positivity within 40 steps"
    R.run(ours[0] - 1)
    dn = wn = 0.0
    for s in range(R.nsubs):
        want = R.get_state(s)
        dn += float(((last[s] - want) ** 2).sum())
        wn += float((want ** 2).sum())
    assert (dn / wn) ** 0.5 <= 1e-8, (dn / wn) ** 0.5
    with pytest.raises(Exception) as ei:
        R.run(ours[0] + 5)
    msg = str(ei.value)
    assert R.time()[1] == ours[0] - 1, (R.time(), ours)
    assert f"patch {ours[1]} subpatch {ours[2]} ({ours[3]},{ours[4]})" in msg, (msg, ours)
    print(f"config3 layout: positivity lost at step {ours[0]}, patch {ours[1]} subpatch {ours[2]} "
          f"({ours[3]},{ours[4]}) in both; reference: {msg}")


@pytest.mark.gpu
def test_config2_200_steps_against_reference(gpu_ctx):
    """BASELINE config 2's horizon (200 supersteps of the seeded Riemann
    quadrants, ANN classifier, CFL 0.5) on a 128 x 128 subpatch against the
    reference's own Engine::run: states within 1e-10 relative L2 per field and
    tau equal wherever the reference's logit margin exceeds 1e-9, at steps 100
    and 200. The full 512 x 512 case is scripts/config2_horizon.py (minutes of
    reference CPU time; profiles/r02_config2_200_steps.log: <= 1e-13, tau
    identical at every point)."""
    n = 128
    dec, ic, meta = PR.riemann_quadrants(n=n, seed=2)
    p = dec.patches[0]
    R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], 1, 1, n - 2 * p.nv, p.nv, [5, 5, 5, 5],
                      cfl=meta["cfl"], workers=THREADS, weight_path=EN.DEFAULT_WEIGHTS)
    e0 = PR.initial_state(dec, ic, 0)
    R.set_state(0, e0)
    R.finish_ic()
    E = EN.Engine(gpu_ctx, dec, cfg=EN.EngineConfig(cfl=meta["cfl"]), initial_states=[e0])
    mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)
    done = 0
    for mark in (100, 200):
        R.run(mark - 1)
        assert E.run(mark - 1 - done) == mark - 1 - done
        margin = tau_margins(mlp, R.get_state(0))[1]
        R.run(mark)
        assert E.run(1) == 1
        done = mark
        assert E.time()[0] == pytest.approx(R.time()[0], rel=1e-12)
        g, w = E.get_state(0), R.get_state(0)
        for c in range(4):
            assert rel_l2(g[c], w[c]) < 1e-10, (mark, c)
        sure = margin > 1e-9
        assert sure.mean() > 0.999
        assert np.array_equal(E.get(0, "tau")[sure], R.get(0, "tau")[sure])
        assert (R.get(0, "tau") < 4).any()  # the classifier is active: the run is not a smooth one
