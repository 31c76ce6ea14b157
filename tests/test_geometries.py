"""Curvilinear, periodic, multi-patch and L-shaped geometries (SURVEY §8 a5,
a10, a16, a19, a21) against the compiled reference (oracle/_ref).

The reference builds the geometry and the CommPlan (its own
init_subpatch_data and build_plan, ref_export.cpp ref_engine_testgeom); the
product receives them through its public API (fcsg_engine_add_subpatch with
L-cuts, fcsg_engine_set_plan + fcsg_engine_set_plan_interps) and both engines
then advance the same state:

* annulus   one periodic S patch (AnnulusMap), 3 subpatches with wrap-around
            copies, curved no-slip wall: general metric passes, BCs on a
            curved boundary
* two-patch a Cartesian I patch and a bilinear S patch with non-coincident
            lattices: 6x6 Lagrange interpolation in the exchange and in the
            viscosity blend, two subpatch shapes in one engine (a Cartesian
            and a curvilinear group), inflow / slip / supersonic outflow
* corner    a C1 corner patch: an L-shaped subpatch (ragged lines, the
            classifier's row/column segments, BCs at segment ends)

(The reference's own multi-patch problems -- flow-cylinder, wedge, prism --
fail its minimum-overlap checks.)
"""
import numpy as np
import pytest

from oracle import ref
from paper_2506_19370_b200 import engine as EN

from .helpers import RefDecomposition, engine_from_reference, rel_err

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]
GEOMS = [pytest.param(0, id="annulus"), pytest.param(1, id="two-patch"), pytest.param(2, id="corner")]


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


def _compare(E, R, tol=1e-12):
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < tol, k
        assert np.array_equal(E.get(k, "tau"), R.get(k, "tau")), k
        assert rel_err(E.get(k, "mu"), R.get(k, "mu")) < tol, k


@pytest.mark.parametrize("which", GEOMS)
@pytest.mark.parametrize("refo", [False, True], ids=["flux", "reforder"])
def test_reference_geometry_steps(backend, which, refo):
    """3 supersteps (the first one with the t=0 smear) of both engines."""
    kind, ctx = backend
    R = ref.RefEngine.testgeom(which, 30, weight_path=EN.DEFAULT_WEIGHTS)
    E, dec = engine_from_reference(ctx, R, EN.EngineConfig(cfl=0.5, reference_order=refo))
    if which == 2:
        assert dec.subs[0].cut_i > 0 and (dec.subs[0].mask == 0).any()
    if which == 1:
        assert len(dec.plan.sol_interps["dst"]) > 0 and len(dec.plan.visc_interps["dst"]) > 0
    for _ in range(3):
        R.step()
        assert E.run(1) == 1
        _compare(E, R)
    t, st = E.time()
    assert st == 3 and t == pytest.approx(R.time()[0], rel=1e-14)


def test_reference_geometry_phases(backend):
    """Two-patch geometry phase by phase: the viscosity blend with
    interpolated mu_hat (phase 1) and the interpolating exchange (phase 6)."""
    kind, ctx = backend
    R = ref.RefEngine.testgeom(1, 30, weight_path=EN.DEFAULT_WEIGHTS)
    E, _ = engine_from_reference(ctx, R)
    E.step_phase(0)
    R.phase(0)
    E.step_phase(1)
    R.phase(1)
    for k in range(R.nsubs):
        assert np.array_equal(E.get(k, "tau"), R.get(k, "tau"))
        assert rel_err(E.get(k, "mu"), R.get(k, "mu")) < 1e-14
    E.step_phase(2)
    R.phase(2)
    assert E.reduce_dt() == pytest.approx(R.reduce_dt(), rel=1e-14)
    for s in range(5):
        E.step_phase(3, s)
        R.phase(3, s)
        E.step_phase(6)
        R.phase(6)
        for k in range(R.nsubs):
            assert rel_err(E.get_state(k), R.get_state(k)) < 1e-12, (s, k)


def test_mixed_shapes_storage_order(backend):
    """Subpatch ids whose shapes interleave (54, 48, 54): the engine stores
    them by shape group; per-id access, bulk state and results are unchanged."""
    kind, ctx = backend
    R = ref.RefEngine.testgeom(1, 30, weight_path=EN.DEFAULT_WEIGHTS)
    dec = RefDecomposition(R)
    perm = [1, 0, 2]  # new id -> reference id
    inv = np.argsort(perm)
    dec.subs = [dec.subs[p] for p in perm]
    pl = dec.plan
    for a in ("sol_dst_sub", "sol_src_sub", "v_dst_sub", "v_src_sub"):
        setattr(pl, a, inv[getattr(pl, a)].astype(np.int32))
    for ip in (pl.sol_interps, pl.visc_interps):
        ip["dst_sub"] = inv[ip["dst_sub"]].astype(np.int32)
        ip["src_sub"] = inv[ip["src_sub"]].astype(np.int32)
    E = EN.Engine(ctx, dec, cfg=EN.EngineConfig(cfl=0.5))
    states = [R.get_state(p) for p in perm]
    bulk = np.concatenate([s.reshape(4, -1) for s in states], axis=1)
    E.set_state_bulk(bulk)
    for k, p in enumerate(perm):
        assert np.array_equal(E.get_state(k), R.get_state(p))
    for _ in range(2):
        R.step()
        E.run(1)
    out = np.empty_like(bulk)
    E.get_state_bulk(out)
    ref_bulk = np.concatenate([R.get_state(p).reshape(4, -1) for p in perm], axis=1)
    assert rel_err(out, ref_bulk) < 1e-12
