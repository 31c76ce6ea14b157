"""The from-scratch multi-patch builder (paper_2506_19370_b200/multipatch.py,
SURVEY.md section 8(f) item 1) against the compiled reference's own init on
the same three geometries (ref_export.cpp ref_engine_testgeom): periodic
annulus, two patches with non-coincident lattices (6x6 interpolation), C1
corner with an L-shaped subpatch.

Geometry, masks, metrics, windows and BC tables agree to round-off; the
plans agree entry for entry, except that a donor stencil choice can differ
where two candidate stencils tie to round-off (build_plan's penalty
comparison, src/runtime.cpp:121-140) -- at most 0.1% of the entries. The
engine on the builder's data then tracks the reference's run.
"""
import math

import numpy as np
import pytest

from oracle import ref
from paper_2506_19370_b200 import engine as EN, multipatch as M, problems as PR

from .helpers import RefDecomposition, rel_err

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]
GEOMS = [pytest.param(0, id="annulus"), pytest.param(1, id="two-patch"), pytest.param(2, id="corner")]
N0, NV = 30, 9


def _bcs():
    inflow = tuple(float(v) for v in PR.conservative(1.0, 0.5, 0.0, 0.7))
    return {"wall": M.BcSpec(M_SLIP), "cyl": M.BcSpec(3), "outer": M.BcSpec(5), "out": M.BcSpec(4),
            "in": M.BcSpec(0, inflow)}


M_SLIP = 2


def _geometry(which):
    """the same patches ref_engine_testgeom builds (oracle/ref_export.cpp)"""
    SI = M.SideInfo
    if which == 0:
        p = M.Patch(M.S, M.AnnulusMap((0.0, 0.0), 0.5, 1.0, -math.pi, 2 * math.pi),
                    [SI(), SI(), SI(True, "cyl"), SI(True, "outer")], periodic1=True)
        M.subdivide_Q(p, 3, 1, N0, NV)
        return [p], True
    if which == 1:
        a = M.Patch(M.I, M.AffineMap((0.0, 0.0), (1.0, 0.0), (0.0, 1.05)),
                    [SI(True, "in"), SI(), SI(True, "wall"), SI(True, "wall")])
        b = M.Patch(M.S, M.BilinearMap((0.5, 0.0), (1.8, 0.0), (0.5, 1.05), (1.5, 1.05)),
                    [SI(), SI(True, "out"), SI(True, "wall"), SI(True, "wall")])
        a.index, b.index = 0, 1
        M.subdivide_Q(a, 1, 1, N0, NV)
        M.subdivide_Q(b, 2, 1, N0 + 6, NV)
        return [a, b], True
    c, arm, ang = (0.5, 0.5), 0.3, 70.0 * math.pi / 180.0
    da, db = (1.0, 0.0), (math.cos(ang), math.sin(ang))
    A = M.Segment((c[0] + arm * da[0], c[1] + arm * da[1]), (c[0] - arm * da[0], c[1] - arm * da[1]))
    B = M.Segment((c[0] + arm * db[0], c[1] + arm * db[1]), (c[0] - arm * db[0], c[1] - arm * db[1]))
    p = M.build_c1_patch(A, B, c, "wall")
    p.sides = [SI(True, "outer") for _ in range(4)]
    p.index = 0
    M.subdivide_L(p, 2, N0, NV)
    return [p], False


def _ic(which):
    bump, u0, v0 = {0: ((0.75, 0.0), 0.2, 0.1), 1: ((0.85, 0.5), 0.5, 0.0), 2: ((0.6, 0.6), 0.3, 0.2)}[which]

    def ic(x, y):
        r2 = (x - bump[0]) * (x - bump[0]) + (y - bump[1]) * (y - bump[1])
        rho = 1.0 + 0.2 * np.exp(-r2 / 0.02)
        return PR.conservative(rho, u0, v0, 0.7)
    return ic


@pytest.mark.parametrize("which", GEOMS)
def test_builder_matches_reference_init(which):
    patches, validate = _geometry(which)
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    R = ref.RefEngine.testgeom(which, N0, weight_path=EN.DEFAULT_WEIGHTS)
    RD = RefDecomposition(R)
    assert len(D.subs) == len(RD.subs)
    for d, r in zip(D.subs, RD.subs):
        assert (d.ni, d.nj, d.cut_i, d.cut_j) == (r.ni, r.nj, r.cut_i, r.cut_j)
        assert (d.sp.i0, d.sp.j0, d.patch) == (r.sp.i0, r.sp.j0, r.patch)
        assert np.array_equal(d.mask, r.mask)
        for f in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm"):
            assert rel_err(getattr(d, f), getattr(r, f)) < 1e-13, f
        for f in ("bc_row_lo", "bc_row_hi", "bc_col_lo", "bc_col_hi"):
            assert getattr(d, f) == getattr(r, f), f
    P1, P2 = D.plan, RD.plan
    for a in ("sol_dst_sub", "sol_dst", "sol_src_sub", "sol_src", "v_dst_sub", "v_dst", "v_src_sub", "v_src"):
        assert np.array_equal(getattr(P1, a), getattr(P2, a)), a
    if len(P2.v_w):
        assert rel_err(P1.v_w, P2.v_w) < 1e-13
    for nm in ("sol_interps", "visc_interps"):
        a, b = getattr(P1, nm), getattr(P2, nm)
        for key in ("dst_sub", "dst", "src_sub"):
            assert np.array_equal(a[key], b[key]), (nm, key)
        same = (a["si0"] == b["si0"]) & (a["sj0"] == b["sj0"])
        assert (~same).sum() <= max(1, len(same) // 1000), nm
        if same.any():
            assert rel_err(a["wx"][same], b["wx"][same]) < 1e-12
            assert rel_err(a["wy"][same], b["wy"][same]) < 1e-12
        if "w" in b and len(b["w"]):
            assert rel_err(a["w"], b["w"]) < 1e-13


@pytest.mark.parametrize("which", GEOMS)
def test_engine_on_builder_tracks_reference(backend, which):
    """The product engine on the builder's decomposition and initial state
    (apply_ic) against the reference's run: 2 supersteps."""
    kind, ctx = backend
    patches, validate = _geometry(which)
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    E = EN.Engine(ctx, D, _ic(which), EN.EngineConfig(cfl=0.5))
    R = ref.RefEngine.testgeom(which, N0, weight_path=EN.DEFAULT_WEIGHTS)
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-13
    for _ in range(2):
        R.step()
        E.run(1)
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-9


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


def test_engine_rejects_inconsistent_inputs(emu_ctx):
    """Usage errors of the general engine inputs (include/fcsg.h): an L-cut
    that disagrees with the mask, a malformed cut, interpolation stencils
    outside the donor, interpolation donors on another rank."""
    from paper_2506_19370_b200 import _native as N

    patches, validate = _geometry(2)
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    d = D.subs[0]
    bad = M.SubData(**{**d.__dict__, "cut_i": d.cut_i - 1})  # mask says otherwise
    with pytest.raises(N.UsageError):
        EN.Engine(emu_ctx, M.MultiPatchDecomposition(D.patches, [bad], D.plan, D.bcs))
    bad = M.SubData(**{**d.__dict__, "cut_j": 0})  # only one of the two cuts
    with pytest.raises(N.UsageError):
        EN.Engine(emu_ctx, M.MultiPatchDecomposition(D.patches, [bad], D.plan, D.bcs))
    patches, validate = _geometry(1)
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    si = {k: v.copy() for k, v in D.plan.sol_interps.items()}
    si["si0"][0] = D.subs[si["src_sub"][0]].ni - 3  # stencil would leave the donor
    plan = M.Plan(**{**D.plan.__dict__, "sol_interps": si})
    with pytest.raises(N.UsageError):
        EN.Engine(emu_ctx, M.MultiPatchDecomposition(D.patches, D.subs, plan, D.bcs))
    si = {k: v.copy() for k, v in D.plan.sol_interps.items()}
    si["src_sub"][0] = -1  # donors must be local
    plan = M.Plan(**{**D.plan.__dict__, "sol_interps": si})
    with pytest.raises(N.UsageError):
        EN.Engine(emu_ctx, M.MultiPatchDecomposition(D.patches, D.subs, plan, D.bcs))


@pytest.mark.parametrize("which", GEOMS)
def test_vectorised_builder_equals_scalar(which):
    """build_decomposition(fast=True) -- the numpy path used for large
    decompositions -- produces the scalar path's geometry and plan."""
    patches, validate = _geometry(which)
    A = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    patches, validate = _geometry(which)
    B = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate, fast=True)
    for a, b in zip(A.subs, B.subs):
        assert np.array_equal(a.mask, b.mask)
        for f in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm"):
            assert rel_err(getattr(b, f), getattr(a, f)) < 1e-14, f
        for f in ("bc_row_lo", "bc_row_hi", "bc_col_lo", "bc_col_hi"):
            assert getattr(a, f) == getattr(b, f)
    for f in ("sol_dst_sub", "sol_dst", "sol_src_sub", "sol_src", "v_dst_sub", "v_dst", "v_src_sub", "v_src"):
        assert np.array_equal(getattr(A.plan, f), getattr(B.plan, f)), f
    assert np.array_equal(A.plan.v_w, B.plan.v_w)
    for nm in ("sol_interps", "visc_interps"):
        a, b = getattr(A.plan, nm), getattr(B.plan, nm)
        for k in a:
            if k in ("wx", "wy", "w"):
                assert rel_err(b[k], a[k]) < 1e-13 if len(a[k]) else len(b[k]) == 0
            else:
                assert np.array_equal(a[k], b[k]), (nm, k)


@pytest.mark.gpu
@pytest.mark.parametrize("full", [False, True], ids=["0.70M", "2.57M"])
def test_config3_cylinder_against_reference(gpu_ctx, full):
    """BASELINE config 3's layout (problems.cylinder_flow; the full size and
    a 0.70M-point variant): the builder reproduces the reference's init
    (which builds the same patches, ref_engine_testgeom 3 / 4) -- geometry,
    masks, windows, BCs and every plan entry -- and the engine on it tracks
    the reference's run for 2 supersteps of Mach 3 flow (impulsive start,
    t = 0 smear). The full size runs the annulus group (147 x 147
    subpatches) on the compile-time n_ext = 171 = 9 x 19 plan."""
    import os
    dec, ic, meta = PR.cylinder_flow(full=full)
    R = ref.RefEngine.testgeom(4 if full else 3, 0, workers=os.cpu_count() or 1, weight_path=EN.DEFAULT_WEIGHTS)
    RD = RefDecomposition(R)
    for d, r in zip(dec.subs, RD.subs):
        assert np.array_equal(d.mask, r.mask)
        # (the vectorised builder's cos / sin may differ from libm's by an ulp;
        # the local spacings are differences of neighbouring points)
        for f in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm"):
            assert rel_err(getattr(d, f), getattr(r, f)) < 1e-12, f
    for f in ("sol_dst_sub", "sol_dst", "sol_src_sub", "sol_src", "v_dst_sub", "v_dst", "v_src_sub", "v_src"):
        assert np.array_equal(getattr(dec.plan, f), getattr(RD.plan, f)), f
    for nm in ("sol_interps", "visc_interps"):
        a, b = getattr(dec.plan, nm), getattr(RD.plan, nm)
        assert np.array_equal(a["si0"], b["si0"]) and np.array_equal(a["sj0"], b["sj0"])
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=meta["cfl"]))
    assert not E.is_cartesian()
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-14
    R.run(2)
    assert E.run(2) == 2
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-10, k


@pytest.mark.gpu
def test_config4_step_against_reference(gpu_ctx):
    """BASELINE config 4's layout (problems.step_flow(1): convex C1 corner
    patch with an L-shaped subpatch at the step's top, concave C2 corner patch
    at its foot, S and I patches of 256 x 256 subpatches; 0.80M points): the
    reference builds the same patches
    (ref_engine_testgeom 5, its overlap checks including the S-C1 corner rule
    pass), the builder reproduces its init (up to viscosity stencils tied to
    round-off), and the engine tracks its run for 2 supersteps of Mach 3
    flow."""
    import os
    dec, ic, meta = PR.step_flow(1)
    R = ref.RefEngine.testgeom(5, 0, cfl=meta["cfl"], workers=os.cpu_count() or 1, weight_path=EN.DEFAULT_WEIGHTS)
    RD = RefDecomposition(R)
    assert any(d.cut_i > 0 for d in dec.subs)
    for d, r in zip(dec.subs, RD.subs):
        assert (d.cut_i, d.cut_j) == (r.cut_i, r.cut_j)
        assert np.array_equal(d.mask, r.mask)
        for f in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm"):
            assert rel_err(getattr(d, f), getattr(r, f)) < 1e-12, f
    for f in ("sol_dst_sub", "sol_dst", "sol_src_sub", "sol_src", "v_dst_sub", "v_dst", "v_src_sub", "v_src"):
        assert np.array_equal(getattr(dec.plan, f), getattr(RD.plan, f)), f
    ties = 0
    for nm in ("sol_interps", "visc_interps"):
        a, b = getattr(dec.plan, nm), getattr(RD.plan, nm)
        same = (a["si0"] == b["si0"]) & (a["sj0"] == b["sj0"])
        ties += int((~same).sum())
        # donor stencils tied to round-off: recipients on the donor's lattice
        # lines, located through the corner patches' Newton inversion
        assert (~same).sum() <= max(1, len(same) // 200), nm
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=meta["cfl"]))
    for k in range(R.nsubs):  # after apply_ic's BCs (slip-wall normals from the metrics)
        assert rel_err(E.get_state(k), R.get_state(k)) < 1e-12
    R.run(2)
    assert E.run(2) == 2
    for k in range(R.nsubs):
        assert rel_err(E.get_state(k), R.get_state(k)) < (1e-10 if ties == 0 else 1e-8), k
