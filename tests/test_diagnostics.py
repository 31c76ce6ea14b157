"""Measurements and writers (src/workbench.cpp:187-412)
against the reference's own functions (oracle/_ref), on the B200 and in the
CPU emulation of the kernels: window-quadrature energy and area integrals,
the |grad rho| raster (device gradient + device sampling on the host-built
pixel plan), Schlieren PGM bytes, the shock-angle fit and the per-subpatch
CSV text."""
import json
import math

import numpy as np
import pytest

from oracle import ref
from paper_2506_19370_b200 import diagnostics as DG, engine as EN, multipatch as M

from .helpers import engine_from_reference, rel_err
from .test_multipatch import N0, NV, _bcs, _geometry

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]
GEOMS = [pytest.param(0, id="annulus"), pytest.param(1, id="two-patch"), pytest.param(2, id="corner")]


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


def _pair(ctx, which, steps=2):
    """reference engine and product engine (on the builder's decomposition of
    the same geometry) at the same state after `steps` supersteps"""
    R = ref.RefEngine.testgeom(which, N0, weight_path=EN.DEFAULT_WEIGHTS)
    patches, validate = _geometry(which)
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=validate)
    E = EN.Engine(ctx, D, cfg=EN.EngineConfig(cfl=0.5))
    for k in range(R.nsubs):
        E.set_state(k, R.get_state(k))
    for _ in range(steps):
        R.step()
    E.run(steps)
    return R, E, D


@pytest.mark.parametrize("which", GEOMS)
def test_integrals_match_reference(backend, which):
    kind, ctx = backend
    R, E, D = _pair(ctx, which)
    DG.set_quadrature(E, D)
    energy, area = R.integrals()
    assert DG.area_integral(E) == pytest.approx(area, rel=1e-12)
    assert DG.energy_integral(E) == pytest.approx(energy, rel=1e-11)
    for k, d in enumerate(D.subs):  # the builder's |det J| is the reference's
        assert rel_err(d.det, R.get(k, "det")) < 1e-12


@pytest.mark.parametrize("which", GEOMS)
def test_gradient_raster_matches_reference(backend, which):
    kind, ctx = backend
    R, E, D = _pair(ctx, which)
    nx, ny = 64, 48
    rv, meta = R.raster(nx, ny)
    ours = DG.density_gradient_raster(E, D, nx, ny)
    assert np.allclose([ours.x0, ours.y0, ours.dx, ours.dy], meta, rtol=1e-12, atol=1e-14)
    # |grad rho| at the points themselves (FC derivatives + metrics)
    for k in range(R.nsubs):
        g = E.get(k, "grad")
        rg = R.get(k, "grad")
        assert rel_err(g * (D.subs[k].mask != 0), rg * (D.subs[k].mask != 0)) < 1e-9, k
    diff = np.abs(ours.v - rv)
    scale = np.abs(rv).max()
    assert scale > 0
    # pixels whose containing patch / deepest subpatch is decided by a
    # round-off-level tie may differ; nothing else
    assert (diff > 1e-9 * scale).mean() < 0.005
    assert np.median(diff) <= 1e-12 * scale


def test_schlieren_pgm_bytes_and_shock_angle(tmp_path):
    rng = np.random.default_rng(3)
    ny, nx = 40, 64
    meta = np.array([-1.0, 0.5, 0.05, 0.025])
    xs = meta[0] + np.arange(nx) * meta[2]
    ys = meta[1] + np.arange(ny) * meta[3]
    # a ramp of |grad| along an oblique line plus noise
    Y, X = np.meshgrid(ys, xs, indexing="ij")
    v = np.exp(-((Y - (0.8 + 0.3 * (X + 1.0))) / 0.05) ** 2) + 0.01 * rng.random((ny, nx))
    r = DG.Raster(nx, ny, *meta, v)
    for beta in (10.0, 3.5):
        DG.write_pgm(DG.schlieren(r, beta), str(tmp_path / "ours.pgm"))
        ref.write_schlieren_pgm(v, meta, beta, str(tmp_path / "ref.pgm"))
        assert (tmp_path / "ours.pgm").read_bytes() == (tmp_path / "ref.pgm").read_bytes()
    flat = DG.Raster(nx, ny, *meta, np.full((ny, nx), 2.0))
    assert (DG.schlieren(flat).v == 1.0).all()
    box = (-0.5, 1.5, 0.6, 1.4)
    # the reference is built with FMA contraction (x86-64-v3): round-off only
    assert DG.fit_shock_angle(r, *box) == pytest.approx(ref.fit_shock_angle(v, meta, *box), rel=1e-13)
    assert DG.fit_shock_angle(r, *box) == pytest.approx(math.degrees(math.atan(0.3)), abs=1.0)
    with pytest.raises(ValueError, match="fewer than 5"):
        DG.fit_shock_angle(r, -0.99, -0.9, 0.6, 1.4)


@pytest.mark.parametrize("which", [pytest.param(1, id="two-patch"), pytest.param(2, id="corner")])
def test_subpatch_csv_matches_reference(backend, which, tmp_path):
    """write_subpatch_csv of the same state (the reference's right after
    Engine::init, written by a child process): same header, same points in
    the same order, every column printed identically (17 significant digits)
    except p, which the reference computes with FMA contraction (round-off)"""
    kind, ctx = backend
    R = ref.RefEngine.testgeom(which, N0, weight_path=EN.DEFAULT_WEIGHTS)
    E, dec = engine_from_reference(ctx, R)
    DG.write_subpatch_csv(E, dec, str(tmp_path / "ours"))
    ref.testgeom_write_csv(which, N0, str(tmp_path / "ref"), EN.DEFAULT_WEIGHTS)
    for k in range(R.nsubs):
        a = (tmp_path / "ours" / f"sub_{k}.csv").read_text().splitlines()
        b = (tmp_path / "ref" / f"sub_{k}.csv").read_text().splitlines()
        assert a[0] == b[0] == "x,y,rho,u,v,p,mu,tau"
        assert len(a) == len(b) > 100, k
        ca = [r.split(",") for r in a[1:]]
        cb = [r.split(",") for r in b[1:]]
        for col in (0, 1, 2, 3, 4, 6, 7):
            assert [r[col] for r in ca] == [r[col] for r in cb], (k, col)
        pa = np.array([float(r[5]) for r in ca])
        pb = np.array([float(r[5]) for r in cb])
        assert np.abs(pa - pb).max() <= 4e-16 * np.abs(pb).max(), k


def test_manifest(tmp_path):
    DG.write_manifest(str(tmp_path), "vortex", 10, 0.25, 1.5, 0.15, 4096, 4, energy_series=[(0.0, 1.0), (0.1, 0.99)])
    j = json.loads((tmp_path / "manifest.json").read_text())
    assert j["format"] == "fcs-manifest" and j["version"] == 1 and j["energy_series"] == "energy.csv"
    assert (tmp_path / "energy.csv").read_text() == "t,E\n0,1\n0.10000000000000001,0.98999999999999999\n"


def test_quadrature_requires_all_weights(backend):
    kind, ctx = backend
    R = ref.RefEngine.testgeom(1, N0, weight_path=EN.DEFAULT_WEIGHTS)
    E, dec = engine_from_reference(ctx, R)
    with pytest.raises(Exception, match="quadrature"):
        E.integrals(3)
    dec.subs[0].det = R.get(0, "det")
    E.set_quadrature(0, DG.quadrature_weights(dec.subs[0]))
    with pytest.raises(Exception, match="quadrature"):
        E.integrals(3)
    with pytest.raises(Exception, match="gradient"):
        E.get(0, "grad")
