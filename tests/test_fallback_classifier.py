"""FC-spectrum ("fallback") classifier -- ClassifierConfig's default variant
(include/fcs/viscosity.hpp:45-52; Classifier::classify_line,
src/viscosity.cpp:161-208, over FcOperator::spectrum, src/fc_core.cpp:308-316).
SURVEY.md §8(f) item 3.

Pins: the numpy restatement (oracle/fcs_oracle.py classify_lines_spectrum)
against the reference's own classify_line (committed fixture
tests/golden/classifier_golden.npz, and the compiled reference when present).
Product: the engine with EngineConfig(classifier="fallback") against the
reference engine with the fallback variant (empty weight path) on geometries
the reference builds, phase by phase and over whole supersteps, on the B200
and in the CPU emulation of the kernels. Class decisions are compared where
the decision variables (decay exponent, tail peak) are more than 1e-9 from a
threshold; the product computes continuation + DFT of the tail modes as one
matrix product, so its round-off differs from FFTW's.
"""
import os

import numpy as np
import pytest

from oracle import fcs_oracle as O
from oracle import ref
from paper_2506_19370_b200 import engine as EN, problems as P

from .helpers import engine_from_reference, rel_err

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "classifier_golden.npz")
BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


def test_oracle_matches_reference_golden():
    g = np.load(GOLDEN)
    n_lines = len([k for k in g.files if k.endswith("_w32")])
    checked = 0
    for k in range(n_lines):
        v = g[f"line{k}"]
        for w in (32, 16):
            tau, margin = O.classify_lines_spectrum(v[None, :], w)
            ok = margin[0] > 1e-9
            assert np.array_equal(tau[0][ok], g[f"line{k}_w{w}"][ok]), (k, w)
            checked += int(ok.sum())
    assert checked > 0.99 * sum(len(g[f"line{k}"]) for k in range(n_lines)) * 2
    classes = np.concatenate([g[f"line{k}_w32"] for k in range(n_lines)])
    assert set(np.unique(classes)) == {1, 2, 3, 4}


@needs_ref
def test_oracle_matches_compiled_reference():
    rng = np.random.default_rng(11)
    for n in (12, 25, 32, 48, 64, 150):
        for _ in range(6):
            x = np.linspace(0.0, 1.0, n)
            v = np.tanh((x - rng.uniform(0.2, 0.8)) * 10 ** rng.uniform(0, 2.5)) + rng.normal(0, 1e-4, n)
            for w in (32, 20, 64, 11):
                tau, margin = O.classify_lines_spectrum(v[None, :], w)
                r = ref.classify_line_fallback(v, w)
                ok = margin[0] > 1e-9
                assert np.array_equal(tau[0][ok], r[ok]), (n, w)
                if w == 11:
                    assert (r == 4).all()


def _fallback_cfg(**kw):
    return EN.EngineConfig(cfl=0.5, classifier="fallback", **kw)


@needs_ref
@pytest.mark.parametrize("which", [pytest.param(0, id="annulus"), pytest.param(1, id="two-patch"),
                                   pytest.param(2, id="corner")])
def test_fallback_engine_reference_geometry(backend, which):
    """Phase 0 (tau, mu_hat) and 3 supersteps on reference-built geometries,
    both engines with the fallback classifier (lines of 30..48 points: window
    lengths below and at 32)."""
    kind, ctx = backend
    R = ref.RefEngine.testgeom(which, 30, weight_path="")
    E, _ = engine_from_reference(ctx, R, _fallback_cfg())
    E.step_phase(0)
    R.phase(0)
    for k in range(R.nsubs):
        assert np.array_equal(E.get(k, "tau"), R.get(k, "tau")), k
        assert rel_err(E.get(k, "mu_hat"), R.get(k, "mu_hat")) < 1e-14, k
    R2 = ref.RefEngine.testgeom(which, 30, weight_path="")
    E2, _ = engine_from_reference(ctx, R2, _fallback_cfg())
    for _ in range(3):
        R2.step()
        assert E2.run(1) == 1
        for k in range(R2.nsubs):
            assert np.array_equal(E2.get(k, "tau"), R2.get(k, "tau")), k
            assert rel_err(E2.get_state(k), R2.get_state(k)) < 1e-12, k


def _ref_vortex(n0, r=2, s=2):
    dec, ic, _ = P.vortex_tiles(r=r, s=s, n0=n0)
    p = dec.patches[0]
    kinds = [5 if sd.on_gamma else -1 for sd in p.sides]
    R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], r, s, n0, p.nv, kinds, cfl=0.5, workers=1,
                      weight_path="")
    for k in range(len(dec.subs)):
        R.set_state(k, P.initial_state(dec, ic, k))
    R.finish_ic()
    return R


@needs_ref
@pytest.mark.parametrize("n0", [pytest.param(30, id="48x48"),
                                pytest.param(238, id="256x256", marks=pytest.mark.gpu)])
def test_fallback_engine_vortex_tiles(backend, n0):
    """Vortex + 1e-3 noise on 2x2 subpatches (config-5 layout at n0 = 238):
    every class occurs; t = 0 smear (the classifier also runs on rho) and two
    steady supersteps track the reference."""
    kind, ctx = backend
    if kind == "emu" and n0 > 30:
        pytest.skip("full-size tiles on the GPU only")
    R = _ref_vortex(n0)
    E, _ = engine_from_reference(ctx, R, _fallback_cfg())
    seen = set()
    for _ in range(3):
        R.step()
        assert E.run(1) == 1
        for k in range(R.nsubs):
            t = E.get(k, "tau")
            seen |= set(np.unique(t).astype(int))
            assert np.array_equal(t, R.get(k, "tau")), k
            assert rel_err(E.get_state(k), R.get_state(k)) < 1e-12, k
    assert len(seen) >= 3


def test_fallback_needs_no_weights_but_ann_does(backend, tmp_path):
    kind, ctx = backend
    dec, ic, _ = P.vortex_tiles(r=1, s=1, n0=30)
    E = EN.Engine(ctx, dec, ic, _fallback_cfg(weights=str(tmp_path / "missing.bin")))
    assert E.run(1) == 1
    with pytest.raises(Exception, match="weights"):
        EN.Engine(ctx, dec, ic, EN.EngineConfig(weights=str(tmp_path / "missing.bin")))


def test_fallback_window_limits(backend):
    kind, ctx = backend
    dec, ic, _ = P.vortex_tiles(r=1, s=1, n0=30)
    with pytest.raises(Exception, match="64"):
        EN.Engine(ctx, dec, ic, _fallback_cfg(classifier_window=65))
    # window < 12: every window shorter than 12 points -> class 4 everywhere
    E = EN.Engine(ctx, dec, ic, _fallback_cfg(classifier_window=8))
    E.step_phase(0)
    assert (E.get(0, "tau") == 4).all()
