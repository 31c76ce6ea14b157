"""Pin the numpy oracle (oracle/fcs_oracle.py) to the unmodified reference:
against the committed golden fixtures (always) and against oracle/_ref live
(when it is built). CPU only."""
import math

import numpy as np
import pytest

from oracle import fcs_oracle as O
from oracle import ref
from paper_2506_19370_b200 import problems as P

from .helpers import line_rel_l2, oracle_engine, rel_err

NS = (50, 64, 100, 101, 128, 147, 256, 512)


def test_blend_matrix_matches_reference(fc_golden):
    A = O.blend_matrix(25)
    assert A.shape == (24, 3)
    assert rel_err(A, fc_golden["blend_25"]) < 1e-15


@pytest.mark.parametrize("n", NS)
def test_operator_sizes_and_profiles(fc_golden, n):
    op = O.get_op(n)
    ne, per = fc_golden[f"n{n}_info"]
    assert op.n_ext == int(ne) == n + 24
    assert op.period == pytest.approx(per, rel=1e-15)
    assert np.abs(op.filter_profile - fc_golden[f"n{n}_filter_profile"]).max() < 1e-15
    assert np.abs(op.smear_profile - fc_golden[f"n{n}_smear_profile"]).max() < 1e-15


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("mode", ["d1", "d2", "filter", "smear", "cont"])
def test_line_operators_match_reference(fc_golden, n, mode):
    op = O.get_op(n)
    f = fc_golden[f"n{n}_in"]
    fn = {"d1": lambda x: op.derivative(x, 1), "d2": lambda x: op.derivative(x, 2), "filter": op.filter,
          "smear": op.strong_filter, "cont": op.continuation}[mode]
    # d2 (unused by the step) amplifies round-off by (2 pi k / period)^2 ~ 1e6
    tol = 1e-10 if mode == "d2" else 1e-13
    assert line_rel_l2(fn(f), fc_golden[f"n{n}_{mode}"]).max() < tol


def test_reference_known_answers_on_oracle():
    """tests/test_fc_core.cpp KATs restated on the oracle (the analytic ones)."""
    op = O.get_op(64)
    x = np.arange(64) / 63
    assert np.abs(op.derivative(np.full(64, 4.25))).max() < 1e-10  # :95-100
    assert np.abs(op.derivative(x) - 1.0).max() < 1e-8  # :102-109
    op = O.get_op(128)
    x = np.arange(128) / 127
    f = np.sin(2 * x + 0.3)
    assert np.abs(op.derivative(f) - 2 * np.cos(2 * x + 0.3)).max() < 5e-4  # :111-121
    assert np.abs(op.derivative(f, 2) + 4 * np.sin(2 * x + 0.3)).max() < 0.1  # :122-128
    prev = None  # spectral convergence :151-170
    for n in (32, 64, 128):
        o = O.get_op(n)
        x = np.arange(n) / (n - 1)
        e = np.abs(o.derivative(np.exp(np.sin(2 * np.pi * x))) -
                   2 * np.pi * np.cos(2 * np.pi * x) * np.exp(np.sin(2 * np.pi * x))).max()
        if prev is not None:
            assert e < prev / 8.0
        prev = e
    assert prev < 6e-4
    op = O.get_op(72)
    assert np.abs(op.filter(np.full(72, -2.5)) + 2.5).max() < 1e-12  # :172-177
    op = O.get_op(50)
    assert op.filter_profile[-1] == pytest.approx(math.exp(-23.025850929940457), rel=1e-12)  # :38-53
    assert np.all(np.diff(op.filter_profile) <= 0)
    with pytest.raises(ValueError):
        O.FcOp(5)
    with pytest.raises(ValueError):
        O.FcOp(50, 2)


def test_degree4_operator_analytic():
    """BASELINE config-1 operator (5 matching points, C=27 gap points): not
    constructible by the reference -- pinned analytically."""
    x, f, df = P.fc_lines_config1(n_lines=16, n=256, seed=7)
    op = O.get_op(256, n_cont=28, degree=4)
    assert op.n_ext == 283
    got = op.derivative(f)
    assert np.median(line_rel_l2(got, df)) < 1e-6
    op2 = O.get_op(256)
    got2 = op2.derivative(f)
    assert np.median(line_rel_l2(got2, df)) < 3e-4
    # degree-4 polynomial exactness of the continuation derivative
    p4 = 1 + x - 2 * x ** 2 + 0.5 * x ** 3 - 0.25 * x ** 4
    dp4 = 1 - 4 * x + 1.5 * x ** 2 - x ** 3
    assert np.abs(op.derivative(p4) - dp4).max() < 1e-6


def test_engine_phases_match_reference(engine_golden):
    """One step of the Riemann-quadrant problem on a 64x64 subpatch, phase by
    phase, against the reference Engine (src/runtime.cpp:316-458)."""
    g = engine_golden
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    E = oracle_engine(dec, states=[g["r64_e_init"]])
    d = E.subs[0]
    E.phase0()
    assert np.array_equal(d.tau, g["r64_s1_tau"])
    assert rel_err(d.mu_hat, g["r64_s1_mu_hat"]) < 1e-13
    E.phase1()
    assert rel_err(d.mu, g["r64_s1_mu"]) < 1e-13
    E.phase2()
    assert np.array_equal(d.m01, g["r64_s1_m01"])
    assert rel_err(d.e, g["r64_s1_e_p2"]) < 1e-13
    assert E.reduce_dt() == pytest.approx(float(g["r64_s1_dt"][0]), rel=1e-14)
    for s in range(5):
        E.stage(s)
        assert rel_err(d.rhs, g[f"r64_s1_rhs{s}"]) < 1e-11
        assert rel_err(d.e, g[f"r64_s1_e{s}"]) < 1e-13
    E.t += E.dt
    E.step_count += 1
    E.step()
    E.step()
    assert rel_err(d.e, g["r64_s3_e"]) < 1e-12


def test_engine_tiles_match_reference(engine_golden):
    """2x2 overlapping subpatches (intra-patch copy exchange and viscosity blend)."""
    g = engine_golden
    dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=30)
    E = oracle_engine(dec, states=[g[f"v2_sub{k}_e_init"] for k in range(4)])
    E.step()
    E.step()
    for k in range(4):
        assert rel_err(E.subs[k].e, g[f"v2_sub{k}_e2"]) < 1e-12
        assert np.array_equal(E.subs[k].tau, g[f"v2_sub{k}_tau2"])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_oracle_against_live_reference():
    rng = np.random.default_rng(3)
    for n in (88, 200):
        f = rng.standard_normal((4, n)).cumsum(1)
        op = O.get_op(n)
        assert line_rel_l2(op.derivative(f), ref.fc_apply(f, "d1")).max() < 1e-13
        assert line_rel_l2(op.filter(f), ref.fc_apply(f, "filter")).max() < 1e-13


def test_engine_rotated_channel_matches_reference(engine_golden):
    """Rotated affine channel (every metric term nonzero; inflow, outflow
    pressure, slip and no-slip walls): 3 supersteps against the reference."""
    g = engine_golden
    dec, ic, _ = P.rotated_channel()
    for k, d in enumerate(dec.subs):
        for f in ("iq1x", "iq2x", "iq1y", "iq2y", "w_norm"):
            assert rel_err(getattr(d, f), g[f"rc_sub{k}_geo_{f}"]) < 1e-14
        assert np.array_equal(d.mask, g[f"rc_sub{k}_geo_mask"].astype(np.uint8))
    E = oracle_engine(dec, states=[g[f"rc_sub{k}_e_init"] for k in range(len(dec.subs))])
    for _ in range(3):
        E.step()
    for k in range(len(dec.subs)):
        assert rel_err(E.subs[k].e, g[f"rc_sub{k}_e3"]) < 1e-12
        assert np.array_equal(E.subs[k].tau, g[f"rc_sub{k}_tau3"])
