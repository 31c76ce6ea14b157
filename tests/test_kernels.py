"""Parity of the product kernels (through the C ABI) against the oracle.

Every test runs twice: on the CPU emulation harness (same kernel source,
one emulated thread per CTA; small sizes, part of the CPU suite) and on the
B200 (``-m gpu``; full BASELINE sizes). Tolerances are the north_star's:
FC first derivatives <= 1e-11 relative L2 per line, solutions <= 1e-8
relative, tau bit-exact where the oracle's logit margin exceeds 1e-9.
"""
import math

import numpy as np
import pytest

from oracle import fcs_oracle as O
from paper_2506_19370_b200 import _native as N, engine as EN, fc, problems as P

from .helpers import line_rel_l2, oracle_engine, rel_err

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


def _apply(op, f, mode, axis=-1, device=False):
    if device:
        import torch

        t = torch.from_numpy(np.ascontiguousarray(f)).cuda()
        out = op.apply(t, mode, 1.0, axis)
        torch.cuda.synchronize()
        return out.cpu().numpy()
    return op.apply(f, mode, 1.0, axis)


# ---------------------------------------------------------------------------
# FC line operator


@pytest.mark.parametrize("n", [50, 64, 101, 128, 147, 256, 512])
def test_fc_lines_match_oracle_all_modes(backend, n):
    kind, ctx = backend
    n_lines = 12 if kind == "emu" else 2048
    _, f, _ = P.fc_lines_config1(n_lines=n_lines, n=n, seed=n)
    op = fc.FcOperator(ctx, n)
    o = O.get_op(n)
    for mode, ref, tol in [(1, o.derivative(f, 1), 1e-11), (2, o.derivative(f, 2), 1e-10),
                           (3, o.filter(f), 1e-13), (4, o.strong_filter(f), 1e-13)]:
        got_rows = op.apply(f, mode)
        assert line_rel_l2(got_rows, ref).max() < tol, (mode, "rows")
        got_cols = op.apply(np.ascontiguousarray(f.T), mode, axis=0).T
        assert line_rel_l2(got_cols, ref).max() < tol, (mode, "cols")


def test_fc_config1_full_size(backend):
    """BASELINE config 1 at full size on the GPU (4096 x N=256), reference
    operator: parity with the oracle and accuracy against f'."""
    kind, ctx = backend
    n_lines = 16 if kind == "emu" else 4096
    x, f, df = P.fc_lines_config1(n_lines=n_lines, n=256, seed=1)
    op = fc.FcOperator(ctx, 256)
    got = _apply(op, f, 1, device=(kind == "gpu"))
    ref = O.get_op(256).derivative(f)
    assert line_rel_l2(got, ref).max() < 1e-11
    assert np.median(line_rel_l2(got, df)) < 3e-4  # measured 8e-5
    if kind == "gpu":  # column (strided) layout of the same lines
        gotc = _apply(op, np.ascontiguousarray(f.T), 1, axis=0, device=True).T
        assert line_rel_l2(gotc, ref).max() < 1e-11


@pytest.mark.parametrize("n_lines", [1, 7, 13, 4093])
def test_fc_ragged_batches(backend, n_lines):
    """line counts that leave a warp's line group partly empty (the row
    kernels take 8 lines per warp, the column kernel 2): rows and columns
    against the oracle"""
    kind, ctx = backend
    if kind == "emu" and n_lines > 100:
        n_lines = 29
    _, f, _ = P.fc_lines_config1(n_lines=n_lines, n=256, seed=n_lines)
    op = fc.FcOperator(ctx, 256)
    ref = O.get_op(256).derivative(f)
    assert line_rel_l2(_apply(op, f, 1, device=(kind == "gpu")), ref).max() < 1e-11
    gotc = _apply(op, np.ascontiguousarray(f.T), 1, axis=0, device=(kind == "gpu")).T
    assert line_rel_l2(gotc, ref).max() < 1e-11


@pytest.mark.parametrize("n_cont,degree,n_ext", [(28, 4, 283), (27, 4, 282)])
def test_fc_degree4_config1_operator(backend, n_cont, degree, n_ext):
    """config 1's 5-point / C=27 operator (prime and 2*3*47 FFT lengths): oracle
    parity and the analytic derivative."""
    kind, ctx = backend
    n_lines = 8 if kind == "emu" else 4096
    x, f, df = P.fc_lines_config1(n_lines=n_lines, n=256, seed=3)
    op = fc.FcOperator(ctx, 256, n_cont=n_cont, degree=degree)
    assert op.n_ext() == n_ext
    o = O.get_op(256, n_cont=n_cont, degree=degree)
    assert np.abs(op.blend_matrix() - o.A).max() < 1e-13 * np.abs(o.A).max()
    got = op.apply(f, 1)
    assert line_rel_l2(got, o.derivative(f)).max() < 1e-11
    assert np.median(line_rel_l2(got, df)) < 1e-6


def test_fc_known_answers(backend):
    """tests/test_fc_core.cpp cases run through the product operator."""
    kind, ctx = backend
    op = fc.build_fc_operator(ctx, 64)
    h = 1.0 / 63
    x = np.arange(64) * h
    assert np.abs(fc.fc_derivative(op, np.full(64, 4.25), h)).max() < 1e-10
    assert np.abs(fc.fc_derivative(op, x, h) - 1.0).max() < 1e-8
    op = fc.build_fc_operator(ctx, 128)
    h = 1.0 / 127
    x = np.arange(128) * h
    f = np.sin(2 * x + 0.3)
    assert np.abs(fc.fc_derivative(op, f, h) - 2 * np.cos(2 * x + 0.3)).max() < 5e-4
    assert np.abs(fc.fc_derivative(op, f, h, 2) + 4 * np.sin(2 * x + 0.3)).max() < 0.1
    with pytest.raises(N.UsageError):
        fc.fc_derivative(op, f, h, 3)
    op = fc.build_fc_operator(ctx, 72)
    assert np.abs(fc.apply_filter(op, np.full(72, -2.5)) + 2.5).max() < 1e-12
    op = fc.build_fc_operator(ctx, 50)
    assert op.n_ext() == 74
    assert op.period() == pytest.approx((50 - 1 + 25) / 49, rel=1e-15)
    prof = op.filter_profile()
    assert prof[0] == 1.0 and np.all(np.diff(prof) <= 0)
    assert prof[-1] == pytest.approx(math.exp(-23.025850929940457), rel=1e-12)
    with pytest.raises(N.ConfigError):
        fc.build_fc_operator(ctx, 5)
    with pytest.raises(N.ConfigError):
        fc.build_fc_operator(ctx, 50, 2)
    # linearity
    op = fc.build_fc_operator(ctx, 80)
    x = np.arange(80) / 79
    a, b = np.exp(x), np.cos(5 * x)
    dfg = op.derivative(1.7 * a - 0.6 * b)
    lin = 1.7 * op.derivative(a) - 0.6 * op.derivative(b)
    assert np.abs(dfg - lin).max() / np.abs(dfg).max() < 1e-10
    # zero input continues to zero; empty batch is a no-op
    assert np.all(op.derivative(np.zeros((3, 80))) == 0.0)
    assert op.apply(np.zeros((0, 80)), 1).shape == (0, 80)


# ---------------------------------------------------------------------------
# full superstep


# stage-pass families: (force_general, reference_order). The default is the
# flux form (Cartesian: 2 passes / 16 derivatives per stage); reference_order
# keeps euler_rhs's own accumulation (3 passes / 24 or 40).
PASSES = [(False, False), (True, False), (False, True), (True, True)]
PASS_IDS = ["cartesian", "general", "cartesian-reforder", "general-reforder"]


def _compare_engines(E, OE, nsub, atol_tau_margin=1e-9):
    for k in range(nsub):
        d = OE.subs[k]
        assert rel_err(E.get_state(k), d.e) < 1e-12
        tau = E.get(k, "tau")
        sure = d.margin > atol_tau_margin
        assert np.array_equal(tau[sure], d.tau[sure])


@pytest.mark.parametrize("general,refo", PASSES, ids=PASS_IDS)
def test_superstep_phases_riemann(backend, engine_golden, general, refo):
    """Riemann quadrants on one 64x64 subpatch: every phase of two steps
    against the oracle, and step 1 against the reference's own snapshots.
    Run with every stage-pass family (Cartesian / general, flux form /
    reference accumulation order)."""
    kind, ctx = backend
    g = engine_golden
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, debug_rhs=True, force_general=general,
                                                 reference_order=refo))
    assert E.is_cartesian() == (not general)
    OE = oracle_engine(dec, ic)
    assert rel_err(E.get_state(0), g["r64_e_init"]) < 1e-15
    d = OE.subs[0]
    for step in range(2):
        E.step_phase(0)
        OE.phase0()
        assert np.array_equal(E.get(0, "tau"), d.tau)
        assert rel_err(E.get(0, "mu_hat"), d.mu_hat) < 1e-13
        E.step_phase(1)
        OE.phase1()
        assert rel_err(E.get(0, "mu"), d.mu) < 1e-13
        E.step_phase(2)
        OE.phase2()
        assert rel_err(E.get_state(0), d.e) < 1e-13
        assert E.reduce_dt() == pytest.approx(OE.reduce_dt(), rel=1e-13)
        for s in range(5):
            E.step_phase(3, s)
            E.step_phase(6)
            OE.stage(s)
            assert rel_err(E.get_state(0, "rhs"), d.rhs) < 1e-11
            assert rel_err(E.get_state(0), d.e) < 1e-13
            if step == 0:
                assert rel_err(E.get_state(0), g[f"r64_s1_e{s}"]) < 1e-13
        E.advance()
        OE.t += OE.dt
        OE.step_count += 1
    t, st = E.time()
    assert st == 2 and t == pytest.approx(OE.t, rel=1e-14)


@pytest.mark.parametrize("general,refo", PASSES, ids=PASS_IDS)
def test_superstep_tiles_exchange(backend, engine_golden, general, refo):
    """2x2 overlapping 48x48 subpatches: fringe copies + viscosity blend; graph
    path equals the phase path bit for bit; state vs the reference run."""
    kind, ctx = backend
    g = engine_golden
    dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=30)
    states = [g[f"v2_sub{k}_e_init"] for k in range(4)]
    cfg = EN.EngineConfig(cfl=0.5, force_general=general, reference_order=refo)
    E = EN.Engine(ctx, dec, cfg=cfg, initial_states=states)
    E2 = EN.Engine(ctx, dec, cfg=cfg, initial_states=states)
    E.step_by_phases()
    E.step_by_phases()
    E2.run(2)
    for k in range(4):
        assert np.array_equal(E.get_state(k), E2.get_state(k))
        assert rel_err(E.get_state(k), g[f"v2_sub{k}_e2"]) < 1e-12
        assert np.array_equal(E.get(k, "tau"), g[f"v2_sub{k}_tau2"])


@pytest.mark.gpu
@pytest.mark.parametrize("general,refo", PASSES, ids=PASS_IDS)
def test_superstep_config2_full_size(gpu_ctx, general, refo):
    """BASELINE config 2 at full size (one 512x512 subpatch, seeded quadrants,
    ANN classifier, CFL 0.5): 3 supersteps against the oracle."""
    dec, ic, _ = P.riemann_quadrants(n=512, seed=2)
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5, force_general=general, reference_order=refo))
    OE = oracle_engine(dec, ic)
    for _ in range(3):
        OE.step()
    assert E.run(3) == 3
    _compare_engines(E, OE, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("general,refo", PASSES, ids=PASS_IDS)
def test_superstep_config5_subpatch_size(gpu_ctx, general, refo):
    """config 5 geometry (256x256 subpatches, 19-point overlap) on a 2x2 tiling,
    vortex + 1e-3 noise, 2 supersteps against the oracle."""
    dec, ic, _ = P.vortex_tiles(r=2, s=2)
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5, force_general=general, reference_order=refo))
    OE = oracle_engine(dec, ic)
    OE.step()
    OE.step()
    assert E.run(2) == 2
    _compare_engines(E, OE, 4)


@pytest.mark.gpu
def test_config2_200_steps_free_stream(gpu_ctx):
    """Size-independent property at the full config-2 size and step count: a
    uniform state (zero stencil span -> class 4 -> no viscosity; FC derivatives
    of constants vanish; zero_normal_all keeps constants) is preserved for
    200 supersteps to round-off. (Mirror/transpose symmetries do NOT hold for
    the reference itself: the MLP is not reflection-symmetric and the t=0
    smear sweeps rows before columns.)"""
    dec, _, _ = P.riemann_quadrants(n=512, seed=2)
    state = np.asarray(P.conservative(0.9, 0.3, -0.2, 0.7), dtype=np.float64)
    ic = lambda x, y: np.broadcast_to(state[:, None, None], (4,) + x.shape).copy()
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    assert E.run(200) == 200
    e = E.get_state(0)
    dev = np.abs(e - state[:, None, None]).max(axis=(1, 2)) / np.abs(state)
    assert dev.max() < 1e-10
    assert np.all(E.get(0, "tau") == 4.0)
    t, st = E.time()
    assert st == 200 and t > 0


@pytest.mark.gpu
def test_config2_full_run_is_deterministic(gpu_ctx):
    """Bitwise reproducibility of the whole config-2 run (graph replay vs the
    eager launch sequence), 50 supersteps at full size."""
    dec, ic, _ = P.riemann_quadrants(n=512, seed=2)
    A = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    B = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    assert A.run(50, use_graph=True) == 50
    assert B.run(50, use_graph=False) == 50
    assert np.array_equal(A.get_state(0), B.get_state(0))
    assert np.all(np.isfinite(A.get_state(0)))


def test_invalid_state_is_reported(backend):
    """Nonpositive density raises InvalidStateError with the location
    (include/fcs/errors.hpp:32-39, src/viscosity.cpp:14)."""
    kind, ctx = backend
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    e = P.initial_state(dec, ic, 0)
    e[0, 20, 30] = -1.0
    E = EN.Engine(ctx, dec, cfg=EN.EngineConfig(cfl=0.5), initial_states=[e])
    with pytest.raises(N.InvalidStateError) as ei:
        E.step_phase(0)
    assert ei.value.subpatch == 0 and (ei.value.i, ei.value.j) == (30, 20)


def test_bad_weights_rejected(backend, tmp_path):
    kind, ctx = backend
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    bad = tmp_path / "w.bin"
    bad.write_bytes(b"XXXX" + b"\0" * 32)
    with pytest.raises(N.ConfigError):
        EN.Engine(ctx, dec, ic, EN.EngineConfig(weights=str(bad)))
    with pytest.raises(N.ConfigError):
        EN.Engine(ctx, dec, ic, EN.EngineConfig(weights=str(tmp_path / "missing.bin")))


def test_superstep_256_subpatch_compile_time_plan(emu_ctx):
    """The compile-time n_ext = 280 plan in the emulation harness: one 256x256 Riemann subpatch, 1 superstep."""
    dec, ic, _ = P.riemann_quadrants(n=256, seed=4)
    E = EN.Engine(emu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    OE = oracle_engine(dec, ic)
    OE.step()
    assert E.run(1) == 1
    _compare_engines(E, OE, 1)


@pytest.mark.parametrize("refo", [False, True], ids=["flux", "reforder"])
def test_superstep_rotated_channel_general_metrics(backend, engine_golden, refo):
    """General (curvilinear-metric) stage passes with every metric term nonzero
    and all four BC kinds (inflow, outflow pressure, slip wall, no-slip
    adiabatic wall): 3 supersteps against the reference's own run."""
    kind, ctx = backend
    g = engine_golden
    dec, ic, _ = P.rotated_channel()
    states = [g[f"rc_sub{k}_e_init"] for k in range(len(dec.subs))]
    E = EN.Engine(ctx, dec, cfg=EN.EngineConfig(cfl=0.5, reference_order=refo), initial_states=states)
    assert not E.is_cartesian()
    assert E.run(3) == 3
    for k in range(len(dec.subs)):
        assert rel_err(E.get_state(k), g[f"rc_sub{k}_e3"]) < 1e-12
        assert np.array_equal(E.get(k, "tau"), g[f"rc_sub{k}_tau3"])


@pytest.mark.parametrize("n0,n_ext", [(52, 94), (60, 102), (61, 103), (121, 163)],
                         ids=["n_ext94", "n_ext102", "n_ext103", "n_ext163"])
@pytest.mark.parametrize("general", [False, True], ids=["cartesian", "general"])
def test_superstep_small_compile_time_plans(backend, n0, n_ext, general):
    """the compile-time plans of the config-4 corner patch's line lengths
    (prime last radices 47, 17, 103 and 163 on the tensor cores):
    one subpatch of (n0 + 18)^2 points, 2 supersteps against the oracle"""
    kind, ctx = backend
    dec, ic, _ = P.vortex_tiles(r=1, s=1, n0=n0)
    assert dec.subs[0].ni + 24 == n_ext
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, force_general=general))
    OE = oracle_engine(dec, ic)
    OE.step()
    OE.step()
    assert E.run(2) == 2
    _compare_engines(E, OE, 1)


_CT_SCRIPT = """
import os, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P
ctx = N.Context(emulate=True) if {emu} else N.Context(0)
dec, ic, _ = P.vortex_tiles(r=2, s=1)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
assert E.run(2, use_graph=False) == 2
np.savez({out!r}, *[E.get_state(k) for k in range(len(dec.subs))])
"""


@pytest.mark.parametrize("kind", [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)])
def test_register_resident_passes_match_default(kind, tmp_path):
    """The Cartesian flux passes on the register-resident 8 x 35 transform
    (wctpass.cu, FCSG_WPASS_CT=1: an A/B variant read once per process, hence
    the subprocesses) against the default prime-factor passes: two 256 x 256
    vortex tiles, 2 supersteps (all five stage classes of the update)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if kind == "emu":
        from paper_2506_19370_b200 import build
        build.build(emulate=True)
    states = {}
    for ct in ("0", "1"):
        out = str(tmp_path / f"ct{ct}.npz")
        env = dict(os.environ, FCSG_WPASS_CT=ct)
        r = subprocess.run([sys.executable, "-c", _CT_SCRIPT.format(root=root, emu=(kind == "emu"), out=out)],
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        z = np.load(out)
        states[ct] = [z[k] for k in z.files]
    for a, b in zip(states["0"], states["1"]):
        assert rel_err(b, a) < 1e-13


_W20_SCRIPT = """
import os, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2506_19370_b200 import _native as N, fc, problems as P
ctx = N.Context(emulate=True) if {emu} else N.Context(0)
op = fc.FcOperator(ctx, 256)
_, f, _ = P.fc_lines_config1(n_lines=37, n=256, seed=5)
np.savez({out!r}, *[op.apply(f, mode) for mode in (1, 2, 3, 4)])
"""


@pytest.mark.parametrize("kind", [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)])
def test_line_kernel_variants_agree(kind, tmp_path):
    """The FC line batch on the 14 x 20 register-resident transform
    (w20lines.cu, FCSG_LINES_KERNEL=20: an A/B variant read once per process,
    hence the subprocesses) against the default 8 x 35 kernel: a ragged batch
    of 37 lines, all four multiplier modes."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if kind == "emu":
        from paper_2506_19370_b200 import build
        build.build(emulate=True)
    res = {}
    for k in ("35", "20"):
        out = str(tmp_path / f"k{k}.npz")
        env = dict(os.environ, FCSG_LINES_KERNEL=k)
        r = subprocess.run([sys.executable, "-c", _W20_SCRIPT.format(root=root, emu=(kind == "emu"), out=out)],
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        z = np.load(out)
        res[k] = [z[n] for n in z.files]
    # two factorisations of the same DFT: round-off apart (the derivative amplifies it by ~N)
    for a, b in zip(res["35"], res["20"]):
        assert rel_err(b, a) < 1e-11


@pytest.mark.gpu
def test_line_kernel_tma_staging_bitwise(tmp_path):
    """The 8 x 35 line kernel with its rows staged by TMA bulk copies
    (FCSG_LINES_TMA=1, an A/B variant): the same arithmetic on the same
    values, so bitwise equal to the direct-load kernel (ragged batch of 37
    lines, all four multiplier modes)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for tma in ("0", "1"):
        out = str(tmp_path / f"tma{tma}.npz")
        env = dict(os.environ, FCSG_LINES_TMA=tma)
        env.pop("FCSG_LINES_KERNEL", None)
        r = subprocess.run([sys.executable, "-c", _W20_SCRIPT.format(root=root, emu=False, out=out)],
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        z = np.load(out)
        res[tma] = [z[n] for n in z.files]
    for a, b in zip(res["0"], res["1"]):
        assert np.array_equal(a, b)
