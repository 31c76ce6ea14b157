"""Host-side logic on CPU: init-time geometry/plan against the reference
fixtures, the C-ABI surface of the product library, problem generators."""
import os
import re

import numpy as np
import pytest

from paper_2506_19370_b200 import geometry as G, problems as P

from .helpers import rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_geometry_single_subpatch_matches_reference(engine_golden):
    g = engine_golden
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    d = dec.subs[0]
    assert (d.ni, d.nj) == (64, 64)
    for k in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm"):
        assert np.abs(getattr(d, k) - g[f"r64_geo_{k}"]).max() <= 4e-16 * max(1.0, np.abs(g[f"r64_geo_{k}"]).max()), k
    assert np.array_equal(d.mask, g["r64_geo_mask"].astype(np.uint8))
    # the fixture's initial state is the IC after enforce_bc (apply_ic); interior points are the raw IC
    assert np.array_equal(P.initial_state(dec, ic, 0)[:, 1:-1, 1:-1], g["r64_e_init"][:, 1:-1, 1:-1])
    assert len(dec.plan.sol_dst) == 0 and len(dec.plan.v_dst) == 0


def test_geometry_tiles_match_reference(engine_golden):
    """subdivide_Q(2,2,30,9): fringe masks, local spacing and the normalised
    window w_norm of every subpatch equal the reference's."""
    g = engine_golden
    dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=30)
    for k, d in enumerate(dec.subs):
        assert np.array_equal(d.mask, g[f"v2_sub{k}_geo_mask"].astype(np.uint8))
        assert rel_err(d.w_norm, g[f"v2_sub{k}_geo_w_norm"]) < 1e-14
        assert rel_err(d.h_min, g[f"v2_sub{k}_geo_h_min"]) < 1e-15
        assert rel_err(d.x, g[f"v2_sub{k}_geo_x"]) < 1e-15


def test_plan_copies_cover_fringe_with_interior_donors():
    dec, ic, _ = P.vortex_tiles(r=3, s=2, n0=30)
    pl = dec.plan
    for k, d in enumerate(dec.subs):
        fr = np.flatnonzero(d.mask.ravel() == 2)
        dst = np.sort(pl.sol_dst[pl.sol_dst_sub == k])
        assert np.array_equal(fr, dst), "every fringe point gets exactly one copy"
    for s, src in zip(pl.sol_src_sub, pl.sol_src):
        assert dec.subs[s].mask.ravel()[src] == 1, "donor purity (src/runtime.cpp:239-247)"
    # the blend weights form a partition of unity at every point
    tot = [d.w_norm.ravel().copy() for d in dec.subs]
    for ds, dst, w in zip(pl.v_dst_sub, pl.v_dst, pl.v_w):
        tot[ds][dst] += w
    for t in tot:
        assert np.abs(t - 1.0).max() < 1e-14
    # copied donors sit on the same lattice point
    for ds, dst, ss, src in zip(pl.sol_dst_sub, pl.sol_dst, pl.sol_src_sub, pl.sol_src):
        a, b = dec.subs[ds], dec.subs[ss]
        assert a.x.ravel()[dst] == pytest.approx(b.x.ravel()[src], abs=1e-12)
        assert a.y.ravel()[dst] == pytest.approx(b.y.ravel()[src], abs=1e-12)


def test_decomposition_errors():
    with pytest.raises(ValueError):
        G.rect_decomposition((0, 0), 1, 1, 1, 1, 40, 5, [G.BcSpec()] * 4, nf=5)  # nv <= nf
    # a 10-point overlap leaves 2 points per row where every
    # window vanishes (src/viscosity.cpp:253-260) -> "window partition vanishes"
    p = G.AffinePatch((0, 0), (1, 0), (0, 1), [G.SideInfo(True, "w")] * 4)
    G.subdivide_Q(p, 2, 1, 30, 9)
    p.subpatches[1].i0 += 9
    assert p.subpatches[0].i1 - p.subpatches[1].i0 + 1 == 10
    subs = [G.init_subpatch_data(p, sp, 5, {"w": G.BcSpec()}) for sp in p.subpatches]
    with pytest.raises(G.DecompositionError):
        G.build_plan(p, subs, 5)
    # the native 2nv+1 = 19-point overlap is fine
    G.subdivide_Q(p, 2, 1, 30, 9)
    subs = [G.init_subpatch_data(p, sp, 5, {"w": G.BcSpec()}) for sp in p.subpatches]
    G.build_plan(p, subs, 5)


def test_splitmix_matches_reference_rng():
    # src/viscosity.cpp:300-313; first outputs of seed 1 (standard splitmix64 sequence)
    r = P.SplitMix64(1)
    assert r.next() == 0x910A2DEC89025CC1
    assert r.next() == 0xBEEB8DA1658EEC67
    u = P.splitmix_uniform_array(np.array([5, 7], dtype=np.uint64), 3)
    for k, s in enumerate((5, 7)):
        rr = P.SplitMix64(s)
        assert np.allclose(u[k], [rr.uniform() for _ in range(3)], rtol=0, atol=0)


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fcsg.h")).read()
    return sorted(set(re.findall(r"\bint\s+(fcsg_\w+)\s*\(", src)))


def test_abi_library_exports_every_declared_symbol():
    """libfcsg.so (the sm_100a build) loads and exports every entry point
    include/fcsg.h declares. No compute call is made (no GPU here)."""
    import ctypes

    from paper_2506_19370_b200 import _native as N

    if not os.path.exists(N.LIB_PATH):
        from paper_2506_19370_b200 import build

        build.build()
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.fcsg_is_cuda_build() == 1


def test_emulation_harness_exports_same_abi(emu_ctx):
    syms = _header_symbols()
    missing = [s for s in syms if not hasattr(emu_ctx.lib, s)]
    assert not missing, missing
    assert emu_ctx.lib.fcsg_is_cuda_build() == 0


def test_product_refuses_to_run_without_cuda():
    """No CPU fallback: the product context requires a CUDA device."""
    import torch

    from paper_2506_19370_b200 import _native as N

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises((RuntimeError, ImportError)):
        N.Context(0)
