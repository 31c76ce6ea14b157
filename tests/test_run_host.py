"""fcsg_engine_run_host: supersteps with host I/O every step, the copies
pipelined against the neighbouring steps' kernels (staging buffers, two copy
streams). The results must be bitwise those of the plain sequence
set_state_bulk -> run(1) -> get_state_bulk on a second engine."""
import numpy as np
import pytest

from paper_2506_19370_b200 import engine as EN, problems as P

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def backend(request):
    if request.param == "emu":
        return "emu", request.getfixturevalue("emu_ctx")
    return "gpu", request.getfixturevalue("gpu_ctx")


@pytest.mark.parametrize("n0", [pytest.param(30, id="4x48x48"),
                                pytest.param(238, id="4x256x256", marks=pytest.mark.gpu)])
def test_run_host_equals_sequential(backend, n0):
    kind, ctx = backend
    if kind == "emu" and n0 > 30:
        pytest.skip("GPU size")
    dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=n0)
    A = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    B = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    npts = A.total_points()
    base = np.empty((4, npts))
    A.get_state_bulk(base)
    K = 5
    rng = np.random.default_rng(0)
    ins = np.stack([base * (1.0 + 1e-3 * rng.standard_normal(base.shape) * (k > 0)) for k in range(K)])
    ins = np.ascontiguousarray(ins)
    outs = np.zeros_like(ins)
    assert A.run_host(ins, outs, steps=K, in_stride=4 * npts, out_stride=4 * npts) == K
    ref_out = np.empty((4, npts))
    for k in range(K):
        B.set_state_bulk(np.ascontiguousarray(ins[k]))
        assert B.run(1) == 1
        B.get_state_bulk(ref_out)
        assert np.array_equal(outs[k], ref_out), k
    assert A.time() == B.time()
    # stride 0: the same input every step, the last result left in place
    one = np.zeros((4, npts))
    assert A.run_host(np.ascontiguousarray(ins[0]), one, steps=3) == 3
    for _ in range(3):
        B.set_state_bulk(np.ascontiguousarray(ins[0]))
        B.run(1)
    B.get_state_bulk(ref_out)
    assert np.array_equal(one, ref_out)


def test_run_host_reports_invalid_state(backend):
    kind, ctx = backend
    dec, ic, _ = P.vortex_tiles(r=1, s=1, n0=30)
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    npts = E.total_points()
    bad = np.empty((4, npts))
    E.get_state_bulk(bad)
    bad[0, npts // 2] = -1.0  # negative density at an interior point
    out = np.zeros_like(bad)
    with pytest.raises(Exception):
        E.run_host(bad, out, steps=2)
