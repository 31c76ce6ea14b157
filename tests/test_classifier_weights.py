"""FCNN v1 weight files (MlpClassifier::load / save, src/viscosity.cpp:63-106;
SURVEY.md §8(f) item 4): the product reads and writes the reference's format
byte for byte, and the reference and the engine read what it writes."""
import numpy as np
import pytest

from oracle import ref
from paper_2506_19370_b200 import classifier as CL, engine as EN, problems as P

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def test_load_save_round_trip_is_byte_exact(tmp_path):
    m = CL.load_fcnn(EN.DEFAULT_WEIGHTS)
    assert m.shape == [(16, 7), (16, 16), (16, 16), (16, 16), (4, 16)]
    CL.save_fcnn(str(tmp_path / "w.bin"), m)
    assert (tmp_path / "w.bin").read_bytes() == open(EN.DEFAULT_WEIGHTS, "rb").read()
    assert m.packed().size == sum(r * c + r for r, c in m.shape)


@needs_ref
def test_reference_reads_written_weights(tmp_path):
    m = CL.load_fcnn(EN.DEFAULT_WEIGHTS)
    rng = np.random.default_rng(4)
    for w in m.weights:
        w += 1e-3 * rng.standard_normal(w.shape)
    path = str(tmp_path / "perturbed.bin")
    CL.save_fcnn(path, m)
    x = rng.uniform(-1, 1, (64, 7))
    logits, cls = ref.mlp_forward(path, x)
    # the same forward pass by hand (MlpClassifier::forward: tanh on hidden layers)
    h = x.T
    for k, (w, b) in enumerate(zip(m.weights, m.biases)):
        h = w @ h + b[:, None]
        if k + 1 < len(m.weights):
            h = np.tanh(h)
    assert np.allclose(logits, h.T, rtol=0, atol=1e-13)
    assert np.array_equal(cls, np.argmax(h.T, axis=1) + 1)


@pytest.mark.parametrize("bad,msg", [
    (lambda b: b"XXXX" + b[4:], "bad weight file magic"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "unsupported weight file version"),
    (lambda b: b[:-8], "truncated weight file"),
], ids=["magic", "version", "truncated"])
def test_bad_files_rejected_like_the_reference(tmp_path, bad, msg):
    path = tmp_path / "bad.bin"
    path.write_bytes(bad(open(EN.DEFAULT_WEIGHTS, "rb").read()))
    with pytest.raises(CL.WeightFileError, match=msg):
        CL.load_fcnn(str(path))
    if ref.available():
        with pytest.raises(ref.RefError, match=msg):
            ref.mlp_forward(str(path), np.zeros((1, 7)))


def test_wrong_dimensions_rejected(tmp_path):
    m = CL.load_fcnn(EN.DEFAULT_WEIGHTS)
    m.weights[-1] = m.weights[-1][:3]
    m.biases[-1] = m.biases[-1][:3]
    CL.save_fcnn(str(tmp_path / "w3.bin"), m)
    with pytest.raises(CL.WeightFileError, match="dimensions"):
        CL.load_fcnn(str(tmp_path / "w3.bin"))


def test_engine_runs_on_written_weights(emu_ctx, tmp_path):
    """the engine's own loader (fcsg_engine_load_mlp) takes a file written here"""
    path = str(tmp_path / "w.bin")
    CL.save_fcnn(path, CL.load_fcnn(EN.DEFAULT_WEIGHTS))
    dec, ic, _ = P.vortex_tiles(r=1, s=1, n0=30)
    A = EN.Engine(emu_ctx, dec, ic, EN.EngineConfig(cfl=0.5, weights=path))
    B = EN.Engine(emu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    A.run(2)
    B.run(2)
    assert np.array_equal(A.get_state(0), B.get_state(0))
