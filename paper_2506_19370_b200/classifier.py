"""FCNN v1 classifier weight files (MlpClassifier::load / save,
src/viscosity.cpp:63-106): read and write the
reference's format so weights move between the two codes unchanged. The
engine loads the same files itself (fcsg_engine_load_mlp); training stays
with the reference (`train_classifier`)."""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"FCNN"
K_INPUT, K_CLASSES = 7, 4  # include/fcs/viscosity.hpp (stencil width 7, classes 1..4)


class WeightFileError(ValueError):
    """ConfigError of MlpClassifier::load"""


@dataclass
class FcnnWeights:
    activation: int = 0                         # stored, as in the reference (tanh on hidden layers)
    weights: list = field(default_factory=list)  # per layer (rows, cols), row-major as in the file
    biases: list = field(default_factory=list)   # per layer (rows,)

    @property
    def shape(self):
        return [(w.shape[0], w.shape[1]) for w in self.weights]

    def packed(self) -> np.ndarray:
        """per layer W then b, the engine's packed order"""
        return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(self.weights, self.biases)])


def load_fcnn(path: str) -> FcnnWeights:
    try:
        f = open(path, "rb")
    except OSError:
        raise WeightFileError("classifier weights not found: " + path) from None
    with f:
        data = f.read()
    if data[:4] != MAGIC:
        raise WeightFileError("bad weight file magic")
    pos = 4

    def u32():
        nonlocal pos
        if pos + 4 > len(data):
            raise WeightFileError("truncated weight file: " + path)
        v = struct.unpack_from("<I", data, pos)[0]
        pos += 4
        return v

    if u32() != 1:
        raise WeightFileError("unsupported weight file version")
    m = FcnnWeights(activation=u32())
    for _ in range(u32()):
        r, c = u32(), u32()
        need = 8 * (r * c + r)
        if pos + need > len(data):
            raise WeightFileError("truncated weight file: " + path)
        w = np.frombuffer(data, dtype="<f8", count=r * c, offset=pos).reshape(r, c).copy()
        pos += 8 * r * c
        b = np.frombuffer(data, dtype="<f8", count=r, offset=pos).copy()
        pos += 8 * r
        m.weights.append(w)
        m.biases.append(b)
    if not m.weights or m.weights[0].shape[1] != K_INPUT or m.weights[-1].shape[0] != K_CLASSES:
        raise WeightFileError("weight file has wrong input/output dimensions")
    return m


def save_fcnn(path: str, m: FcnnWeights):
    out = [MAGIC, struct.pack("<III", 1, m.activation, len(m.weights))]
    for w, b in zip(m.weights, m.biases):
        w = np.ascontiguousarray(w, dtype="<f8")
        out.append(struct.pack("<II", w.shape[0], w.shape[1]))
        out.append(w.tobytes())
        out.append(np.ascontiguousarray(b, dtype="<f8").tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(out))
