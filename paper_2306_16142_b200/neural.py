"""Network weights on the host: the reference's MlpModel layout and the DDFN
checkpoint (ddfield/neural.py:41-95, 378-431), plus the BASELINE configs'
Kaiming-uniform synthetic weights.

The GPU consumes ``effective_weights()`` (W = g V/|V| row-wise, computed once
in float64 on the host, neural.py:69-74) and the biases; the encoding is
signalled out of band (DDFN has no field for it): 65 inputs mean the 6-octave
sin/cos encoding of configs 3-5, 5 inputs the reference encoding.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import DataError

CHECKPOINT_MAGIC = b"DDFN"
CHECKPOINT_VERSION = 1
PE_INPUTS = 65


@dataclass
class MlpModel:
    """Same fields as ddfield.neural.MlpModel (neural.py:41-56); any object
    with ``widths``, ``v``, ``g``, ``b`` is accepted where a model is needed."""
    widths: tuple
    v: list
    g: list
    b: list
    dropout: float = 0.0

    @property
    def n_layers(self) -> int:
        return len(self.v)

    def effective_weights(self):
        return effective_weights(self)


def effective_weights(model):
    """neural.py:69-74 in float64."""
    out = []
    for v, g in zip(model.v, model.g):
        v = np.asarray(v, dtype=np.float64)
        g = np.asarray(g, dtype=np.float64)
        out.append(g[:, None] * v / np.linalg.norm(v, axis=1)[:, None])
    return out


def encoding_of(model) -> int:
    from ._lib import ENC_PE6, ENC_RAW5
    return ENC_PE6 if int(model.widths[0]) == PE_INPUTS else ENC_RAW5


def kaiming_uniform(widths, seed: int) -> MlpModel:
    """BASELINE synthetic weights: per layer, in order, V ~ U(+-sqrt(6/fan_in))
    with shape (out, in) from np.random.default_rng(seed); g = |V| row-wise
    (W == V); b = 0."""
    rng = np.random.default_rng(seed)
    vs, gs, bs = [], [], []
    for i in range(len(widths) - 1):
        lim = np.sqrt(6.0 / widths[i])
        v = rng.uniform(-lim, lim, size=(widths[i + 1], widths[i]))
        vs.append(v)
        gs.append(np.linalg.norm(v, axis=1))
        bs.append(np.zeros(widths[i + 1]))
    return MlpModel(tuple(int(w) for w in widths), vs, gs, bs)


def save_model(model, delta: float, path) -> None:
    """neural.py:378-390 byte layout."""
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(struct.pack("<II", CHECKPOINT_VERSION, len(model.widths)))
        fh.write(struct.pack(f"<{len(model.widths)}I", *model.widths))
        fh.write(struct.pack("<d", float(delta)))
        for v, g, b in zip(model.v, model.g, model.b):
            for a in (v, g, b):
                fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def load_model(path):
    """neural.py:393-431: widths in the file are authoritative; DataError on a
    bad magic, version, truncation or trailing bytes.  Returns (model, delta)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != CHECKPOINT_MAGIC:
        raise DataError(f"{path}: not a DDFN checkpoint")
    try:
        version, n = struct.unpack_from("<II", blob, 4)
        if version != CHECKPOINT_VERSION:
            raise DataError(f"{path}: unsupported checkpoint version {version}")
        widths = struct.unpack_from(f"<{n}I", blob, 12)
        (delta,) = struct.unpack_from("<d", blob, 12 + 4 * n)
    except struct.error as exc:
        raise DataError(f"{path}: truncated checkpoint header") from exc
    off = 20 + 4 * n
    vs, gs, bs = [], [], []
    for i in range(n - 1):
        o, k = widths[i + 1], widths[i]
        need = 8 * (o * k + 2 * o)
        if off + need > len(blob):
            raise DataError(f"{path}: truncated checkpoint (layer {i})")
        flat = np.frombuffer(blob, dtype="<f8", count=o * k + 2 * o, offset=off)
        vs.append(flat[:o * k].reshape(o, k).copy())
        gs.append(flat[o * k:o * k + o].copy())
        bs.append(flat[o * k + o:].copy())
        off += need
    if off != len(blob):
        raise DataError(f"{path}: {len(blob) - off} trailing bytes in checkpoint")
    return MlpModel(tuple(int(w) for w in widths), vs, gs, bs), float(delta)
