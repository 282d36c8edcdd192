"""CudaNeuralField: the reference's DDF backend protocol on the B200.

Drop-in for ``ddfield.field.NeuralField`` (field.py:218-317): same attributes
(``model``, ``delta``, ``bounds``, ``grid_bounds``, ``normal_eval_backoff``,
``exact_udf``), same batch methods and return types, same classmethod
``from_checkpoint``.  Each method copies its numpy inputs to the device, runs
one C-ABI call (include/ddf_b200.h) and copies the result back, so the
reference's own ``render.render_depth/normal/shaded/path`` work unchanged on
top of it; ``paper_2306_16142_b200.render.render_path`` keeps the whole
wavefront on the device instead.

EXTENSION (config 5): ``CudaNeuralField.scene(models, centers, scale,
albedos)`` composes several networks by min distance.
"""

from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from . import _lib
from .neural import effective_weights, encoding_of, load_model


def _dev(a, dtype=torch.float64, device="cuda"):
    """numpy -> device tensor through pinned memory (the host<->device copy a
    protocol call pays).  Measured in situ against a direct pageable copy and
    against one shared pinned buffer for both inputs: both were slower
    (query_raw 314 us here vs 423 and 418 us; scratch/e2e_ab.py)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    if torch.cuda.is_available():
        t = t.pin_memory()
    return t.to(device, non_blocking=True)


PINNED_READBACK_BYTES = 8 << 20


def _host(stream, *ts):
    """Device tensors -> numpy, ordered on ``stream`` (the field's device).
    Small results (<= 8 MB in all) go through pinned buffers: asynchronous
    copies and one synchronize, the blocks recycled by PyTorch's host
    allocator.  Larger ones use pageable copies, so a big protocol call does
    not leave page-locked memory behind.  The arrays are plain numpy either
    way, as the reference returns."""
    if sum(t.numel() * t.element_size() for t in ts) > PINNED_READBACK_BYTES:
        with torch.cuda.stream(stream):
            return [t.cpu().numpy() for t in ts]
    outs = []
    for t in ts:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        with torch.cuda.stream(stream):
            h.copy_(t, non_blocking=True)
        outs.append(h)
    stream.synchronize()
    return [np.array(h.numpy()) for h in outs]


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class CudaNeuralField:
    """Trained network(s) as a field backend evaluated by libddf_b200."""

    exact_udf = False
    DEFAULT_BOUNDS = np.array([[-1.1, -1.1, -1.1], [1.1, 1.1, 1.1]])  # field.py:229

    def __init__(self, model, delta: float, bounds=None, precision: str = "fp32", device: int | None = None):
        self._h = None
        self._init_field(delta, bounds, precision, device)
        self.model = model
        self.models = [model]
        self._add(model, (0.0, 0.0, 0.0), 1.0, 0.0)

    def _init_field(self, delta, bounds, precision, device):
        self.delta = float(delta)
        self.bounds = (np.asarray(bounds, dtype=np.float64) if bounds is not None
                       else self.DEFAULT_BOUNDS.copy())
        self.grid_bounds = self.bounds
        self.normal_eval_backoff = 0.5 * self.delta           # field.py:237
        if precision not in _lib.PRECISIONS:
            raise ValueError("precision must be 'fp32', 'bf16' or 'fp32_simt'")
        self.precision = precision
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.torch_device = torch.device("cuda", self.device)
        L = _lib.lib()
        h = ctypes.c_void_p()
        b6 = (ctypes.c_double * 6)(*self.bounds.reshape(-1).tolist())
        _lib.check(L.ddf_field_create(self.delta, b6, _lib.PRECISIONS[precision],
                                      self.device, ctypes.byref(h)))
        self._h = h
        self.albedos = None
        self.centers = None
        self.scale = 1.0

    def _add(self, model, center, scale, albedo):
        ws = effective_weights(model)
        flat_w = np.concatenate([w.reshape(-1) for w in ws]).astype(np.float64)
        flat_b = np.concatenate([np.asarray(b, dtype=np.float64).reshape(-1) for b in model.b])
        widths = (ctypes.c_int32 * len(model.widths))(*[int(w) for w in model.widths])
        c3 = (ctypes.c_double * 3)(*[float(c) for c in center])
        _lib.check(_lib.lib().ddf_field_add_network(
            self._h, widths, len(model.widths),
            flat_w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            flat_b.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            encoding_of(model), c3, float(scale), float(albedo)))

    @classmethod
    def from_checkpoint(cls, path, bounds=None, precision: str = "fp32"):
        """field.py:239-242."""
        model, delta = load_model(path)
        return cls(model, delta, bounds=bounds, precision=precision)

    @classmethod
    def scene(cls, models, centers, scale, albedos, delta, bounds=None, precision="fp32"):
        """EXTENSION (config 5): distance = min_j scale * f_j((x - c_j)/scale)."""
        self = cls.__new__(cls)
        self._h = None
        self._init_field(delta, bounds, precision, None)
        self.model = models[0]
        self.models = list(models)
        self.centers = np.asarray(centers, dtype=np.float64)
        self.scale = float(scale)
        self.albedos = np.asarray(albedos, dtype=np.float64)
        for m, c, a in zip(models, self.centers, self.albedos):
            self._add(m, c, scale, a)
        return self

    def set_precision(self, precision: str) -> None:
        if precision not in _lib.PRECISIONS:
            raise ValueError("precision must be 'fp32', 'bf16' or 'fp32_simt'")
        _lib.check(_lib.lib().ddf_field_set_precision(self._h, _lib.PRECISIONS[precision]))
        self.precision = precision

    def __del__(self):
        h = getattr(self, "_h", None)
        # at interpreter exit the module globals may already be gone
        if h is not None and _lib is not None and getattr(_lib, "_lib", None) is not None:
            _lib._lib.ddf_field_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------ protocol
    @contextlib.contextmanager
    def _call(self):
        """Make the field's device current for one protocol call (restored
        afterwards, so a C call's cudaSetDevice does not leak) and yield that
        device's current stream."""
        with torch.cuda.device(self.torch_device):
            yield torch.cuda.current_stream(self.torch_device)

    def _rows(self, *arrays):
        n = None
        out = []
        for a in arrays:
            a = np.atleast_2d(np.asarray(a, dtype=np.float64))
            if n is None:
                n = len(a)
            elif len(a) != n:
                raise ValueError("row count mismatch")
            out.append(a)
        return n, out

    def _empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.torch_device)

    def forward_inputs(self, inputs, net: int = 0):
        """neural.forward_batch (neural.py:138-157) on raw network inputs."""
        x = np.atleast_2d(np.asarray(inputs, dtype=np.float64))
        with self._call() as st:
            xd = _dev(x, device=self.torch_device)
            out = self._empty(len(x))
            _lib.check(_lib.lib().ddf_mlp_forward(self._h, net, _ptr(xd), len(x), _ptr(out),
                                                  ctypes.c_void_p(st.cuda_stream)))
            return _host(st, out)[0]

    def input_gradient_inputs(self, inputs, net: int = 0):
        """neural.input_gradient_batch (neural.py:229-249) on raw inputs."""
        x = np.atleast_2d(np.asarray(inputs, dtype=np.float64))
        with self._call() as st:
            xd = _dev(x, device=self.torch_device)
            out = self._empty(x.shape)
            _lib.check(_lib.lib().ddf_mlp_input_grad(self._h, net, _ptr(xd), len(x), _ptr(out),
                                                     ctypes.c_void_p(st.cuda_stream)))
            return _host(st, out)[0]

    def query_raw(self, positions, dir_vecs):
        """(pred, t, hit, obj): the raw network distance next to query_batch."""
        n, (p, d) = self._rows(positions, dir_vecs)
        with self._call() as st:
            pd, dd = _dev(p, device=self.torch_device), _dev(d, device=self.torch_device)
            t, pred = self._empty(n), self._empty(n)
            hit, obj = self._empty(n, torch.uint8), self._empty(n, torch.int32)
            _lib.check(_lib.lib().ddf_query(self._h, _ptr(pd), _ptr(dd), n, _ptr(t), _ptr(hit), _ptr(pred),
                                            _ptr(obj), ctypes.c_void_p(st.cuda_stream)))
            pred, t, hit, obj = _host(st, pred, t, hit, obj)
        return pred, t, hit.astype(bool), obj

    def query_batch(self, positions, dir_vecs):
        """field.py:257-258 -> (t, hit)."""
        _, t, hit, _ = self.query_raw(positions, dir_vecs)
        return t, hit

    def query_batch_angles(self, positions, angles):
        """field.py:248-255 (angles -> unit vectors; the kernel re-canonicalises)."""
        a = np.atleast_2d(np.asarray(angles, dtype=np.float64))
        s = np.sin(a[:, 1])
        d = np.stack([np.cos(a[:, 0]) * s, np.sin(a[:, 0]) * s, np.cos(a[:, 1])], axis=1)
        return self.query_batch(positions, d)

    def trace_with_objects(self, origins, dir_vecs):
        """trace_batch plus the id of the object each ray hit (0 for one net)."""
        n, (o, d) = self._rows(origins, dir_vecs)
        with self._call() as st:
            od, dd = _dev(o, device=self.torch_device), _dev(d, device=self.torch_device)
            t, hit, obj = self._empty(n), self._empty(n, torch.uint8), self._empty(n, torch.int32)
            _lib.check(_lib.lib().ddf_trace(self._h, _ptr(od), _ptr(dd), n, _ptr(t), _ptr(hit), _ptr(obj),
                                            ctypes.c_void_p(st.cuda_stream)))
            t, hit, obj = _host(st, t, hit, obj)
        return t, hit.astype(bool), obj

    def trace_batch(self, origins, dir_vecs):
        """field.py:260-289 -> (t with inf on miss, hit)."""
        t, hit, _ = self.trace_with_objects(origins, dir_vecs)
        return t, hit

    def normal_batch(self, origins, dir_vecs, t_hit=None, obj=None):
        """field.py:295-317 -> (normals, valid).

        Composite fields (config 5) take the gradient of one object per row:
        ``obj`` (the hit object from trace_with_objects) when given.  Called
        through the plain protocol, as the reference's render loop does
        (render.py:131), there is no object id, so the row's object is the
        scene's argmin at the evaluation point itself."""
        n, (o, d) = self._rows(origins, dir_vecs)
        th = None if t_hit is None else np.asarray(t_hit, dtype=np.float64).reshape(n)
        if obj is None and self.albedos is not None and n:
            back = np.zeros(n) if th is None else np.maximum(th - self.normal_eval_backoff, 0.0)
            _, _, _, obj = self.query_raw(o + back[:, None] * d, d)
        with self._call() as st:
            od, dd = _dev(o, device=self.torch_device), _dev(d, device=self.torch_device)
            thd = _dev(th, device=self.torch_device) if th is not None else None
            ob = _dev(np.asarray(obj).reshape(n), dtype=torch.int32, device=self.torch_device) if obj is not None \
                else None
            nr, valid = self._empty((n, 3)), self._empty(n, torch.uint8)
            _lib.check(_lib.lib().ddf_normal(self._h, _ptr(od), _ptr(dd), _ptr(thd), _ptr(ob), n, _ptr(nr),
                                             _ptr(valid), ctypes.c_void_p(st.cuda_stream)))
            nr, valid = _host(st, nr, valid)
        return nr, valid.astype(bool)

    def input_gradients(self, positions, angles):
        """field.py:291-293: (N, 5) gradient w.r.t. the encoded inputs
        (single-network fields, reference encoding)."""
        if int(self.model.widths[0]) != 5:
            raise ValueError("input_gradients on raw inputs needs a 5-input network")
        p = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        a = np.atleast_2d(np.asarray(angles, dtype=np.float64))
        x = np.concatenate([p, a[:, :1] / np.pi - 1.0, 2.0 * a[:, 1:2] / np.pi - 1.0], axis=1)  # neural.py:26-38
        return self.input_gradient_inputs(x)
