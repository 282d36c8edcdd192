"""Exact triangle-mesh backend on the GPU: the reference's OracleField
(field.py:144-200) over its mesh substrate (mesh.py:94-330).

``CudaMeshField`` takes any mesh the reference builds -- a
``ddfield.mesh.TriangleMesh``, a ``Bvh`` or ``OracleField`` wrapping one
(anything with ``.mesh``), or a plain ``(vertices, faces)`` pair -- and answers
the backend protocol on the device through the C ABI (ddf_mesh_create,
ddf_mesh_intersect, ddf_query / ddf_trace / ddf_normal, ddf_render_path,
ddf_udf).  The library builds a median-split BVH on the host and walks it with
one thread per ray in float64, using the reference's Moller-Trumbore and slab
arithmetic, so hits are the reference's bit for bit.  Reading and writing mesh
files stays with the reference (mesh.py:186-253): it is not on the hot path.
"""

from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from . import _lib
from .field import _dev, _host, _ptr


def mesh_arrays(geom):
    """(vertices (N, 3) float64, faces (M, 3) int32), C-contiguous."""
    mesh = getattr(geom, "mesh", geom)
    if isinstance(mesh, tuple):
        v, f = mesh
    else:
        v, f = mesh.vertices, mesh.faces
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    f = np.ascontiguousarray(np.asarray(f, dtype=np.int32))
    if v.ndim != 2 or v.shape[1] != 3 or f.ndim != 2 or f.shape[1] != 3:
        raise ValueError(f"mesh arrays must be (N, 3) and (M, 3), got {v.shape} and {f.shape}")
    return v, f


class CudaMeshField:
    """OracleField (field.py:144-200) on the device: the same protocol
    (query_batch, trace_batch, normal_batch, exact_distance), bounds and
    grid_bounds, and ``intersect_rays`` (mesh.py:264-279)."""

    exact_udf = True
    normal_eval_backoff = 0.0

    def __init__(self, geom, device: int | None = None):
        self._h = None
        self.vertices, self.faces = mesh_arrays(geom)
        # DataError (empty mesh, face index out of range) comes from the C side
        if len(self.vertices):
            lo, hi = self.vertices.min(axis=0), self.vertices.max(axis=0)
        else:
            lo = hi = np.zeros(3)
        diag = float(np.linalg.norm(hi - lo))
        self.bounds = np.stack([lo - diag, hi + diag])                  # field.py:154-157
        self.grid_bounds = np.stack([lo - 0.05 * diag, hi + 0.05 * diag])
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.torch_device = torch.device("cuda", self.device)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().ddf_mesh_create(self.vertices.ctypes.data, len(self.vertices), self.faces.ctypes.data,
                                              len(self.faces), self.device, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None and getattr(_lib, "_lib", None) is not None:
            _lib._lib.ddf_field_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @contextlib.contextmanager
    def _call(self):
        with torch.cuda.device(self.torch_device):
            yield torch.cuda.current_stream(self.torch_device)

    def _rays(self, origins, dirs):
        o = np.atleast_2d(np.asarray(origins, dtype=np.float64))
        d = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
        if len(o) != len(d):
            raise ValueError("row count mismatch")
        return len(o), _dev(o, device=self.torch_device), _dev(d, device=self.torch_device)

    def _empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.torch_device)

    def intersect_rays(self, origins, dirs, t_min: float = 0.0, t_max: float = np.inf):
        """mesh.py:264-279 -> (face int64, t, u, v); face = -1 on a miss."""
        with self._call() as st:
            n, od, dd = self._rays(origins, dirs)
            face = self._empty(n, torch.int64)
            t, u, v = self._empty(n), self._empty(n), self._empty(n)
            if n:
                _lib.check(_lib.lib().ddf_mesh_intersect(self._h, _ptr(od), _ptr(dd), n, float(t_min), float(t_max),
                                                         _ptr(face), _ptr(t), _ptr(u), _ptr(v),
                                                         ctypes.c_void_p(st.cuda_stream)))
            return tuple(_host(st, face, t, u, v))

    def trace_with_objects(self, origins, dirs):
        """(t with inf on a miss, hit, hit face id)."""
        with self._call() as st:
            n, od, dd = self._rays(origins, dirs)
            t, hit, face = self._empty(n), self._empty(n, torch.uint8), self._empty(n, torch.int32)
            if n:
                _lib.check(_lib.lib().ddf_trace(self._h, _ptr(od), _ptr(dd), n, _ptr(t), _ptr(hit), _ptr(face),
                                                ctypes.c_void_p(st.cuda_stream)))
            t, hit, face = _host(st, t, hit, face)
        return t, hit.astype(bool), face

    def query_batch(self, positions, dir_vecs):
        """field.py:161-165 -> (t with inf on a miss, hit)."""
        t, hit, _ = self.trace_with_objects(positions, dir_vecs)
        return t, hit

    trace_batch = query_batch   # field.py:168

    def normal_batch(self, origins, dir_vecs, t_hit=None, obj=None):
        """field.py:172-189 -> (normals, valid): re-intersect, face normal
        flipped against the ray."""
        with self._call() as st:
            n, od, dd = self._rays(origins, dir_vecs)
            nr, valid = self._empty((n, 3)), self._empty(n, torch.uint8)
            if n:
                _lib.check(_lib.lib().ddf_normal(self._h, _ptr(od), _ptr(dd), None, None, n, _ptr(nr), _ptr(valid),
                                                 ctypes.c_void_p(st.cuda_stream)))
            nr, valid = _host(st, nr, valid)
        return nr, valid.astype(bool)

    def exact_distance(self, points):
        """OracleField.exact_distance (field.py:198-200) = mesh.closest_distance
        (mesh.py:324-330): exact point-to-surface distance."""
        p = np.atleast_2d(np.asarray(points, dtype=np.float64))
        with self._call() as st:
            out = self._empty(len(p))
            if len(p):
                pd = _dev(p, device=self.torch_device)
                _lib.check(_lib.lib().ddf_mesh_closest(self._h, _ptr(pd), len(p), _ptr(out),
                                                       ctypes.c_void_p(st.cuda_stream)))
            return _host(st, out)[0]


OracleField = CudaMeshField
