"""Unsigned distance from the DDF on the GPU (paper Eq. 5).

Mirrors the reference's entry points with the same names, arguments,
results and errors:

  udf(backend, x, n_dirs, exact, polish)            field.py:388-403
  udf_many(backend, points, n_dirs, exact, polish)   field.py:418-488
  udf_grid(backend, resolution, n_dirs, bounds, ...) recon.py:61-81
  ScalarGrid, grid_points                            recon.py:17-58

The whole computation (direction scan, first argmin, golden-section polish)
runs on the device through ``ddf_udf`` / ``ddf_udf_grid``; there is no host
fallback.  Exact backends (the mesh field, ``exact_udf = True``) take the
reference's shortcut to the closest-point distance, also on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .field import _dev, _ptr


@dataclass
class ScalarGrid:
    """recon.py:17-44: UDF values over a box; +inf marks all-miss vertices."""
    bbox: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.bbox = np.asarray(self.bbox, dtype=np.float64).reshape(2, 3)
        if self.values.ndim != 3:
            raise ValueError("grid values must be 3-D")
        finite = self.values[np.isfinite(self.values)]
        if finite.size and finite.min() < 0.0:
            raise ValueError("UDF grid values must be non-negative")

    @property
    def resolution(self):
        return self.values.shape

    @property
    def voxel(self):
        return (self.bbox[1] - self.bbox[0]) / (np.asarray(self.values.shape) - 1)

    def axes(self):
        return [np.linspace(self.bbox[0, k], self.bbox[1, k], self.values.shape[k]) for k in range(3)]


def grid_points(bbox, resolution: int) -> np.ndarray:
    """recon.py:47-51 (host copy, for callers; the device builds its own)."""
    bbox = np.asarray(bbox, dtype=np.float64).reshape(2, 3)
    ax = np.linspace(bbox[0], bbox[1], resolution)
    g = np.meshgrid(ax[:, 0], ax[:, 1], ax[:, 2], indexing="ij")
    return np.stack([c.ravel() for c in g], axis=1)


def _exact(backend, exact) -> bool:
    """field.py:428-433: exact backends (meshes) shortcut to closest-point distances."""
    ex = bool(getattr(backend, "exact_udf", False) if exact is None else exact)
    if not ex and getattr(backend, "exact_udf", False):
        raise ValueError("the sampled UDF over a mesh backend is not on the GPU; use exact=True")
    return ex


def udf_many_device(backend, points, n_dirs: int = 512, polish: bool = True, out=None, stream=None):
    """Device in, device out: points (P, 3) float64 CUDA tensor -> (P,) float64."""
    if out is None:
        out = torch.empty(points.shape[0], dtype=torch.float64, device=points.device)
    s = stream if stream is not None else torch.cuda.current_stream(points.device)
    _lib.check(_lib.lib().ddf_udf(backend.handle, _ptr(points), points.shape[0], int(n_dirs), int(bool(polish)),
                                  _ptr(out), ctypes.c_void_p(s.cuda_stream)))
    return out


def udf_many(backend, points, n_dirs: int = 512, exact: bool | None = None, polish: bool = True,
             chunk: int = 250_000) -> np.ndarray:
    """field.py:418-488: (P, 3) points -> (P,) distances, +inf = all directions miss.
    ``chunk`` is accepted for signature parity; the device chunks by itself."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    if _exact(backend, exact):
        return backend.exact_distance(pts)
    if len(pts) == 0:
        return np.empty(0)
    with torch.cuda.device(backend.torch_device):
        d = _dev(pts, device=backend.torch_device)
        return udf_many_device(backend, d, n_dirs, polish).cpu().numpy()


def udf(backend, x, n_dirs: int = 512, exact: bool | None = None, polish: bool = True):
    """field.py:388-403: the distance at one point, None when every direction misses."""
    if n_dirs < 2:
        raise ValueError("need n_dirs >= 2")
    v = float(udf_many(backend, np.asarray(x, dtype=np.float64)[None, :], n_dirs=n_dirs, exact=exact,
                       polish=polish)[0])
    return None if np.isinf(v) else v


def udf_grid(backend, resolution: int = 64, n_dirs: int = 512, bounds=None, exact: bool | None = None,
             polish: bool = True, chunk_points: int = 32_768) -> ScalarGrid:
    """recon.py:61-81: the UDF at every vertex of a resolution^3 grid over
    ``bounds`` (default ``backend.grid_bounds``)."""
    if resolution < 8:
        raise ValueError("resolution must be >= 8")
    box = np.asarray(bounds if bounds is not None else backend.grid_bounds, dtype=np.float64).reshape(2, 3)
    if _exact(backend, exact) and not getattr(backend, "exact_udf", False):
        return ScalarGrid(box, backend.exact_distance(grid_points(box, resolution)).reshape((resolution,) * 3))
    with torch.cuda.device(backend.torch_device):
        out = torch.empty(resolution ** 3, dtype=torch.float64, device=backend.torch_device)
        b6 = (ctypes.c_double * 6)(*box.reshape(-1))
        st = torch.cuda.current_stream(backend.torch_device)
        _lib.check(_lib.lib().ddf_udf_grid(backend.handle, b6, int(resolution), int(n_dirs), int(bool(polish)),
                                           _ptr(out), ctypes.c_void_p(st.cuda_stream)))
        return ScalarGrid(box, out.cpu().numpy().reshape(resolution, resolution, resolution))
