"""Exact triangle-mesh backend on the GPU: the reference's OracleField
(field.py:144-200) and its mesh substrate (mesh.py:19-279).

Host side (construction, file formats) mirrors the reference names and errors:
TriangleMesh, load_mesh, save_obj, normalize.  Queries run on the device
through the C ABI (ddf_mesh_create / ddf_mesh_intersect / ddf_query /
ddf_trace / ddf_normal / ddf_render_path): a median-split BVH walked by one
thread per ray in float64 with the reference's Moller-Trumbore and slab
arithmetic, so hits are the reference's bit for bit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .field import _dev, _ptr, _stream


@dataclass(frozen=True, eq=False)
class TriangleMesh:
    """mesh.py:19-67: vertices (N, 3) float64, faces (M, 3) int32, bbox."""
    vertices: np.ndarray
    faces: np.ndarray
    bbox: np.ndarray = dc_field(init=False)

    def __post_init__(self):
        v = np.ascontiguousarray(np.asarray(self.vertices, dtype=np.float64))
        f = np.ascontiguousarray(np.asarray(self.faces, dtype=np.int32))
        if v.ndim != 2 or v.shape[1] != 3:
            raise DataError(f"vertices must be (N, 3), got {v.shape}")
        if f.ndim != 2 or f.shape[1] != 3:
            raise DataError(f"faces must be (M, 3), got {f.shape}")
        if f.size and (f.min() < 0 or f.max() >= len(v)):
            raise DataError("face index out of range")
        bbox = np.stack([v.min(axis=0), v.max(axis=0)]) if len(v) else np.zeros((2, 3))
        for a in (v, f, bbox):
            a.flags.writeable = False
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "faces", f)
        object.__setattr__(self, "bbox", bbox)

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_faces(self) -> int:
        return len(self.faces)

    def face_normal(self, face_index: int) -> np.ndarray:
        a, b, c = self.vertices[self.faces[face_index]]
        n = np.cross(b - a, c - a)
        norm = np.linalg.norm(n)
        if norm == 0.0:
            raise DataError(f"degenerate face {face_index}")
        return n / norm

    def face_areas(self) -> np.ndarray:
        tri = self.vertices[self.faces]
        return 0.5 * np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)


def load_mesh(path) -> TriangleMesh:
    """mesh.py:186-230: ASCII OBJ (v / f records, polygons fan-triangulated,
    negative indices relative, vn/vt/material records ignored); DataError
    names the offending line."""
    verts, tris, where = [], [], []
    try:
        with open(path, "r", encoding="ascii", errors="replace") as fh:
            lines = fh.readlines()
    except OSError as exc:
        raise DataError(f"cannot read {path}: {exc}") from exc
    for lineno, raw in enumerate(lines, start=1):
        tok = raw.split()
        if not tok or tok[0].startswith("#"):
            continue
        if tok[0] == "v":
            if len(tok) < 4:
                raise DataError(f"{path}:{lineno}: vertex needs 3 coordinates")
            try:
                verts.append(tuple(float(x) for x in tok[1:4]))
            except ValueError as exc:
                raise DataError(f"{path}:{lineno}: bad vertex: {exc}") from exc
        elif tok[0] == "f":
            if len(tok) < 4:
                raise DataError(f"{path}:{lineno}: face needs >= 3 vertices")
            idx = []
            for t in tok[1:]:
                try:
                    k = int(t.split("/")[0])
                except ValueError as exc:
                    raise DataError(f"{path}:{lineno}: bad face index {t!r}") from exc
                if k < 0:
                    k = len(verts) + k + 1
                if k < 1:
                    raise DataError(f"{path}:{lineno}: face index out of range")
                idx.append(k - 1)
            for k in range(1, len(idx) - 1):
                tris.append((idx[0], idx[k], idx[k + 1]))
                where.append(lineno)
    n = len(verts)
    for tri, lineno in zip(tris, where):
        if max(tri) >= n:
            raise DataError(f"{path}:{lineno}: face index out of range")
    return TriangleMesh(np.asarray(verts, dtype=np.float64).reshape(-1, 3),
                        np.asarray(tris, dtype=np.int32).reshape(-1, 3))


def save_obj(mesh: TriangleMesh, path) -> None:
    """mesh.py:233-239 (deterministic bytes)."""
    with open(path, "w", encoding="ascii") as fh:
        for x, y, z in mesh.vertices:
            fh.write(f"v {float(x)!r} {float(y)!r} {float(z)!r}\n")
        for a, b, c in mesh.faces:
            fh.write(f"f {a + 1} {b + 1} {c + 1}\n")


def normalize(mesh: TriangleMesh) -> TriangleMesh:
    """mesh.py:242-253: centre at the origin, longest bbox edge -> 2."""
    if mesh.n_vertices == 0:
        raise DataError("cannot normalize an empty mesh")
    longest = float((mesh.bbox[1] - mesh.bbox[0]).max())
    if longest <= 0.0:
        raise DataError("degenerate mesh: zero-extent bounding box")
    centre = 0.5 * (mesh.bbox[0] + mesh.bbox[1])
    return TriangleMesh((mesh.vertices - centre) * (2.0 / longest), mesh.faces)


class CudaMeshField:
    """OracleField (field.py:144-200) on the device: the same protocol
    (query_batch, trace_batch, normal_batch), bounds / grid_bounds, and
    ``intersect_rays`` (mesh.py:264-279)."""

    exact_udf = True
    normal_eval_backoff = 0.0

    def __init__(self, geom: TriangleMesh, device: int | None = None):
        mesh = getattr(geom, "mesh", geom)
        if not isinstance(mesh, TriangleMesh):
            mesh = TriangleMesh(mesh.vertices, mesh.faces)
        self.mesh = mesh
        diag = float(np.linalg.norm(mesh.bbox[1] - mesh.bbox[0]))
        self.bounds = np.stack([mesh.bbox[0] - diag, mesh.bbox[1] + diag])          # field.py:154-157
        self.grid_bounds = np.stack([mesh.bbox[0] - 0.05 * diag, mesh.bbox[1] + 0.05 * diag])
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = device
        self.torch_device = torch.device("cuda", device)
        self._h = ctypes.c_void_p()
        if mesh.n_faces == 0:
            raise DataError("cannot build a BVH over an empty mesh")
        _lib.check(_lib.lib().ddf_mesh_create(mesh.vertices.ctypes.data, mesh.n_vertices, mesh.faces.ctypes.data,
                                              mesh.n_faces, device, ctypes.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().ddf_field_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def _rays(self, origins, dirs):
        o = np.atleast_2d(np.asarray(origins, dtype=np.float64))
        d = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
        if len(o) != len(d):
            raise ValueError("row count mismatch")
        return len(o), _dev(o, device=self.torch_device), _dev(d, device=self.torch_device)

    def intersect_rays(self, origins, dirs, t_min: float = 0.0, t_max: float = np.inf):
        """mesh.py:264-279 -> (face int64, t, u, v); face = -1 on a miss."""
        n, od, dd = self._rays(origins, dirs)
        face = torch.empty(n, dtype=torch.int64, device=self.torch_device)
        t, u, v = (torch.empty(n, dtype=torch.float64, device=self.torch_device) for _ in range(3))
        if n:
            _lib.check(_lib.lib().ddf_mesh_intersect(self._h, _ptr(od), _ptr(dd), n, float(t_min), float(t_max),
                                                     _ptr(face), _ptr(t), _ptr(u), _ptr(v), _stream()))
        return face.cpu().numpy(), t.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()

    def trace_with_objects(self, origins, dirs):
        n, od, dd = self._rays(origins, dirs)
        t = torch.empty(n, dtype=torch.float64, device=self.torch_device)
        hit = torch.empty(n, dtype=torch.uint8, device=self.torch_device)
        face = torch.empty(n, dtype=torch.int32, device=self.torch_device)
        if n:
            _lib.check(_lib.lib().ddf_trace(self._h, _ptr(od), _ptr(dd), n, _ptr(t), _ptr(hit), _ptr(face), _stream()))
        return t.cpu().numpy(), hit.cpu().numpy().astype(bool), face.cpu().numpy()

    def query_batch(self, positions, dir_vecs):
        """field.py:161-165 -> (t with inf on a miss, hit)."""
        t, hit, _ = self.trace_with_objects(positions, dir_vecs)
        return t, hit

    trace_batch = query_batch   # field.py:168

    def normal_batch(self, origins, dir_vecs, t_hit=None, obj=None):
        """field.py:172-189 -> (normals, valid)."""
        n, od, dd = self._rays(origins, dir_vecs)
        nr = torch.empty((n, 3), dtype=torch.float64, device=self.torch_device)
        valid = torch.empty(n, dtype=torch.uint8, device=self.torch_device)
        if n:
            _lib.check(_lib.lib().ddf_normal(self._h, _ptr(od), _ptr(dd), None, None, n, _ptr(nr), _ptr(valid),
                                             _stream()))
        return nr.cpu().numpy(), valid.cpu().numpy().astype(bool)

    def exact_distance(self, points):
        """OracleField.exact_distance (field.py:198-200) = mesh.closest_distance
        (mesh.py:324-330): exact point-to-surface distance."""
        p = np.atleast_2d(np.asarray(points, dtype=np.float64))
        out = torch.empty(len(p), dtype=torch.float64, device=self.torch_device)
        if len(p):
            pd = _dev(p, device=self.torch_device)
            _lib.check(_lib.lib().ddf_mesh_closest(self._h, _ptr(pd), len(p), _ptr(out), _stream()))
        return out.cpu().numpy()


OracleField = CudaMeshField
