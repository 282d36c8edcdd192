"""render.render_path on the B200 (ddfield/render.py:198-247, drop-in).

``render_path(backend, camera, config)`` has the reference's signature and
returns a ``Framebuffer`` with the (H, W, 3) float64 film.  The whole
wavefront -- camera rays, sphere march, gradient normals, cosine bounces,
compaction and film accumulation -- runs on the device in one
``ddf_render_path`` call; the host only builds the camera basis and the PCG64
seed state exactly as the reference does.

``Camera``, ``RenderConfig`` and ``Framebuffer`` mirror render.py:22-124; the
reference's own objects are accepted too (duck typing).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

RNG_TAG = 0x9A7   # render.py:209
RR_TAG = 0x5252   # EXTENSION: Russian-roulette stream


@dataclass
class Camera:
    """render.py:22-51 pinhole camera (right-handed, y-up default)."""
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray = (0.0, 1.0, 0.0)
    vfov: float = np.pi / 3.0
    width: int = 256
    height: int = 256

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.look_at = np.asarray(self.look_at, dtype=np.float64)
        self.up = np.asarray(self.up, dtype=np.float64)
        if not 0.0 < self.vfov < np.pi:
            raise ValueError("vfov must be in (0, pi)")
        if self.width < 1 or self.height < 1:
            raise ValueError("film dimensions must be >= 1")
        fwd = self.look_at - self.position
        norm = np.linalg.norm(fwd)
        if norm == 0.0:
            raise ValueError("camera position equals look-at target")
        self.forward = fwd / norm
        right = np.cross(self.forward, self.up)
        rnorm = np.linalg.norm(right)
        if rnorm < 1e-12:
            raise ValueError("up vector is parallel to the view direction")
        self.right = right / rnorm
        self.up_ortho = np.cross(self.right, self.forward)


@dataclass
class Framebuffer:
    """render.py:92-103."""
    width: int
    height: int
    data: np.ndarray

    def __post_init__(self):
        if self.data.shape[:2] != (self.height, self.width):
            raise ValueError("framebuffer shape does not match the film")


@dataclass
class RenderConfig:
    """render.py:106-124 (path-mode fields) plus the EXTENSION knobs."""
    mode: str = "path"
    spp: int = 16
    bounces: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    light_dir: np.ndarray = field(default_factory=lambda: np.array([1.0, 1.0, 1.0]) / np.sqrt(3.0))
    albedo: float = 0.7
    env_radiance: float = 1.0
    ambient: bool = False
    seed: int = 0
    rr_start: int = -1          # EXTENSION: Russian roulette from this bounce index
    tile: int = 0               # image-tile sharding (config 4)
    rank: int = 0
    world: int = 1
    max_wave_paths: int = 0
    profile: int = 0            # 1: per-kernel-class CUDA-event timing in the stats
    graph: int = 1              # 1: replay the waves as a captured CUDA graph (same camera/config/accumulator)
    no_fuse: int = 0            # 1: never fuse a bounce's first march step with the next normal (same results)
    tile_owner: object = None   # per-tile rank array (dist.balanced_tile_owners); None = tile k -> rank k % world

    def __post_init__(self):
        if self.spp < 1:
            raise ValueError("spp must be >= 1")
        if self.bounces < 0:
            raise ValueError("bounces must be >= 0")


def _split128(v: int):
    return (v & (2 ** 64 - 1), v >> 64)


def pcg_state(seed: int, tag: int):
    """(state, inc) of np.random.default_rng([seed, tag]) -- numpy's own
    SeedSequence hashing, taken on the host."""
    st = np.random.PCG64(np.random.SeedSequence([int(seed), int(tag)])).state["state"]
    return int(st["state"]), int(st["inc"])


def camera_struct(camera) -> _lib.Camera_t:
    c = _lib.Camera_t()
    c.position[:] = [float(x) for x in camera.position]
    c.forward[:] = [float(x) for x in camera.forward]
    c.right[:] = [float(x) for x in camera.right]
    c.up_ortho[:] = [float(x) for x in camera.up_ortho]
    c.tan_half = float(np.tan(camera.vfov / 2.0))     # render.py:66
    c.aspect = camera.width / camera.height           # render.py:67
    c.width, c.height = int(camera.width), int(camera.height)
    return c


def path_struct(config) -> _lib.PathConfig_t:
    p = _lib.PathConfig_t()
    p.spp, p.bounces = int(config.spp), int(config.bounces)
    p.albedo, p.env_radiance = float(config.albedo), float(config.env_radiance)
    s, inc = pcg_state(config.seed, RNG_TAG)
    p.rng_state[:] = list(_split128(s))
    p.rng_inc[:] = list(_split128(inc))
    p.rr_start = int(getattr(config, "rr_start", -1))
    s, inc = pcg_state(config.seed, RR_TAG)
    p.rr_state[:] = list(_split128(s))
    p.rr_inc[:] = list(_split128(inc))
    p.tile = int(getattr(config, "tile", 0))
    p.rank = int(getattr(config, "rank", 0))
    p.world = int(getattr(config, "world", 1))
    p.max_wave_paths = int(getattr(config, "max_wave_paths", 0))
    p.profile = int(getattr(config, "profile", 0))
    p.graph = int(getattr(config, "graph", 1))
    p.no_fuse = int(getattr(config, "no_fuse", 0))
    owner = getattr(config, "tile_owner", None)
    if owner is not None:
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        p._owner_ref = owner   # the struct borrows it for the duration of the call
        p.tile_owner = owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    return p


def render_path_device(backend, camera, config, accum=None, stream=None):
    """Run the wavefront; returns (accum device tensor (W*H,) float64 holding
    the per-pixel radiance summed over spp, stats dict).  No host copies."""
    if config.bounces < 1:
        raise ValueError("path mode needs bounces >= 1")   # render.py:207-208
    n_pix = camera.width * camera.height
    if accum is None:
        accum = torch.empty(n_pix, dtype=torch.float64, device=backend.torch_device)
    owner = getattr(config, "tile_owner", None)
    tile = int(getattr(config, "tile", 0))
    if owner is not None and tile > 0:
        n_tiles = -(-camera.width // tile) * -(-camera.height // tile)
        if np.size(owner) != n_tiles:
            raise ValueError(f"tile_owner has {np.size(owner)} entries, the film has {n_tiles} tiles")
    st = _lib.RenderStats_t()
    cam = camera_struct(camera)
    cfg = path_struct(config)
    s = stream if stream is not None else torch.cuda.current_stream(backend.torch_device)
    _lib.check(_lib.lib().ddf_render_path(backend.handle, ctypes.byref(cam), ctypes.byref(cfg),
                                          ctypes.c_void_p(accum.data_ptr()), ctypes.byref(st),
                                          ctypes.c_void_p(s.cuda_stream)))
    stats = {k: getattr(st, k) for k, _ in _lib.RenderStats_t._fields_}
    return accum, stats


def film_from_accum(accum, camera, spp):
    """render.py:244-247: value = accum / spp, grey replicated to RGB."""
    value = accum.cpu().numpy() / spp
    rgb = np.repeat(value[:, None], 3, axis=1)
    return Framebuffer(camera.width, camera.height, rgb.reshape(camera.height, camera.width, 3))


def render_path(backend, camera, config=None):
    """render.py:198-247 with the reference's signature and result."""
    config = config or RenderConfig(mode="path")
    accum, _ = render_path_device(backend, camera, config)
    return film_from_accum(accum, camera, config.spp)


def pixel_rays(camera, offsets=None):
    """render.py:54-75 on the host (float64, row-major pixel index)."""
    w, h = camera.width, camera.height
    px = np.tile(np.arange(w), h).astype(np.float64)
    py = np.repeat(np.arange(h), w).astype(np.float64)
    ox, oy = (0.5, 0.5) if offsets is None else (offsets[:, 0], offsets[:, 1])
    tan_half = np.tan(camera.vfov / 2.0)
    sx = (2.0 * (px + ox) / w - 1.0) * tan_half * (w / h)
    sy = (1.0 - 2.0 * (py + oy) / h) * tan_half
    d = camera.forward[None, :] + sx[:, None] * camera.right[None, :] + sy[:, None] * camera.up_ortho[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(camera.position, d.shape).copy(), d


def _hit_normals(backend, origins, dirs, t, hit, obj=None):
    """render.py:127-141: degenerate gradients face the ray; the sign rule
    n . d < 0 raises NumericError."""
    from .errors import NumericError
    normals = np.zeros((len(origins), 3))
    if hit.any():
        n, valid = backend.normal_batch(origins[hit], dirs[hit], t_hit=t[hit],
                                        obj=None if obj is None else obj[hit])
        bad = ~valid
        if bad.any():
            n[bad] = -dirs[hit][bad]
        if not (np.einsum("ij,ij->i", n, dirs[hit]) < 0.0).all():
            raise NumericError("normal sign rule violated: n . dir >= 0")
        normals[hit] = n
    return normals


def _trace_with_obj(backend, o, d):
    if hasattr(backend, "trace_with_objects"):
        return backend.trace_with_objects(o, d)
    t, hit = backend.trace_batch(o, d)
    return t, hit, None


_MODE_IDS = {"depth": 0, "normal": 1, "shaded": 2}


def _device_backend(backend) -> bool:
    return getattr(backend, "handle", None) is not None and hasattr(backend, "torch_device")


def render_mode_device(backend, camera, config, mode: str, out=None, to_host: bool = True):
    """render.py:144-184 on the device (ddf_render_mode): pixel-centre rays,
    trace, hit normals and shading without host round trips.  Returns the
    (H, W) depth or (H, W, 3) RGB array (a device tensor with to_host=False)."""
    m = _lib.ModeConfig_t()
    m.mode = _MODE_IDS[mode]
    m.ambient = int(bool(getattr(config, "ambient", False)))
    for k in range(3):
        m.background[k] = float(config.background[k])
        m.light_dir[k] = float(np.asarray(config.light_dir, dtype=np.float64)[k])
    m.albedo = float(config.albedo)
    m.env_radiance = float(config.env_radiance)
    W, H = camera.width, camera.height
    if out is None:
        out = torch.empty(W * H * (1 if mode == "depth" else 3), dtype=torch.float64, device=backend.torch_device)
    cam = camera_struct(camera)
    _lib.check(_lib.lib().ddf_render_mode(backend.handle, ctypes.byref(cam), ctypes.byref(m),
                                          ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(torch.cuda.current_stream(backend.torch_device).cuda_stream)))
    if not to_host:
        return out
    a = out.cpu().numpy()
    return a.reshape(H, W) if mode == "depth" else a.reshape(H, W, 3)


def render_depth(backend, camera, config=None):
    """render.py:144-150: field values per pixel, non-finite on a miss."""
    if _device_backend(backend):
        return Framebuffer(camera.width, camera.height,
                           render_mode_device(backend, camera, config or RenderConfig(mode="depth"), "depth"))
    o, d = pixel_rays(camera)
    t, hit, _ = _trace_with_obj(backend, o, d)
    return Framebuffer(camera.width, camera.height, np.where(hit, t, np.inf).reshape(camera.height, camera.width))


def render_normal(backend, camera, config=None):
    """render.py:153-164: normals mapped (n + 1)/2, misses get the background."""
    config = config or RenderConfig(mode="normal")
    if _device_backend(backend):
        return Framebuffer(camera.width, camera.height, render_mode_device(backend, camera, config, "normal"))
    o, d = pixel_rays(camera)
    t, hit, obj = _trace_with_obj(backend, o, d)
    nrm = _hit_normals(backend, o, d, t, hit, obj)
    rgb = np.empty((len(d), 3))
    rgb[:] = np.asarray(config.background)
    rgb[hit] = 0.5 * (nrm[hit] + 1.0)
    return Framebuffer(camera.width, camera.height, rgb.reshape(camera.height, camera.width, 3))


def render_shaded(backend, camera, config=None):
    """render.py:167-184: Lambertian under a directional light (used as
    given, render.py:181) or the flat ambient term."""
    config = config or RenderConfig(mode="shaded")
    if _device_backend(backend):
        return Framebuffer(camera.width, camera.height, render_mode_device(backend, camera, config, "shaded"))
    o, d = pixel_rays(camera)
    t, hit, obj = _trace_with_obj(backend, o, d)
    nrm = _hit_normals(backend, o, d, t, hit, obj)
    rgb = np.empty((len(d), 3))
    rgb[:] = np.asarray(config.background)
    if config.ambient:
        shade = np.full(int(hit.sum()), config.albedo * config.env_radiance)
    else:
        shade = config.albedo * np.maximum(nrm[hit] @ np.asarray(config.light_dir, dtype=np.float64), 0.0)
    rgb[hit] = shade[:, None]
    return Framebuffer(camera.width, camera.height, rgb.reshape(camera.height, camera.width, 3))


_MODES = {"depth": render_depth, "normal": render_normal, "shaded": render_shaded, "path": render_path}


def render(backend, camera, config):
    """render.py:258-263 dispatch."""
    try:
        fn = _MODES[config.mode]
    except KeyError:
        raise ValueError(f"unknown render mode {config.mode!r}") from None
    return fn(backend, camera, config)


def bench(backends: dict, camera, config, frames: int):
    """render.py:266-280 (the paper's Fig. 5 timing convention): wall-clock
    per frame per backend, first frame flagged warm-up.  Rows (backend,
    frame, ms, warmup)."""
    import time
    if frames < 2:
        raise ValueError("need frames >= 2 to separate warm-up")
    rows = []
    for name, backend in backends.items():
        for i in range(frames):
            if torch.cuda.is_available():
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            render(backend, camera, config)
            if torch.cuda.is_available():
                torch.cuda.synchronize()
            rows.append((name, i, (time.perf_counter() - t0) * 1e3, 1 if i == 0 else 0))
    return rows


def write_ppm(fb, path, gamma: float = 2.2) -> None:
    """render.py:283-293 binary P6, 8-bit, gamma-encoded (misses write 0)."""
    data = fb.data
    if data.ndim == 2:
        data = np.repeat(data[:, :, None], 3, axis=2)
    data = np.where(np.isfinite(data), data, 0.0)
    u8 = (np.clip(data, 0.0, 1.0) ** (1.0 / gamma) * 255.0 + 0.5).astype(np.uint8)
    with open(path, "wb") as fh:
        fh.write(f"P6\n{fb.width} {fb.height}\n255\n".encode("ascii"))
        fh.write(u8.tobytes())


def write_pfm(fb, path) -> None:
    """render.py:296-303 grayscale little-endian PFM, rows bottom to top."""
    if fb.data.ndim != 2:
        raise ValueError("PFM output is for scalar framebuffers")
    data = np.where(np.isfinite(fb.data), fb.data, 0.0).astype("<f4")
    with open(path, "wb") as fh:
        fh.write(f"Pf\n{fb.width} {fb.height}\n-1.0\n".encode("ascii"))
        fh.write(data[::-1].tobytes())
