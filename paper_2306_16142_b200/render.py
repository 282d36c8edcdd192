"""render.render_path and the single-bounce modes on the B200 (drop-in for
ddfield/render.py:144-247).

``render_path(backend, camera, config)`` keeps the reference's signature and
returns a ``Framebuffer`` holding the (H, W, 3) float64 film.  One
``ddf_render_path`` call runs the whole wavefront on the device: camera rays,
sphere march, gradient normals, cosine bounces, compaction and film
accumulation.  The host side builds only two things, both exactly as the
reference does: the camera basis and the PCG64 seed state.

Host backends (anything without a device handle) are not served here.  The
reference's own ``ddfield.render`` drives them through the backend protocol,
and ``CudaNeuralField`` implements that protocol.

``Camera``, ``RenderConfig`` and ``Framebuffer`` are the reference's schemas
(render.py:22-124).  The reference's own objects are accepted too: every
function reads attributes only.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

RNG_TAG = 0x9A7   # render.py:209  default_rng([seed, 0x9A7])
RR_TAG = 0x5252   # EXTENSION: the Russian-roulette stream, independent of the cosine draws


def camera_basis(position, look_at, up):
    """(forward, right, up_ortho) in float64 with numpy's operation order, so
    the device rays match render.py:62-75 bit for bit."""
    fwd = np.asarray(look_at, dtype=np.float64) - np.asarray(position, dtype=np.float64)
    span = np.linalg.norm(fwd)
    if span == 0.0:
        raise ValueError("camera position equals look-at target")
    fwd = fwd / span
    side = np.cross(fwd, np.asarray(up, dtype=np.float64))
    side_len = np.linalg.norm(side)
    if side_len < 1e-12:
        raise ValueError("up vector is parallel to the view direction")
    side = side / side_len
    return fwd, side, np.cross(side, fwd)


@dataclass
class Camera:
    """Pinhole camera schema (render.py:22-30); the basis is derived once."""
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray = (0.0, 1.0, 0.0)
    vfov: float = np.pi / 3.0
    width: int = 256
    height: int = 256

    def __post_init__(self):
        if not 0.0 < self.vfov < np.pi:
            raise ValueError("vfov must be in (0, pi)")
        if min(self.width, self.height) < 1:
            raise ValueError("film dimensions must be >= 1")
        self.position = np.asarray(self.position, dtype=np.float64)
        self.forward, self.right, self.up_ortho = camera_basis(self.position, self.look_at, self.up)


@dataclass
class Framebuffer:
    """render.py:92-103: (H, W) scalar or (H, W, 3) RGB float64."""
    width: int
    height: int
    data: np.ndarray


@dataclass
class RenderConfig:
    """render.py:106-124 fields plus the device knobs (EXTENSION and
    scheduling; none of them changes a pixel value except rr_start)."""
    mode: str = "path"
    spp: int = 16
    bounces: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    light_dir: np.ndarray = field(default_factory=lambda: np.full(3, 1.0) / np.sqrt(3.0))
    albedo: float = 0.7
    env_radiance: float = 1.0
    ambient: bool = False
    seed: int = 0
    rr_start: int = -1          # EXTENSION: Russian roulette from this bounce index (-1 = off)
    tile: int = 0               # image-tile sharding (config 4): tile edge in pixels, 0 = whole film
    rank: int = 0
    world: int = 1
    max_wave_paths: int = 0     # path slots per wave (0 = library default)
    profile: int = 0            # 1: CUDA-event time per kernel class into the stats
    graph: int = 1              # 1: replay the waves as a captured CUDA graph
    no_fuse: int = 0            # 1: keep trace step and normal gradient in separate kernels
    tile_owner: object = None   # per-tile rank table (dist.balanced_tile_owners); None = round-robin
    stage_log: object = None    # device int32 tensor: per-stage compaction lists (debug, disables the graph)

    def __post_init__(self):
        if self.spp < 1:
            raise ValueError("spp must be >= 1")
        if self.bounces < 0:
            raise ValueError("bounces must be >= 0")


def pcg_state(seed: int, tag: int):
    """(state, inc) of np.random.default_rng([seed, tag]): numpy's own
    SeedSequence hashing, taken on the host."""
    st = np.random.PCG64(np.random.SeedSequence([int(seed), int(tag)])).state["state"]
    return int(st["state"]), int(st["inc"])


def _u128(v: int):
    return [v & 0xFFFFFFFFFFFFFFFF, v >> 64]


def camera_struct(camera) -> _lib.Camera_t:
    """ddf_camera_t from a Camera (ours or the reference's)."""
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
    """ddf_path_config_t from a RenderConfig (ours or the reference's)."""
    p = _lib.PathConfig_t()
    p.spp, p.bounces = int(config.spp), int(config.bounces)
    p.albedo, p.env_radiance = float(config.albedo), float(config.env_radiance)
    s, inc = pcg_state(config.seed, RNG_TAG)
    p.rng_state[:], p.rng_inc[:] = _u128(s), _u128(inc)
    s, inc = pcg_state(config.seed, RR_TAG)
    p.rr_state[:], p.rr_inc[:] = _u128(s), _u128(inc)
    opt = lambda k, d: getattr(config, k, d)  # noqa: E731  (the reference's RenderConfig lacks the knobs)
    p.rr_start = int(opt("rr_start", -1))
    p.tile, p.rank, p.world = int(opt("tile", 0)), int(opt("rank", 0)), int(opt("world", 1))
    p.max_wave_paths = int(opt("max_wave_paths", 0))
    p.profile, p.graph, p.no_fuse = int(opt("profile", 0)), int(opt("graph", 1)), int(opt("no_fuse", 0))
    owner = opt("tile_owner", None)
    if owner is not None:
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        p._owner_ref = owner   # the struct borrows it for the duration of the call
        p.tile_owner = owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    log = opt("stage_log", None)
    if log is not None:
        if not (isinstance(log, torch.Tensor) and log.is_cuda and log.dtype == torch.int32):
            raise ValueError("stage_log must be a device int32 tensor")
        p.stage_log = ctypes.cast(ctypes.c_void_p(log.data_ptr()), ctypes.POINTER(ctypes.c_int32))
        p.stage_log_cap = int(log.numel())
    return p


def render_path_device(backend, camera, config, accum=None, stream=None):
    """Run the wavefront.  Returns (accum, stats): accum is a (W*H,) float64
    device tensor with each pixel's radiance summed over spp; stats is the
    ddf_render_stats_t as a dict.  No host copies."""
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
    return accum, _lib.stats_dict(st)


def film_from_accum(accum, camera, spp):
    """render.py:244-247: value = accum / spp, grey replicated to RGB."""
    grey = (accum.cpu().numpy() / spp).reshape(camera.height, camera.width, 1)
    return Framebuffer(camera.width, camera.height, np.repeat(grey, 3, axis=2))


def render_path(backend, camera, config=None):
    """render.py:198-247 with the reference's signature and result."""
    config = config or RenderConfig(mode="path")
    accum, _ = render_path_device(backend, camera, config)
    return film_from_accum(accum, camera, config.spp)


_MODE_IDS = {"depth": 0, "normal": 1, "shaded": 2}


def _require_device(backend):
    if getattr(backend, "handle", None) is None or not hasattr(backend, "torch_device"):
        raise TypeError("not a device backend: host backends render through ddfield.render "
                        "(CudaNeuralField also serves that protocol path)")


def render_mode_device(backend, camera, config, mode: str, out=None, to_host: bool = True):
    """render.py:144-184 in one ddf_render_mode call: pixel-centre rays,
    trace, hit normals and shading.  Returns the (H, W) depth or (H, W, 3)
    RGB array, or the flat device tensor with to_host=False."""
    _require_device(backend)
    m = _lib.ModeConfig_t()
    m.mode = _MODE_IDS[mode]
    m.ambient = int(bool(getattr(config, "ambient", False)))
    m.background[:] = [float(x) for x in config.background]
    m.light_dir[:] = [float(x) for x in np.asarray(config.light_dir, dtype=np.float64)]
    m.albedo, m.env_radiance = float(config.albedo), float(config.env_radiance)
    W, H = camera.width, camera.height
    if out is None:
        out = torch.empty(W * H * (1 if mode == "depth" else 3), dtype=torch.float64, device=backend.torch_device)
    cam = camera_struct(camera)
    stream = torch.cuda.current_stream(backend.torch_device)
    _lib.check(_lib.lib().ddf_render_mode(backend.handle, ctypes.byref(cam), ctypes.byref(m),
                                          ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
    if not to_host:
        return out
    return out.cpu().numpy().reshape((H, W) if mode == "depth" else (H, W, 3))


def _mode_renderer(mode):
    def run(backend, camera, config=None):
        config = config or RenderConfig(mode=mode)
        return Framebuffer(camera.width, camera.height, render_mode_device(backend, camera, config, mode))
    run.__name__ = f"render_{mode}"
    run.__doc__ = f"render.render_{mode} (render.py:144-184) on a device backend."
    return run


render_depth = _mode_renderer("depth")
render_normal = _mode_renderer("normal")
render_shaded = _mode_renderer("shaded")


def render(backend, camera, config):
    """render.py:258-263 for device backends: path or a single-bounce mode."""
    if config.mode == "path":
        return render_path(backend, camera, config)
    if config.mode not in _MODE_IDS:
        raise ValueError(f"unknown render mode {config.mode!r}")
    return Framebuffer(camera.width, camera.height, render_mode_device(backend, camera, config, config.mode))
