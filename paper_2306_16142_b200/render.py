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
    return p


def render_path_device(backend, camera, config, accum=None, stream=None):
    """Run the wavefront; returns (accum device tensor (W*H,) float64 holding
    the per-pixel radiance summed over spp, stats dict).  No host copies."""
    if config.bounces < 1:
        raise ValueError("path mode needs bounces >= 1")   # render.py:207-208
    n_pix = camera.width * camera.height
    if accum is None:
        accum = torch.empty(n_pix, dtype=torch.float64, device=backend.torch_device)
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


def render(backend, camera, config):
    """render.py:258-263 dispatch (path mode is the device wavefront)."""
    if config.mode == "path":
        return render_path(backend, camera, config)
    raise ValueError(f"unknown render mode {config.mode!r}")
