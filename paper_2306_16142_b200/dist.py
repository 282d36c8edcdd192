"""Multi-GPU rendering: image-tile sharding with one collective (the film).

The path shards by pixel: a path touches only its own film entry
(render.py:215-243) and every random draw is addressed by the GLOBAL pixel
index, so splitting the film changes nothing but who renders what.  64x64
tiles of the row-major film go round-robin to ranks (tile k -> rank k % world);
each rank renders its tiles on its own GPU (ddf_render_path with tile / rank /
world) into a full-size float64 accumulator that is zero elsewhere, and one
all-reduce(sum) over NCCL gathers the film exactly (x + 0 = x).
"""

from __future__ import annotations

import copy

import numpy as np


def owned_pixels(width: int, height: int, tile: int, rank: int, world: int) -> np.ndarray:
    """Ascending global pixel ids owned by `rank` -- the same rule as
    ddf_render_path (csrc/ddf_api.cu)."""
    idx = np.arange(width * height)
    if tile > 0:
        ntx = (width + tile - 1) // tile
        tid = (idx // width // tile) * ntx + (idx % width) // tile
        return idx[tid % world == rank]
    return idx[idx % world == rank] if world > 1 else idx


def tile_config(config, rank: int, world: int, tile: int = 64):
    cfg = copy.copy(config)
    cfg.tile = getattr(config, "tile", 0) or tile
    cfg.rank, cfg.world = rank, world
    return cfg


def render_path_distributed(backend, camera, config, group=None):
    """render.render_path over every rank of the default process group.

    Returns (Framebuffer on every rank, per-rank stats)."""
    import torch.distributed as dist

    from .render import film_from_accum, render_path_device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cfg = tile_config(config, rank, world)
    accum, stats = render_path_device(backend, camera, cfg)
    if world > 1:
        dist.all_reduce(accum, op=dist.ReduceOp.SUM, group=group)
    return film_from_accum(accum, camera, cfg.spp), stats
