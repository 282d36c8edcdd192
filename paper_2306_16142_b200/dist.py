"""Multi-GPU rendering: image-tile sharding with one collective (the film).

The path shards by pixel: a path touches only its own film entry
(render.py:215-243) and every random draw is addressed by the GLOBAL pixel
index, so splitting the film changes nothing but who renders what.  64x64
tiles of the row-major film go round-robin to ranks (tile k -> rank k % world),
or, with a tile_owner table, to the rank balanced_tile_owners picks for them;
each rank renders its tiles on its own GPU (ddf_render_path with tile / rank /
world) into a full-size float64 accumulator that is zero elsewhere, and one
all-reduce(sum) over NCCL gathers the film exactly (x + 0 = x).
"""

from __future__ import annotations

import copy

import numpy as np


def owned_pixels(width: int, height: int, tile: int, rank: int, world: int,
                 tile_owner: np.ndarray | None = None) -> np.ndarray:
    """Ascending global pixel ids owned by `rank` -- the same rule as
    ddf_render_path (csrc/ddf_api.cu)."""
    idx = np.arange(width * height)
    if tile > 0:
        ntx = (width + tile - 1) // tile
        tid = (idx // width // tile) * ntx + (idx % width) // tile
        owner = tid % world if tile_owner is None else np.asarray(tile_owner)[tid]
        return idx[owner == rank]
    return idx[idx % world == rank] if world > 1 else idx


def measure_tile_costs(backend, camera, config, tile: int = 64, spp: int = 1) -> np.ndarray:
    """Per-tile cost (row-major tile order) from a pilot render: each tile is
    rendered alone at `spp` samples (the prefix of the config's stream;
    tile k of n_tiles is "rank k of world n_tiles" under round-robin) and
    costed at its MLP rows, forward + 2 x gradient (a gradient row
    is 2F).  Box-coverage estimates miss the variation that matters (how
    long paths survive inside the bounds), so the pilot measures it."""
    import torch

    from .render import render_path_device
    ntx = (camera.width + tile - 1) // tile
    nty = (camera.height + tile - 1) // tile
    n = ntx * nty
    accum = torch.empty(camera.width * camera.height, dtype=torch.float64, device=backend.torch_device)
    cost = np.empty(n)
    for k in range(n):
        cfg = copy.copy(config)
        cfg.tile, cfg.rank, cfg.world, cfg.tile_owner = tile, k, n, None
        cfg.spp, cfg.graph, cfg.profile = min(spp, config.spp), 0, 0
        _, st = render_path_device(backend, camera, cfg, accum=accum)
        cost[k] = st["forward_rows"] + 2.0 * st["gradient_rows"] + 1e-3 * st["path_samples"]
    return cost


def balanced_tile_owners(costs: np.ndarray, world: int) -> np.ndarray:
    """Longest-processing-time assignment: tiles in descending cost (ties by
    tile id) each go to the least-loaded rank (ties to the rank with fewer
    tiles, then the lowest rank, so equal costs deal out round-robin).
    Deterministic: the same costs give the same table on every rank."""
    costs = np.asarray(costs, dtype=np.float64)
    owner = np.empty(len(costs), dtype=np.int32)
    load = [0.0] * world
    count = [0] * world
    for k in np.lexsort((np.arange(len(costs)), -costs)):
        r = min(range(world), key=lambda q: (load[q], count[q], q))
        owner[k] = r
        load[r] += float(costs[k])
        count[r] += 1
    return owner


def tile_config(config, rank: int, world: int, tile: int = 64, tile_owner=None):
    """Per-rank copy of `config`; tiles round-robin unless a tile_owner table
    (balanced_tile_owners) is given."""
    cfg = copy.copy(config)
    cfg.tile = getattr(config, "tile", 0) or tile
    cfg.rank, cfg.world = rank, world
    if world > 1 and tile_owner is not None:
        cfg.tile_owner = np.asarray(tile_owner, dtype=np.int32)
    return cfg


def balanced_owners_distributed(backend, camera, config, world: int, tile: int = 64, group=None):
    """Rank 0 runs the pilot (measure_tile_costs) and broadcasts the
    balanced table, so every rank holds the identical partition (a table
    computed per rank could differ if the pilots did).  Setup work: done once
    per scene and camera, outside any timed render."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    ntx = (camera.width + tile - 1) // tile
    nty = (camera.height + tile - 1) // tile
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.empty(ntx * nty, dtype=torch.int32, device=dev)
    if rank == 0:
        cost = measure_tile_costs(backend, camera, config, tile)
        t.copy_(torch.from_numpy(balanced_tile_owners(cost, world)))
    dist.broadcast(t, src=0, group=group)
    return t.cpu().numpy()


def render_path_distributed(backend, camera, config, group=None, tile_owner=None):
    """render.render_path over every rank of the default process group;
    `tile_owner` = "balanced" runs balanced_owners_distributed first, an
    array is used as given, None is round-robin.

    Returns (Framebuffer on every rank, per-rank stats)."""
    import torch.distributed as dist

    from .render import film_from_accum, render_path_device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if isinstance(tile_owner, str) and tile_owner == "balanced":
        tile_owner = (balanced_owners_distributed(backend, camera, config, world, group=group)
                      if world > 1 else None)
    cfg = tile_config(config, rank, world, tile_owner=tile_owner)
    accum, stats = render_path_device(backend, camera, cfg)
    if world > 1:
        dist.all_reduce(accum, op=dist.ReduceOp.SUM, group=group)
    return film_from_accum(accum, camera, cfg.spp), stats
