"""Multi-GPU rendering: image-tile sharding with one collective (the film).

The path shards by pixel.  A path touches only its own film entry
(render.py:215-243), and every random draw is addressed by the GLOBAL pixel
index, so splitting the film changes who renders a pixel, never its value.

* Partition: 64x64 tiles of the row-major film.  Tile k goes to rank
  k % world (round-robin, config 4's rule and the default), or to the rank a
  ``tile_owner`` table names (``balanced_tile_owners``, optional).
* Each rank renders its tiles on its own GPU (ddf_render_path with tile /
  rank / world) into a full-size float64 accumulator that is zero elsewhere.
* The one collective is a sum-reduce of that film to rank 0 over NCCL.  It is
  exact, because x + 0 = x: the film equals the 1-GPU film bit for bit.
"""

from __future__ import annotations

import copy
import time

import numpy as np

DEFAULT_TILE = 64


def effective_tile(config, tile: int | None = None) -> int:
    """The tile edge a distributed render uses: the config's, else ``tile``,
    else 64.  Every table and config of one render must agree on it."""
    return int(getattr(config, "tile", 0) or tile or DEFAULT_TILE)


def tile_grid(width: int, height: int, tile: int):
    return (width + tile - 1) // tile, (height + tile - 1) // tile


def owned_pixels(width: int, height: int, tile: int, rank: int, world: int,
                 tile_owner: np.ndarray | None = None) -> np.ndarray:
    """Ascending global pixel ids owned by ``rank`` -- the rule
    ddf_render_path applies (csrc/ddf_api.cu)."""
    idx = np.arange(width * height)
    if tile > 0:
        ntx, _ = tile_grid(width, height, tile)
        tid = (idx // width // tile) * ntx + (idx % width) // tile
        owner = tid % world if tile_owner is None else np.asarray(tile_owner)[tid]
        return idx[owner == rank]
    return idx[idx % world == rank] if world > 1 else idx


def measure_tile_costs(backend, camera, config, tile: int = DEFAULT_TILE, spp: int = 1, tiles=None) -> np.ndarray:
    """Per-tile cost (row-major tile order) from a pilot render.  Each tile
    in ``tiles`` (default: all) is rendered alone at ``spp`` samples, the
    prefix of the config's stream (tile k of n is "rank k of world n" under
    round-robin), and costed at its MLP rows, forward + 2 x gradient (a
    gradient row is 2F).  Tiles not measured cost 0."""
    import torch

    from .render import render_path_device
    ntx, nty = tile_grid(camera.width, camera.height, tile)
    n = ntx * nty
    accum = torch.empty(camera.width * camera.height, dtype=torch.float64, device=backend.torch_device)
    cost = np.zeros(n)
    for k in (range(n) if tiles is None else tiles):
        cfg = copy.copy(config)
        cfg.tile, cfg.rank, cfg.world, cfg.tile_owner = tile, int(k), n, None
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


def tile_config(config, rank: int, world: int, tile: int | None = None, tile_owner=None):
    """Per-rank copy of ``config`` with the effective tile; tiles go
    round-robin unless a tile_owner table is given."""
    cfg = copy.copy(config)
    cfg.tile = effective_tile(config, tile)
    cfg.rank, cfg.world = rank, world
    cfg.tile_owner = np.asarray(tile_owner, dtype=np.int32) if world > 1 and tile_owner is not None else None
    return cfg


def _collective_device(group):
    import torch.distributed as dist
    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def balanced_owners_distributed(backend, camera, config, world: int, tile: int | None = None, group=None):
    """Pilot on every rank, then one exact sum of the cost vector.

    Rank r measures the tiles it owns under round-robin (k % world == r), so
    the pilot's 1-spp renders split across the GPUs.  The cost vectors are
    disjoint, so their sum is exact, and every rank derives the identical LPT
    table from it.  Returns (table, setup seconds on this rank)."""
    import torch
    import torch.distributed as dist
    t0 = time.perf_counter()
    tile = effective_tile(config, tile)
    rank = dist.get_rank(group)
    ntx, nty = tile_grid(camera.width, camera.height, tile)
    mine = [k for k in range(ntx * nty) if k % world == rank]
    cost = torch.from_numpy(measure_tile_costs(backend, camera, config, tile, tiles=mine))
    cost = cost.to(_collective_device(group))
    dist.all_reduce(cost, op=dist.ReduceOp.SUM, group=group)
    return balanced_tile_owners(cost.cpu().numpy(), world), time.perf_counter() - t0


def reduce_film(accum, group=None, dst: int = 0, force_collective: bool = False):
    """Sum the per-rank films onto rank ``dst`` in place (NCCL reduce; gloo
    reduces a host copy).  Exact: every pixel has one non-zero term.  A
    one-rank group skips the collective unless ``force_collective`` (tests
    run the NCCL reduce itself on the one GPU of the test box)."""
    import torch.distributed as dist
    if dist.get_world_size(group) == 1 and not force_collective:
        return accum
    if _collective_device(group) == "cpu" and accum.is_cuda:
        host = accum.cpu()
        dist.reduce(host, dst=dst, op=dist.ReduceOp.SUM, group=group)
        accum.copy_(host)
    else:
        dist.reduce(accum, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return accum


def render_path_distributed(backend, camera, config, group=None, tile_owner=None):
    """render.render_path over every rank of ``group``.

    ``tile_owner``: None = round-robin (config 4), "balanced" = the pilot
    table of balanced_owners_distributed, or an explicit table.  Returns
    (Framebuffer on rank 0 and None elsewhere, this rank's stats, with
    "pilot_s" when a pilot ran)."""
    import torch.distributed as dist

    from .render import film_from_accum, render_path_device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    pilot_s = None
    if isinstance(tile_owner, str):
        if tile_owner != "balanced":
            raise ValueError(f"unknown tile_owner mode {tile_owner!r}")
        tile_owner = None
        if world > 1:
            tile_owner, pilot_s = balanced_owners_distributed(backend, camera, config, world, group=group)
    cfg = tile_config(config, rank, world, tile_owner=tile_owner)
    accum, stats = render_path_device(backend, camera, cfg)
    reduce_film(accum, group=group)
    if pilot_s is not None:
        stats["pilot_s"] = pilot_s
    return (film_from_accum(accum, camera, cfg.spp) if rank == 0 else None), stats
