"""Multi-rank host logic on CPU (gloo, world sizes 2 and 8): tile ownership,
per-rank renders of owned tiles (the CPU oracle stands in for each rank's
GPU), the pilot's cost sum and the single film reduce to rank 0 reproduce the
1-rank film bit-exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu_ddf as O
from paper_2306_16142_b200.dist import balanced_tile_owners, owned_pixels, reduce_film

W, H, TILE = 24, 16, 8


def _field_cam():
    net = O.kaiming_uniform_net((5, 32, 32, 1), 4)
    f = O.Field([net], 10.0 / 0.98, bounds=np.array([[-1.0] * 3, [1.0] * 3]))
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
    return f, cam, O.PathConfig(spp=2, bounces=3, albedo=0.7, env=1.0, seed=42, rr_start=1)


def _worker(rank, world, port, out, owner=None, pilot=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f, cam, cfg = _field_cam()
    if pilot:
        # dist.balanced_owners_distributed's exchange: each rank costs its
        # round-robin tiles (here: owned path samples x alive rows of a 1-spp
        # oracle render), one sum makes the vector identical on every rank
        ntx, nty = -(-W // TILE), -(-H // TILE)
        cost = torch.zeros(ntx * nty, dtype=torch.float64)
        for k in range(rank, ntx * nty, world):
            px = owned_pixels(W, H, TILE, k, ntx * nty)
            cost[k] = float(np.sum(O.render_path(f, cam, O.PathConfig(spp=1, bounces=3, seed=42), pixels=px) > 0))
            cost[k] += 1.0 + k % 3
        dist.all_reduce(cost, op=dist.ReduceOp.SUM)
        owner = balanced_tile_owners(cost.numpy(), world)
        out.put(("owner", rank, owner.tobytes()))
    mine = owned_pixels(W, H, TILE, rank, world, owner)
    film = torch.zeros(W * H, dtype=torch.float64)
    film[torch.from_numpy(mine)] = torch.from_numpy(O.render_path(f, cam, cfg, pixels=mine))
    reduce_film(film)
    if rank == 0:
        out.put(("film", rank, film.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_owned_pixels_partition():
    for world in (1, 2, 3, 8):
        parts = [owned_pixels(150, 70, 64, r, world) for r in range(world)]
        allp = np.concatenate(parts)
        assert len(allp) == 150 * 70 and len(np.unique(allp)) == 150 * 70
        for p in parts:
            assert np.all(np.diff(p) > 0)
    # tile k -> rank k % world
    p = owned_pixels(130, 70, 64, 1, 2)
    assert 64 in p and 0 not in p and 128 not in p


def test_pixel_subset_render_matches_full():
    f, cam, cfg = _field_cam()
    full = O.render_path(f, cam, cfg)
    sub = owned_pixels(W, H, TILE, 1, 3)
    assert np.array_equal(O.render_path(f, cam, cfg, pixels=sub), full[sub])


def test_balanced_tile_owners_lpt():
    cost = np.array([5.0, 1.0, 4.0, 4.0, 2.0, 0.0, 3.0])
    o = balanced_tile_owners(cost, 3)
    assert o.dtype == np.int32 and o.shape == cost.shape
    # LPT by hand: 5->r0, 4->r1, 4->r2, 3->r1, 2->r2, 1->r0, 0->r0
    assert list(o) == [0, 0, 1, 2, 2, 0, 1]
    load = np.bincount(o, weights=cost, minlength=3)
    assert load.max() - load.min() <= cost.max()
    assert np.array_equal(o, balanced_tile_owners(cost, 3))          # deterministic
    assert np.array_equal(balanced_tile_owners(np.zeros(10), 4), np.arange(10) % 4)   # ties -> round-robin
    rng = np.random.default_rng(3)
    c = rng.gamma(2.0, 1.0, 510)
    for world in (2, 4, 8):
        o = balanced_tile_owners(c, world)
        lb = np.bincount(o, weights=c, minlength=world)
        rr = np.bincount(np.arange(510) % world, weights=c, minlength=world)
        assert lb.max() <= rr.max() and lb.max() / lb.mean() < 1.01
        parts = [owned_pixels(1920, 1080, 64, r, world, o) for r in range(world)]
        allp = np.concatenate(parts)
        assert len(allp) == 1920 * 1080 and len(np.unique(allp)) == 1920 * 1080


@pytest.mark.parametrize("world,balanced,pilot", [(2, False, False), (2, True, False), (8, False, False),
                                                  (8, False, True)])
def test_gloo_film_reduce_is_exact(world, balanced, pilot):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    owner = None
    if balanced:   # a skewed table from a made-up cost: one heavy tile alone on rank 0
        owner = balanced_tile_owners(np.array([9.0, 1.0, 1.0, 1.0, 1.0, 1.0]), 2)
        assert list(np.bincount(owner)) == [1, 5]
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, owner, pilot)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(1 + (world if pilot else 0))]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    films = [m for m in msgs if m[0] == "film"]
    assert len(films) == 1 and films[0][1] == 0
    got = np.frombuffer(films[0][2], dtype=np.float64)
    if pilot:   # every rank derived the same table; 6 tiles land on 6 distinct ranks
        tables = {np.frombuffer(m[2], dtype=np.int32).tobytes() for m in msgs if m[0] == "owner"}
        assert len(tables) == 1
        n_tiles = -(-W // TILE) * -(-H // TILE)
        assert set(np.frombuffer(tables.pop(), dtype=np.int32)) == set(range(min(world, n_tiles)))
    f, cam, cfg = _field_cam()
    assert np.array_equal(got, O.render_path(f, cam, cfg))
