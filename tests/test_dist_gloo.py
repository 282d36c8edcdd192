"""Multi-rank host logic on CPU (gloo, world size 2): tile ownership, per-rank
renders of owned tiles (CPU oracle stands in for each rank's GPU), and the
single all-reduce of the film reproduce the 1-rank film bit-exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu_ddf as O
from paper_2306_16142_b200.dist import balanced_tile_owners, owned_pixels

W, H, TILE = 24, 16, 8


def _field_cam():
    net = O.kaiming_uniform_net((5, 32, 32, 1), 4)
    f = O.Field([net], 10.0 / 0.98, bounds=np.array([[-1.0] * 3, [1.0] * 3]))
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
    return f, cam, O.PathConfig(spp=2, bounces=3, albedo=0.7, env=1.0, seed=42, rr_start=1)


def _worker(rank, world, port, out, owner=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f, cam, cfg = _field_cam()
    mine = owned_pixels(W, H, TILE, rank, world, owner)
    film = torch.zeros(W * H, dtype=torch.float64)
    film[torch.from_numpy(mine)] = torch.from_numpy(O.render_path(f, cam, cfg, pixels=mine))
    dist.all_reduce(film, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put(film.numpy().tobytes())
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


@pytest.mark.parametrize("balanced", [False, True])
def test_gloo_world2_film_allreduce_is_exact(balanced):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    owner = None
    if balanced:   # a skewed table from a made-up cost: one heavy tile alone on rank 0
        owner = balanced_tile_owners(np.array([9.0, 1.0, 1.0, 1.0, 1.0, 1.0]), 2)
        assert list(np.bincount(owner)) == [1, 5]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, owner)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=np.float64)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    f, cam, cfg = _field_cam()
    assert np.array_equal(got, O.render_path(f, cam, cfg))
