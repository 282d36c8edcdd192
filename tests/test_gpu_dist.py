"""dist.render_path_distributed with a real 2-rank process group.

Both ranks share cuda:0 (the test box has one GPU) and reduce over gloo; the
ranks' kernels never wait on each other, only the host-side reduce does.
The film reduced onto rank 0 must equal the 1-rank film bit-exactly."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

W, H = 150, 70


def _setup(precision, tile=0):
    from paper_2306_16142_b200 import render as R
    from paper_2306_16142_b200.field import CudaNeuralField
    from paper_2306_16142_b200.neural import kaiming_uniform
    net = kaiming_uniform((65, 128, 128, 1), 6)
    f = CudaNeuralField(net, 10.0 / 0.98, bounds=np.array([[-1.0] * 3, [1.0] * 3]), precision=precision)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
    cfg = R.RenderConfig(spp=2, bounces=3, seed=5, rr_start=1, tile=tile)
    return f, cam, cfg


def _worker(rank, world, port, precision, out, tile_owner=None, tile=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_16142_b200.dist import render_path_distributed
    f, cam, cfg = _setup(precision, tile)
    fb, stats = render_path_distributed(f, cam, cfg, tile_owner=tile_owner)
    assert (fb is None) == (rank != 0)
    out.put((rank, None if fb is None else np.asarray(fb.data).tobytes(), int(stats["path_samples"]),
             stats.get("pilot_s")))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("precision,balance,tile", [("fp32", None, 0), ("bf16", None, 0), ("bf16", "balanced", 0),
                                                   ("bf16", "balanced", 32)])
def test_two_rank_render_equals_single_rank(precision, balance, tile):
    from paper_2306_16142_b200 import render as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, precision, q, balance, tile)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    f, cam, cfg = _setup(precision)
    want = np.asarray(R.render_path(f, cam, cfg).data)
    films = {r: b for r, b, _, _ in got}
    assert films[1] is None
    assert np.array_equal(np.frombuffer(films[0], dtype=want.dtype).reshape(want.shape), want)
    assert sum(n for _, _, n, _ in got) == W * H * cfg.spp
    if balance:   # the pilot ran on both ranks and reports its setup time
        assert all(p is not None and p > 0 for _, _, _, p in got)


def _nccl_worker(port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    from paper_2306_16142_b200 import render as R
    from paper_2306_16142_b200.dist import balanced_owners_distributed, reduce_film, tile_config
    f, cam, cfg = _setup("bf16", tile=32)
    accum, _ = R.render_path_device(f, cam, tile_config(cfg, 0, 1))
    want = accum.clone()
    reduce_film(accum, force_collective=True)          # ncclReduce of the float64 film
    table, pilot_s = balanced_owners_distributed(f, cam, cfg, 1)   # ncclAllReduce of the cost vector
    torch.cuda.synchronize()
    out.put((bool(torch.equal(accum, want)), sorted(set(int(x) for x in table)), float(pilot_s), dist.get_backend()))
    dist.destroy_process_group()


def test_nccl_collectives_on_one_rank():
    """The box has one GPU and NCCL refuses two ranks on one device, so the
    multi-GPU path's two collectives (the float64 film reduce and the pilot's
    cost all-reduce) run here over NCCL in a one-rank group: the calls, dtypes
    and device placement the N-GPU run makes, with nothing to sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    same, owners, pilot_s, backend = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert backend == "nccl" and same and owners == [0] and pilot_s > 0


def test_tile_owner_table_partitions_film_exactly():
    """Three ranks under a pilot-balanced table (and a hand-made one): the
    per-rank films are disjoint and sum bit-exactly to the 1-rank film; a bad
    table entry is a usage error."""
    import torch as T

    from paper_2306_16142_b200 import render as R
    from paper_2306_16142_b200.dist import balanced_tile_owners, measure_tile_costs, owned_pixels, tile_config
    f, cam, cfg = _setup("bf16")
    want, _ = R.render_path_device(f, cam, R.RenderConfig(**{**cfg.__dict__, "graph": 0}))
    want = want.cpu().numpy()
    cost = measure_tile_costs(f, cam, cfg, tile=32)
    assert cost.shape == (((W + 31) // 32) * ((H + 31) // 32),) and np.all(cost > 0)
    for owner in (balanced_tile_owners(cost, 3), np.array([2, 2, 2, 2, 2, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1])):
        total = np.zeros_like(want)
        for rank in range(3):
            c = tile_config(cfg, rank, 3, tile=32, tile_owner=owner)
            c.tile = 32
            acc, st = R.render_path_device(f, cam, c)
            acc = acc.cpu().numpy()
            mine = owned_pixels(W, H, 32, rank, 3, owner)
            assert st["path_samples"] == len(mine) * cfg.spp
            other = np.ones(W * H, bool)
            other[mine] = False
            assert np.all(acc[other] == 0.0)
            total += acc
        assert np.array_equal(total, want)
    bad = tile_config(cfg, 0, 3, tile=32, tile_owner=np.full(15, 3))
    bad.tile = 32
    with pytest.raises(ValueError, match="tile_owner"):
        R.render_path_device(f, cam, bad)
    short = tile_config(cfg, 0, 3, tile=32, tile_owner=np.zeros(14))
    short.tile = 32
    with pytest.raises(ValueError, match="tile_owner has 14"):
        R.render_path_device(f, cam, short)
    T.cuda.synchronize()
