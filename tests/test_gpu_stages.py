"""Compaction and pixel-index parity INSIDE the render (render.py:225,
field.py:277): every slot list the wavefront compacts, read back through
ddf_path_config_t.stage_log, against the oracle's np.nonzero lists for the
same render.  The oracle's stage lengths are pinned to the unmodified
reference (tests/test_oracle_golden.py::test_render_stage_lists_match_reference_lengths).

Bars:
  primary march step 0 (box entry, f64 geometry)   identical lists
  march regime (delta = 0.1, exact fp32 engine)     identical lists (measured: all 184 stages)
  config 2, fp32 engines                            <= 0.002 % (FFMA) / 0.01 % (3xTF32) of
                                                    entries differ (measured 1 and 17 of 274,105)
  per-stage counts in ddf_render_stats_t            = the logged list lengths
  fused vs unfused bf16 march                       identical lists
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import cpu_ddf as O  # noqa: E402
from paper_2306_16142_b200 import render as R  # noqa: E402
from paper_2306_16142_b200.field import CudaNeuralField  # noqa: E402
from paper_2306_16142_b200.neural import MlpModel, kaiming_uniform  # noqa: E402

CFG_DELTA = 10.0 / 0.98
BOX = np.array([[-1.0] * 3, [1.0] * 3])


def march_net():
    net = O.kaiming_uniform_net((5, 64, 64, 1), seed=7)
    net.g[-1] = net.g[-1] * 0.05
    net.b[-1] = net.b[-1] + 0.12
    return net


def parse_stage_log(log, spp):
    """stage_log words -> {(kind, bounce, step, sample): ascending local pixel
    ids}; kinds 2 and 3 (the two halves of a fused march step) are merged
    into kind 2."""
    w = log.cpu().numpy()
    assert w[1] == 0, "stage log overflowed"
    end, pos, out = 2 + int(w[0]), 2, {}
    while pos < end:
        kind, b, step, s0, n_own, n = (int(x) for x in w[pos:pos + 6])
        ids = w[pos + 6:pos + 6 + n].astype(np.int64)
        pos += 6 + n
        kind = 2 if kind == 3 else kind
        for s in range(s0, spp):
            sel = ids[(ids // n_own) == s - s0]
            if len(sel) or (kind, b, step, s) not in out:
                key = (kind, b, step, s)
                out[key] = np.union1d(out.get(key, np.empty(0, np.int64)), sel % n_own)
    return out


def oracle_stages(log):
    out = {}
    for s, rec in enumerate(log):
        for j, lst in enumerate(rec["primary_march"]):
            out[(0, -1, j, s)] = np.asarray(lst, np.int64)
        for b, lst in enumerate(rec["bounce_alive"]):
            out[(1, b, 0, s)] = np.asarray(lst, np.int64)
        for b, steps in enumerate(rec["bounce_march"]):
            for j, lst in enumerate(steps):
                out[(2, b, j, s)] = np.asarray(lst, np.int64)
    return out


def compare(gpu, ref):
    """(identical stages, total stages, entries in only one of the lists,
    total entries).  A stage missing on one side is an empty list."""
    same = total = diff = entries = 0
    for k in set(gpu) | set(ref):
        a = gpu.get(k, np.empty(0, np.int64))
        b = ref.get(k, np.empty(0, np.int64))
        if not len(a) and not len(b):
            continue
        total += 1
        same += int(np.array_equal(a, b))
        diff += len(np.setxor1d(a, b))
        entries += max(len(a), len(b))
    return same, total, diff, entries


def render_logged(f, w, h, cfg, cap=1 << 24):
    log = torch.zeros(cap, dtype=torch.int32, device="cuda")
    cfg.stage_log = log
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=w, height=h)
    acc, stats = R.render_path_device(f, cam, cfg)
    return acc.cpu().numpy() / cfg.spp, stats, parse_stage_log(log, cfg.spp)


def oracle_render(f, w, h, cfg):
    log = []
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=w, height=h)
    img = O.render_path(f, cam, cfg, log=log)
    return img, oracle_stages(log)


def check_stats(stats, lists):
    """ddf_render_stats_t per-stage counts == the lengths of the logged lists."""
    prim = np.zeros(64, np.int64)
    alive = np.zeros(32, np.int64)
    bmarch = np.zeros(32, np.int64)
    for (kind, b, j, _), ids in lists.items():
        if kind == 0:
            prim[j] += len(ids)
        elif kind == 1:
            alive[b] += len(ids)
        else:
            bmarch[b] += len(ids)
    assert list(prim) == stats["primary_march_rows"]
    assert list(alive) == stats["bounce_alive_rows"]
    assert list(bmarch) == stats["bounce_march_rows"]


@pytest.mark.parametrize("prec", ["fp32_simt", "fp32"])
def test_config2_stage_lists(prec):
    net = kaiming_uniform((5,) + (256,) * 8 + (1,), 1)
    f = CudaNeuralField(net, CFG_DELTA, bounds=BOX, precision=prec)
    img, stats, gpu = render_logged(f, 128, 128, R.RenderConfig(spp=4, bounces=2, albedo=0.7, seed=42))
    of = O.Field([O.Net(net.widths, net.v, net.g, net.b)], CFG_DELTA, bounds=BOX)
    _, ref = oracle_render(of, 128, 128, O.PathConfig(spp=4, bounces=2, albedo=0.7, env=1.0, seed=42))
    check_stats(stats, gpu)
    for s in range(4):
        assert np.array_equal(gpu[(0, -1, 0, s)], ref[(0, -1, 0, s)])
    same, total, diff, entries = compare(gpu, ref)
    print(f"config 2 {prec}: {same}/{total} stages identical, {diff} of {entries} entries differ")
    assert diff <= (2e-5 if prec == "fp32_simt" else 1e-4) * entries


def test_march_regime_stage_lists():
    """delta = 0.1 (the reference default): rays march up to 47 steps and
    every step's list is compacted on the device."""
    net = march_net()
    f = CudaNeuralField(MlpModel(net.widths, net.v, net.g, net.b), 0.1, bounds=BOX, precision="fp32")
    cfg = R.RenderConfig(spp=2, bounces=3, albedo=0.6, env_radiance=1.5, seed=9)
    img, stats, gpu = render_logged(f, 48, 32, cfg)
    ref_img, ref = oracle_render(O.Field([net], 0.1, bounds=BOX), 48, 32,
                                 O.PathConfig(spp=2, bounces=3, albedo=0.6, env=1.5, seed=9))
    check_stats(stats, gpu)
    for s in range(2):
        assert np.array_equal(gpu[(0, -1, 0, s)], ref[(0, -1, 0, s)])
    same, total, diff, entries = compare(gpu, ref)
    print(f"march regime: {same}/{total} stages identical, {diff} of {entries} entries differ; "
          f"film RMSE {np.sqrt(np.mean((img - ref_img) ** 2)):.3g}")
    assert total > 40
    assert same == total


def test_fused_and_unfused_lists_identical():
    """bf16 on a 512-wide PE network fuses a bounce ray's first march step
    with its next normal; the lists (kind 3 + kind 2) equal the unfused run's."""
    net = kaiming_uniform((65, 512, 512, 512, 1), 2)
    f = CudaNeuralField(net, CFG_DELTA, bounds=BOX, precision="bf16")
    cfg = dict(spp=2, bounces=4, seed=42, rr_start=2)
    img_a, st_a, a = render_logged(f, 40, 30, R.RenderConfig(**cfg))
    img_b, st_b, b = render_logged(f, 40, 30, R.RenderConfig(**cfg, no_fuse=1))
    assert st_a["fused_rows"] > 0 and st_b["fused_rows"] == 0
    assert np.array_equal(img_a, img_b)
    same, total, _, _ = compare(a, b)
    assert same == total
    for k in ("primary_march_rows", "bounce_alive_rows", "bounce_march_rows"):
        assert st_a[k] == st_b[k]


def test_stage_log_overflow_is_flagged():
    f = CudaNeuralField(kaiming_uniform((5, 32, 32, 1), 3), CFG_DELTA, bounds=BOX)
    log = torch.zeros(64, dtype=torch.int32, device="cuda")
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=16, height=16)
    R.render_path_device(f, cam, R.RenderConfig(spp=1, bounces=1, seed=1, stage_log=log))
    w = log.cpu().numpy()
    assert w[1] == 1 and w[0] <= 62
