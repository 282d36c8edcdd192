"""Fused normal reuse ("fused normal-reuse optimisation"): a
bounce ray's first march step and the next bounce's normal evaluate the
network at the same input whenever t_acc == max(t_hit - delta/2, 0)
(field.py:274-285 vs field.py:305-309), so the bf16 engine runs the forward
and the backward chain of those rows in one kernel (TraceGradOp).

The bar is bit-identity with the unfused passes: same film, same per-stage
row counts, same degenerate-normal count -- the reference's count of normal
evaluations stays in `gradient_rows`, only where they execute changes.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2306_16142_b200 import render as R  # noqa: E402
from paper_2306_16142_b200.field import CudaNeuralField  # noqa: E402
from paper_2306_16142_b200.neural import kaiming_uniform  # noqa: E402

BOX = np.array([[-1.0] * 3, [1.0] * 3])
D = 10.0 / 0.98


def _render(f, cam, cfg):
    acc, st = R.render_path_device(f, cam, cfg)
    torch.cuda.synchronize()
    return acc.cpu().numpy().copy(), st


@pytest.mark.parametrize("widths", [(65, 384, 384, 384, 1), (5, 512, 512, 1)])
@pytest.mark.parametrize("rr,waves,graph", [(-1, 0, 0), (2, 0, 1), (1, 1500, 0)])
def test_fused_render_bit_identical(widths, rr, waves, graph):
    net = kaiming_uniform(widths, 3)
    f = CudaNeuralField(net, D, bounds=BOX, precision="bf16")
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=40, height=36)
    base = dict(spp=3, bounces=4, seed=42, rr_start=rr, max_wave_paths=waves, graph=graph)
    a0, s0 = _render(f, cam, R.RenderConfig(no_fuse=1, **base))
    a1, s1 = _render(f, cam, R.RenderConfig(no_fuse=0, **base))
    if graph:   # the replayed graph gives the same film again
        a1, s1 = _render(f, cam, R.RenderConfig(no_fuse=0, **base))
    assert s0["fused_rows"] == 0 and s0["gradient_rows_executed"] == s0["gradient_rows"]
    assert s1["fused_rows"] > 0
    assert s1["gradient_rows_executed"] < s1["gradient_rows"]
    for k in ("forward_rows", "gradient_rows", "degenerate", "path_samples"):
        assert s0[k] == s1[k], k
    np.testing.assert_array_equal(a0, a1)


def test_fusion_off_in_march_regime():
    """delta = 0.1: a bounce ray's first step is rarely where its normal is
    taken, so the engine keeps the unfused passes (and the same film)."""
    net = kaiming_uniform((5, 384, 384, 1), 4)
    f = CudaNeuralField(net, 0.1, bounds=BOX, precision="bf16")
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=16, height=16)
    a, s = _render(f, cam, R.RenderConfig(spp=1, bounces=2, seed=42))
    assert s["fused_rows"] == 0 and s["gradient_rows_executed"] == s["gradient_rows"]
    b, _ = _render(f, cam, R.RenderConfig(spp=1, bounces=2, seed=42, no_fuse=1))
    np.testing.assert_array_equal(a, b)


def test_fusion_not_used_for_fp32_or_narrow():
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=16, height=16)
    for widths, prec in (((5, 384, 384, 1), "fp32"), ((5, 256, 256, 1), "bf16")):
        f = CudaNeuralField(kaiming_uniform(widths, 5), D, bounds=BOX, precision=prec)
        _, s = _render(f, cam, R.RenderConfig(spp=1, bounces=3, seed=42))
        assert s["fused_rows"] == 0, (widths, prec)
