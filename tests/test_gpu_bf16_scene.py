"""GPU parity for the tcgen05 bf16 engine, the 65-D encoding and the
multi-object scene (EXTENSIONS, parity against the oracle restatement).

bf16 tolerance (stated, measured; SURVEY App. B probe 3e-2..1.1e-1):
  distances              max |d| / rms(ref) <= 0.15, median <= 0.02
  input gradients        kernel == numpy bf16 emulation (median 1e-4); vs
                         float64 the per-row error median is <= 0.5 of rms:
                         bf16 rounding flips ReLU masks near kinks and deep
                         nets' gradients change discretely (emulation shows
                         the same; measured medians 0.01 (3 layers) to 0.37
                         (9 layers))
  bf16 image (config-2 net)  RMSE <= 0.12 (probe 9.5e-2), mean within 0.02
fp32 engine on the PE / scene paths keeps the fp32 tolerance 1e-4.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import cpu_ddf as O  # noqa: E402
from paper_2306_16142_b200 import configs as C  # noqa: E402
from paper_2306_16142_b200 import render as R  # noqa: E402
from paper_2306_16142_b200.field import CudaNeuralField  # noqa: E402
from paper_2306_16142_b200.neural import MlpModel, kaiming_uniform  # noqa: E402

BOX = np.array([[-1.0] * 3, [1.0] * 3])
D = 10.0 / 0.98


def onet(m):
    return O.Net(m.widths, m.v, m.g, m.b)


def err_stats(x, ref):
    rms = np.sqrt(np.mean(ref ** 2))
    e = np.abs(x - ref) / rms
    return float(e.max()), float(np.median(e))


def fp32_ok(x, ref, tol=1e-4):
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref ** 2)))
    return np.max(np.abs(x - ref) / scale) <= tol


def bf16(x):
    """Round-to-nearest-even float32 -> bfloat16 (kept as float32)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)


def bf16_emulation(m, x):
    """What the tcgen05 engine computes: bf16 operands, fp32 accumulate, fp32
    bias/ReLU epilogue, fp32 head dot; gradient chain with bf16 d_h."""
    ws = [w.astype(np.float32) for w in onet(m).effective()]
    bs = [b.astype(np.float32) for b in m.b]
    L = len(ws)
    a, masks = bf16(x), []
    for l in range(L - 1):
        z = a @ bf16(ws[l]).T + bs[l]
        masks.append(z > 0)
        r = np.maximum(z, 0)
        a = bf16(r)
    y = r @ ws[L - 1][0] + bs[L - 1][0]
    G = bf16(ws[L - 1][0][None, :] * masks[L - 2])
    for l in range(L - 2, 0, -1):
        G = bf16((G @ bf16(ws[l])) * masks[l - 1])
    return y, G @ bf16(ws[0])


@pytest.mark.parametrize("widths", [(5, 128, 128, 128, 128, 1), (5,) + (256,) * 8 + (1,), (65,) + (512,) * 8 + (1,),
                                    (65,) + (256,) * 6 + (1,), (5, 64, 64, 1), (65, 100, 200, 1), (65, 128, 256, 1),
                                    (5, 192, 192, 1), (65, 384, 384, 1), (5, 320, 448, 1)])
def test_bf16_forward_and_gradient(widths):
    m = kaiming_uniform(widths, 3)
    f = CudaNeuralField(m, D, bounds=BOX, precision="bf16")
    n = 3000
    if widths[0] == 65:
        o, d = C.query_rays(n, 2)
        x = O.pe_encode(O.encode5(o, O.dirs_to_angles(d)))
    else:
        x = np.random.default_rng(1).uniform(-1, 1, (n, widths[0]))
    y, g = f.forward_inputs(x), f.input_gradient_inputs(x)
    ye, ge = bf16_emulation(m, x)
    # 1) the kernel computes exactly the bf16 arithmetic (up to fp32 summation
    #    order, which can flip a ReLU mask at an exact kink in deep nets)
    ey = np.abs(y - ye) / np.sqrt(np.mean(ye ** 2))
    eg = np.max(np.abs(g - ge), axis=1) / np.sqrt(np.mean(ge ** 2))
    assert np.median(ey) <= 1e-4 and ey.max() <= 0.05
    assert np.median(eg) <= 1e-4 and np.mean(eg > 1e-2) <= 0.10
    # 2) bf16 vs the float64 reference: the stated bf16 tolerance
    ref = O.mlp_forward(onet(m), x)
    mx, med = err_stats(y, ref)
    gref = O.mlp_input_grad(onet(m), x)
    e = np.max(np.abs(g - gref), axis=1) / np.sqrt(np.mean(gref ** 2))
    print(f"bf16 {widths[:3]}.. L={len(widths) - 1}: distance max {mx:.3g} median {med:.3g}; "
          f"gradient median {np.median(e):.3g} p90 {np.percentile(e, 90):.3g}")
    assert mx <= 0.15 and med <= 0.02
    assert np.median(e) <= 0.5
    # fp32 engine on the same net is within the fp32 tolerance
    f.set_precision("fp32")
    assert fp32_ok(f.forward_inputs(x), ref)


@pytest.mark.parametrize("widths", [(5, 128, 128, 128, 1), (5, 64, 96, 1), (5, 192, 256, 1), (5, 160, 192, 1),
                                    (65, 512, 512, 512, 1), (5, 320, 448, 1), (65, 128, 128, 1)])
def test_bf16_nonzero_biases(widths):
    """Trained checkpoints carry biases; the BASELINE's synthetic networks have
    none.  The <= 128-wide and > 256-wide engines fold the bias into the
    accumulator (a bf16 hi/mid/lo bias chunk against a ones block), the
    129..256-wide engine adds it in the epilogue: all three against the bf16
    emulation (fp32 bias add) and the float64 reference, forward and gradient,
    plus the fp32 engines on the same network."""
    m = kaiming_uniform(widths, 5)
    rng = np.random.default_rng(17)
    m.b = [rng.normal(0.0, 0.3, size=np.shape(b)) for b in m.b]
    f = CudaNeuralField(m, D, bounds=BOX, precision="bf16")
    n = 2500
    if widths[0] == 65:
        o, d = C.query_rays(n, 4)
        x = O.pe_encode(O.encode5(o, O.dirs_to_angles(d)))
    else:
        x = rng.uniform(-1, 1, (n, widths[0]))
    y, g = f.forward_inputs(x), f.input_gradient_inputs(x)
    ye, ge = bf16_emulation(m, x)
    ey = np.abs(y - ye) / np.sqrt(np.mean(ye ** 2))
    eg = np.max(np.abs(g - ge), axis=1) / np.sqrt(np.mean(ge ** 2))
    print(f"bf16 with biases {widths}: vs emulation median {np.median(ey):.3g} max {ey.max():.3g}")
    assert np.median(ey) <= 1e-4 and ey.max() <= 0.05
    assert np.median(eg) <= 1e-4 and np.mean(eg > 1e-2) <= 0.10
    ref = O.mlp_forward(onet(m), x)
    mx, med = err_stats(y, ref)
    assert mx <= 0.15 and med <= 0.02
    f.set_precision("fp32")
    assert fp32_ok(f.forward_inputs(x), ref)
    gref = O.mlp_input_grad(onet(m), x)
    e = np.max(np.abs(f.input_gradient_inputs(x) - gref), axis=1) / np.sqrt(np.mean(gref ** 2))
    assert np.mean(e > 1e-4) <= 1e-3


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_pe65_query_trace_normal(prec):
    m = kaiming_uniform((65,) + (128,) * 3 + (1,), 2)
    f = CudaNeuralField(m, D, bounds=BOX, precision=prec)
    of = O.Field([onet(m)], D, bounds=BOX)
    o, d = C.query_rays(4096, 5)
    o2 = o * 2.5
    pred, t, hit, _ = f.query_raw(o, d)
    ang = O.dirs_to_angles(O.angles_to_dirs(O.dirs_to_angles(d)))
    pref, _ = of.predict(o, ang)
    if prec == "fp32":
        assert fp32_ok(pred, pref)
    else:
        assert err_stats(pred, pref)[0] <= 0.15
    tt, hh = f.trace_batch(o2, d)
    tr, hr, _ = of.trace(o2, d)
    assert (hh == hr).mean() >= 0.999
    both = hh & hr
    th = np.where(np.isfinite(tr), tr, 0.0)
    n, v = f.normal_batch(o2, d, t_hit=th)
    nr, vr = of.normal(o2, d, t_hit=th)
    cos = np.clip(np.einsum("ij,ij->i", n, nr), -1, 1)
    ang_err = np.degrees(np.arccos(cos))
    print(f"PE65 {prec} normals: angular error median {np.median(ang_err):.2e} p99 {np.percentile(ang_err, 99):.2e}"
          f" max {ang_err.max():.2e} deg")
    if prec == "fp32":
        # the PE chain multiplies fp32 gradient errors by up to 2^5 pi; rays whose
        # spatial gradient nearly cancels show it as a larger angle
        assert np.max(np.abs(tt[both] - tr[both])) <= 1e-4
        assert np.percentile(ang_err, 99) < 0.05 and ang_err.max() < 2.0
    else:
        assert np.median(np.abs(tt[both] - tr[both])) <= 2e-2
        assert np.median(ang_err) < 5.0


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_scene_composite(prec):
    ms = [kaiming_uniform((65, 64, 64, 1), s) for s in range(10, 18)]
    centers, scale, albedos = C.scene_layout()
    f = CudaNeuralField.scene(ms, centers, scale, albedos, D, bounds=C.SCENE_BOX, precision=prec)
    of = O.Field([onet(m) for m in ms], D, bounds=C.SCENE_BOX, centers=centers, scale=scale, albedos=albedos)
    o, d = C.query_rays(2048, 9)
    o = o * 3.0
    pred, t, hit, obj = f.query_raw(o, d)
    ang = O.dirs_to_angles(O.angles_to_dirs(O.dirs_to_angles(d)))
    pref, oref = of.predict(o, ang)
    if prec == "fp32":
        assert fp32_ok(pred, pref)
        assert (obj == oref).mean() >= 0.999
    else:
        assert err_stats(pred, pref)[0] <= 0.15
        assert (obj == oref).mean() >= 0.9
    tt, hh, ob = f.trace_with_objects(o, d)
    tr, hr, obr = of.trace(o, d)
    assert (hh == hr).mean() >= 0.99
    th = np.where(np.isfinite(tr), tr, 0.0)
    n, v = f.normal_batch(o, d, t_hit=th, obj=obr)
    nr, vr = of.normal(o, d, t_hit=th, obj=obr)
    cos = np.clip(np.einsum("ij,ij->i", n, nr), -1, 1)
    ang_err = np.degrees(np.arccos(cos))
    assert (ang_err.max() < 0.05) if prec == "fp32" else (np.median(ang_err) < 5.0)


@pytest.mark.parametrize("hidden", [96, 256])
def test_scene_composite_nonzero_biases(hidden):
    """Several networks per tile with biases in every layer: the quad (96) and
    ping-pong (256) engines switch network between tiles' layers, each with
    its own folded bias chunks and head weights read in place."""
    rng = np.random.default_rng(23)
    ms = [kaiming_uniform((65, hidden, hidden, 1), s) for s in range(30, 33)]
    for m in ms:
        m.b = [rng.normal(0.0, 0.25, size=np.shape(b)) for b in m.b]
    centers, scale, albedos = C.scene_layout()
    centers, albedos = centers[:3], albedos[:3]
    f = CudaNeuralField.scene(ms, centers, scale, albedos, D, bounds=C.SCENE_BOX, precision="bf16")
    of = O.Field([onet(m) for m in ms], D, bounds=C.SCENE_BOX, centers=centers, scale=scale, albedos=albedos)
    o, d = C.query_rays(3000, 12)
    o = o * 3.0
    pred, t, hit, obj = f.query_raw(o, d)
    ang = O.dirs_to_angles(O.angles_to_dirs(O.dirs_to_angles(d)))
    pref, oref = of.predict(o, ang)
    assert err_stats(pred, pref)[0] <= 0.15 and err_stats(pred, pref)[1] <= 0.02
    assert (obj == oref).mean() >= 0.9
    f.set_precision("fp32")
    p32, _, _, o32 = f.query_raw(o, d)
    assert fp32_ok(p32, pref)
    assert (o32 == oref).mean() >= 0.999


def _cam(w, h):
    return R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=w, height=h)


def test_bf16_render_config2_statistics(golden):
    m = kaiming_uniform((5,) + (256,) * 8 + (1,), 1)
    f = CudaNeuralField(m, D, bounds=BOX, precision="bf16")
    cfg = R.RenderConfig(spp=4, bounces=2, albedo=0.7, env_radiance=1.0, seed=42)
    img = R.render_path(f, _cam(128, 128), cfg).data[:, :, 0]
    ref = golden["r2_film"]
    rmse = float(np.sqrt(np.mean((img - ref) ** 2)))
    print(f"bf16 config-2 image: RMSE {rmse:.3g}, mean {img.mean():.4f} vs {ref.mean():.4f}")
    assert rmse <= 0.12
    assert abs(img.mean() - ref.mean()) <= 0.02


def test_render_scene_and_rr_vs_oracle():
    """Config-5-style scene and config-4-style Russian roulette, small film,
    fp32 engine vs the oracle restatement with identical streams."""
    ms = [kaiming_uniform((65, 64, 64, 1), s) for s in range(10, 18)]
    centers, scale, albedos = C.scene_layout()
    f = CudaNeuralField.scene(ms, centers, scale, albedos, D, bounds=C.SCENE_BOX)
    of = O.Field([onet(m) for m in ms], D, bounds=C.SCENE_BOX, centers=centers, scale=scale, albedos=albedos)
    cam = _cam(40, 30)
    oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=40, height=30)
    img = R.render_path(f, cam, R.RenderConfig(spp=3, bounces=5, seed=42, rr_start=2)).data[:, :, 0].reshape(-1)
    ref = O.render_path(of, oc, O.PathConfig(spp=3, bounces=5, albedo=0.7, env=1.0, seed=42, rr_start=2))
    rmse = float(np.sqrt(np.mean((img - ref) ** 2)))
    print("scene+RR RMSE", rmse)
    assert rmse <= 5e-3
