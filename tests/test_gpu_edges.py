"""Edge cases on the GPU path: empty and single-row batches,
axis-aligned directions (zero components: the slab test's special branch,
field.py:332-336), rays starting inside the box, tiny films, odd tilings,
bounces = 1, Russian roulette from bounce 0, and the error classes."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import cpu_ddf as O  # noqa: E402
from paper_2306_16142_b200 import render as R  # noqa: E402
from paper_2306_16142_b200.dist import owned_pixels  # noqa: E402
from paper_2306_16142_b200.errors import DataError  # noqa: E402
from paper_2306_16142_b200.field import CudaNeuralField  # noqa: E402
from paper_2306_16142_b200.neural import kaiming_uniform, save_model  # noqa: E402

BOX = np.array([[-1.0] * 3, [1.0] * 3])
D = 10.0 / 0.98


@pytest.fixture(scope="module")
def pair():
    m = kaiming_uniform((5, 64, 64, 64, 1), 12)
    return m, CudaNeuralField(m, D, bounds=BOX), O.Field([O.Net(m.widths, m.v, m.g, m.b)], D, bounds=BOX)


def test_empty_batches(pair):
    _, f, _ = pair
    e = np.zeros((0, 3))
    t, h = f.trace_batch(e, e)
    assert t.shape == (0,) and h.shape == (0,)
    t, h = f.query_batch(e, e)
    assert t.shape == (0,)
    n, v = f.normal_batch(e, e)
    assert n.shape == (0, 3)
    assert f.forward_inputs(np.zeros((0, 5))).shape == (0,)


def test_single_row_and_axis_aligned_rays(pair):
    _, f, of = pair
    o = np.array([[0.0, 0.0, 3.0], [0.5, -0.2, 3.0], [2.0, 0.0, 0.0], [0.0, 1.0, 0.5], [0.3, 0.3, 0.3],
                  [1.5, 1.5, 0.0], [1.0, 0.2, 0.1]])
    d = np.array([[0.0, 0.0, -1.0], [0.0, 0.0, -1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 1.0, 0.0],
                  [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    t, h = f.trace_batch(o, d)
    tr, hr, _ = of.trace(o, d)
    assert np.array_equal(h, hr)
    assert np.allclose(t[h], tr[hr], atol=1e-4)
    t1, h1 = f.trace_batch(o[:1], d[:1])
    assert h1[0] == h[0] and (not h[0] or abs(t1[0] - t[0]) < 1e-12)


def test_rays_starting_inside_box(pair):
    _, f, of = pair
    rng = np.random.default_rng(3)
    o = rng.uniform(-0.9, 0.9, (500, 3))
    d = rng.normal(size=(500, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, h = f.trace_batch(o, d)
    tr, hr, _ = of.trace(o, d)
    assert (h == hr).mean() >= 0.999
    both = h & hr
    assert np.max(np.abs(t[both] - tr[both])) <= 1e-4
    n, v = f.normal_batch(o, d)           # t_hit=None: gradient at the origin
    nr, vr = of.normal(o, d)
    assert np.degrees(np.arccos(np.clip(np.einsum("ij,ij->i", n, nr), -1, 1))).max() < 0.05


@pytest.mark.parametrize("w,h,spp,b", [(1, 1, 1, 1), (3, 5, 2, 1), (17, 1, 3, 2), (1, 9, 1, 4)])
def test_tiny_films(pair, w, h, spp, b):
    m, f, of = pair
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=w, height=h)
    img = R.render_path(f, cam, R.RenderConfig(spp=spp, bounces=b, seed=4)).data[:, :, 0].reshape(-1)
    oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=w, height=h)
    ref = O.render_path(of, oc, O.PathConfig(spp=spp, bounces=b, albedo=0.7, env=1.0, seed=4))
    assert np.sqrt(np.mean((img - ref) ** 2)) <= 3e-3


def test_odd_tiles_and_rr_from_zero(pair):
    _, f, of = pair
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=37, height=23)
    full, _ = R.render_path_device(f, cam, R.RenderConfig(spp=2, bounces=3, seed=8, rr_start=0))
    full = full.cpu().numpy()
    acc = np.zeros_like(full)
    for rank in range(3):
        part, _ = R.render_path_device(f, cam, R.RenderConfig(spp=2, bounces=3, seed=8, rr_start=0, tile=7,
                                                              rank=rank, world=3))
        part = part.cpu().numpy()
        mine = owned_pixels(37, 23, 7, rank, 3)
        assert np.all(part[np.setdiff1d(np.arange(37 * 23), mine)] == 0.0)
        acc += part
    assert np.array_equal(acc, full)
    oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=37, height=23)
    ref = O.render_path(of, oc, O.PathConfig(spp=2, bounces=3, albedo=0.7, env=1.0, seed=8, rr_start=0))
    assert np.sqrt(np.mean((full / 2 - ref) ** 2)) <= 3e-3


def test_from_checkpoint_and_bad_checkpoint(tmp_path, pair):
    m, _, _ = pair
    p = tmp_path / "m.ddfn"
    save_model(m, D, p)
    f = CudaNeuralField.from_checkpoint(p, bounds=BOX)
    assert f.delta == D and f.normal_eval_backoff == 0.5 * D
    (tmp_path / "bad.ddfn").write_bytes(b"DDFN" + b"\0" * 3)
    with pytest.raises(DataError):
        CudaNeuralField.from_checkpoint(tmp_path / "bad.ddfn")


def test_reference_render_modes_run_on_the_shim(pair, reference):
    """The drop-in: the reference's own render_depth / render_normal /
    render_shaded (render.py:144-184, host loop, backend protocol calls) run
    on CudaNeuralField unchanged and equal the one-call device modes (depth
    and normal bit for bit, shading to the last ulp of numpy's light dot)."""
    _, f, _ = pair
    _, _, render = reference
    cam = render.Camera(position=(0.3, 0.5, 3.0), look_at=(0.0, 0.1, 0.0), vfov=np.pi / 4, width=41, height=27)
    for mode in ("depth", "normal", "shaded"):
        cfg = render.RenderConfig(mode=mode, background=(0.1, 0.2, 0.3), light_dir=np.array([0.3, -2.0, 1.1]),
                                  albedo=0.6)
        host = render.render(f, cam, cfg).data                # the reference's loop over the protocol
        dev = R.render(f, cam, cfg).data                      # ddf_render_mode (the reference's Camera as-is)
        assert host.shape == dev.shape
        if mode == "shaded":
            np.testing.assert_allclose(dev, host, rtol=0, atol=1e-15)
        else:
            assert np.array_equal(dev, host)


def test_reference_render_path_runs_on_the_shim(pair, reference):
    """render.render_path (render.py:198-247) of the unmodified reference on
    CudaNeuralField (host loop: numpy camera rays, _hit_normals, _cosine_dirs,
    one trace_batch / normal_batch call per stage) against the one-call device
    wavefront.  Both draw the same PCG64 stream; they can differ only where
    CUDA's f64 sin/cos/acos (1-2 ulp from libm) move a bounce direction."""
    _, f, _ = pair
    _, _, render = reference
    cam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=32, height=24)
    cfg = render.RenderConfig(mode="path", spp=3, bounces=3, albedo=0.7, env_radiance=1.0, seed=42)
    host = render.render(f, cam, cfg).data[:, :, 0]
    dev = R.render(f, cam, cfg).data[:, :, 0]
    d = np.abs(host - dev)
    print(f"reference loop on the shim vs device wavefront: RMSE {np.sqrt(np.mean(d ** 2)):.3g}, "
          f"pixels differing {np.mean(d > 1e-12):.2%}")
    assert np.sqrt(np.mean(d ** 2)) <= 1e-3 and np.mean(d > 1e-12) <= 0.02


def test_reference_image_writers_take_device_framebuffers(pair, reference, tmp_path):
    """write_pfm / write_ppm and the bench harness stay the reference's
    (render.py:266-303); they consume the device renders unchanged."""
    _, f, _ = pair
    _, _, render = reference
    cam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=8, height=6)
    render.write_pfm(R.render(f, cam, render.RenderConfig(mode="depth")), tmp_path / "d.pfm")
    render.write_ppm(R.render(f, cam, render.RenderConfig(mode="path", spp=1, bounces=1)), tmp_path / "p.ppm")
    assert (tmp_path / "d.pfm").read_bytes().startswith(b"Pf\n8 6\n-1.0\n")
    assert len((tmp_path / "p.ppm").read_bytes()) == len(b"P6\n8 6\n255\n") + 8 * 6 * 3
    with pytest.raises(ValueError):
        R.render(f, cam, R.RenderConfig(mode="bogus"))


def test_sign_rule_raises_numeric_error(reference):
    """render.py:137-139: a normal exactly perpendicular to its ray violates
    n . d < 0.  A linear net pred = z + 0.5 has gradient (0, 0, 1); a camera
    on the x axis with z up and an odd film height sends its centre row with
    d_z = 0 exactly.  The device modes raise NumericError from the device
    error word; the reference's own loop on the shim raises its own class."""
    from paper_2306_16142_b200.errors import NumericError
    from paper_2306_16142_b200.neural import MlpModel
    v = np.array([[0.0, 0.0, 1.0, 0.0, 0.0]])
    m = MlpModel((5, 1), [v], [np.array([1.0])], [np.array([0.5])])
    f = CudaNeuralField(m, D, bounds=BOX)
    cam = R.Camera(position=(3.0, 0.0, 0.0), look_at=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0), vfov=np.pi / 4,
                   width=9, height=7)
    for mode in ("normal", "shaded"):
        with pytest.raises(NumericError, match="sign rule"):
            R.render(f, cam, R.RenderConfig(mode=mode))
    assert np.all(np.isfinite(R.render(f, cam, R.RenderConfig(mode="depth")).data))
    _, _, render = reference
    rcam = render.Camera(position=(3.0, 0.0, 0.0), look_at=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0), vfov=np.pi / 4,
                         width=9, height=7)
    from ddfield.errors import NumericError as RefNumericError
    with pytest.raises(RefNumericError):
        render.render(f, rcam, render.RenderConfig(mode="normal"))


@pytest.mark.parametrize("mode", ["depth", "normal", "shaded", "ambient"])
def test_single_bounce_render_modes(pair, mode):
    """render.py:144-184 on the GPU backend vs the oracle restatement."""
    _, f, of = pair
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=40, height=30)
    oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=40, height=30)
    cfg = R.RenderConfig(mode="shaded" if mode == "ambient" else mode, ambient=mode == "ambient")
    img = R.render(f, cam, cfg).data
    ref = O.render_mode(of, oc, "shaded" if mode == "ambient" else mode, ambient=mode == "ambient")
    fin = np.isfinite(ref)
    assert np.array_equal(fin, np.isfinite(img))
    assert np.max(np.abs(img[fin] - ref[fin])) <= 1e-3


def test_config4_network_path_parity_fp32():
    """Config 3/4's 65->8x512->1 network with PE, fp32 engine vs the oracle
    with identical streams.  The first two bounces are bit-identical; from
    bounce 3 single paths decorrelate chaotically (the 2^5 pi PE features turn
    ~1e-5 degree fp32-vs-f64 normal differences into different hits), so deep
    renders (8 bounces, Russian roulette from 3) agree in distribution:
    image mean within 1 %, most pixels identical."""
    from paper_2306_16142_b200 import configs as C
    m = C.models("c4")[0]
    f = CudaNeuralField(m, D, bounds=BOX, precision="fp32")
    of = O.Field([O.Net(m.widths, m.v, m.g, m.b)], D, bounds=BOX)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=24, height=14)
    oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=24, height=14)
    img = R.render_path(f, cam, R.RenderConfig(spp=2, bounces=2, seed=42)).data[:, :, 0].reshape(-1)
    ref = O.render_path(of, oc, O.PathConfig(spp=2, bounces=2, albedo=0.7, env=1.0, seed=42))
    assert np.sqrt(np.mean((img - ref) ** 2)) <= 3e-3
    img = R.render_path(f, cam, R.RenderConfig(spp=4, bounces=8, seed=42, rr_start=3)).data[:, :, 0].reshape(-1)
    ref = O.render_path(of, oc, O.PathConfig(spp=4, bounces=8, albedo=0.7, env=1.0, seed=42, rr_start=3))
    d = np.abs(img - ref)
    print(f"config-4 net, 8 bounces + RR: mean {img.mean():.4f} vs {ref.mean():.4f}, "
          f"pixels differing {np.mean(d > 1e-6):.1%}, RMSE {np.sqrt(np.mean(d ** 2)):.3g}")
    assert abs(img.mean() - ref.mean()) <= 0.01 * ref.mean()
    assert np.mean(d > 1e-6) <= 0.25


def test_device_render_modes_scene_vs_oracle():
    """Composite scene (config 5 layout): the device modes use the hit
    object's gradient, as the oracle (and the reference subclass of
    tests/golden/make_golden.py) does."""
    from paper_2306_16142_b200 import configs as C
    centers, scale, albedos = C.scene_layout()
    ms = [kaiming_uniform((5, 32, 32, 1), s) for s in range(10, 18)]
    f = CudaNeuralField.scene(ms, centers, scale, albedos, D, bounds=C.SCENE_BOX)
    of = O.Field([O.Net(m.widths, m.v, m.g, m.b) for m in ms], D, bounds=C.SCENE_BOX, centers=centers,
                 scale=scale, albedos=albedos)
    cam = R.Camera(position=(0.3, 0.5, 3.0), look_at=(0.0, 0.1, 0.0), vfov=np.pi / 4, width=41, height=27)
    oc = O.Cam((0.3, 0.5, 3.0), (0.0, 0.1, 0.0), vfov=np.pi / 4, width=41, height=27)
    for mode in ("depth", "normal", "shaded"):
        img = R.render(f, cam, R.RenderConfig(mode=mode)).data
        ref = O.render_mode(of, oc, mode)
        fin = np.isfinite(ref)
        assert np.array_equal(fin, np.isfinite(img))
        assert np.max(np.abs(img[fin] - ref[fin])) <= 1e-3


def test_device_render_mode_degenerate_normals():
    """render.py:133-136 on the device path: a zero-gradient network (W = 0,
    constant distance) hits every in-box pixel and every normal falls back to
    -d, so the normal image is 0.5 * (1 - d)."""
    m = kaiming_uniform((5, 16, 1), 0)
    m.g[0] = np.zeros_like(m.g[0])          # W = 0: constant output, zero gradient
    m.b[1] = np.array([0.5])
    f = CudaNeuralField(m, D, bounds=BOX)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=9, height=7)
    img = R.render(f, cam, R.RenderConfig(mode="normal")).data.reshape(-1, 3)
    _, d = O.camera_rays(O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=9, height=7),
                         np.full((63, 2), 0.5), np.arange(63))
    o = np.broadcast_to(cam.position, d.shape)
    t, hit = f.trace_batch(o, d)
    assert hit.all()
    assert np.array_equal(img, 0.5 * (-d + 1.0))


def test_graph_replay_identical_and_invalidated():
    """cfg.graph: the second call with the same camera / config
    replays the captured waves.  Replays equal eager renders; a precision
    change (field generation) or a scratch reallocation by another call
    (buffer epoch) forces a fresh capture instead of a stale replay."""
    import torch
    f = CudaNeuralField(kaiming_uniform((5, 64, 64, 1), 9), D, bounds=BOX)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=48, height=32)
    acc = torch.empty(48 * 32, dtype=torch.float64, device="cuda")
    cfg = R.RenderConfig(spp=3, bounces=3, seed=4, rr_start=1, graph=1)
    eager = R.render_path_device(f, cam, R.RenderConfig(spp=3, bounces=3, seed=4, rr_start=1, graph=0))[0].clone()
    for _ in range(3):                                   # capture, then replays
        assert torch.equal(R.render_path_device(f, cam, cfg, accum=acc)[0], eager)
    f.set_precision("bf16")                              # new generation
    bf = R.render_path_device(f, cam, R.RenderConfig(spp=3, bounces=3, seed=4, rr_start=1, graph=0))[0].clone()
    assert not torch.equal(bf, eager)
    assert torch.equal(R.render_path_device(f, cam, cfg, accum=acc)[0], bf)
    big = np.random.default_rng(0).uniform(-1, 1, (300_000, 3))
    dirs = big / np.linalg.norm(big, axis=1, keepdims=True)
    f.trace_batch(big * 2.5, dirs)                       # grows (reallocates) the shared scratch
    assert torch.equal(R.render_path_device(f, cam, cfg, accum=acc)[0], bf)
    assert torch.equal(R.render_path_device(f, cam, cfg, accum=acc)[0], bf)
    # the graph renders into the field's own film: a new accumulator per call
    # (what the public render_path does) replays the same graph
    launches = R.render_path_device(f, cam, cfg)[1]["kernel_launches"]
    for _ in range(2):
        other = torch.full((48 * 32,), 7.0, dtype=torch.float64, device="cuda")
        got, st = R.render_path_device(f, cam, cfg, accum=other)
        assert torch.equal(got, bf) and st["kernel_launches"] == launches and st["graph_replayed"] == 1
    assert np.array_equal(R.render_path(f, cam, cfg).data[:, :, 0].reshape(-1), bf.cpu().numpy() / 3)
