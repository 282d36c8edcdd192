"""The reference's SPEC known-answer cases for the hot path (SURVEY §4 and
§8(c): SPEC.md:182-190 normals, :342-350 forward, :369-377 input gradient,
:417 kink filter, :447-455 camera, :483-506 path tracer, weight-norm
invariance), on the CPU oracle and, marked gpu, on the CUDA path through the
C ABI.

The furnace scene: one hidden layer whose prediction is exactly
pred = -K*u4 + z - 0.5 on the box [-1, 1]^3 (u4 = 2*polar/pi - 1 > 0 for
downward rays).  A camera at (0, 0, 3) looking down sees only the top face:
every primary ray clamps to -delta at box entry and hits there (t = t_enter),
the normal is +z, the bounce origin lies 1e-6 above the box, so every
cosine-sampled bounce ray leaves the bounds and escapes.  Each path sample is
then albedo * env exactly -- the SPEC's "furnace limit within 2% at spp=4096"
(render.py:215-243) becomes an exact identity at any spp."""

import numpy as np
import pytest

from oracle import cpu_ddf as O
from paper_2306_16142_b200 import render as R
from paper_2306_16142_b200.neural import MlpModel

K_STEEP = 1.0e4
BOX = np.array([[-1.0] * 3, [1.0] * 3])


def furnace_net(hidden=16):
    """pred = -K*u4 + z - 0.5: both hidden units stay in ReLU's linear range
    for every encoded input in [-1.1, 1.1]^3 x [-1, 1]^2."""
    v1 = np.zeros((hidden, 5))
    v1[:, 0] = 1.0
    g1 = np.zeros(hidden)
    b1 = np.zeros(hidden)
    v1[0] = [0, 0, 0, 0, -1.0]
    g1[0], b1[0] = K_STEEP, K_STEEP + 1.0          # h0 = -K*u4 + K + 1 >= 1
    v1[1] = [0, 0, 1.0, 0, 0]
    g1[1], b1[1] = 1.0, 2.0                          # h1 = z + 2 >= 0.9
    v2 = np.zeros((1, hidden))
    v2[0, :2] = 1.0
    g2 = np.array([np.sqrt(2.0)])
    b2 = np.array([-(K_STEEP + 3.0) - 0.5])
    return (5, hidden, 1), [v1, v2], [g1, g2], [b1, b2]


def zero_net(widths=(5, 32, 32, 1), head_bias=0.37):
    """g = 0 everywhere: W_eff = 0, the output is the head bias."""
    rng = np.random.default_rng(7)
    vs = [rng.normal(size=(widths[i + 1], widths[i])) for i in range(len(widths) - 1)]
    gs = [np.zeros(widths[i + 1]) for i in range(len(widths) - 1)]
    bs = [rng.normal(size=widths[i + 1]) for i in range(len(widths) - 1)]
    bs[-1] = np.array([head_bias])
    return widths, vs, gs, bs


def linear_net():
    rng = np.random.default_rng(8)
    v = rng.normal(size=(1, 5))
    return (5, 1), [v], [np.array([1.7])], [np.array([0.25])]


def as_oracle(spec):
    return O.Net(*spec)


def as_model(spec):
    return MlpModel(*spec)


def smooth_points(net, n, margin=1e-3, seed=0):
    """probe points whose every pre-activation is >= margin from 0."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.9, 0.9, (4 * n, 5))
    keep = np.ones(len(x), bool)
    h = x
    ws = net.effective()
    for w, b in zip(ws[:-1], net.b[:-1]):
        z = h @ w.T + b
        keep &= np.all(np.abs(z) >= margin, axis=1)
        h = np.maximum(z, 0.0)
    return x[keep][:n]


def fd_grad(f, x, h):
    g = np.empty_like(x)
    for j in range(x.shape[1]):
        e = np.zeros(x.shape[1])
        e[j] = h
        g[:, j] = (f(x + e) - f(x - e)) / (2 * h)
    return g


def furnace_camera(size=33):
    return (O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=size, height=size),
            R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=size, height=size))


# --------------------------------------------------------------------- oracle

def test_zero_weight_model_is_bias_only_with_zero_gradient():
    net = as_oracle(zero_net())
    x = np.random.default_rng(1).uniform(-1, 1, (64, 5))
    assert np.all(O.mlp_forward(net, x) == 0.37)
    assert np.all(O.mlp_input_grad(net, x) == 0.0)


def test_forward_matches_straight_line_matmul():
    net = O.kaiming_uniform_net((5, 48, 1), 3)
    x = np.random.default_rng(2).uniform(-1, 1, (128, 5))
    w1, w2 = net.effective()
    ref = np.array([sum(w2[0, j] * max(0.0, sum(w1[j, i] * r[i] for i in range(5)) + net.b[0][j])
                        for j in range(48)) + net.b[1][0] for r in x])
    np.testing.assert_allclose(O.mlp_forward(net, x), ref, rtol=0, atol=1e-12)


def test_linear_model_gradient_is_w_row():
    net = as_oracle(linear_net())
    x = np.random.default_rng(3).uniform(-1, 1, (32, 5))
    w = net.effective()[0][0]
    assert np.all(O.mlp_input_grad(net, x) == w)


def test_input_gradient_matches_central_differences():
    net = O.kaiming_uniform_net((5, 64, 64, 1), 4)
    x = smooth_points(net, 64)
    assert len(x) >= 32
    fd = fd_grad(lambda y: O.mlp_forward(net, y), x, 1e-5)
    g = O.mlp_input_grad(net, x)
    assert np.max(np.abs(g - fd) / np.maximum(np.abs(fd), 1e-3)) < 1e-5


def _normal_fd_check(normals, valid, o, d, t, net):
    """κ rule (n·d < 0) and the normal vs central differences (h = 1e-4) of
    the same network at the back-off point."""
    assert np.all(np.einsum("ij,ij->i", normals[valid], d[valid]) < 0)
    back = np.maximum(t - 0.5 * 1.0, 0.0)
    p = o + back[:, None] * d
    ang = O.dirs_to_angles(d)
    pred = lambda q: O.mlp_forward(net, O.encode5(q, ang))
    g = fd_grad(pred, p, 1e-4)
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    g = np.where((np.einsum("ij,ij->i", g, d) > 0)[:, None], -g, g)
    cosang = np.clip(np.einsum("ij,ij->i", g[valid], normals[valid]), -1, 1)
    return np.degrees(np.arccos(cosang))


def _normal_probe(net, n=200, seed=5):
    """Random rays inside the box whose hidden pre-activations at the origin
    stay >= 1e-3 from the ReLU kink."""
    rng = np.random.default_rng(seed)
    o = rng.uniform(-0.8, 0.8, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    z = O.encode5(o, O.dirs_to_angles(d)) @ net.effective()[0].T + net.b[0]
    keep = np.all(np.abs(z) >= 1e-3, axis=1)
    return o[keep], d[keep]


def film_value(x, spp):
    """The film entry when every sample is x: f64 sum in spp order, / spp."""
    acc = 0.0
    for _ in range(spp):
        acc += x
    return acc / spp


def test_oracle_normals_kappa_rule_and_finite_differences():
    net = O.kaiming_uniform_net((5, 64, 1), 6)
    fld = O.Field([net], 1.0, bounds=BOX)
    o, d = _normal_probe(net)
    t = np.zeros(len(o))              # back = 0: the gradient is taken at o
    nrm, valid = fld.normal(o, d, t_hit=t)
    err = _normal_fd_check(nrm, valid, o, d, t, net)
    assert valid.mean() > 0.99 and np.max(err) < 0.5


def test_camera_centre_on_axis_corners_mirrored():
    for cam in (O.Cam((0.3, -0.2, 3.0), (0.1, 0.2, -0.4), vfov=np.pi / 4, width=33, height=21),):
        o, d = O.camera_rays(cam, np.full((33 * 21, 2), 0.5), np.arange(33 * 21))
        c = (cam.height // 2) * cam.width + cam.width // 2
        assert np.max(np.abs(d[c] - cam.forward)) < 1e-9
        W, H = cam.width, cam.height
        tl, tr, bl, br = d[0], d[W - 1], d[(H - 1) * W], d[H * W - 1]
        f = cam.forward
        for a, b in ((tl, br), (tr, bl)):
            # mirror about the view axis: a + b is parallel to the axis
            s = a + b
            assert np.linalg.norm(s - (s @ f) * f) < 1e-9
        rt = O.angles_to_dirs(O.dirs_to_angles(d))
        assert np.max(np.abs(rt - d)) < 1e-9


def test_oracle_furnace_is_exact():
    fld = O.Field([as_oracle(furnace_net())], 1.0, bounds=BOX)
    ocam, _ = furnace_camera(9)
    for bounces in (1, 3):
        v = O.render_path(fld, ocam, O.PathConfig(spp=4, bounces=bounces, albedo=0.7, env=1.3, seed=3))
        assert np.all(v == film_value(0.7 * 1.3, 4))
    amb = O.render_mode(fld, ocam, "shaded", background=(1.3,) * 3, albedo=0.7, env=1.3, ambient=True)
    assert np.all(amb == 0.7 * 1.3)
    v = O.render_path(fld, ocam, O.PathConfig(spp=2, bounces=2, albedo=0.0, env=1.0, seed=3))
    assert np.all(v == 0.0)


# ----------------------------------------------------------------------- GPU

@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2306_16142_b200.field import CudaNeuralField
    return CudaNeuralField


PRECS = ["fp32", "bf16"]


@pytest.mark.gpu
@pytest.mark.parametrize("prec", PRECS)
def test_gpu_zero_weight_model(cuda, prec):
    f = cuda(as_model(zero_net()), 1.0, bounds=BOX, precision=prec)
    x = np.random.default_rng(1).uniform(-1, 1, (300, 5))
    y = f.forward_inputs(x)
    assert np.all(y == np.float32(0.37))
    assert np.all(f.input_gradient_inputs(x) == 0.0)
    assert np.array_equal(f.forward_inputs(x), y)          # eval mode is deterministic


@pytest.mark.gpu
@pytest.mark.parametrize("prec", PRECS)
def test_gpu_linear_model_gradient_is_w_row(cuda, prec):
    spec = linear_net()
    f = cuda(as_model(spec), 1.0, bounds=BOX, precision=prec)
    w = as_oracle(spec).effective()[0][0]
    x = np.random.default_rng(3).uniform(-1, 1, (257, 5))
    g = f.input_gradient_inputs(x)
    # no hidden layer -> no GEMM: both precisions run the fp32 SIMT kernel
    assert np.all(g == w.astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(f.forward_inputs(x), O.mlp_forward(as_oracle(spec), x), rtol=0, atol=1e-5)


@pytest.mark.gpu
def test_gpu_forward_and_gradient_vs_matmul_and_fd(cuda):
    net = O.kaiming_uniform_net((5, 48, 1), 3)
    f = cuda(as_model((net.widths, net.v, net.g, net.b)), 1.0, bounds=BOX)
    x = smooth_points(net, 200, seed=9)
    np.testing.assert_allclose(f.forward_inputs(x), O.mlp_forward(net, x), rtol=0, atol=2e-6)
    fd = fd_grad(lambda y: O.mlp_forward(net, y), x, 1e-5)
    g = f.input_gradient_inputs(x)
    assert np.max(np.abs(g - fd) / np.maximum(np.abs(fd), 1e-2)) < 1e-4


@pytest.mark.gpu
def test_gpu_weight_norm_scale_invariance(cuda):
    net = O.kaiming_uniform_net((5, 64, 64, 1), 11)
    scaled = [v * c for v, c in zip(net.v, (3.0, 0.25, 7.5))]
    f1 = cuda(as_model((net.widths, net.v, net.g, net.b)), 1.0, bounds=BOX)
    f2 = cuda(as_model((net.widths, scaled, net.g, net.b)), 1.0, bounds=BOX)
    x = np.random.default_rng(4).uniform(-1, 1, (500, 5))
    a, b = f1.forward_inputs(x), f2.forward_inputs(x)
    assert np.max(np.abs(a - b)) <= 1e-6 * max(1.0, np.max(np.abs(a)))


@pytest.mark.gpu
def test_gpu_normals_kappa_rule_and_finite_differences(cuda):
    net = O.kaiming_uniform_net((5, 64, 1), 6)
    f = cuda(as_model((net.widths, net.v, net.g, net.b)), 1.0, bounds=BOX)
    o, d = _normal_probe(net)
    t = np.zeros(len(o))
    nrm, valid = f.normal_batch(o, d, t_hit=t)
    err = _normal_fd_check(nrm, valid, o, d, t, net)
    assert valid.mean() > 0.99 and np.max(err) < 0.5


@pytest.mark.gpu
@pytest.mark.parametrize("prec", PRECS)
def test_gpu_furnace_ambient_and_absorbing(cuda, prec):
    f = cuda(as_model(furnace_net()), 1.0, bounds=BOX, precision=prec)
    _, cam = furnace_camera(33)
    for bounces in (1, 4):
        fb = R.render_path(f, cam, R.RenderConfig(spp=16, bounces=bounces, albedo=0.7, env_radiance=1.3, seed=3))
        assert np.all(fb.data == film_value(0.7 * 1.3, 16))
    # N_b = 1 == ambient-shaded render (background = env)
    amb = R.render_shaded(f, cam, R.RenderConfig(mode="shaded", ambient=True, albedo=0.7, env_radiance=1.3,
                                                   background=(1.3, 1.3, 1.3)))
    fb = R.render_path(f, cam, R.RenderConfig(spp=8, bounces=1, albedo=0.7, env_radiance=1.3, seed=4))
    assert np.all(amb.data == 0.7 * 1.3) and np.all(fb.data == film_value(0.7 * 1.3, 8))
    np.testing.assert_allclose(amb.data, fb.data, rtol=1e-15)
    # depth: every pixel hits the top face at t_enter = (3 - 1) / |d_z|
    oc = O.Cam(cam.position, cam.look_at, vfov=cam.vfov, width=cam.width, height=cam.height)
    o, d = O.camera_rays(oc, np.full((cam.width * cam.height, 2), 0.5), np.arange(cam.width * cam.height))
    depth = R.render_depth(f, cam).data.reshape(-1)
    np.testing.assert_allclose(depth, 2.0 / np.abs(d[:, 2]), rtol=1e-12)
    # zero-emission / all-absorbing -> black
    fb = R.render_path(f, cam, R.RenderConfig(spp=4, bounces=3, albedo=0.0, env_radiance=1.0, seed=5))
    assert np.all(fb.data == 0.0)


@pytest.mark.gpu
def test_gpu_furnace_with_russian_roulette_is_unbiased(cuda):
    """RR (p = min(1, throughput)) keeps the furnace mean: each surviving
    sample is env*albedo/p, so the film mean stays albedo*env within 3 sigma."""
    f = cuda(as_model(furnace_net()), 1.0, bounds=BOX, precision="bf16")
    _, cam = furnace_camera(64)
    cfg = R.RenderConfig(spp=64, bounces=3, albedo=0.6, env_radiance=1.0, seed=9, rr_start=0)
    v = R.render_path(f, cam, cfg).data[..., 0].reshape(-1)
    n = v.size * cfg.spp
    sigma = np.sqrt(0.6 * 0.4 / n)       # per-sample value is Bernoulli(0.6) * 1.0
    assert abs(v.mean() - 0.6) < 3 * sigma


@pytest.mark.gpu
@pytest.mark.parametrize("prec", PRECS)
def test_gpu_energy_bound_and_determinism(cuda, prec):
    from paper_2306_16142_b200.neural import kaiming_uniform
    f = cuda(kaiming_uniform((5, 64, 64, 1), 12), 10.0 / 0.98, bounds=BOX, precision=prec)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=48, height=40)
    cfg = R.RenderConfig(spp=8, bounces=4, albedo=0.9, env_radiance=2.0, seed=21)
    a = R.render_path(f, cam, cfg).data
    assert np.all(a <= 2.0) and np.all(a >= 0.0)          # every sample <= env (no RR)
    assert np.array_equal(a, R.render_path(f, cam, cfg).data)
    cfg.seed = 22
    assert not np.array_equal(a, R.render_path(f, cam, cfg).data)


@pytest.mark.gpu
def test_gpu_all_miss_depth_is_uniform_background(cuda):
    from paper_2306_16142_b200.neural import kaiming_uniform
    f = cuda(kaiming_uniform((5, 32, 1), 1), 10.0 / 0.98, bounds=BOX)
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 6.0), vfov=np.pi / 4, width=16, height=12)
    assert np.all(np.isinf(R.render_depth(f, cam).data))
    fb = R.render_path(f, cam, R.RenderConfig(spp=2, bounces=2, env_radiance=0.8, seed=1))
    assert np.all(fb.data == 0.8)
