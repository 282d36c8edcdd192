"""Pin the CPU oracle (oracle/cpu_ddf.py) before trusting it.

Every fixture in tests/golden/reference_golden.npz was produced by the
unmodified reference (tests/golden/make_golden.py).  The oracle must
reproduce each one bit-for-bit (same float64 operation order); the live
reference is re-checked where it is importable.
"""

import os
import tempfile

import numpy as np
import pytest

from oracle import cpu_ddf as O

CFG_DELTA = 10.0 / 0.98
BOX = np.array([[-1.0] * 3, [1.0] * 3])


def march_net():
    net = O.kaiming_uniform_net((5, 64, 64, 1), seed=7)
    net.g[-1] = net.g[-1] * 0.05
    net.b[-1] = net.b[-1] + 0.12
    return net


@pytest.fixture(scope="module")
def cfg1_field():
    return O.Field([O.kaiming_uniform_net((5, 128, 128, 128, 128, 1), 0)], CFG_DELTA, bounds=BOX)


def test_encoding_matches(golden):
    x = O.encode5(golden["q_origins"], O.dirs_to_angles(golden["q_dirs"]))
    assert np.array_equal(x, golden["q_inputs"])


def test_forward_and_gradient_bit_exact(golden, cfg1_field):
    net = cfg1_field.nets[0]
    x = golden["q_inputs"]
    assert np.array_equal(O.mlp_forward(net, x), golden["q_forward"])
    assert np.array_equal(O.mlp_input_grad(net, x), golden["q_grad"])


def test_query_trace_normal(golden, cfg1_field):
    t, h = cfg1_field.query(golden["q_origins"], golden["q_dirs"])
    assert np.array_equal(t, golden["q_query_t"]) and np.array_equal(h, golden["q_query_hit"])
    t, h, _ = cfg1_field.trace(golden["q_trace_origins"], golden["q_dirs"])
    assert np.array_equal(t, golden["q_trace_t"]) and np.array_equal(h, golden["q_trace_hit"])
    th = np.where(np.isfinite(t), t, 0.0)
    n, v = cfg1_field.normal(golden["q_trace_origins"], golden["q_dirs"], th)
    assert np.array_equal(n, golden["q_normal"]) and np.array_equal(v, golden["q_normal_valid"])
    n0, _ = cfg1_field.normal(golden["q_origins"], golden["q_dirs"])
    assert np.array_equal(n0, golden["q_normal_noback"])


def test_multistep_march(golden):
    f = O.Field([march_net()], 0.1, bounds=BOX)
    log = []
    t, h, _ = f.trace(golden["m_origins"], golden["m_dirs"], log)
    assert np.array_equal(t, golden["m_trace_t"]) and np.array_equal(h, golden["m_trace_hit"])
    assert len(log) > 10  # really marches several steps
    for a, b in zip(log, log[1:]):
        assert set(b) <= set(a) and np.all(np.diff(a) > 0)
    t, h = f.query(golden["m_origins"] * 0.5, golden["m_dirs"])
    assert np.array_equal(t, golden["m_query_t"]) and np.array_equal(h, golden["m_query_hit"])


def test_camera_and_cosine(golden):
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=24, height=16)
    o, d = O.camera_rays(cam, golden["cam_jitter"], np.arange(24 * 16))
    assert np.array_equal(d, golden["cam_dirs"]) and np.array_equal(o, golden["cam_origins"])
    assert np.array_equal(O.cosine_dirs(golden["cos_normals"], golden["cos_u"]), golden["cos_dirs"])


def test_pcg64_counter_formula(golden):
    s = O.pcg_seed_state(42)
    ref = golden["rng_first"]
    assert np.array_equal(O.stream_block(42, O.RNG_TAG, 0, 64), ref)
    for k in (0, 1, 7, 33, 63):
        assert O.pcg_double(s, k) == ref[k]
    # jump-ahead == numpy's advance far into the stream
    k = 3 * 2 * 16384 * 5 + 12345
    assert O.pcg_double(s, k) == O.stream_block(42, O.RNG_TAG, k, 1)[0]


def test_render_config2_bit_exact(golden):
    """Config 2 at its full size (128x128, 4 spp, 2 bounces) vs the reference."""
    f = O.Field([O.kaiming_uniform_net((5,) + (256,) * 8 + (1,), 1)], CFG_DELTA, bounds=BOX)
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=128, height=128)
    img = O.render_path(f, cam, O.PathConfig(spp=4, bounces=2, albedo=0.7, env=1.0, seed=42))
    assert np.array_equal(img.reshape(128, 128), golden["r2_film"])
    part = O.render_path(f, cam, O.PathConfig(spp=4, bounces=2, albedo=0.7, env=1.0, seed=42),
                         pix_range=(7000, 7300))
    assert np.array_equal(part, img[7000:7300])


def test_render_march_regime(golden):
    f = O.Field([march_net()], 0.1, bounds=BOX)
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=20, height=12)
    img = O.render_path(f, cam, O.PathConfig(spp=3, bounces=3, albedo=0.6, env=1.5, seed=9))
    assert np.array_equal(img.reshape(12, 20), golden["rm_film"])


def test_ddfn_roundtrip_and_errors(golden):
    blob = golden["ddfn_bytes"].tobytes()
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "m.ddfn")
        with open(p, "wb") as fh:
            fh.write(blob)
        net, delta = O.read_ddfn(p)
        ref = march_net()
        assert delta == 0.1 and net.widths == ref.widths
        for a, b in zip(net.v + net.g + net.b, ref.v + ref.g + ref.b):
            assert np.array_equal(a, b)
        q = os.path.join(td, "w.ddfn")
        O.write_ddfn(net, delta, q)
        assert open(q, "rb").read() == blob
        for bad in (b"XXXX" + blob[4:], blob[:30], blob + b"\0"):
            with open(q, "wb") as fh:
                fh.write(bad)
            with pytest.raises(O.OracleDataError):
                O.read_ddfn(q)


def test_pe_gradient_matches_finite_difference():
    """EXTENSION pin: the 65-D encoding's chain rule vs central differences."""
    net = O.kaiming_uniform_net((65, 32, 32, 1), seed=3)
    rng = np.random.default_rng(0)
    u = rng.uniform(-0.9, 0.9, (64, 5))
    g = O.pe_chain(u, O.mlp_input_grad(net, O.pe_encode(u)))
    h = 1e-6
    for j in range(5):
        e = np.zeros(5)
        e[j] = h
        fd = (O.mlp_forward(net, O.pe_encode(u + e)) - O.mlp_forward(net, O.pe_encode(u - e))) / (2 * h)
        ok = np.abs(fd - g[:, j]) <= 1e-4 * (1 + np.abs(fd))
        assert ok.mean() > 0.95  # ReLU kinks may break a few rows


def test_oracle_matches_live_reference(reference):
    neural, field, render = reference
    net = O.kaiming_uniform_net((65, 48, 48, 1), seed=4)
    m = neural.MlpModel(widths=net.widths, v=net.v, g=net.g, b=net.b)
    x = np.random.default_rng(1).normal(size=(300, 65))
    assert np.array_equal(neural.forward_batch(m, x), O.mlp_forward(net, x))
    f = field.NeuralField(m, 2.0)  # default bounds
    assert np.array_equal(f.bounds, O.Field([net], 2.0).bounds)


# ------------------------------------------------------------------ extensions
# tests/golden/reference_golden_ext.npz comes from the reference with App. A's
# subclasses layered on it (make_golden.py: EncodedNeuralField,
# SceneNeuralField, render_path_ext): the reference still marches, takes
# normals, samples bounces and builds camera rays.

@pytest.fixture(scope="module")
def ext():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_ext.npz"))


def pe_field():
    return O.Field([O.kaiming_uniform_net((65, 128, 128, 1), 6)], CFG_DELTA, bounds=BOX)


def scene_field():
    import itertools
    centers = np.array(list(itertools.product((-0.75, 0.75), repeat=3)), dtype=np.float64)
    albedos = np.random.default_rng(5).uniform(0.2, 0.9, 8)
    nets = [O.kaiming_uniform_net((65, 32, 32, 1), s) for s in range(10, 18)]
    return O.Field(nets, CFG_DELTA, bounds=np.array([[-1.25] * 3, [1.25] * 3]), centers=centers, scale=0.5,
                   albedos=albedos)


def test_pe_field_matches_encoded_reference(ext):
    f = pe_field()
    o, d = ext["pe_o"], ext["pe_d"]
    ang = O.dirs_to_angles(d)
    net = f.nets[0]
    assert np.array_equal(O.mlp_forward(net, O.pe_encode(O.encode5(o, ang))), ext["pe_forward"])
    assert np.array_equal(O.net_grad5(net, o, ang), ext["pe_grad5"])
    t, h = f.query(o, d)
    assert np.array_equal(t, ext["pe_query_t"]) and np.array_equal(h, ext["pe_query_hit"])
    t, h, _ = f.trace(o * 2.5, d)
    assert np.array_equal(t, ext["pe_trace_t"]) and np.array_equal(h, ext["pe_trace_hit"])
    n, v = f.normal(o * 2.5, d, np.where(np.isfinite(t), t, 0.0))
    assert np.array_equal(n, ext["pe_normal"]) and np.array_equal(v, ext["pe_normal_valid"])


def test_pe_and_rr_renders_match_reference_loop(ext):
    f = pe_field()
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=24, height=16)
    v = O.render_path(f, cam, O.PathConfig(spp=2, bounces=2, albedo=0.7, env=1.0, seed=42))
    assert np.array_equal(v.reshape(16, 24), ext["pe_film"])
    v = O.render_path(f, cam, O.PathConfig(spp=3, bounces=6, albedo=0.7, env=1.0, seed=8, rr_start=1))
    assert np.array_equal(v.reshape(16, 24), ext["pe_rr_film"])


def test_scene_matches_reference_subclass(ext):
    f = scene_field()
    t, h, obj = f.trace(ext["sc_o"], ext["sc_d"])
    assert np.array_equal(t, ext["sc_trace_t"]) and np.array_equal(h, ext["sc_trace_hit"])
    assert np.array_equal(obj[h], ext["sc_trace_obj"][h])
    n, v = f.normal(ext["sc_o"][h], ext["sc_d"][h], t[h], obj[h])
    assert np.array_equal(n, ext["sc_normal"]) and np.array_equal(v, ext["sc_normal_valid"])
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=20, height=14)
    for rr, key in ((-1, "sc_film"), (2, "sc_rr_film")):
        v = O.render_path(f, cam, O.PathConfig(spp=2, bounces=4, albedo=0.7, env=1.0, seed=42, rr_start=rr))
        assert np.array_equal(v.reshape(14, 20), ext[key])


def test_render_stage_lists_match_reference_lengths():
    """The oracle's per-stage lists have the lengths the unmodified
    reference's render loop produced (make_golden.main_stages logs them from
    a NeuralField subclass), stage by stage, for the config-2 render and the
    march regime; each list is ascending (np.nonzero order)."""
    st = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_stages.npz"))
    cases = [
        (O.Field([O.kaiming_uniform_net((5,) + (256,) * 8 + (1,), 1)], CFG_DELTA, bounds=BOX), 128, 128,
         O.PathConfig(spp=4, bounces=2, albedo=0.7, env=1.0, seed=42), "r2_stages", None),
        (O.Field([march_net()], 0.1, bounds=BOX), 20, 12,
         O.PathConfig(spp=3, bounces=3, albedo=0.6, env=1.5, seed=9), "rm_stages", None),
        (O.Field([march_net()], 0.1, bounds=BOX), 48, 32,
         O.PathConfig(spp=2, bounces=3, albedo=0.6, env=1.5, seed=9), "rmb_stages", "rmb_film"),
    ]
    for f, w, h, cfg, key, film in cases:
        log = []
        img = O.render_path(f, O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=w, height=h), cfg,
                            log=log)
        assert O.stage_sequence(log) == [tuple(r) for r in st[key].tolist()]
        for rec in log:
            for lst in rec["primary_march"] + rec["bounce_alive"] + [x for b in rec["bounce_march"] for x in b]:
                assert np.all(np.diff(lst) > 0)
        if film:
            assert np.array_equal(img.reshape(h, w), st[film])
