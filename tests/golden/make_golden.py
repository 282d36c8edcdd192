"""Generate golden fixtures by running the UNMODIFIED reference.

Run in the build container (the reference is importable there, not on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every array written here comes out of the reference's own public API
(``ddfield.neural``, ``ddfield.field.NeuralField``, ``ddfield.render``); the
synthetic inputs and the Kaiming-uniform weights are built by
``oracle.cpu_ddf.kaiming_uniform_net`` (seeded, deterministic) and handed to
the reference as an ``MlpModel``.  Fixtures are committed; tests regenerate
weights from (widths, seed) rather than storing them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import cpu_ddf as O  # noqa: E402

from ddfield import neural, field, render  # noqa: E402  (reference)

DELTA_CFG = 10.0 / 0.98
UNIT_BOX = np.array([[-1.0, -1.0, -1.0], [1.0, 1.0, 1.0]])


def ref_model(net: O.Net):
    return neural.MlpModel(widths=net.widths, v=[v.copy() for v in net.v],
                           g=[g.copy() for g in net.g], b=[b.copy() for b in net.b])


def rays(n, seed):
    """Config-1 synthetic rays: origins U[-1,1]^3, directions = normalised
    N(0, I3) draws, both from default_rng(seed) (origins drawn first)."""
    rng = np.random.default_rng(seed)
    o = rng.uniform(-1.0, 1.0, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


def march_net():
    """A net whose head is scaled so predictions straddle a small delta,
    exercising the multi-step sphere march (field.py:274-288)."""
    net = O.kaiming_uniform_net((5, 64, 64, 1), seed=7)
    net.g[-1] = net.g[-1] * 0.05
    net.b[-1] = net.b[-1] + 0.12
    return net


def main():
    out = {}
    # --- config-1 query batch: forward / gradient / protocol (small N) ---
    w1 = (5, 128, 128, 128, 128, 1)
    n1 = O.kaiming_uniform_net(w1, seed=0)
    m1 = ref_model(n1)
    o, d = rays(1024, seed=0)
    x = neural.encode_inputs(o, field.vecs_to_angles(d))
    out["q_origins"], out["q_dirs"] = o, d
    out["q_inputs"] = x
    out["q_forward"] = neural.forward_batch(m1, x)
    out["q_grad"] = neural.input_gradient_batch(m1, x)
    nf = field.NeuralField(m1, DELTA_CFG, bounds=UNIT_BOX)
    out["q_query_t"], out["q_query_hit"] = nf.query_batch(o, d)
    # trace from points outside the box towards it, plus random rays
    o2 = o * 2.5
    out["q_trace_t"], out["q_trace_hit"] = nf.trace_batch(o2, d)
    th = np.where(np.isfinite(out["q_trace_t"]), out["q_trace_t"], 0.0)
    out["q_normal"], out["q_normal_valid"] = nf.normal_batch(o2, d, t_hit=th)
    out["q_normal_noback"], _ = nf.normal_batch(o, d)
    out["q_trace_origins"] = o2

    # --- multi-step march regime (small delta) ---
    mn = march_net()
    mf = field.NeuralField(ref_model(mn), 0.1, bounds=UNIT_BOX)
    o3, d3 = rays(512, seed=3)
    o3 = o3 * 1.8
    out["m_origins"], out["m_dirs"] = o3, d3
    out["m_trace_t"], out["m_trace_hit"] = mf.trace_batch(o3, d3)
    out["m_query_t"], out["m_query_hit"] = mf.query_batch(o3 * 0.5, d3)

    # --- camera rays and cosine sampling ---
    cam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0),
                        vfov=np.pi / 4.0, width=24, height=16)
    jit = np.random.default_rng(5).random((24 * 16, 2))
    out["cam_jitter"] = jit
    out["cam_origins"], out["cam_dirs"] = render.pixel_rays(cam, offsets=jit)
    nrm = np.random.default_rng(6).normal(size=(257, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[0] = (0.0, 0.0, 1.0)
    nrm[1] = (1.0, 0.0, 0.0)
    uu = np.random.default_rng(8).random((257, 2))
    out["cos_normals"], out["cos_u"] = nrm, uu
    out["cos_dirs"] = render._cosine_dirs(nrm, uu)

    # --- RNG: the reference's stream ---
    rng = np.random.default_rng([42, 0x9A7])
    out["rng_first"] = rng.random(64)

    # --- renders through render.render_path ---
    w2 = (5,) + (256,) * 8 + (1,)
    n2 = O.kaiming_uniform_net(w2, seed=1)
    f2 = field.NeuralField(ref_model(n2), DELTA_CFG, bounds=UNIT_BOX)
    cam2 = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0),
                         vfov=np.pi / 4.0, width=128, height=128)
    cfg2 = render.RenderConfig(mode="path", spp=4, bounces=2, albedo=0.7,
                               env_radiance=1.0, seed=42)
    out["r2_film"] = render.render(f2, cam2, cfg2).data[:, :, 0]

    cams = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0),
                         vfov=np.pi / 4.0, width=20, height=12)
    cfgs = render.RenderConfig(mode="path", spp=3, bounces=3, albedo=0.6,
                               env_radiance=1.5, seed=9)
    out["rm_film"] = render.render(mf, cams, cfgs).data[:, :, 0]

    # --- DDFN bytes ---
    tmp = os.path.join("/tmp", "golden_small.ddfn")
    neural.save_model(ref_model(mn), 0.1, tmp)
    with open(tmp, "rb") as fh:
        out["ddfn_bytes"] = np.frombuffer(fh.read(), dtype=np.uint8)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})
    main_udf()
    main_mesh()


def main_udf():
    """field.udf_many (field.py:418-488) and recon.udf_grid (recon.py:61-81).
    recon imports scikit-image for marching cubes, which is not installed and
    not on this path: a stub module stands in for that import only."""
    import types
    if "skimage" not in sys.modules:
        sk, skm = types.ModuleType("skimage"), types.ModuleType("skimage.measure")
        skm.marching_cubes = None
        sk.measure = skm
        sys.modules["skimage"], sys.modules["skimage.measure"] = sk, skm
    from ddfield import recon
    out = {}
    mf = field.NeuralField(ref_model(march_net()), 0.1, bounds=UNIT_BOX)
    pts = np.random.default_rng(4).uniform(-1.0, 1.0, (300, 3))
    out["u_points"] = pts
    out["u_dirs64"] = field.sphere_directions(64)
    out["u_many64_raw"] = field.udf_many(mf, pts, n_dirs=64, polish=False)
    out["u_many64"] = field.udf_many(mf, pts, n_dirs=64, polish=True)
    out["u_many16"] = field.udf_many(mf, pts, n_dirs=16, polish=True)
    out["u_grid8"] = recon.udf_grid(mf, resolution=8, n_dirs=32).values
    n1 = O.kaiming_uniform_net((5, 128, 128, 128, 128, 1), seed=0)
    f1 = field.NeuralField(ref_model(n1), DELTA_CFG, bounds=UNIT_BOX)
    out["u_cfg1_many32"] = field.udf_many(f1, pts[:100], n_dirs=32, polish=True)
    path = os.path.join(HERE, "reference_golden_udf.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


def mesh_rays(n, seed):
    """Half random rays from a [-2.5, 2.5]^3 shell, half aimed at the origin
    with jitter; both from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    o = rng.uniform(-2.5, 2.5, (n, 3))
    d = rng.normal(size=(n, 3))
    half = n // 2
    d[:half] = -o[:half] + 0.3 * rng.normal(size=(half, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


def main_mesh():
    """Exact mesh backend: mesh.intersect_rays over the BVH and the linear
    scan, OracleField query / normal, render_path / render_depth /
    render_normal with an OracleField backend (field.py:144-200,
    mesh.py:264-279, render.py:144-247)."""
    from ddfield import mesh as rmesh
    from ddfield import meshes
    out = {}
    for name, m in (("blob", meshes.blob(3, 0)), ("cube", meshes.cube(0.8)), ("ico", meshes.icosphere(2))):
        o, d = mesh_rays(2048, {"blob": 1, "cube": 2, "ico": 3}[name])
        bvh = rmesh.Bvh(m)
        f, t, u, v = rmesh.intersect_rays(bvh, o, d)
        fl, tl, ul, vl = rmesh.intersect_rays(m, o, d)
        assert np.array_equal(f, fl) and np.array_equal(t, tl)
        out[f"{name}_o"], out[f"{name}_d"] = o, d
        out[f"{name}_face"], out[f"{name}_t"], out[f"{name}_u"], out[f"{name}_v"] = f, t, u, v
        fw, tw, _, _ = rmesh.intersect_rays(bvh, o, d, 0.5, 3.0)
        out[f"{name}_face_win"], out[f"{name}_t_win"] = fw, tw
        of = field.OracleField(m)
        out[f"{name}_q_t"], out[f"{name}_q_hit"] = of.query_batch(o, d)
        out[f"{name}_n"], out[f"{name}_n_valid"] = of.normal_batch(o, d)
    of = field.OracleField(meshes.blob(3, 0))
    cam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=40, height=30)
    cfg = render.RenderConfig(mode="path", spp=3, bounces=3, albedo=0.6, env_radiance=1.2, seed=7)
    out["blob_film"] = render.render(of, cam, cfg).data[:, :, 0]
    cube = field.OracleField(meshes.cube(0.8))
    cc = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=21, height=21)
    out["cube_depth"] = render.render_depth(cube, cc).data
    out["cube_normal"] = render.render_normal(cube, cc, render.RenderConfig(mode="normal")).data
    # exact distance (mesh.closest_distance) and the exact UDF grid (recon.udf_grid)
    import types
    if "skimage" not in sys.modules:
        sk, skm = types.ModuleType("skimage"), types.ModuleType("skimage.measure")
        skm.marching_cubes = None
        sk.measure = skm
        sys.modules["skimage"], sys.modules["skimage.measure"] = sk, skm
    from ddfield import recon
    pts = np.random.default_rng(21).uniform(-2.0, 2.0, (3000, 3))
    pts[:600] *= 0.55                                   # many near / inside the surface
    bm = meshes.blob(3, 0)
    out["closest_pts"] = pts
    out["closest_blob"] = field.OracleField(bm).exact_distance(pts)
    assert np.array_equal(out["closest_blob"], field.BruteForceField(bm).exact_distance(pts))
    out["closest_cube"] = field.OracleField(meshes.cube(0.8)).exact_distance(pts)
    out["udf_grid_blob"] = recon.udf_grid(field.OracleField(bm), resolution=12).values
    path = os.path.join(HERE, "reference_golden_mesh.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


if __name__ == "__main__":
    if sys.argv[1:] == ["udf"]:
        main_udf()
    elif sys.argv[1:] == ["mesh"]:
        main_mesh()
    else:
        main()
