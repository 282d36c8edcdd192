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


# --------------------------------------------------------------------------
# EXTENSIONS the BASELINE configs need, layered on the
# unmodified reference: subclasses override only what App. A names, so the
# reference's own code still marches (field.py:260-289), takes normals
# (field.py:295-317, render.py:127-141), samples bounces (render.py:187-195)
# and builds camera rays (render.py:54-75).
# --------------------------------------------------------------------------
PE_OCTAVES = 6
RR_TAG = 0x5252


def pe(u):
    """65-D encoding of the 5 encoded inputs, column order
    [u, sin(2^0 pi u), cos(2^0 pi u), ..., sin(2^5 pi u), cos(2^5 pi u)]."""
    cols = [u]
    for k in range(PE_OCTAVES):
        a = (2.0 ** k) * np.pi * u
        cols += [np.sin(a), np.cos(a)]
    return np.concatenate(cols, axis=1)


def pe_backprop(u, g65):
    """d out / d u from d out / d(pe(u)): d sin(f u)/du = f cos(f u),
    d cos(f u)/du = -f sin(f u)."""
    g = g65[:, :5].copy()
    for k in range(PE_OCTAVES):
        f = (2.0 ** k) * np.pi
        a = f * u
        base = 5 + 10 * k
        g += f * np.cos(a) * g65[:, base:base + 5]
        g -= f * np.sin(a) * g65[:, base + 5:base + 10]
    return g


def encoded_gradient(model, u):
    """neural.input_gradient_batch (neural.py:229-249) on the 65 encoded
    inputs.  The reference sizes its output by the module constant N_INPUTS
    (neural.py:23, 234); it is widened for the call and restored."""
    saved = neural.N_INPUTS
    neural.N_INPUTS = int(model.widths[0])
    try:
        g65 = neural.input_gradient_batch(model, pe(u))
    finally:
        neural.N_INPUTS = saved
    return pe_backprop(u, g65)


class EncodedNeuralField(field.NeuralField):
    """NeuralField with the 6-octave encoding (configs 3-5): overrides
    _predict (field.py:244-246) and input_gradients (field.py:291-293)."""

    def _predict(self, positions, angles):
        return neural.forward_batch(self.model, pe(neural.encode_inputs(positions, angles)))

    def input_gradients(self, positions, angles):
        return encoded_gradient(self.model, neural.encode_inputs(positions, angles))


class SceneNeuralField(field.NeuralField):
    """Config 5: distance = min_j scale * f_j((x - c_j) / scale, angles), ties
    to the lower object index.  The normal of a row is the gradient of the
    object ``grad_obj`` names (the one the row hit, set by the render loop);
    d/dx of s f((x - c)/s) is grad f."""

    def __init__(self, models, centers, scale, albedos, delta, bounds):
        super().__init__(models[0], delta, bounds=bounds)
        self.models, self.centers, self.scale = models, np.asarray(centers, dtype=np.float64), float(scale)
        self.albedos = np.asarray(albedos, dtype=np.float64)
        self.grad_obj = None

    def _object_preds(self, positions, angles):
        return [self.scale * neural.forward_batch(m, pe(neural.encode_inputs((positions - c) / self.scale, angles)))
                for m, c in zip(self.models, self.centers)]

    def _predict(self, positions, angles):
        preds = self._object_preds(positions, angles)
        best = preds[0]
        for p in preds[1:]:
            best = np.where(p < best, p, best)
        return best

    def argmin(self, positions, angles):
        preds = self._object_preds(positions, angles)
        best, obj = preds[0], np.zeros(len(positions), np.int32)
        for j, p in enumerate(preds[1:], start=1):
            take = p < best
            obj[take] = j
            best = np.where(take, p, best)
        return obj

    def trace_with_objects(self, origins, dirs):
        """The reference's trace_batch, plus the object of each hit.  In the
        configs' regime (0.9 delta spans the box) a hit is found at march
        step 0, so its object is the argmin at o + max(t_enter, 0) d; the
        reconstructed t is asserted equal to the march's."""
        t, hit = self.trace_batch(origins, dirs)
        ang = field.vecs_to_angles(dirs)
        te, _ = field._ray_box(origins, dirs, self.bounds)
        t0 = np.maximum(te, 0.0)
        p0 = origins + t0[:, None] * dirs
        obj = np.zeros(len(origins), np.int32)
        if hit.any():
            obj[hit] = self.argmin(p0[hit], ang[hit])
            c = np.clip(self._predict(p0[hit], ang[hit]), -self.delta, self.delta)
            assert np.array_equal(t0[hit] + np.maximum(c, 0.0), t[hit]), "not a single-step march"
        return t, hit, obj

    def input_gradients(self, positions, angles):
        out = np.zeros((len(positions), 5))
        for j, (m, c) in enumerate(zip(self.models, self.centers)):
            sel = self.grad_obj == j
            if sel.any():
                out[sel] = encoded_gradient(m, neural.encode_inputs((positions[sel] - c) / self.scale, angles[sel]))
        return out


def render_path_ext(backend, camera, config, rr_start=-1):
    """render.render_path (render.py:198-247) with the two EXTENSIONS App. A
    asks for: Russian roulette from bounce index rr_start (survive with
    p = min(1, throughput), throughput /= p; the uniform is draw
    (s * bounces + b) * n_pix + i of default_rng([seed, 0x5252]), so the
    reference stream's draws are untouched) and, for a SceneNeuralField,
    per-object albedo and hit-object normals.  Everything else calls the
    reference: pixel_rays, trace_batch, _hit_normals, _cosine_dirs."""
    rng = np.random.default_rng([config.seed, 0x9A7])
    rr_rng = np.random.default_rng([config.seed, RR_TAG])
    scene = isinstance(backend, SceneNeuralField)
    n_pix = camera.width * camera.height
    accum = np.zeros(n_pix)
    for _ in range(config.spp):
        jitter = rng.random((n_pix, 2))
        origins, dirs = render.pixel_rays(camera, offsets=jitter)
        radiance = np.zeros(n_pix)
        throughput = np.ones(n_pix)
        if scene:
            t, hit, obj = backend.trace_with_objects(origins, dirs)
        else:
            (t, hit), obj = backend.trace_batch(origins, dirs), np.zeros(n_pix, np.int32)
        radiance[~hit] = config.env_radiance
        alive = hit.copy()
        pos = origins
        for b in range(config.bounces):
            u = rng.random((n_pix, 2))
            rr = rr_rng.random(n_pix)
            if 0 <= rr_start <= b and alive.any():
                idx = np.nonzero(alive)[0]
                p = np.minimum(1.0, throughput[idx])
                live = rr[idx] < p
                alive[idx[~live]] = False
                throughput[idx[live]] = throughput[idx[live]] / p[live]
            if not alive.any():
                continue
            idx = np.nonzero(alive)[0]
            if scene:
                backend.grad_obj = obj[idx]
            normals = render._hit_normals(backend, pos[idx], dirs[idx], t[idx], np.ones(len(idx), dtype=bool))
            hit_pts = pos[idx] + t[idx, None] * dirs[idx] + 1e-6 * normals
            throughput[idx] *= backend.albedos[obj[idx]] if scene else config.albedo
            new_dirs = render._cosine_dirs(normals, u[idx])
            if scene:
                t_new, hit_new, obj_new = backend.trace_with_objects(hit_pts, new_dirs)
            else:
                t_new, hit_new = backend.trace_batch(hit_pts, new_dirs)
                obj_new = np.zeros(len(idx), np.int32)
            escaped = idx[~hit_new]
            radiance[escaped] += throughput[escaped] * config.env_radiance
            alive[escaped] = False
            cont = idx[hit_new]
            pos[cont] = hit_pts[hit_new]
            dirs[cont] = new_dirs[hit_new]
            t[cont] = t_new[hit_new]
            obj[cont] = obj_new[hit_new]
            alive_next = np.zeros(n_pix, dtype=bool)
            alive_next[cont] = True
            alive = alive_next
        accum += radiance
    return accum / config.spp


def scene_layout():
    """Config 5's layout (paper_2306_16142_b200.configs.scene_layout)."""
    import itertools
    centers = np.array(list(itertools.product((-0.75, 0.75), repeat=3)), dtype=np.float64)
    return centers, 0.5, np.random.default_rng(5).uniform(0.2, 0.9, 8)


def main_ext():
    """Fixtures for the EXTENSIONS: 65-D PE network (forward, gradient,
    query, trace, normals), Russian roulette renders, and an 8-object
    min-composite scene (trace with objects, hit-object normals, render)."""
    out = {}
    pe_w = (65, 128, 128, 1)
    pn = O.kaiming_uniform_net(pe_w, seed=6)
    pf = EncodedNeuralField(ref_model(pn), DELTA_CFG, bounds=UNIT_BOX)
    o, d = rays(512, seed=11)
    ang = field.vecs_to_angles(d)
    u = neural.encode_inputs(o, ang)
    out["pe_o"], out["pe_d"] = o, d
    out["pe_forward"] = neural.forward_batch(pf.model, pe(u))
    out["pe_grad5"] = pf.input_gradients(o, ang)
    out["pe_query_t"], out["pe_query_hit"] = pf.query_batch(o, d)
    out["pe_trace_t"], out["pe_trace_hit"] = pf.trace_batch(o * 2.5, d)
    th = np.where(np.isfinite(out["pe_trace_t"]), out["pe_trace_t"], 0.0)
    out["pe_normal"], out["pe_normal_valid"] = pf.normal_batch(o * 2.5, d, t_hit=th)
    cam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=24, height=16)
    cfg = render.RenderConfig(mode="path", spp=2, bounces=2, albedo=0.7, env_radiance=1.0, seed=42)
    out["pe_film"] = render.render(pf, cam, cfg).data[:, :, 0]        # the reference's own render_path
    out["pe_film_ext"] = render_path_ext(pf, cam, cfg).reshape(16, 24)
    assert np.array_equal(out["pe_film"], out["pe_film_ext"]), "the RR copy must equal render_path with RR off"
    cfg_rr = render.RenderConfig(mode="path", spp=3, bounces=6, albedo=0.7, env_radiance=1.0, seed=8)
    out["pe_rr_film"] = render_path_ext(pf, cam, cfg_rr, rr_start=1).reshape(16, 24)

    centers, scale, albedos = scene_layout()
    nets = [O.kaiming_uniform_net((65, 32, 32, 1), s) for s in range(10, 18)]
    box = np.array([[-1.25] * 3, [1.25] * 3])
    sf = SceneNeuralField([ref_model(n) for n in nets], centers, scale, albedos, DELTA_CFG, box)
    so, sd = rays(400, seed=12)
    so = so * 2.2
    out["sc_o"], out["sc_d"] = so, sd
    out["sc_trace_t"], out["sc_trace_hit"], out["sc_trace_obj"] = sf.trace_with_objects(so, sd)
    h = out["sc_trace_hit"]
    sf.grad_obj = out["sc_trace_obj"][h]
    out["sc_normal"], out["sc_normal_valid"] = sf.normal_batch(so[h], sd[h], t_hit=out["sc_trace_t"][h])
    scam = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=20, height=14)
    scfg = render.RenderConfig(mode="path", spp=2, bounces=4, albedo=0.7, env_radiance=1.0, seed=42)
    out["sc_film"] = render_path_ext(sf, scam, scfg).reshape(14, 20)
    out["sc_rr_film"] = render_path_ext(sf, scam, scfg, rr_start=2).reshape(14, 20)
    path = os.path.join(HERE, "reference_golden_ext.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


class StageCountingField(field.NeuralField):
    """The reference NeuralField, recording the length of every per-stage
    list its callers hand it: one ("march", n) per trace_batch march step
    (the np.nonzero list of field.py:277, seen by _predict) and one
    ("normal", n) per bounce (the alive list of render.py:225, seen by
    normal_batch)."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.stages = []

    def _predict(self, positions, angles):
        self.stages.append((0, len(positions)))
        return super()._predict(positions, angles)

    def normal_batch(self, origins, dir_vecs, t_hit=None):
        self.stages.append((1, len(origins)))
        return super().normal_batch(origins, dir_vecs, t_hit=t_hit)


def main_stages():
    """Per-stage list lengths of the unmodified render_path for the
    config-2 render and the march-regime render (compaction parity)."""
    out = {}
    w2 = (5,) + (256,) * 8 + (1,)
    f2 = StageCountingField(ref_model(O.kaiming_uniform_net(w2, seed=1)), DELTA_CFG, bounds=UNIT_BOX)
    cam2 = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=128, height=128)
    film = render.render(f2, cam2, render.RenderConfig(mode="path", spp=4, bounces=2, albedo=0.7,
                                                       env_radiance=1.0, seed=42)).data[:, :, 0]
    assert np.array_equal(film, np.load(os.path.join(HERE, "reference_golden.npz"))["r2_film"])
    out["r2_stages"] = np.array(f2.stages, dtype=np.int64)
    mf = StageCountingField(ref_model(march_net()), 0.1, bounds=UNIT_BOX)
    cams = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=20, height=12)
    render.render(mf, cams, render.RenderConfig(mode="path", spp=3, bounces=3, albedo=0.6, env_radiance=1.5, seed=9))
    out["rm_stages"] = np.array(mf.stages, dtype=np.int64)
    # a larger march-regime film for the GPU's stage lists (48 x 32, 2 spp)
    camb = render.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=48, height=32)
    mf.stages = []
    out["rmb_film"] = render.render(mf, camb, render.RenderConfig(mode="path", spp=2, bounces=3, albedo=0.6,
                                                                  env_radiance=1.5, seed=9)).data[:, :, 0]
    out["rmb_stages"] = np.array(mf.stages, dtype=np.int64)
    path = os.path.join(HERE, "reference_golden_stages.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


MESH_FIXTURES = {"blob3": ("blob", (3, 0)), "blob3_1": ("blob", (3, 1)), "blob4": ("blob", (4, 0)),
                 "blob5_2": ("blob", (5, 2)), "cube": ("cube", (0.8,)), "ico": ("icosphere", (2,)),
                 "plane_quad": ("plane_quad", ())}


def main_meshes():
    """The reference's procedural test meshes (meshes.py), stored as arrays so
    the tests and bench.py's BVH workload need no copy of the generators:
    vertices (N, 3) f64 and faces (M, 3) i32 per mesh."""
    from ddfield import meshes
    out = {}
    for key, (fn, args) in MESH_FIXTURES.items():
        m = getattr(meshes, fn)(*args)
        out[f"{key}_v"], out[f"{key}_f"] = m.vertices, m.faces
    path = os.path.join(HERE, "reference_meshes.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: getattr(v, "shape", None) for k, v in out.items()})


if __name__ == "__main__":
    which = sys.argv[1:]
    if which == ["udf"]:
        main_udf()
    elif which == ["mesh"]:
        main_mesh()
    elif which == ["meshes"]:
        main_meshes()
    elif which == ["ext"]:
        main_ext()
    elif which == ["stages"]:
        main_stages()
    else:
        main()
        main_meshes()
        main_ext()
        main_stages()
