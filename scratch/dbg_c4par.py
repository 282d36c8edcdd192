import sys, numpy as np
sys.path.insert(0, '.')
from oracle import cpu_ddf as O
from paper_2306_16142_b200 import configs as C, render as R
from paper_2306_16142_b200.field import CudaNeuralField
D = 10/0.98; BOX = np.array([[-1.0]*3, [1.0]*3])
m = C.models("c4")[0]
f = CudaNeuralField(m, D, bounds=BOX, precision="fp32")
of = O.Field([O.Net(m.widths, m.v, m.g, m.b)], D, bounds=BOX)
W, H = 24, 14
cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
oc = O.Cam((0, 0, 3.0), (0, 0, 0.0), vfov=np.pi / 4, width=W, height=H)
for b, rr in [(1, -1), (2, -1), (3, -1), (5, -1), (8, -1), (8, 3)]:
    img = R.render_path(f, cam, R.RenderConfig(spp=2, bounces=b, seed=42, rr_start=rr)).data[:, :, 0].reshape(-1)
    ref = O.render_path(of, oc, O.PathConfig(spp=2, bounces=b, albedo=0.7, env=1.0, seed=42, rr_start=rr))
    d = np.abs(img - ref)
    print(f"bounces {b} rr {rr}: RMSE {np.sqrt(np.mean(d**2)):.3g} max {d.max():.3g} pixels>1e-6 {np.mean(d > 1e-6):.3f} mean {img.mean():.4f} vs {ref.mean():.4f}")
# normals at primary hits
n = W * H
o, d = O.camera_rays(oc, np.full((n, 2), 0.5), np.arange(n))
t, hit, _ = of.trace(o, d)
tg, hg = f.trace_batch(o, d)
print("primary hit agree", (hit == hg).mean(), "t maxdiff", np.max(np.abs(t[hit & hg] - tg[hit & hg])))
nr, vr = of.normal(o[hit], d[hit], t[hit])
ng, vg = f.normal_batch(o[hit], d[hit], t_hit=t[hit])
ang = np.degrees(np.arccos(np.clip(np.einsum('ij,ij->i', nr, ng), -1, 1)))
print("normal angle err max", ang.max(), "median", np.median(ang))
