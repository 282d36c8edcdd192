"""3xTF32 vs FFMA vs f64 oracle on the config-2 network: per-row error
distributions of forward and input gradient, and the config-2 image."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cpu_ddf as O
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform, MlpModel
from paper_2306_16142_b200 import render as R

BOX = np.array([[-1.0] * 3, [1.0] * 3]); DELTA = 10.0 / 0.98
net = kaiming_uniform((5,) + (256,) * 8 + (1,), 1)
onet = O.Net(net.widths, net.v, net.g, net.b)
x = np.random.default_rng(0).uniform(-1, 1, (20000, 5))
ref = O.mlp_forward(onet, x); gref = O.mlp_input_grad(onet, x)
def rel(a, r):
    s = np.maximum(np.abs(r), np.sqrt(np.mean(r ** 2)))
    return np.abs(a - r) / s
for prec in ("fp32", "fp32_simt"):
    f = CudaNeuralField(net, DELTA, bounds=BOX, precision=prec)
    y = f.forward_inputs(x); g = f.input_gradient_inputs(x)
    e = rel(y, ref); eg = np.stack([rel(g[:, j], gref[:, j]) for j in range(5)], 1)
    print(prec, "fwd max %.2e p99.9 %.2e med %.2e" % (e.max(), np.quantile(e, .999), np.median(e)),
          "| grad max %.2e p99.9 %.2e med %.2e" % (eg.max(), np.quantile(eg, .999), np.median(eg)))
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4.0, width=128, height=128)
    cfg = R.RenderConfig(mode="path", spp=4, bounces=2, albedo=0.7, env_radiance=1.0, seed=42)
    img = R.render_path(f, cam, cfg).data[:, :, 0]
    gold = np.load("tests/golden/reference_golden.npz")["r2_film"]
    d = np.abs(img - gold)
    print(prec, "image rmse %.3e  pixels differing %d (%.3f%%)  max %.3f" % (np.sqrt(np.mean(d ** 2)), (d > 1e-9).sum(), 100 * (d > 1e-9).mean(), d.max()))
