import sys, numpy as np
sys.path.insert(0, '.')
from oracle import cpu_ddf as O
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform, MlpModel
BOX = np.array([[-1.0]*3,[1.0]*3])
def run(widths, n=512, zero_bias=True):
    m = kaiming_uniform(widths, 3)
    f = CudaNeuralField(m, 1.0, bounds=BOX, precision="bf16")
    x = np.random.default_rng(1).uniform(-1,1,(n, widths[0]))
    on = O.Net(m.widths, m.v, m.g, m.b)
    y = f.forward_inputs(x); yr = O.mlp_forward(on, x)
    g = f.input_gradient_inputs(x); gr = O.mlp_input_grad(on, x)
    rms = np.sqrt(np.mean(gr**2))
    e = np.abs(g-gr)/rms
    print(widths, "fwd max", np.abs(y-yr).max()/np.sqrt(np.mean(yr**2)), "grad max", e.max(), "median", np.median(e))
    bad = np.argwhere(e > 0.2)
    print("  bad rows", np.unique(bad[:,0])[:20], "cols", np.unique(bad[:,1]), "nbad rows", len(np.unique(bad[:,0])))
    print("  g[0]", g[0][:6], "\n  r[0]", gr[0][:6])
    f.set_precision("fp32")
    g2 = f.input_gradient_inputs(x)
    print("  fp32 grad max", (np.abs(g2-gr)/rms).max())
run((5,64,64,1))
run((5,64,1))  if False else None
run((5,128,128,1))
run((5,128,128,128,128,1))

run((5,64,64,64,1))
