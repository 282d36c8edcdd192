import sys, numpy as np
sys.path.insert(0, '.')
from oracle import cpu_ddf as O
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform
for widths in [(65, 512, 512, 1), (65, 256, 256, 1), (5, 512, 512, 1), (65,) + (512,) * 8 + (1,), (5, 300, 1)]:
    m = kaiming_uniform(widths, 3)
    f = CudaNeuralField(m, 1.0, precision="fp32")
    x = np.random.default_rng(1).uniform(-1, 1, (700, widths[0]))
    on = O.Net(m.widths, m.v, m.g, m.b)
    y = f.forward_inputs(x); yr = O.mlp_forward(on, x)
    g = f.input_gradient_inputs(x); gr = O.mlp_input_grad(on, x)
    e = np.abs(g - gr).max(1) / np.sqrt(np.mean(gr ** 2))
    print(widths[:3], len(widths), "fwd", np.abs(y - yr).max() / np.sqrt(np.mean(yr ** 2)), "grad max", e.max(), "bad rows", np.sum(e > 1e-3), "first bad", np.argmax(e > 1e-3))
