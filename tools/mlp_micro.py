import sys, ctypes, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import _lib, configs as C
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform
widths = eval(sys.argv[1]); n = int(sys.argv[2]); prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
m = kaiming_uniform(widths, 2)
f = CudaNeuralField(m, 10/0.98, precision=prec)
x = torch.rand(n, widths[0], dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty(n, dtype=torch.float64, device="cuda"); g = torch.empty(n, widths[0], dtype=torch.float64, device="cuda")
L = _lib.lib(); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
F = C.mlp_flops(widths)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
tf = t(lambda: L.ddf_mlp_forward(f.handle, 0, ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(y.data_ptr()), s))
tg = t(lambda: L.ddf_mlp_input_grad(f.handle, 0, ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(g.data_ptr()), s))
print(f"{str(widths[:3]):16s} n={n} {prec} dbg={os.environ.get('DDF_DEBUG_UMMA','0')}: fwd {tf:.2f} ms {n/tf/1e3:.3g} Mrows/s {F*n/tf/1e9:.0f} TF/s | grad {tg:.2f} ms {2*F*n/tg/1e9:.0f} TF/s")
