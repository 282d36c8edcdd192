import sys, ctypes, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import _lib, configs as C
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform
widths = eval(sys.argv[1]); n = int(sys.argv[2])
f = CudaNeuralField(kaiming_uniform(widths, 2), 10/0.98, precision="bf16")
o = torch.rand(n, 3, dtype=torch.float64, device="cuda") * 2 - 1
d = torch.nn.functional.normalize(torch.randn(n, 3, dtype=torch.float64, device="cuda"), dim=1)
t = torch.empty(n, dtype=torch.float64, device="cuda"); hit = torch.empty(n, dtype=torch.uint8, device="cuda")
L = _lib.lib(); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda x: ctypes.c_void_p(x.data_ptr())
q = lambda: L.ddf_query(f.handle, P(o), P(d), n, P(t), P(hit), None, None, s)
q(); torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)(); L.ddf_debug_counters(buf, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); q(); e1.record(); torch.cuda.synchronize()
L.ddf_debug_counters(buf, 1); c = list(buf)
ms = e0.elapsed_time(e1)
print(f"{widths} n={n} query {ms:.3f} ms  {C.mlp_flops(widths)*n/ms/1e9:.0f} TF/s")
names = {0: "mma wait A_READY", 1: "mma wait FULL", 4: "mma total", 6: "prod wait EMPTY", 2: "row wait ACC", 3: "row load", 5: "row encode", 7: "row epilogue", 8: "row params", 10: "row store", 9: "row total"}
for i in (4, 0, 1, 6, 9, 3, 5, 2, 7, 8, 10):
    print(f"  {names[i]:18s} {c[i]/148/1e3:10.1f} kcyc/CTA")
