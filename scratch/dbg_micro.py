import sys, ctypes, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import _lib, configs as C
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform
widths = eval(sys.argv[1]); n = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "fwd"
_lib.LIB_PATH = os.environ.get("DDF_LIB", _lib.LIB_PATH)
f = CudaNeuralField(kaiming_uniform(widths, 2), 10/0.98, precision="bf16")
buf0 = (ctypes.c_uint64 * 16)(); _lib.lib().ddf_debug_counters(buf0, 1)
x = torch.rand(n, widths[0], dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty(n, dtype=torch.float64, device="cuda") if mode == "fwd" else torch.empty(n, widths[0], dtype=torch.float64, device="cuda")
_lib.LIB_PATH = os.environ.get("DDF_LIB", _lib.LIB_PATH); L = _lib.lib(); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
(L.ddf_mlp_forward if mode == "fwd" else L.ddf_mlp_input_grad)(f.handle, 0, ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(y.data_ptr()), s); torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)(); L.ddf_debug_counters(buf, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
(L.ddf_mlp_forward if mode == "fwd" else L.ddf_mlp_input_grad)(f.handle, 0, ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(y.data_ptr()), s); e1.record(); torch.cuda.synchronize()
L.ddf_debug_counters(buf, 1); c = list(buf)
names = ["mma_wait_a_ready", "mma_wait_w_full", "epi_wait_acc", "epi_wait_a_free", "mma_total", "mma_steps", "prod_wait_empty", "epi_busy", "mma_issue_blocks", "epi_compute", "epi_free_wait", "epi_store_arrive"]
F = C.mlp_flops(widths) * (1 if mode == "fwd" else 2); ms = e0.elapsed_time(e1)
print(widths[:3], mode, f"{ms:.2f} ms {F*n/ms/1e9:.0f} TF/s")
for i, nm in enumerate(names): print(f"  {nm:18s} {c[i]/148:14.0f} per CTA  {100*c[i]/max(c[4],1):6.1f}%")
