# Timing experiment (diagnostics build only): is the 512-wide engine bound by
# shared-memory bandwidth?  dbg 1 drops the weight stream's smem writes (wrong
# results), dbg 128 drops the MMAs (epilogue-only time).
import sys, os, ctypes, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import _lib
_lib.LIB_PATH = os.path.abspath('scratch/statslib/libddf_b200.so')
from paper_2306_16142_b200 import configs as C
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform
widths = eval(sys.argv[1]); n = int(sys.argv[2])
m = kaiming_uniform(widths, 2)
f = CudaNeuralField(m, 10/0.98, precision="bf16")
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
print(f"{str(widths[:3]):16s} n={n} dbg={os.environ.get('DDF_DEBUG_UMMA','0')}: fwd {tf:.2f} ms {F*n/tf/1e9:.0f} TF/s | grad {tg:.2f} ms {2*F*n/tg/1e9:.0f} TF/s", flush=True)
if os.environ.get("STATS"):
    buf = (ctypes.c_uint64 * 16)()
    L.ddf_debug_counters(buf, 1)
    L.ddf_mlp_forward(f.handle, 0, ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(y.data_ptr()), s); torch.cuda.synchronize()
    L.ddf_debug_counters(buf, 1)
    c = list(buf)
    names = ["mma_wait_a_ready", "mma_wait_w_full", "epi_wait_acc(w2)", "epi_wait_a_free(w2)", "mma_total", "mma_steps", "prod_wait_empty", "epi_busy(w2)", "mma_issue"]
    tiles = (n + 127) // 128
    per_sm_steps = c[5] / 148
    print("  forward counters, cycles per (SM x step):", flush=True)
    for i, nm in enumerate(names):
        if i == 5: continue
        print(f"    {nm:22s} {c[i] / max(c[5],1):10.0f}")
