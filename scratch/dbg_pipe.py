import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C, render as R, _lib
name = sys.argv[1]
f = C.build_field(name); cam = C.camera(name); cfg = C.render_config(name)
R.render_path_device(f, cam, cfg); torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)()
_lib.lib().ddf_debug_counters(buf, 1)
cfg.profile = 1
acc, st = R.render_path_device(f, cam, cfg); torch.cuda.synchronize()
_lib.lib().ddf_debug_counters(buf, 1)
c = list(buf)
names = ["mma_wait_a_ready", "mma_wait_w_full", "epi_wait_acc (warp2)", "epi_wait_a_free (warp2)", "mma_total", "mma_steps", "prod_wait_empty", "epi_busy (warp2)", "mma_issue_blocks"]
print(name, "ms fwd %.1f grad %.1f total %.1f" % (st["ms_forward"], st["ms_gradient"], st["ms_total"]))
tot = c[4]
for i, n in enumerate(names):
    print(f"  {n:26s} {c[i]:16d}  {100*c[i]/max(tot,1):6.1f}% of MMA-warp cycles")
