import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C, render as R
for name, prec in (("c2", "bf16"), ("c2", "fp32"), ("c5", "bf16"), ("c3", "bf16")):
    f = C.build_field(name, precision=prec); cam = C.camera(name)
    acc = torch.empty(cam.width * cam.height, dtype=torch.float64, device="cuda")
    res = {}
    for gr in (0, 1):
        cfg = C.render_config(name, graph=gr)
        R.render_path_device(f, cam, cfg, accum=acc); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); _, st = R.render_path_device(f, cam, cfg, accum=acc); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[gr] = (min(ts), acc.clone())
    print(name, prec, "eager %.3f ms  graph %.3f ms  identical %s  launches %d" % (res[0][0], res[1][0], torch.equal(res[0][1], res[1][1]), st["kernel_launches"]), flush=True)
