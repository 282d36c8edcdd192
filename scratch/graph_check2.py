import sys, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C, render as R
name = sys.argv[1]; reps = int(sys.argv[2])
f = C.build_field(name); cam = C.camera(name)
acc = torch.empty(cam.width * cam.height, dtype=torch.float64, device="cuda")
for rnd in range(2):
    for gr in (0, 1):
        cfg = C.render_config(name, graph=gr)
        R.render_path_device(f, cam, cfg, accum=acc); torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); R.render_path_device(f, cam, cfg, accum=acc); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(name, "graph", gr, "min %.2f mean %.2f" % (min(ts), sum(ts) / len(ts)), flush=True)
