import sys, time, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C, render as R
name = sys.argv[1]
f = C.build_field(name); cam = C.camera(name)
for mw in [int(x) for x in sys.argv[2:]]:
    cfg = C.render_config(name, max_wave_paths=mw)
    acc, st = R.render_path_device(f, cam, cfg); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); acc, st = R.render_path_device(f, cam, cfg, accum=acc); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "max_wave_paths", mw, "waves", st["waves"], "ms", min(ts), "Msamples/s", cam.width * cam.height * cfg.spp / min(ts) / 1e3, "launches", st["kernel_launches"], flush=True)
