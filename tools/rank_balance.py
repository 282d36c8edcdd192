"""Per-rank load of the config-4 tile sharding, measured on ONE GPU.

For world = 1, 2, 4, 8 each rank's share (ddf_path_config_t.rank/world) is
rendered on its own, one after another, and timed with CUDA events; the
predicted strong-scaling efficiency at that world size (ignoring the film
all-reduce) is T(world=1) / (world * max_r T_r).  No rank waits on another.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16142_b200 import configs as C  # noqa: E402
from paper_2306_16142_b200 import render as R  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    torch.cuda.set_device(0)
    fld = C.build_field(name)
    cam = C.camera(name)
    accum = torch.empty(cam.width * cam.height, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    mode = sys.argv[3] if len(sys.argv) > 3 else "rr"
    out = {"workload": name, "mode": mode, "worlds": {}}
    cost = None
    if mode == "pilot":
        from paper_2306_16142_b200.dist import balanced_tile_owners, measure_tile_costs
        import time
        t0 = time.perf_counter()
        cost = measure_tile_costs(fld, cam, C.render_config(name), 64)
        out["pilot_s"] = time.perf_counter() - t0
        print("pilot", out["pilot_s"], flush=True)
    t1 = None
    for world in (1, 2, 4, 8):
        times, rows = [], []
        owner = balanced_tile_owners(cost, world) if cost is not None and world > 1 else None
        for rank in range(world):
            cfg = C.render_config(name, rank=rank, world=world, tile=64, tile_owner=owner)
            R.render_path_device(fld, cam, cfg, accum=accum, stream=s)
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                _, st = R.render_path_device(fld, cam, cfg, accum=accum, stream=s)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            times.append(float(np.median(ts)))
            rows.append(int(st["forward_rows"]))
        if world == 1:
            t1 = times[0]
        mx = max(times)
        out["worlds"][world] = {"ms_per_rank": times, "forward_rows_per_rank": rows,
                                "max_over_mean": mx / float(np.mean(times)),
                                "predicted_efficiency": t1 / (world * mx)}
        print(world, json.dumps(out["worlds"][world]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
