"""Pipeline counters of the <= 128-wide (quad) and <= 256-wide (ping-pong)
tcgen05 engines: needs a library built with -DDDF_PIPE_STATS=1, e.g.

  DDF_NVCC_EXTRA=-DDDF_PIPE_STATS=1 DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_stats.so \\
      python -c "from paper_2306_16142_b200 import _lib; _lib.build()"
  DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_stats.so python tools/quad_stats.py [rows]

Runs the config-1 query (QueryOp, f64 geometry) and the raw forward on the
same network, and prints each role's cycle counters as a share of its total."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_16142_b200 import _lib  # noqa: E402
from paper_2306_16142_b200 import configs as C  # noqa: E402

NAMES = {0: "issuer waits A_READY", 1: "issuer waits weights (FULL)", 2: "row warp waits accumulator", 3: "row: load path state",
         4: "issuer total", 5: "row: encode + store A", 6: "producer waits EMPTY", 7: "row: epilogues", 8: "row: stage params",
         9: "row total", 10: "row: store result"}


def counters(reset=True):
    buf = (ctypes.c_uint64 * 16)()
    _lib.lib().ddf_debug_counters(buf, int(reset))
    return list(buf)


def show(title, c, ms):
    print(f"== {title}: {ms:.3f} ms")
    for i, v in enumerate(c):
        if v:
            tot = c[4] if i in (0, 1, 4) else c[9] if i in (2, 3, 5, 7, 8, 9, 10) else 0
            print(f"  [{i:2d}] {NAMES.get(i, '?'):32s} {v:>16d}" + (f"  {100.0 * v / tot:5.1f}% of role" if tot else ""))


def timed(fn):
    fn()
    torch.cuda.synchronize()
    counters(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    name = sys.argv[2] if len(sys.argv) > 2 else "c1"
    torch.cuda.set_device(0)
    f = C.build_field(name, precision="bf16")
    o, d = C.query_rays(1 << 16, 0)
    reps = -(-n // (1 << 16))
    od = torch.from_numpy(o).cuda().repeat(reps, 1)[:n].contiguous()
    dd = torch.from_numpy(d).cuda().repeat(reps, 1)[:n].contiguous()
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    hit = torch.empty(n, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ms = timed(lambda: _lib.check(L.ddf_query(f.handle, P(od), P(dd), n, P(t), P(hit), None, None, s)))
    show(f"{name} query, {n} rows ({n / ms / 1e3:.0f} M queries/s)", counters(True), ms)
    if name == "c1":
        w = C.WORKLOADS["c1"]["widths"]
        x = torch.rand(n, w[0], dtype=torch.float64, device="cuda") * 2 - 1
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        ms = timed(lambda: _lib.check(L.ddf_mlp_forward(f.handle, 0, P(x), n, P(y), s)))
        show(f"raw forward, {n} rows ({n / ms / 1e3:.0f} M rows/s)", counters(True), ms)
        g = torch.empty(n, w[0], dtype=torch.float64, device="cuda")
        ms = timed(lambda: _lib.check(L.ddf_mlp_input_grad(f.handle, 0, P(x), n, P(g), s)))
        show(f"raw gradient, {n} rows ({n / ms / 1e3:.0f} M rows/s)", counters(True), ms)


if __name__ == "__main__":
    main()
