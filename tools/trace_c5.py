"""Event timeline of the ping-pong engine on config 5's scene (8 networks per
tile, 65-D encoding): needs a -DDDF_TRACE=1 library (see tools/trace_mlp.py).

  DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_trace.so python tools/trace_c5.py [rays]

Prints CTA 0's events for one pair of tiles in time order: issuer (role 1) and
two row warps (roles 2, 3); step = layer step * 2 + slot."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_16142_b200 import configs as C  # noqa: E402
from tools.trace_quad import read_trace  # noqa: E402

EV = {1: "I.waitA", 2: "I.gotA", 7: "I.issued", 16: "R.pair", 17: "R.waitAcc", 18: "R.acc", 19: "R.done", 20: "R.enc"}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    torch.cuda.set_device(0)
    f = C.build_field("c5", precision="bf16")
    o, d = C.query_rays(n, 3)
    read_trace(True)
    f.query_raw(o * 0.9, d)
    ev = read_trace(True)
    if not ev:
        print("no events (not a DDF_TRACE build?)")
        return
    t0 = min(t for t, e, s, r in ev if e == 16)
    last = {}
    for t, e, s, role in ev:
        if t - t0 > 120000:
            break
        dt = t - last.get(role, t)
        last[role] = t
        print(f"{t - t0:8d}  role {role}  {EV.get(e, e):10s} step {s >> 1:2d} slot {s & 1}   (+{dt})")


if __name__ == "__main__":
    main()
