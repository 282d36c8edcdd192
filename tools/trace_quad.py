"""Event timeline of the <= 128-wide (quad) tcgen05 engine for CTA 0: needs a
library built with -DDDF_TRACE=1 (see tools/trace_mlp.py for the recipe).

  DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_trace.so python tools/trace_quad.py [rows] [widths]

Prints, per layer step and slot, when the MMA issuer waited for / got the A
tile and finished issuing the layer, and when slot 0's and slot 3's row warps
saw the accumulator and finished the epilogue (cycles from the pack start)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_16142_b200 import _lib  # noqa: E402
from paper_2306_16142_b200.field import CudaNeuralField  # noqa: E402
from paper_2306_16142_b200.neural import kaiming_uniform  # noqa: E402

NSL = 4   # slots per CTA: 4 (quad engine, <= 128 wide) or 2 (ping-pong engine, <= 256 wide); set from the widths


def read_trace(reset=True):
    buf = (ctypes.c_uint64 * 16384)()
    n = _lib.lib().ddf_debug_trace(buf, 16384, int(reset))
    out = []
    for v in list(buf)[:n]:
        tag = v & 0xFFFF
        out.append((v >> 16, tag & 31, (tag >> 5) & 63, tag >> 12))
    return sorted(out)


def show(title, ev):
    if not ev:
        print(title, ": no events (not a DDF_TRACE build?)")
        return
    starts = [e[0] for e in ev if e[1] == 16]
    t0 = min(starts) if starts else ev[0][0]
    print(f"== {title}: {len(ev)} events; pack starts at +{sorted(s - t0 for s in starts)}")
    rows = {}
    for t, e, step, role in ev:
        if e in (16, 20):
            print(f"   slot {step}: {'pack start' if e == 16 else 'encoding stored'} +{t - t0}")
            continue
        rows.setdefault(step, {}).setdefault(e, []).append(t - t0)
    print(" step slot |   I.waitA     I.gotA   I.issued |  R.waitAcc      R.acc     R.done   (epilogue)")
    for key in sorted(rows):
        r = rows[key]
        g = lambda e: r[e] if e in r else []  # noqa: E731
        n = max(len(g(e)) for e in (1, 2, 7, 17, 18, 19))
        for i in range(n):
            c = [(str(g(e)[i]) if i < len(g(e)) else "-") for e in (1, 2, 7, 17, 18, 19)]
            epi = (g(19)[i] - g(18)[i]) if i < len(g(19)) and i < len(g(18)) else ""
            print(f" {key // NSL:4d} {key % NSL:4d} | " + " ".join(f"{x:>10s}" for x in c[:3]) + " | " +
                  " ".join(f"{x:>10s}" for x in c[3:]) + f"   {epi}")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
    widths = eval(sys.argv[2]) if len(sys.argv) > 2 else (5, 128, 128, 128, 128, 1)
    global NSL
    NSL = 4 if max(widths[1:-1]) <= 128 else 2
    torch.cuda.set_device(0)
    f = CudaNeuralField(kaiming_uniform(widths, 2), 10 / 0.98, precision="bf16")
    x = torch.rand(n, widths[0], dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    g = torch.empty(n, widths[0], dtype=torch.float64, device="cuda")
    L = _lib.lib()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    read_trace(True)
    _lib.check(L.ddf_mlp_forward(f.handle, 0, P(x), n, P(y), s))
    torch.cuda.synchronize()
    show("raw forward", read_trace(True))
    _lib.check(L.ddf_mlp_input_grad(f.handle, 0, P(x), n, P(g), s))
    torch.cuda.synchronize()
    show("raw gradient", read_trace(True))


if __name__ == "__main__":
    main()
