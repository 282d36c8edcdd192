"""Event timeline of the 512-wide tcgen05 engine (mlp_umma.cuh mlp_kernel)
for CTA 0: needs a library built with -DDDF_TRACE=1, e.g.

  DDF_NVCC_EXTRA=-DDDF_TRACE=1 DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_trace.so \\
      python -c "from paper_2306_16142_b200 import _lib; _lib.build()"
  DDF_B200_LIB=$PWD/paper_2306_16142_b200/lib/libddf_trace.so python tools/trace_mlp.py [rows]

Runs one forward (query_batch) and one gradient (normal_batch) pass of the
config-4 network and prints, per layer step and N-half, when the MMA issuer
waited for / got the A tile, issued the first and last K chunk, and when the
row warps saw the accumulator and finished the epilogue (cycles from the
tile start)."""

import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_16142_b200 import _lib  # noqa: E402
from paper_2306_16142_b200 import configs as C  # noqa: E402

EV = {8: "I.chunk", 9: "I.wfull", 1: "I.waitA0", 2: "I.gotA0", 3: "I.waitA1", 4: "I.gotA1", 5: "I.waitW", 6: "I.first", 7: "I.last",
      16: "R.tile", 17: "R.waitAcc", 18: "R.acc", 19: "R.done", 20: "R.enc"}


def read_trace(reset=True):
    buf = (ctypes.c_uint64 * 16384)()
    n = _lib.lib().ddf_debug_trace(buf, 16384, int(reset))
    out = []
    for v in list(buf)[:n]:
        tag = v & 0xFFFF
        out.append((v >> 16, tag & 31, (tag >> 5) & 63, (tag >> 11) & 1, tag >> 12))
    return sorted(out)


def show(title, ev):
    if not ev:
        print(title, ": no events (not a DDF_TRACE build?)")
        return
    starts = [e for e in ev if e[1] == 16 and e[4] == 2]
    t0 = starts[0][0] if starts else ev[0][0]
    print(f"== {title}: {len(ev)} events; tile starts at +{[s[0] - t0 for s in starts]}")
    rows = {}
    for t, e, s, h, role in ev:
        key = (s, h)
        rows.setdefault(key, {})
        name = EV.get(e, str(e)) + ("" if role != 3 else "(w9)")
        rows[key].setdefault(name, []).append(t - t0)
    cols = ["I.waitA0", "I.gotA0", "I.waitA1", "I.gotA1", "I.first", "I.last", "R.acc", "R.done", "R.done(w9)"]
    print("step h " + " ".join(f"{c:>11s}" for c in cols) + "   per K chunk: issue/FULL-wait cycles")
    for key in sorted(rows):
        r = rows[key]
        ch = r.get("I.chunk", [])[:8]
        wf = r.get("I.wfull", [])[:8]
        # per chunk: cycles from "weights present" to "issued" (issue blocked on a full MMA queue) /
        # cycles from the previous chunk's issue to "weights present"
        gaps = " ".join(f"{b - a}/{a - p}" for p, a, b in zip([ch[0]] + ch, wf, ch))
        print(f"{key[0]:4d} {key[1]} " + " ".join(
            f"{(str(r[c][0]) if c in r else '-'):>11s}" for c in cols) + "   " + gaps)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
    torch.cuda.set_device(0)
    f = C.build_field("c4", precision="bf16")
    o, d = C.query_rays(n, 3)
    read_trace(True)
    f.query_raw(o, d)
    show("forward (QueryOp)", read_trace(True))
    f.normal_batch(o, d)
    show("gradient (NormalOp)", read_trace(True))


if __name__ == "__main__":
    main()
