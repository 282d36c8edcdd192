import sys, numpy as np
sys.path.insert(0, '.')
from oracle import cpu_ddf as O
from paper_2306_16142_b200.field import CudaNeuralField
from paper_2306_16142_b200.neural import kaiming_uniform

def bf(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)

def emu(m, x):
    ws = [w.astype(np.float32) for w in O.Net(m.widths, m.v, m.g, m.b).effective()]
    bs = [b.astype(np.float32) for b in m.b]
    L = len(ws)
    a = bf(x); masks = []
    for l in range(L - 1):
        z = a @ bf(ws[l]).T + bs[l]
        masks.append(z > 0)
        r = np.maximum(z, 0)
        a = bf(r)
    y = r @ ws[L-1][0] + bs[L-1][0]
    G = bf(ws[L-1][0][None, :] * masks[L-2])
    for l in range(L - 2, 0, -1):
        D = G @ bf(ws[l])
        G = bf(D * masks[l-1])
    g = G @ bf(ws[0])
    return y, g

def run(widths, n=1024):
    m = kaiming_uniform(widths, 3)
    f = CudaNeuralField(m, 1.0, precision="bf16")
    x = np.random.default_rng(1).uniform(-1, 1, (n, widths[0]))
    y = f.forward_inputs(x); g = f.input_gradient_inputs(x)
    ye, ge = emu(m, x)
    ry = np.abs(y - ye) / np.sqrt(np.mean(ye**2)); rg = np.abs(g - ge).max(1) / np.sqrt(np.mean(ge**2))
    on = O.Net(m.widths, m.v, m.g, m.b)
    gt = O.mlp_input_grad(on, x); yt = O.mlp_forward(on, x)
    rt = np.abs(ge - gt).max(1) / np.sqrt(np.mean(gt**2))
    print(f"{str(widths[:3]):18s} L={len(widths)-1} kernel-vs-emu fwd max {ry.max():.2e} grad med {np.median(rg):.2e} p99 {np.percentile(rg,99):.2e} max {rg.max():.2e} | emu-vs-f64 grad med {np.median(rt):.3f} fwd max {(np.abs(ye-yt)/np.sqrt(np.mean(yt**2))).max():.3f}")
    if ry.max() > 0.05:
        bad = np.argsort(-ry)[:5]; print("   worst rows", bad, y[bad], ye[bad])
for w in [(5,64,64,1), (5,128,128,128,128,1), (5,)+(256,)*8+(1,), (65,)+(256,)*6+(1,), (65,100,200,1), (65,128,256,1), (65,64,64,1), (65,)+(512,)*8+(1,)]:
    run(w)
