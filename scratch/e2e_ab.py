"""Same-process A/B of the protocol call's input staging: one pinned
buffer for both inputs (_dev_pair) vs pin_memory() per input (_dev)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C
from paper_2306_16142_b200 import field as FL

fld = C.build_field("c1")
n = 65536
rng = np.random.default_rng(0)
p = rng.uniform(-1, 1, (n, 3)); d = rng.normal(size=(n, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
packed = FL._dev_pair
separate = lambda a, b, device="cuda": (FL._dev(a, device=device), FL._dev(b, device=device))
def tm(reps=100):
    for _ in range(5): fld.query_raw(p, d)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fld.query_raw(p, d)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
for r in range(3):
    for name, fn in (("separate", separate), ("packed", packed)):
        FL._dev_pair = fn
        print(name, round(tm(), 1), "us per query_raw", flush=True)
