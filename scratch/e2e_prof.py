"""Where the c1 protocol call (query_batch, numpy in/out) spends its time."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_16142_b200 import configs as C
from paper_2306_16142_b200 import field as FL

fld = C.build_field("c1")
n = 65536
rng = np.random.default_rng(0)
p = rng.uniform(-1, 1, (n, 3)); d = rng.normal(size=(n, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
for _ in range(5): fld.query_batch(p, d)
torch.cuda.synchronize()
def tm(f, reps=50):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
print("query_batch us", tm(lambda: fld.query_batch(p, d)), flush=True)
print("_rows us", tm(lambda: fld._rows(p, d)))
print("_dev x2 us", tm(lambda: (FL._dev(p), FL._dev(d))))
td = torch.empty(n, dtype=torch.float64, device="cuda")
print("cpu() 1 f64 us", tm(lambda: td.cpu().numpy()))
print("empty x4 us", tm(lambda: [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]))
