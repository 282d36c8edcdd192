"""numpy -> device: pinned staging (torch pin_memory) vs direct pageable copy."""
import time
import numpy as np, torch
n = 65536
a = np.random.default_rng(0).uniform(-1, 1, (n, 3)); b = a.copy()
def tm(f, reps=50):
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
pin = lambda x: torch.from_numpy(x).pin_memory().to("cuda", non_blocking=True)
direct = lambda x: torch.from_numpy(x).to("cuda")
def packed():
    h = torch.empty((2, n, 3), dtype=torch.float64, pin_memory=True)
    hn = h.numpy(); hn[0] = a; hn[1] = b
    return h.to("cuda", non_blocking=True)
print("pinned x2 us", tm(lambda: (pin(a), pin(b))))
print("direct x2 us", tm(lambda: (direct(a), direct(b))))
print("packed pinned us", tm(packed))
