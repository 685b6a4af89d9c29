"""First-call vs steady cost of the cluster SVD per cluster size (npairs = ng/32)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context

ctx = Context(0)
rng = np.random.default_rng(0)
order = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5, 6, 7, 8]
for k in order:
    n = 32 * k
    a = torch.tensor(rng.standard_normal((n, n)), device='cuda')
    s = torch.zeros(n, device='cuda', dtype=torch.float64)
    u = torch.zeros((n, n), device='cuda', dtype=torch.float64)
    vt = torch.zeros((n, n), device='cuda', dtype=torch.float64)
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"npairs {k} n {n}: " + " ".join(f"{x:.2f}" for x in ts) + " ms", flush=True)
