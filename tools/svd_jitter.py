"""Run-to-run spread of the device SVD at a C3-like shape (cluster path)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 218
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = torch.Generator(device="cuda").manual_seed(7)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
s = torch.empty(n, dtype=torch.float64, device="cuda")
u = torch.empty(n, n, dtype=torch.float64, device="cuda")
vt = torch.empty(n, n, dtype=torch.float64, device="cuda")
ms = []
for i in range(reps):
    ctx.timer_start()
    sw = ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
    ms.append(ctx.timer_stop())
ms = np.array(ms[5:])
print(f"n={n} sweeps={sw} ms min {ms.min():.3f} p50 {np.median(ms):.3f} p90 {np.percentile(ms, 90):.3f} max {ms.max():.3f}")
