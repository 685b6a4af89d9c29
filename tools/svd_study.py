"""Time the device SVD (inputs resident) for several sizes; print sweeps and ms."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
for n in [int(x) for x in (sys.argv[1:] or ["200", "512", "1024", "2048", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.svd_batched_device(a.data_ptr(), 1, n, n, s.data_ptr())
    ms = []
    for _ in range(3):
        ctx.timer_start()
        sw = ctx.svd_batched_device(a.data_ptr(), 1, n, n, s.data_ptr())
        ms.append(ctx.timer_stop())
    ref = torch.linalg.svdvals(a)
    err = float((s - ref).abs().max() / ref[0])
    print(f"n={n} sweeps={sw} ms={min(ms):.2f} err={err:.2e}", flush=True)
