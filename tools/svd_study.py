"""Time the device SVD (inputs resident) for several sizes; print sweeps and ms.

values: achi_svd_batched_device (singular values only); full: achi_svd_device
(U, sigma, V^T).  ACHI_JACOBI_PROF=1 adds the per-round clock64 phase split.
"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
for n in [int(x) for x in (sys.argv[1:] or ["200", "512", "1024", "2048", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    u = torch.empty(n, n, dtype=torch.float64, device="cuda")
    vt = torch.empty(n, n, dtype=torch.float64, device="cuda")
    ref = torch.linalg.svdvals(a)
    for mode in ("values", "full"):
        def run():
            if mode == "values":
                return ctx.svd_batched_device(a.data_ptr(), 1, n, n, s.data_ptr())
            return ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
        run()
        ms = []
        for _ in range(3):
            ctx.timer_start()
            sw = run()
            ms.append(ctx.timer_stop())
        err = float((s - ref).abs().max() / ref[0])
        extra = ""
        if mode == "full":
            extra = f" recon={float(((u * s) @ vt - a).abs().max() / ref[0]):.2e}"
        print(f"n={n} {mode} sweeps={sw} ms={min(ms):.2f} err={err:.2e}{extra}", flush=True)
