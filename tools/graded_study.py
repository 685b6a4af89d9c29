"""Jacobi convergence on graded spectra (sigma log-spaced from 1 to lo) at cluster and
stream sizes; ACHI_JACOBI_CONVLOG=1 prints the stream path's per-sweep measures."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context, AchiError

ctx = Context(0)
for n in (200, 400, 800):
    for lo in (1e-4, 1e-6, 1e-9, 1e-12):
        rng = np.random.default_rng(n)
        qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
        qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
        sv = np.logspace(0, np.log10(lo), n)
        an = (qa * sv) @ qb.T
        a = torch.from_numpy(an).cuda()
        s = torch.empty(n, dtype=torch.float64, device="cuda")
        u = torch.empty(n, n, dtype=torch.float64, device="cuda")
        vt = torch.empty(n, n, dtype=torch.float64, device="cuda")
        try:
            sw = ctx.svd_device(a.data_ptr(), n, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
            ref = np.linalg.svd(an, compute_uv=False)
            print(f"n={n} lo={lo:.0e} sweeps={sw} sigma_err={np.abs(s.cpu().numpy() - ref).max():.2e}", flush=True)
        except AchiError as e:
            print(f"n={n} lo={lo:.0e} FAILED {e}", flush=True)
