"""V recovery study (SvdWs::vrecover): time and accuracy of achi_svd_device with the
accumulated factor recovered by GEMM against ACHI_SVD_VRECOVER=0 (run the script once
per setting).  Cases: random square n x n (the chi=2048 metric is n = 4096), wide and
tall shapes, a spectrum with a tail between 1e-5 and 1e-3 sigma_1 (tail projection + Newton-
Schulz) and one reaching below 1e-5 sigma_1 (the fallback)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context

ctx = Context(0)
tag = os.environ.get("ACHI_SVD_VRECOVER", "1")


def graded(m, n, lo, seed):
    rng = np.random.default_rng(seed)
    k = min(m, n)
    qa, _ = np.linalg.qr(rng.standard_normal((m, k)))
    qb, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s = np.logspace(0, np.log10(lo), k)
    return (qa * s) @ qb.T


cases = []
for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096"])]:
    cases.append((f"gauss{n}", np.random.default_rng(1234).standard_normal((n, n))))
cases.append(("wide600x1100", np.random.default_rng(7).standard_normal((600, 1100))))
cases.append(("tall1100x600", np.random.default_rng(8).standard_normal((1100, 600))))
cases.append(("tail1e-4_800", graded(800, 800, 1e-4, 3)))
cases.append(("illcond1e-9_800", graded(800, 800, 1e-9, 4)))
for name, an in cases:
    m, n = an.shape
    k = min(m, n)
    a = torch.from_numpy(an).cuda()
    s = torch.empty(k, dtype=torch.float64, device="cuda")
    u = torch.empty(m, k, dtype=torch.float64, device="cuda")
    vt = torch.empty(k, n, dtype=torch.float64, device="cuda")
    ref = np.linalg.svd(an, compute_uv=False) if max(m, n) <= 2048 else None
    ctx.svd_device(a.data_ptr(), m, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
    ms = []
    for _ in range(3):
        ctx.flush_l2(256 << 20)
        ctx.timer_start()
        sw = ctx.svd_device(a.data_ptr(), m, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
        ms.append(ctx.timer_stop())
    eye = torch.eye(k, dtype=torch.float64, device="cuda")
    ou = float((u.T @ u - eye).abs().max())
    ov = float((vt @ vt.T - eye).abs().max())
    rec = float(((u * s) @ vt - a).abs().max() / s[0])
    serr = float(np.abs(s.cpu().numpy() - ref).max() / ref[0]) if ref is not None else float("nan")
    print(f"[vrec={tag}] {name} sweeps={sw} ms={sorted(ms)[1]:.2f} sigma_err={serr:.2e} "
          f"orthU={ou:.2e} orthV={ov:.2e} recon={rec:.2e}", flush=True)
