"""Jacobi sweeps of the streamed SVD on QR-preconditioned inputs (study for a stream-path
preconditioner): the preconditioner is formed on the host (numpy / scipy), the device
Jacobi runs on theta' whose working matrix is G Q = Pi R^T (G^T Pi = Q R, Pi sorting G's
rows by norm), or on the QRCP variant."""
import sys
import time
import numpy as np
import scipy.linalg as sl
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context

ctx = Context(0)


def sweeps_of(theta):
    m, n = theta.shape
    a = torch.tensor(theta, device='cuda')
    s = torch.zeros(min(m, n), device='cuda', dtype=torch.float64)
    ctx.timer_start()
    sw = ctx.svd_batched_device(a.data_ptr(), 1, m, n, s.data_ptr())
    ms = ctx.timer_stop()
    return sw, ms, s.cpu().numpy()


for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]:
    for kind in ("gauss", "graded"):
        rng = np.random.default_rng(1234)
        if kind == "gauss":
            A = rng.standard_normal((n, n))
        else:
            qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
            qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
            A = (qa * np.logspace(0, -9, n)) @ qb.T
        sw0, ms0, s0 = sweeps_of(A)
        G = A.T  # rows side for a square matrix: G = theta^T
        t = time.time()
        order = np.argsort(-np.sum(G * G, 1))
        Q, R = np.linalg.qr(G[order].T)
        th1 = (G @ Q).T
        t1 = time.time() - t
        sw1, ms1, s1 = sweeps_of(th1)
        t = time.time()
        Q2, R2, P2 = sl.qr(G.T, pivoting=True)  # G^T P = Q R (column pivoting of G^T)
        th2 = (G @ Q2).T
        t2 = time.time() - t
        sw2, ms2, s2 = sweeps_of(th2)
        print(f"n={n} {kind}: plain {sw0} sweeps {ms0:.1f} ms | QR sorted rows {sw1} sweeps {ms1:.1f} ms "
              f"(host QR {t1:.1f} s) | QRCP {sw2} sweeps {ms2:.1f} ms; sigma diff "
              f"{np.abs(s1 - s0).max() / s0[0]:.1e} {np.abs(s2 - s0).max() / s0[0]:.1e}", flush=True)
