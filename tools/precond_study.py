"""Jacobi sweeps of dumped C3 thetas with and without QR preconditioning.

The preconditioner Q (orthogonal) comes from the Householder QR of G^T with
G's rows sorted by norm (host numpy: a study of the convergence effect only);
the GPU Jacobi then runs on G Q, whose column Gram equals R R^T.
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context

ctx = Context(0)


def load(p):
    b = open(p, 'rb').read()
    h = np.frombuffer(b[:24], np.int32)
    a = np.frombuffer(b[24:], np.float64).reshape(h[0], h[1])
    return h, a[:h[2], :h[3]].copy()


def sweeps_of(theta):
    m, n = theta.shape
    a = torch.tensor(theta, device='cuda')
    k = min(m, n)
    s = torch.zeros(k, device='cuda', dtype=torch.float64)
    u = torch.zeros((m, k), device='cuda', dtype=torch.float64)
    vt = torch.zeros((k, n), device='cuda', dtype=torch.float64)
    sw = ctx.svd_device(a.data_ptr(), m, n, s.data_ptr(), u.data_ptr(), vt.data_ptr())
    return sw, s.cpu().numpy()


for f in sys.argv[1:]:
    h, th = load(f)
    right = h[4] == 1
    G = th.T if right else th  # columns to orthogonalise
    order = np.argsort(-np.sum(G * G, 1))
    Q, R = np.linalg.qr(G[order].T, mode='complete')
    Gq = G @ Q
    sw0, s0 = sweeps_of(G.T.copy())   # kRows on G^T == orthogonalise G's columns
    sw1, s1 = sweeps_of(Gq.T.copy())
    print(f, G.shape, "plain", sw0, "precond", sw1, "max dsigma", np.abs(s0 - s1).max() / s0[0])
