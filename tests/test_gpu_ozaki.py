"""Emulated-FP64 GEMM on the int8 tensor cores (Ozaki scheme, tcgen05.mma kind::i8;
SURVEY.md §8 f5) against an exact-enough FP64 reference.

Error model: with s 7-bit digits per entry, every product keeps the digit pairs
p + q <= s + 1, so |C - AB| <= ~ (s + 2) 2^(-7s) (|A| |B|) elementwise (digit
truncation) plus FP64 rounding of the final sum; the reference is numpy's FP64
matmul, itself within ~K eps |A||B|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2604_03960_b200.api import Context
    c = Context(0)
    yield c
    c.close()


def run(ctx, a, b, s, a_trans=False, b_kmajor=False):
    import torch
    M, K = (a.shape[1], a.shape[0]) if a_trans else a.shape
    N = b.shape[0] if b_kmajor else b.shape[1]
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dc = torch.empty(M, N, dtype=torch.float64, device="cuda")
    ctx.dgemm_ozaki_device(M, N, K, da.data_ptr(), a.shape[1], db.data_ptr(), b.shape[1], dc.data_ptr(), N,
                           s, a_trans, b_kmajor)
    ctx.synchronize()  # the call is queued on the library stream
    return dc.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(128, 64, 128), (128, 64, 1), (200, 130, 257), (512, 384, 1024),
                                   (1000, 600, 1300)])
def test_ozaki_fp64_level(ctx, M, N, K):
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)) * np.exp(rng.uniform(-3, 3, (M, 1)))  # rows of different scales
    b = rng.standard_normal((K, N))
    c = run(ctx, a, b, 8)
    bound = np.abs(a) @ np.abs(b)
    if M * N * K <= 3e8:  # extended-precision reference (x86 long double, 64-bit mantissa)
        ref = (a.astype(np.longdouble) @ b.astype(np.longdouble)).astype(np.float64)
        tol = 2e-15
    else:  # FP64 reference: its own rounding is within ~K eps of the product
        ref = a @ b
        tol = 2e-15 + K * 1.2e-16
    err = np.max(np.abs(c - ref) / bound)
    assert err <= tol, err


def test_ozaki_layouts_and_digits(ctx):
    rng = np.random.default_rng(9)
    M, N, K = 300, 200, 700
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N))
    ref = (a.astype(np.longdouble) @ b.astype(np.longdouble)).astype(np.float64)
    bound = np.abs(a) @ np.abs(b)
    for at in (False, True):
        for bk in (False, True):
            c = run(ctx, np.ascontiguousarray(a.T) if at else a, np.ascontiguousarray(b.T) if bk else b, 8,
                    at, bk)
            assert np.max(np.abs(c - ref) / bound) <= 2e-15
    prev = None
    for s in (3, 4, 5, 6, 7, 8):  # the error falls by ~2^-7 per digit
        err = np.max(np.abs(run(ctx, a, b, s) - ref) / bound)
        assert err <= (s + 2) * 2.0 ** (-7 * s) * 4 + 1e-15, (s, err)
        if prev is not None and prev > 1e-13:
            assert err < prev / 16
        prev = err


def test_ozaki_rejects(ctx):
    with pytest.raises(Exception, match="InvalidConfig"):
        run(ctx, np.ones((4, 4)), np.ones((4, 4)), 1)
