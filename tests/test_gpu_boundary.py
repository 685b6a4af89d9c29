"""GPU tests of the boundary entry points added for the reference's complex and
operator-callback interfaces (through the C-ABI):

* achi_svd_complex: svd_full on a complex DenseMatrix (linalg.cpp:11-48,
  67-70; DenseMatrix = MatrixXcd, tensor.hpp:15) against the oracle's LAPACK
  zgesdd; sigma within 1e-11 sigma_1, U / V^dagger unitary, reconstruction,
  the fix_phases convention (linalg.cpp:19-35), complex multiplets, rank
  deficiency, real-valued complex input, non-finite input (InvalidMatrix).
* achi_eigs_lowest_callback: eigs_lowest(LinearMap, ...) (linalg.hpp:64-78)
  with a host operator; the reference's known answers (test_linalg.cpp) and
  the dense-operator path.
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


def crandn(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def check_csvd(a, u, s, vd, s_ref=None):
    m, n = a.shape
    r = min(m, n)
    assert u.shape == (m, r) and s.shape == (r,) and vd.shape == (r, n)
    assert np.all(np.diff(s) <= 1e-14 * s[0])
    if s_ref is not None:
        assert np.abs(s - s_ref).max() <= 1e-11 * s_ref[0], np.abs(s - s_ref).max() / s_ref[0]
    # values at the rounding-noise floor (64 sqrt(m) eps ||A||_F, svd_jacobi.cu zero_floor_kernel)
    # carry no orthonormal completion on the normalised-column side, as on the real path
    nz = s > 1e-10 * s[0]
    k = int(nz.sum())
    assert np.abs(u[:, :k].conj().T @ u[:, :k] - np.eye(k)).max() <= 1e-10
    assert np.abs(vd[:k] @ vd[:k].conj().T - np.eye(k)).max() <= 1e-10
    assert np.linalg.norm(u @ np.diag(s) @ vd - a) <= 1e-12 * max(1.0, np.linalg.norm(a)) * np.sqrt(r)
    # fix_phases: the first largest-|u| entry of each column is real and positive
    for q in range(k):
        col = np.abs(u[:, q])
        i = int(np.flatnonzero(col == col.max())[0])
        assert abs(u[i, q].imag) <= 1e-15 * col.max() and u[i, q].real > 0


@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (3, 5), (8, 8), (12, 9), (9, 12), (64, 64),
                                   (100, 37), (37, 100), (130, 96), (200, 260), (300, 300)])
def test_svd_complex_matches_zgesdd(ctx, oracle, shape):
    rng = np.random.default_rng(sum(shape) + 7)
    a = crandn(rng, shape)
    u, s, vd = ctx.svd_complex(a)
    check_csvd(a, u, s, vd, oracle.svd_complex_sigma(a))


def unitary(rng, n):
    q, r = np.linalg.qr(crandn(rng, (n, n)))
    return q * (np.diag(r) / np.abs(np.diag(r)))


@pytest.mark.parametrize("m,n", [(40, 40), (48, 30), (30, 48)])
def test_svd_complex_multiplets_and_rank_deficiency(ctx, oracle, m, n):
    """Exact complex multiplets (the SU(2) multiplets of DMRG spectra) go through the
    complex Gram-Schmidt of svd_complex.cu; exact zeros through the zero run."""
    rng = np.random.default_rng(m * n)
    r = min(m, n)
    vals = np.array([3.0] * 3 + [2.0] * 4 + [1.5] + [1.0] * 2 + list(np.linspace(0.9, 0.1, r - 14))
                    + [0.0] * 4)
    assert vals.size == r
    a = unitary(rng, m)[:, :r] @ np.diag(vals) @ unitary(rng, n)[:r]
    u, s, vd = ctx.svd_complex(a)
    assert np.abs(s - np.sort(vals)[::-1]).max() <= 1e-12 * 3.0
    check_csvd(a, u, s, vd, oracle.svd_complex_sigma(a))


def test_svd_complex_real_input_equals_real_path(ctx):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((50, 70))
    _, s_c, _ = ctx.svd_complex(a.astype(np.complex128))
    _, s_r, _, _ = ctx.svd_full(a)
    assert np.abs(s_c - s_r).max() <= 1e-12 * s_r[0]


def test_svd_complex_rejects_nonfinite(ctx):
    a = np.ones((4, 4), np.complex128)
    a[1, 2] = complex(0.0, np.nan)
    with pytest.raises(Exception, match="InvalidMatrix"):
        ctx.svd_complex(a)


def test_eigs_callback_known_answers(ctx):  # test_linalg.cpp:182-206
    h = np.array([[2.0, -1.0], [-1.0, 2.0]])
    ev, vec, mv, res = ctx.eigs_lowest(lambda x: h @ x, np.array([1.0, 0.3]))
    assert abs(ev - 1.0) <= 1e-10 and res <= 1e-10
    rng = np.random.default_rng(5)
    a = rng.standard_normal((64, 64))
    hs = 0.5 * (a + a.T)
    ev, vec, mv, res = ctx.eigs_lowest(lambda x: hs @ x, np.ones(64), 1e-10, 400)
    w = np.linalg.eigvalsh(hs)
    assert abs(ev - w[0]) <= 1e-9 * max(1.0, abs(w[0]))
    assert np.linalg.norm(hs @ vec - ev * vec) <= 1e-9 * max(1.0, abs(ev))
    ev_d, vec_d, mv_d, res_d = ctx.eigs_lowest_dense(hs, np.ones(64), 1e-10, 400)
    assert abs(ev - ev_d) <= 1e-12 * max(1.0, abs(ev)) and mv == mv_d


def test_eigs_callback_errors(ctx):
    with pytest.raises(Exception, match="InvalidMatrix"):
        ctx.eigs_lowest(lambda x: x, np.zeros(4))
    with pytest.raises(Exception, match="InvalidMatrix"):
        ctx.eigs_lowest(lambda x: x * np.nan, np.ones(4))
    rng = np.random.default_rng(12)
    a = rng.standard_normal((32, 32))
    h = 0.5 * (a + a.T)
    with pytest.raises(Exception) as ei:
        ctx.eigs_lowest(lambda x: h @ x, np.ones(32), 1e-14, 3)
    assert ei.value.name == "EigenNonConvergence" and ei.value.residual > 0


@pytest.mark.parametrize("n,lo", [(32, -17), (64, -16), (48, -20), (40, -8)])
def test_svd_complex_graded_spectrum(ctx, n, lo):
    """DMRG-like exponentially graded spectra down past the noise floor: the
    orthonormal factor (U for a square matrix) stays unitary across the whole
    spectrum -- the tail and the noise subspace are orthonormalised together by
    the complex Gram-Schmidt of svd_complex.cu; the lone pairs above them carry
    the Jacobi vectors' own ~1e-11 accuracy on such spectra -- and U S V^dagger
    reproduces A."""
    rng = np.random.default_rng(n - lo)
    s = np.logspace(0, lo, n)
    a = unitary(rng, n) @ np.diag(s) @ unitary(rng, n)
    u, sg, vd = ctx.svd_complex(a)
    assert np.abs(u.conj().T @ u - np.eye(n)).max() <= 1e-10
    assert np.linalg.norm(u @ np.diag(sg) @ vd - a) <= 1e-12
    big = s > 1e-10
    assert np.abs(sg[big] - s[big]).max() <= 1e-13
