"""Stream-path SVD with the accumulated factor recovered by GEMM (SvdWs::vrecover,
svd_jacobi.cu v_recover) against the oracle's svd_full (linalg.cpp:67-70: gesdd +
fix_phases), across the three regimes of the recovery:

* every value >= 1e-3 sigma_1: V = G0^T G Sigma^-2 with the first-order correction only;
* a tail in [1e-5, 1e-3) sigma_1: projected off the accurate columns, Newton-Schulz;
* values below 1e-5 sigma_1 (ill-conditioned, rank-deficient): decomposed again with V
  accumulated (the fallback), and strongly graded spectra converge within the stream
  path's sweep cap.

Bars: sigma within 1e-11 sigma_1 (north_star), U and V orthonormal to 1e-10 on the
resolved part (test_linalg.cpp:25-34), reconstruction 1e-10 relative, fix_phases signs.
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


def graded(m, n, lo, seed, rank=None):
    rng = np.random.default_rng(seed)
    k = min(m, n)
    qa, _ = np.linalg.qr(rng.standard_normal((m, k)))
    qb, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s = np.logspace(0, np.log10(lo), k)
    if rank is not None:
        s[rank:] = 0.0
    return (qa * s) @ qb.T


def check(ctx, oracle, a, resolved=1e-8, orth=1e-10):
    u, s, vt, _ = ctx.svd_full(a)
    _, so, _ = oracle.svd(a)
    k = min(a.shape)
    assert np.abs(s - so).max() <= 1e-11 * so[0]
    big = s > resolved * s[0]
    nb = int(big.sum())
    assert np.abs(u[:, big].T @ u[:, big] - np.eye(nb)).max() <= orth
    assert np.abs(vt[big] @ vt[big].T - np.eye(nb)).max() <= orth
    assert np.linalg.norm(a - (u * s) @ vt) / np.linalg.norm(a) <= 1e-10
    assert np.all(np.diff(s) <= 0)
    for j in range(k):
        if s[j] > 0:
            i = int(np.argmax(np.abs(u[:, j])))
            assert u[i, j] > 0
    return u, s, vt


@pytest.mark.parametrize("shape", [(1024, 1024), (700, 1300), (1300, 700), (520, 520)])
def test_gaussian_recovered(ctx, oracle, shape):
    """Well-conditioned inputs: the recovered factor is orthonormal to ~1e-12."""
    a = np.random.default_rng(shape[0] + 3 * shape[1]).standard_normal(shape)
    u, s, vt = check(ctx, oracle, a)
    # the recovered factor (U for m <= n, the rows side; V otherwise) is orthonormal to ~1e-12
    rec = u if shape[0] <= shape[1] else vt.T
    assert np.abs(rec.T @ rec - np.eye(rec.shape[1])).max() <= 5e-12


@pytest.mark.parametrize("lo", [3e-4, 2e-5])
def test_tail_projected(ctx, oracle, lo):
    """Values between 1e-5 and 1e-3 sigma_1: the tail projection + Newton-Schulz keep both
    factors orthonormal across the whole spectrum."""
    a = graded(640, 640, lo, 11)
    u, s, vt = check(ctx, oracle, a, resolved=0.0)
    assert np.abs(u.T @ u - np.eye(640)).max() <= 5e-12  # the recovered factor (rows side)


@pytest.mark.parametrize("lo,rank", [(1e-7, None), (1e-3, 500)])
def test_fallback_accumulates(ctx, oracle, lo, rank):
    """Below 1e-5 sigma_1 (ill-conditioned or rank-deficient) the decomposition is redone
    with V accumulated: same bars as the accumulated path."""
    a = graded(600, 600, lo, 12, rank)
    # the normalised-column factor of values far below sigma_1 carries the Jacobi's residual
    # cosines (the stop test weights them by sqrt(sigma_c / ||G||_F)): 1e-10 from 1e-6 sigma_1
    check(ctx, oracle, a, resolved=1e-6)


def test_strongly_graded_converges(ctx, oracle):
    """sigma over 12 decades at 800 x 800 (the stream path converges linearly for a long
    stretch there; its sweep cap is 100)."""
    a = graded(800, 800, 1e-12, 13)
    check(ctx, oracle, a, resolved=1e-6)


@pytest.mark.parametrize("shape,lo,rank", [((2048, 2048), 1e-4, 900), ((4096, 2048), 1e-1, None)])
def test_stream_rowsplit_deterministic(ctx, oracle, shape, lo, rank):
    """Row-split pairs (2048^2: four CTAs per block pair) with tracked diagonal Grams in the
    cross rounds: every CTA of a pair must rotate its rows with the same J.  The tracked
    blocks are read before the pair's partial-Gram exchange (svd_jacobi.cu, jacobi_stream
    kernel), after which CTA 0 overwrites them; a late read would mix two rounds.  The
    kernel's sums run in a fixed order, so repeated decompositions are bit-identical."""
    a = graded(shape[0], shape[1], lo, 21, rank)
    u0, s0, vt0 = check(ctx, oracle, a, resolved=1e-6)
    for _ in range(4):
        u, s, vt, _ = ctx.svd_full(a)
        assert np.array_equal(s, s0) and np.array_equal(u, u0) and np.array_equal(vt, vt0)


def test_chain_chi1024_stream_svds(ctx):
    """The bench's in-sweep H_eff chain (bench.py heff_insweep): N=100 Heisenberg, fixed
    chi=1024 from the Neel state through sweep 5 -- 2048 x 2048 theta SVDs on the stream
    path, many of them rank-deficient.  Energies stay variational and decrease."""
    from paper_2604_03960_b200 import abi
    from paper_2604_03960_b200.api import Chain
    ctx.set_lanczos_graph(0)
    ch = Chain(ctx, abi.model_spec(100, convention=abi.SPIN_HALF), abi.fixed_config(1024, max_sweeps=6))
    try:
        es = []
        for s in range(6):
            r = ch.sweep(s)
            es.append(r["energy"] / 100)
        assert int(r["chi_profile"].max()) == 1024
    finally:
        ch.close()
        ctx.set_lanczos_graph(-1)
    assert all(np.isfinite(es))
    assert all(b <= a + 1e-12 for a, b in zip(es, es[1:]))
    assert -0.4432 < es[-1] < -0.4412  # N=100 OBC ground state -0.44127739861..., Bethe limit -0.44315
