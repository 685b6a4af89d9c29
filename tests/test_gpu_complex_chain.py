"""GPU parity of the complex128 chain, through the C-ABI.

The reference runs every chain in complex128 and starts the transverse-field
Ising family from the complex random_mps (mps.cpp:75-95, chosen by the
automatic initial state at dmrg.cpp:222-235).  With
achi_dmrg_config.arithmetic = ACHI_ARITH_COMPLEX the chain runs that start in
complex128 (planar 4M DMMA contractions, the complex SVD, the real Lanczos on
[Re; Im]); the oracle runs the reference algorithm in complex128
(complex_mode=True).  Bar: per-sweep energies within 1e-10 relative, identical
chi profiles and kept ranks at every visit, identical controller trace.
"""
import numpy as np
import pytest

from paper_2604_03960_b200 import abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2604_03960_b200.api import Context
    c = Context(0)
    yield c
    c.close()


def tfim(n, h):  # acceptance_main.cpp:39-47
    return abi.model_spec(n, family=abi.TRANSVERSE_ISING, jz=1.0, h=h)


def compare_runs(g, o, e_rel=1e-10, s_tol=1e-8, mv_tol=2):
    assert g["n_sweeps"] == o["n_sweeps"]
    for a, b in zip(g["energies"], o["energies"]):
        assert abs(a - b) <= e_rel * abs(b), (a, b)
    assert np.array_equal(g["chi_profiles"], o["chi_profiles"])
    assert np.abs(g["entropy_profiles"] - o["entropy_profiles"]).max(initial=0.0) <= s_tol
    assert [v.kept for v in g["visits"]] == [v.kept for v in o["visits"]]
    assert [(t.chi, t.delta_chi, t.clamped) for t in g["trace"]] == \
        [(t.chi, t.delta_chi, t.clamped) for t in o["trace"]]
    if mv_tol is not None:  # the realified Lanczos takes the reference's steps
        mg = [v.matvecs for v in g["visits"]]
        mo = [v.matvecs for v in o["visits"]]
        assert max(abs(a - b) for a, b in zip(mg, mo)) <= mv_tol


def complex_cfg(cfg):
    cfg.arithmetic = abi.ARITH_COMPLEX
    return cfg


def test_complex_tfim_criterion4_parity(ctx, oracle):  # acceptance_main.cpp:159-174
    spec = tfim(20, 1.0)
    cfg = complex_cfg(abi.adaptive_config(64, 1e-10))
    g = ctx.run_dmrg(spec, cfg)
    o = oracle.run_dmrg(spec, cfg, complex_mode=True)
    compare_runs(g, o)
    epn = g["energy"] / 20
    assert abs(epn + 1.25539) <= 1e-4
    assert abs(epn - oracle.exact_ground_energy(spec) / 20) <= 1e-4


@pytest.mark.parametrize("n,h", [(8, 1.0), (12, 1.0), (10, 0.5)])
def test_complex_tfim_criterion1_parity(ctx, oracle, n, h):  # acceptance_main.cpp:73-104
    spec = tfim(n, h)
    cfg = complex_cfg(abi.fixed_config(1 << (n // 2), eps_conv=1e-11, max_sweeps=16))
    cfg.eig_tol, cfg.eig_max_iter = 1e-12, 400
    g = ctx.run_dmrg(spec, cfg)
    o = oracle.run_dmrg(spec, cfg, complex_mode=True)
    # eig_tol 1e-12 sits at the rounding level of the residual estimate of a
    # converged state: a stop may move by a few steps (energies and ranks do not)
    compare_runs(g, o, mv_tol=None)
    assert abs(g["energy"] - oracle.exact_ground_energy(spec)) <= 1e-8


def test_complex_random_start_xxz(ctx, oracle):
    """ACHI_INIT_RANDOM on the XXZ family selects complex arithmetic by itself."""
    spec = abi.model_spec(14, jz=1.5)
    cfg = abi.adaptive_config(32, 1e-8, max_sweeps=8)
    cfg.initial_state = abi.INIT_RANDOM
    g = ctx.run_dmrg(spec, cfg)
    o = oracle.run_dmrg(spec, cfg, complex_mode=True)
    # a stop of the restarted Lanczos may move by a few steps where the residual
    # estimate crosses eig_tol at rounding level (energies and ranks do not)
    compare_runs(g, o, mv_tol=4)


def test_complex_neel_equals_real_chain(ctx):
    """A real state in complex storage follows the real chain's trajectory."""
    spec = abi.model_spec(20)
    cfg = abi.fixed_config(32, max_sweeps=4)
    r = ctx.run_dmrg(spec, cfg)
    c = ctx.run_dmrg(spec, complex_cfg(abi.fixed_config(32, max_sweeps=4)))
    assert r["n_sweeps"] == c["n_sweeps"]
    assert np.array_equal(r["chi_profiles"], c["chi_profiles"])
    for a, b in zip(r["energies"], c["energies"]):
        assert abs(a - b) <= 1e-12 * abs(b)


def test_complex_sites_snapshot_and_reload(ctx, oracle, tmp_path):
    """Complex sites come back as complex128 (l, d, r) arrays; expectation_energy
    equals the last eigenvalue with nothing truncated; a complex ACHI snapshot
    (mps.cpp:276-315) reloads into a fresh chain, and the same state in a random
    complex gauge reloads through the device canonicalisation."""
    from paper_2604_03960_b200 import outputs
    from paper_2604_03960_b200.api import Chain
    spec = tfim(10, 1.0)
    cfg = complex_cfg(abi.fixed_config(32, max_sweeps=3, eps_conv=1e-16))
    ch = Chain(ctx, spec, cfg)
    assert ch.is_complex
    start = ch.sites()  # the complex random start, canonicalize(psi, 0) on the device
    assert all(s.dtype == np.complex128 for s in start)
    assert max(np.abs(s.imag).max() for s in start) > 1e-3
    assert abs(np.linalg.norm(start[0]) - 1.0) <= 1e-12
    rec = None
    for s in range(3):
        rec = ch.sweep(s)
    e_last = rec["energy"]
    e_state = ch.energy()
    assert abs(e_state - e_last) <= 1e-10 * abs(e_last)
    assert abs(e_state - oracle.exact_ground_energy(spec)) <= 1e-8
    sites = ch.sites()
    for s in sites[1:]:  # right-canonical: sum_{s,r} B B^dagger = 1
        m = s.reshape(s.shape[0], -1)
        assert np.abs(m @ m.conj().T - np.eye(m.shape[0])).max() <= 1e-10
    p = tmp_path / "psi_c.achi"
    outputs.save_mps(sites, p)
    fresh = Chain(ctx, spec, cfg)
    fresh.load_state(outputs.load_mps(p, real=False))
    assert abs(fresh.energy() - e_state) <= 1e-12 * abs(e_state)
    rng = np.random.default_rng(11)
    g = [s.copy() for s in sites]
    for k in range(len(g) - 1):
        chi = g[k].shape[2]
        G = np.eye(chi) + 0.3 * (rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi)))
        g[k] = np.einsum("lsr,rq->lsq", g[k], G)
        g[k + 1] = np.einsum("qr,rsx->qsx", np.linalg.inv(G), g[k + 1])
    other = Chain(ctx, spec, cfg)
    other.load_state(g, canonicalize=True)
    assert abs(other.energy() - e_state) <= 1e-10 * abs(e_state)
    r2 = other.sweep(3)
    assert abs(r2["energy"] - e_last) <= 1e-10 * abs(e_last)
    with pytest.raises(Exception, match="UnsupportedModel"):
        ch.env(0, 1)


def test_complex_chain_growing_chi_stays_variational(ctx):
    """N=60 Heisenberg, PID chi_max=256, 8 sweeps in complex128 (the graph-mode Lanczos at
    every bond while chi grows): sweep energies never rise and end on the real chain's.
    Regression: a cached Lanczos graph once kept a pointer into the context's shared
    reduction scratch, which a later, larger eigensolve reallocated (the graph then wrote
    into freed memory and broke the orthonormality of a kept SVD factor)."""
    spec = abi.model_spec(60, convention=abi.SPIN_HALF)
    cfg = complex_cfg(abi.adaptive_config(256, 1e-10, max_sweeps=8, eps_conv=1e-16))
    g = ctx.run_dmrg(spec, cfg)
    e = g["energies"]
    assert all(b <= a + 1e-10 * abs(a) for a, b in zip(e, e[1:])), e
    r = ctx.run_dmrg(spec, abi.adaptive_config(256, 1e-10, max_sweeps=8, eps_conv=1e-16))
    assert abs(e[-1] - r["energies"][-1]) <= 1e-10 * abs(r["energies"][-1])
