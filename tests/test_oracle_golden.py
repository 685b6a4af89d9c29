"""Pin the CPU oracle against the reference's own known answers (CPU only).

Every expected value below is taken from the reference test suite or
acceptance criteria (file:line under /root/reference/proj) so that the oracle
used as the GPU parity checker is itself anchored to the reference.
"""
import math

import numpy as np
import pytest

from paper_2604_03960_b200 import abi


def dense_from_mpo(ws):
    """Dense matrix of an MPO (models.cpp:111-138 dense_mpo_matrix)."""
    acc = ws[0]  # (1, O, I, w)
    for w in ws[1:]:
        t = np.einsum("aoiw,wpjv->aopijv", acc, w)
        a, o, p, i, j, v = t.shape
        acc = t.reshape(a, o * p, i * j, v)
    return acc[0, :, :, 0]


# ---------------- linalg (test_linalg.cpp) ----------------

def test_svd_identity_phase_convention(oracle):  # test_linalg.cpp:38-46
    u, s, vt = oracle.svd(np.eye(2))
    assert np.allclose(s, [1, 1], atol=1e-12)
    assert np.abs(u - np.eye(2)).max() <= 1e-12
    assert np.abs(vt - np.eye(2)).max() <= 1e-12


def test_svd_diag(oracle):  # test_linalg.cpp:48-55
    _, s, _ = oracle.svd(np.diag([3.0, 2.0]))
    assert abs(s[0] - 3) <= 3e-13 and abs(s[1] - 2) <= 2e-13


@pytest.mark.parametrize("shape", [(8, 8), (6, 3), (3, 6), (1, 5), (5, 1), (12, 9)])
def test_svd_invariants(oracle, shape):  # test_linalg.cpp:25-82
    rng = np.random.default_rng(sum(shape))
    m = rng.standard_normal(shape)
    u, s, vt = oracle.svd(m)
    k = min(shape)
    assert len(s) == k
    assert np.abs(u.T @ u - np.eye(k)).max() <= 1e-10
    assert np.abs(vt @ vt.T - np.eye(k)).max() <= 1e-10
    assert np.all(np.diff(s) <= 0) and s.min() >= 0
    assert np.linalg.norm(m - (u * s) @ vt) / np.linalg.norm(m) <= 1e-10
    assert abs((s**2).sum() - (m**2).sum()) <= 1e-10 * (m**2).sum()
    # fix_phases: the first largest-|u| entry of each column is positive
    for j in range(k):
        i = int(np.argmax(np.abs(u[:, j])))
        assert u[i, j] > 0


def test_svd_determinism_and_bad_input(oracle):  # test_linalg.cpp:84-96
    m = np.random.default_rng(5).standard_normal((10, 10))
    a, b = oracle.svd(m), oracle.svd(m)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
    bad = np.zeros((2, 2))
    bad[0, 0] = np.nan
    with pytest.raises(Exception, match="InvalidMatrix"):
        oracle.svd(bad)


def test_svd_truncated(oracle):  # test_linalg.cpp:98-144
    s, deg = oracle.svd_truncated(np.diag([3.0, 2.0, 1.0]), 2)
    assert np.allclose(s, [3, 2])
    assert oracle.svd_truncated(np.diag([2.0, 1.0, 1.0]), 2)[1] is True
    assert oracle.svd_truncated(np.diag([2.0, 1.0, 1.0]), 1)[1] is False
    for keep in (0, 5):
        with pytest.raises(Exception, match="InvalidRank"):
            oracle.svd_truncated(np.random.default_rng(1).standard_normal((4, 4)), keep)


def test_eigs_known_answers(oracle):  # test_linalg.cpp:170-193
    ev, vec, _, _ = oracle.eigs_lowest_dense(np.diag([-1.0, 0.0, 1.0]), np.ones(3), 1e-12, 100)
    assert abs(ev + 1) <= 1e-10 and abs(abs(vec[0]) - 1) <= 1e-8
    assert abs(np.linalg.norm(vec) - 1) <= 1e-12
    h = np.zeros((4, 4))
    h[0, 0] = h[3, 3] = 0.25
    h[1, 1] = h[2, 2] = -0.25
    h[1, 2] = h[2, 1] = 0.5
    ev, *_ = oracle.eigs_lowest_dense(h, np.random.default_rng(0).standard_normal(4), 1e-12, 100)
    assert abs(ev + 0.75) <= 1e-10


def test_eigs_dense_64(oracle):  # test_linalg.cpp:195-206
    rng = np.random.default_rng(777)
    a = rng.standard_normal((64, 64))
    h = 0.5 * (a + a.T)
    ev, vec, _, _ = oracle.eigs_lowest_dense(h, rng.standard_normal(64), 1e-11, 400)
    assert abs(ev - np.linalg.eigvalsh(h)[0]) <= 1e-9
    assert np.linalg.norm(h @ vec - ev * vec) <= 1e-11 * max(1, abs(ev))


def test_eigs_nonconvergence_and_zero_start(oracle):  # test_linalg.cpp:208-226
    rng = np.random.default_rng(12)
    a = rng.standard_normal((32, 32))
    h = 0.5 * (a + a.T)
    with pytest.raises(Exception) as ei:
        oracle.eigs_lowest_dense(h, np.ones(32), 1e-14, 3)
    assert ei.value.name == "EigenNonConvergence"
    assert math.isfinite(ei.value.residual) and ei.value.residual > 0
    with pytest.raises(Exception, match="InvalidMatrix"):
        oracle.eigs_lowest_dense(np.eye(4), np.zeros(4), 1e-10, 10)


# ---------------- mps (test_mps.cpp) ----------------

def test_entropy_examples(oracle):  # test_mps.cpp:76-93
    assert oracle.entropy([1.0]) == 0.0
    assert abs(oracle.entropy([math.sqrt(0.5)] * 2) - math.log(2)) <= 1e-12
    assert abs(oracle.entropy([math.sqrt(0.9), math.sqrt(0.1)]) - 0.3250829733914482) <= 1e-12
    assert oracle.entropy([1.0, 1e-15]) == 0.0
    with pytest.raises(Exception, match="DegenerateSpectrum"):
        oracle.entropy([0.0, 0.0])


def test_entropy_bound(oracle):  # test_mps.cpp:95-107
    rng = np.random.default_rng(5)
    for _ in range(50):
        v = np.sort(rng.uniform(size=1 + int(rng.uniform() * 20)))[::-1]
        assert oracle.entropy(v) <= math.log(len(v)) + 1e-12


def test_truncation_error(oracle):  # test_mps.cpp:109-121
    sp = [math.sqrt(0.8), math.sqrt(0.2)]
    assert oracle.truncation_error(sp, 2) == 0.0
    assert abs(oracle.truncation_error(sp, 1) - 0.4472135954999579) <= 1e-12
    for bad in (0, 3):
        with pytest.raises(Exception, match="InvalidRank"):
            oracle.truncation_error(sp, bad)
    big = [0.9, 0.5, 0.3, 0.1, 0.01]
    for k in range(1, 5):
        assert oracle.truncation_error(big, k + 1) <= oracle.truncation_error(big, k) + 1e-15


# ---------------- controller (test_controller.cpp) ----------------

def test_chi_target_direct(oracle):  # test_controller.cpp:85-90
    assert oracle.chi_target_direct(math.log(4), 1.0, 1, 1024) == 4
    assert oracle.chi_target_direct(math.log(4), 1.5, 1, 1024) == 6
    assert oracle.chi_target_direct(10.0, 1.0, 1, 256) == 256
    assert oracle.chi_target_direct(0.0, 1.0, 2, 64) == 2


def test_pid_hand_example(oracle):  # test_controller.cpp:92-110
    cc = abi.controller_config(kp=2.0, ki=0.1, kd=0.5, s_target=0.0, chi_min=1, chi_max=1024)
    st = oracle.state(chi=10, initialized=1, prev_error=0.5, integral=0.0)
    row = oracle.pid_step(st, 0.5, cc)
    assert abs(row.p_term - 1.0) < 1e-12 and abs(st.integral - 0.05) < 1e-12
    assert row.d_term == 0.0 and row.delta_chi == 1 and st.chi == 11 and not row.clamped


def test_pid_antiwindup_and_scales(oracle):  # test_controller.cpp:112-174
    cc = abi.controller_config(s_target=0.8, chi_min=1)
    st = oracle.state(chi=7, initialized=1)
    oracle.pid_step(st, 0.8, cc)
    assert st.chi == 7
    cc = abi.controller_config(kp=2.0, ki=0.1, kd=0.5, s_target=0.0, chi_min=1, chi_max=16)
    st = oracle.state(chi=16, initialized=1, prev_error=1.0)
    row = oracle.pid_step(st, 1.0, cc)
    assert st.chi == 16 and row.clamped and st.integral == 0.0
    cc = abi.controller_config(kp=2.0, ki=0.1, kd=0.5, s_target=0.0, chi_min=1, chi_max=32)
    st = oracle.state(chi=32, initialized=1)
    for _ in range(100):
        oracle.pid_step(st, 0.9, cc)
    assert abs(st.integral) <= 0.1 * 0.9 + 1e-12
    cc = abi.controller_config(kp=2.0, ki=0.0, kd=0.0, s_target=0.0, chi_min=1, chi_max=4096,
                               pid_scale=abi.PID_MULTIPLICATIVE)
    st = oracle.state(chi=100, initialized=1)
    oracle.pid_step(st, 1.0, cc)
    assert st.chi == 120


def test_predict_entropy(oracle):  # test_controller.cpp:176-215
    st = oracle.state(ema=0.5, history=[0.4, 0.5], history_len=2)
    v, fb = oracle.predict_entropy(st, 1.0, abi.PREDICT_LINEAR)
    assert not fb and abs(v - 0.6) <= 1e-14
    v, _ = oracle.predict_entropy(st, 0.0, abi.PREDICT_LINEAR)
    assert v == 0.5
    q = oracle.state(ema=0.5, history=[0.5, 0.5, 0.5], history_len=3)
    assert abs(oracle.predict_entropy(q, 0.8, abi.PREDICT_QUADRATIC)[0] - 0.5) <= 1e-14
    f = oracle.state(ema=0.42, history=[0.42], history_len=1)
    assert oracle.predict_entropy(f, 1.0, abi.PREDICT_LINEAR) == (0.42, True)
    assert oracle.predict_entropy(f, 1.0, abi.PREDICT_QUADRATIC)[1]
    fl = oracle.state(ema=0.1, history=[0.9, 0.1], history_len=2)
    assert oracle.predict_entropy(fl, 2.0, abi.PREDICT_LINEAR)[0] == 0.0


def test_rank_for_discarded_weight(oracle):  # test_controller.cpp:217-225
    v = [0.9, 0.4, 0.1, 0.01]
    got = [oracle.rank_for_discarded_weight(v, e)[0] for e in (1e-6, 1e-3, 0.05, 0.5)]
    assert got == [4, 3, 2, 1]


def test_controller_mode_dispatch(oracle):  # test_controller.cpp:227-275
    cc = abi.controller_config(chi_min=1, chi_max=64, mode=abi.MODE_FIXED)
    st = oracle.state()
    for _ in range(5):
        assert oracle.controller_update(st, [0.9, 0.3, 0.01], cc).chi == 64
    cc = abi.controller_config(chi_min=1, chi_max=64, mode=abi.MODE_DIRECT, gamma_margin=1.0,
                               alpha_ema=0.5, predictor_order=abi.PREDICT_OFF)
    st = oracle.state()
    for _ in range(60):
        chi = oracle.controller_update(st, [math.sqrt(0.5)] * 2, cc).chi
    assert chi == 2
    cc = abi.controller_config(chi_min=1, chi_max=64, mode=abi.MODE_THRESHOLD, eps_trunc=1e-6)
    assert oracle.controller_update(oracle.state(), [1.0, 1e-2, 1e-9], cc).chi == 2
    cc = abi.controller_config(chi_min=1, chi_max=64, mode=abi.MODE_PID, alpha_ema=1.0,
                               predictor_order=abi.PREDICT_OFF, s_target=math.log(2))
    st = oracle.state(chi=8, initialized=1)
    last = [oracle.controller_update(st, [math.sqrt(0.5)] * 2, cc).chi for _ in range(40)]
    assert all(abs(x - last[29]) <= 1 for x in last[30:])


def test_controller_clamp_containment(oracle):  # test_controller.cpp:277-295
    rng = np.random.default_rng(8)
    cc = abi.controller_config(mode=abi.MODE_PID, chi_min=3, chi_max=17, s_target=1.0)
    st = oracle.state(chi=5, initialized=1)
    for _ in range(300):
        v = np.sort(rng.uniform(0, 2.5, 6) + 1e-6)[::-1]
        chi = oracle.controller_update(st, v, cc).chi
        assert 3 <= chi <= 17


def test_beta_zero_bit_equality(oracle):  # test_controller.cpp:297-317
    w = abi.controller_config(mode=abi.MODE_PID, s_target=0.4, predictor_order=abi.PREDICT_LINEAR,
                              beta_predict=0.0)
    wo = abi.controller_config(mode=abi.MODE_PID, s_target=0.4, predictor_order=abi.PREDICT_OFF)
    a, b = oracle.state(chi=4, initialized=1), oracle.state(chi=4, initialized=1)
    rng = np.random.default_rng(3)
    for _ in range(50):
        x = rng.uniform(0.1, 1.4)
        ra = oracle.controller_update(a, [1.0, x, x * x], w)
        rb = oracle.controller_update(b, [1.0, x, x * x], wo)
        assert ra.chi == rb.chi and ra.error == rb.error


# ---------------- models (test_models.cpp) ----------------

@pytest.mark.parametrize("n", [2, 4, 6])
def test_real_gauge_mpo_equals_reference_mpo(oracle, n):  # SURVEY.md §9 probe
    spec = abi.model_spec(n, jz=1.3, h=0.4)
    hr = dense_from_mpo(oracle.build_mpo(spec, real_gauge=True))
    hc = dense_from_mpo(oracle.build_mpo(spec, real_gauge=False))
    assert np.abs(hc.imag).max() == 0.0
    assert np.abs(hr - hc.real).max() <= 1e-15


def test_mpo_bond_dims(oracle):  # test_models.cpp:45-52
    w = oracle.build_mpo(abi.model_spec(4))
    assert w[0].shape == (1, 2, 2, 5) and w[1].shape == (5, 2, 2, 5) and w[3].shape == (5, 2, 2, 1)
    t = oracle.build_mpo(abi.model_spec(4, family=abi.TRANSVERSE_ISING, h=0.5))
    assert t[1].shape == (3, 2, 2, 3)


def test_singlet_and_ed(oracle):  # test_models.cpp:39-43,98-108
    h = dense_from_mpo(oracle.build_mpo(abi.model_spec(2, convention=abi.SPIN_HALF)))
    assert abs(np.linalg.eigvalsh(h)[0] + 0.75) <= 1e-12
    spec = abi.model_spec(8, jz=0.7, h=0.3)
    ed = oracle.exact_ground_energy(spec)
    dense = np.linalg.eigvalsh(dense_from_mpo(oracle.build_mpo(spec)))[0]
    assert abs(ed - dense) <= 1e-9


def test_heff_matches_dense_n2(oracle):  # test_dmrg.cpp:64-82
    spec = abi.model_spec(2, convention=abi.SPIN_HALF)
    w = oracle.build_mpo(spec)
    h = dense_from_mpo(w)
    one = np.ones((1, 1, 1))
    theta = np.random.default_rng(2).standard_normal((1, 2, 2, 1))
    out = oracle.heff_apply(one, w[0], w[1], one, theta)
    assert np.abs(out.ravel() - h @ theta.ravel()).max() <= 1e-12


# ---------------- dmrg (test_dmrg.cpp, acceptance) ----------------

def test_n2_singlet(oracle):  # test_dmrg.cpp:111-115
    r = oracle.run_dmrg(abi.model_spec(2, convention=abi.SPIN_HALF), abi.fixed_config(4))
    assert abs(r["energy"] + 0.75) <= 1e-9 * 0.75


def test_n8_fixed_vs_ed(oracle):  # test_dmrg.cpp:117-126
    spec = abi.model_spec(8)
    r = oracle.run_dmrg(spec, abi.fixed_config(16, eps_conv=1e-10))
    assert r["converged"] and r["n_sweeps"] <= 5
    assert abs(r["energy"] - oracle.exact_ground_energy(spec)) <= 1e-8


def test_monotone_fixed(oracle):  # test_dmrg.cpp:128-134
    r = oracle.run_dmrg(abi.model_spec(10), abi.fixed_config(24))
    e = r["energies"]
    assert all(e[s] <= e[s - 1] + 1e-10 for s in range(1, len(e)))
    assert r["max_monotonicity_violation"] <= 1e-10


def test_variational_and_adaptive_monotonicity(oracle):  # test_dmrg.cpp:136-149
    spec = abi.model_spec(8)
    exact = oracle.exact_ground_energy(spec)
    r = oracle.run_dmrg(spec, abi.adaptive_config(32))
    assert all(e >= exact - 1e-9 for e in r["energies"])
    r = oracle.run_dmrg(abi.model_spec(12), abi.adaptive_config(32, 1e-9))
    assert r["converged"] and r["max_monotonicity_violation"] <= 1e-6 * abs(r["energy"])


def test_strategy_equivalence_at_capacity(oracle):  # test_dmrg.cpp:179-186
    spec = abi.model_spec(8)
    f = oracle.run_dmrg(spec, abi.fixed_config(12))
    pinned = abi.adaptive_config(12)
    pinned.controller.chi_min = 12
    a = oracle.run_dmrg(spec, pinned)
    assert abs(f["energy"] - a["energy"]) <= 1e-10


def test_trace_rows(oracle):  # test_dmrg.cpp:270-279
    cfg = abi.adaptive_config(16, max_sweeps=3, eps_conv=1e-16)
    r = oracle.run_dmrg(abi.model_spec(6), cfg)
    assert r["n_sweeps"] == 3 and len(r["trace"]) == 3 * 2 * 5


def test_real_gauge_run_equals_complex_reference(oracle):  # C1, SURVEY.md §8d
    spec = abi.model_spec(20)
    cfg = abi.fixed_config(32, max_sweeps=5)
    r = oracle.run_dmrg(spec, cfg)
    c = oracle.run_dmrg(spec, cfg, complex_mode=True)
    assert r["n_sweeps"] == c["n_sweeps"]
    assert np.array_equal(r["chi_profiles"], c["chi_profiles"])
    for a, b in zip(r["energies"], c["energies"]):
        assert abs(a - b) <= 1e-12 * abs(b)
    # exact N=20 Pauli E/N: C1's fixed chi=32 sits 1.7e-10 weight off it
    assert abs(r["energy"] / 20 + 1.736494666879792) <= 1e-8


def test_acceptance_criterion_2(oracle):  # acceptance_main.cpp:106-126
    spec = abi.model_spec(20)
    f = oracle.run_dmrg(spec, abi.fixed_config(64))
    p = oracle.run_dmrg(spec, abi.adaptive_config(64, 1e-5))
    assert abs(f["energy"] / 20 + 1.73649) <= 2e-4
    assert abs(f["energy"] / 20 + 1.736494666879792) <= 1e-9
    assert abs(p["energy"] / 20 - f["energy"] / 20) <= 1e-4
    assert p["records"][-1].average_chi <= 10.0 and p["max_chi_used"] <= 14
    assert f["converged"] and p["converged"]


def tfim(n, h):  # acceptance_main.cpp:39-47
    return abi.model_spec(n, family=abi.TRANSVERSE_ISING, jz=1.0, h=h)


def test_tfim_free_fermion_small_n(oracle):  # models.cpp:225-239 vs ED of the dense MPO
    for n, h in [(4, 1.0), (6, 0.2), (8, 0.7)]:
        spec = tfim(n, h)
        hd = dense_from_mpo(oracle.build_mpo(spec))
        assert abs(np.linalg.eigvalsh(hd)[0] - oracle.exact_ground_energy(spec)) <= 1e-10


def test_acceptance_criterion_1_tfim_rows(oracle):  # acceptance_main.cpp:73-104 (Ising rows)
    for n in (4, 6, 8, 10, 12):
        for h in (1.0, 0.2):
            spec = tfim(n, h)
            cfg = abi.fixed_config(1 << (n // 2), eps_conv=1e-11, max_sweeps=16)
            cfg.eig_tol, cfg.eig_max_iter = 1e-12, 400
            r = oracle.run_dmrg(spec, cfg)  # automatic init -> random real on the real path
            assert abs(r["energy"] - oracle.exact_ground_energy(spec)) <= 1e-8


def test_acceptance_criterion_4(oracle):  # acceptance_main.cpp:159-174
    spec = tfim(20, 1.0)
    r = oracle.run_dmrg(spec, abi.adaptive_config(64, 1e-10))
    epn = r["energy"] / 20
    assert abs(epn + 1.25539) <= 1e-4
    assert abs(epn - oracle.exact_ground_energy(spec) / 20) <= 1e-4


def test_random_real_init_real_equals_complex_mode(oracle):
    """ACHI_INIT_RANDOM_REAL: the real-gauge run and the complex128 run of the
    same real random start agree (energies 1e-12 rel, identical chi profiles)."""
    spec = tfim(20, 1.0)
    cfg = abi.adaptive_config(64, 1e-10)
    cfg.initial_state = abi.INIT_RANDOM_REAL
    r = oracle.run_dmrg(spec, cfg)
    c = oracle.run_dmrg(spec, cfg, complex_mode=True)
    assert r["n_sweeps"] == c["n_sweeps"]
    assert np.array_equal(r["chi_profiles"], c["chi_profiles"])
    for a, b in zip(r["energies"], c["energies"]):
        assert abs(a - b) <= 1e-12 * abs(b)
    cfg.initial_state = abi.INIT_RANDOM  # complex random_mps needs complex arithmetic
    with pytest.raises(Exception, match="UnsupportedModel"):
        oracle.run_dmrg(spec, cfg)


def test_acceptance_criteria_3_6_7(oracle):  # acceptance_main.cpp:130-157,206-273 (energies, sweeps)
    for spec, cap in [(abi.model_spec(20), 1e-4), (tfim(20, 1.0), 1e-8), (tfim(20, 0.2), 1e-8),
                      (abi.model_spec(20, jz=1.5), 1e-4)]:
        f = oracle.run_dmrg(spec, abi.fixed_config(64))
        a = oracle.run_dmrg(spec, abi.adaptive_config(64, 1e-10))
        assert f["converged"] and a["converged"] and abs(a["energy"] - f["energy"]) / 20 <= cap
    for spec, eps in [(abi.model_spec(20), 1e-5), (tfim(20, 1.0), 1e-10)]:
        ref = oracle.run_dmrg(spec, abi.adaptive_config(64, eps))
        for scale in (0.5, 0.75, 1.25, 1.5):
            cfg = abi.adaptive_config(64, eps)
            cfg.controller.kp *= scale
            cfg.controller.ki *= scale
            cfg.controller.kd *= scale
            r = oracle.run_dmrg(spec, cfg)
            assert abs(r["energy"] - ref["energy"]) / 20 <= 1e-4 and r["n_sweeps"] == ref["n_sweeps"]
        b0 = abi.adaptive_config(64, eps)
        b0.controller.beta_predict = 0.0
        r0 = oracle.run_dmrg(spec, b0)
        for beta in (0.4, 0.8):
            cfg = abi.adaptive_config(64, eps)
            cfg.controller.beta_predict = beta
            r = oracle.run_dmrg(spec, cfg)
            assert abs(r["energy"] - r0["energy"]) <= 1e-8 and r["n_sweeps"] == r0["n_sweeps"]
