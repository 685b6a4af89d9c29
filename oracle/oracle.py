"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle.

Loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, as
the checker / CPU baseline.  The product package never imports this module.
The oracle restates the reference hot path; see adaptchi_oracle.hpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2604_03960_b200 import abi  # struct layouts only (include/adaptchi_b200.h)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")


class OracleError(RuntimeError):
    def __init__(self, code, msg, residual=None):
        super().__init__(f"{abi.ERROR_NAMES.get(code, code)}: {msg}")
        self.code, self.name, self.residual = code, abi.ERROR_NAMES.get(code, str(code)), residual


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _err():
    return C.create_string_buffer(512), 512


def _check(rc, buf, residual=None):
    if rc != 0:
        raise OracleError(rc, buf.value.decode(), residual)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def set_threads(n):
    lib().oracle_set_threads(C.c_int(n))


def run_dmrg(spec, cfg, complex_mode=False, want_state=False):
    """run_dmrg (dmrg.cpp:216-282); returns dict of records/profiles/trace/visits."""
    n, ms = spec.n, cfg.max_sweeps
    res = abi.DmrgResult()
    recs = (abi.SweepRecord * ms)()
    chi = np.zeros(ms * (n - 1), np.int32)
    ent = np.zeros(ms * (n - 1))
    trace = (abi.TraceRow * (ms * 2 * (n - 1)))()
    visits = (abi.VisitRecord * (ms * 2 * (n - 1)))()
    dims = np.zeros(n - 1, np.int32)
    cap = 0
    sites = None
    if want_state:
        cap = 2 * n * max(1, cfg.controller.chi_max) ** 2 * 2 + 64
        sites = np.zeros(cap)
    buf, bl = _err()
    f = lib().oracle_run_dmrg
    f.restype = C.c_int
    rc = f(C.byref(spec), C.byref(cfg), C.c_int(int(complex_mode)), C.byref(res), recs,
           _ip(chi), _dp(ent), trace, visits, _ip(dims),
           _dp(sites) if sites is not None else None, C.c_size_t(cap), buf, C.c_size_t(bl))
    _check(rc, buf)
    ns = res.n_sweeps
    out = dict(
        energy=res.energy, converged=bool(res.converged), max_chi_used=res.max_chi_used,
        max_monotonicity_violation=res.max_monotonicity_violation, n_sweeps=ns,
        records=[recs[i] for i in range(ns)],
        energies=[recs[i].energy for i in range(ns)],
        chi_profiles=chi[: ns * (n - 1)].reshape(ns, n - 1).copy(),
        entropy_profiles=ent[: ns * (n - 1)].reshape(ns, n - 1).copy(),
        trace=[trace[i] for i in range(ns * 2 * (n - 1))],
        visits=[visits[i] for i in range(ns * 2 * (n - 1))],
        bond_dims=dims.copy(),
    )
    if want_state:
        dd = [1] + list(dims) + [1]
        tens, off = [], 0
        for k in range(n):
            sz = dd[k] * 2 * dd[k + 1]
            tens.append(sites[off:off + sz].reshape(dd[k], 2, dd[k + 1]).copy())
            off += sz
        out["sites"] = tens
    return out


def sample_visits(spec, cfg, warm_sweeps, first, count, complex_mode=True):
    secs = C.c_double()
    dims = np.zeros(spec.n - 1, np.int32)
    buf, bl = _err()
    rc = lib().oracle_sample_visits(C.byref(spec), C.byref(cfg), C.c_int(int(complex_mode)),
                                    C.c_int(warm_sweeps), C.c_int(first), C.c_int(count),
                                    C.byref(secs), _ip(dims), buf, C.c_size_t(bl))
    _check(rc, buf)
    return secs.value, dims


class OracleChain:
    """Step-wise oracle run (run_dmrg setup, then one two_site_sweep per call)."""

    def __init__(self, spec, cfg, complex_mode=True):
        self.n = spec.n
        buf, bl = _err()
        f = lib().oracle_chain_create
        f.restype = C.c_void_p
        self.h = f(C.byref(spec), C.byref(cfg), C.c_int(int(complex_mode)), buf, C.c_size_t(bl))
        if not self.h:
            raise OracleError(1, buf.value.decode())

    def sweep(self, index):
        rec = abi.SweepRecord()
        chi = np.zeros(self.n - 1, np.int32)
        buf, bl = _err()
        _check(lib().oracle_chain_sweep(C.c_void_p(self.h), index, C.byref(rec), _ip(chi), buf,
                                        C.c_size_t(bl)), buf)
        return rec, chi

    def close(self):
        if self.h:
            lib().oracle_chain_destroy(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        self.close()


def time_visits_from_state(spec, cfg, sites, states, first, count, complex_mode=True):
    """Seconds and matvec counts of `count` right-moving visits from a given state."""
    dims = np.array([s.shape[2] for s in sites[:-1]], np.int32)
    flat = [np.ascontiguousarray(s, dtype=np.float64) for s in sites]
    ptrs = (C.POINTER(C.c_double) * len(flat))(*[_dp(a) for a in flat])
    st = (abi.BondState * len(states))(*states)
    secs = np.zeros(count)
    mv = np.zeros(count, np.int32)
    buf, bl = _err()
    rc = lib().oracle_time_visits_from_state(C.byref(spec), C.byref(cfg), C.c_int(int(complex_mode)),
                                             _ip(dims), ptrs, st, first, count, _dp(secs), _ip(mv),
                                             buf, C.c_size_t(bl))
    _check(rc, buf)
    return secs, mv


def heff_apply(L, W1, W2, R, theta):
    chl, D1 = L.shape[0], L.shape[1]
    chr_, D3 = R.shape[0], R.shape[1]
    d, D2 = W1.shape[1], W1.shape[3]
    out = np.zeros((chl, d, d, chr_))
    buf, bl = _err()
    args = [np.ascontiguousarray(x, dtype=np.float64) for x in (L, W1, W2, R, theta)]
    rc = lib().oracle_heff_apply(chl, chr_, d, D1, D2, D3, *[_dp(a) for a in args], _dp(out),
                                 buf, C.c_size_t(bl))
    _check(rc, buf)
    return out


def env_update_left(L, A, W):
    chl, Dl = L.shape[0], L.shape[1]
    d, chn, Dr = A.shape[1], A.shape[2], W.shape[3]
    out = np.zeros((chn, Dr, chn))
    buf, bl = _err()
    args = [np.ascontiguousarray(x, dtype=np.float64) for x in (L, A, W)]
    rc = lib().oracle_env_update_left(chl, chn, d, Dl, Dr, *[_dp(a) for a in args], _dp(out),
                                      buf, C.c_size_t(bl))
    _check(rc, buf)
    return out


def env_update_right(R, B, W):
    chr_, Dr = R.shape[0], R.shape[1]
    chn, d, Dl = B.shape[0], B.shape[1], W.shape[0]
    out = np.zeros((chn, Dl, chn))
    buf, bl = _err()
    args = [np.ascontiguousarray(x, dtype=np.float64) for x in (R, B, W)]
    rc = lib().oracle_env_update_right(chr_, chn, d, Dl, Dr, *[_dp(a) for a in args], _dp(out),
                                       buf, C.c_size_t(bl))
    _check(rc, buf)
    return out


def svd(a):
    """svd_full (linalg.cpp:67-70) + fix_phases: returns (u, sigma, vt)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    r = min(m, n)
    s, u, vt = np.zeros(r), np.zeros((m, r)), np.zeros((r, n))
    buf, bl = _err()
    rc = lib().oracle_svd(m, n, _dp(a), _dp(s), _dp(u), _dp(vt), buf, C.c_size_t(bl))
    _check(rc, buf)
    return u, s, vt


def svd_complex_sigma(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    m, n = a.shape
    s = np.zeros(min(m, n))
    inter = a.view(np.float64)
    buf, bl = _err()
    rc = lib().oracle_svd_complex(m, n, _dp(inter), _dp(s), buf, C.c_size_t(bl))
    _check(rc, buf)
    return s


def svd_truncated(a, keep):
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    s = np.zeros(keep)
    deg = C.c_int()
    buf, bl = _err()
    rc = lib().oracle_svd_truncated(m, n, _dp(a), keep, _dp(s), C.byref(deg), buf, C.c_size_t(bl))
    _check(rc, buf)
    return s, bool(deg.value)


def eigs_lowest_dense(h, v0, tol=1e-10, max_iter=200):
    h = np.ascontiguousarray(h, dtype=np.float64)
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    dim = h.shape[0]
    ev, mv, res = C.c_double(), C.c_int(), C.c_double()
    vec = np.zeros(dim)
    buf, bl = _err()
    rc = lib().oracle_eigs_lowest_dense(dim, _dp(h), _dp(v0), C.c_double(tol), max_iter,
                                        C.byref(ev), _dp(vec), C.byref(mv), C.byref(res),
                                        buf, C.c_size_t(bl))
    _check(rc, buf, res.value)
    return ev.value, vec, mv.value, res.value


def _spec_arr(v):
    return np.ascontiguousarray(v, dtype=np.float64)


def entropy(v):
    v = _spec_arr(v)
    out = C.c_double()
    buf, bl = _err()
    _check(lib().oracle_entropy(len(v), _dp(v), C.byref(out), buf, C.c_size_t(bl)), buf)
    return out.value


def truncation_error(v, kept):
    v = _spec_arr(v)
    out = C.c_double()
    buf, bl = _err()
    _check(lib().oracle_truncation_error(len(v), _dp(v), kept, C.byref(out), buf,
                                         C.c_size_t(bl)), buf)
    return out.value


def rank_for_discarded_weight(v, eps):
    v = _spec_arr(v)
    out, margin = C.c_int(), C.c_double()
    buf, bl = _err()
    _check(lib().oracle_rank_for_discarded_weight(len(v), _dp(v), C.c_double(eps), C.byref(out),
                                                  C.byref(margin), buf, C.c_size_t(bl)), buf)
    return out.value, margin.value


def chi_target_direct(s, gamma, chi_min, chi_max):
    out = C.c_int()
    buf, bl = _err()
    _check(lib().oracle_chi_target_direct(C.c_double(s), C.c_double(gamma), chi_min, chi_max,
                                          C.byref(out), buf, C.c_size_t(bl)), buf)
    return out.value


def ema_update(state, s_raw, alpha):
    buf, bl = _err()
    _check(lib().oracle_ema_update(C.byref(state), C.c_double(s_raw), C.c_double(alpha), buf,
                                   C.c_size_t(bl)), buf)


def pid_step(state, s_input, cc):
    row = abi.TraceRow()
    buf, bl = _err()
    _check(lib().oracle_pid_step(C.byref(state), C.c_double(s_input), C.byref(cc), C.byref(row),
                                 buf, C.c_size_t(bl)), buf)
    return row


def predict_entropy(state, beta, order):
    v, fb = C.c_double(), C.c_int()
    lib().oracle_predict_entropy(C.byref(state), C.c_double(beta), order, C.byref(v), C.byref(fb))
    return v.value, bool(fb.value)


def controller_update(state, spectrum, cc):
    v = _spec_arr(spectrum)
    row = abi.TraceRow()
    buf, bl = _err()
    _check(lib().oracle_controller_update(C.byref(state), len(v), _dp(v), C.byref(cc),
                                          C.byref(row), buf, C.c_size_t(bl)), buf)
    return row


def build_mpo(spec, real_gauge=True):
    """All MPO site tensors (left, out, in, right) (models.cpp:49-97)."""
    sites = []
    for k in range(spec.n):
        dims = (C.c_int64 * 4)()
        buf, bl = _err()
        _check(lib().oracle_build_mpo_site(C.byref(spec), int(real_gauge), k, dims, None, buf,
                                           C.c_size_t(bl)), buf)
        shape = tuple(dims)
        size = int(np.prod(shape))
        out = np.zeros(size if real_gauge else 2 * size)
        _check(lib().oracle_build_mpo_site(C.byref(spec), int(real_gauge), k, dims, _dp(out), buf,
                                           C.c_size_t(bl)), buf)
        sites.append(out.reshape(shape) if real_gauge else out.view(np.complex128).reshape(shape))
    return sites


def tfim_free_fermion_energy(n, coupling_j, field_h, convention):
    """tfim_free_fermion_energy (models.cpp:225-239): E0 = -1/2 sum of the
    singular values of M = 2(h I - j L), L the lower shift (open chain)."""
    j, h = coupling_j, field_h
    if convention == abi.SPIN_HALF:
        j, h = j * 0.25, h * 0.5
    m = np.diag(np.full(n, 2.0 * h)) + np.diag(np.full(n - 1, -2.0 * j), -1)
    return -0.5 * float(np.linalg.svd(m, compute_uv=False).sum())


def exact_ground_energy(spec, cap=14):
    """exact_ground_energy (models.cpp:241-259): free fermions for the
    transverse-field Ising family, matrix-free Lanczos for XXZ (n <= cap)."""
    if spec.family == abi.TRANSVERSE_ISING:
        return tfim_free_fermion_energy(spec.n, spec.jz, spec.h, spec.convention)
    out = C.c_double()
    buf, bl = _err()
    _check(lib().oracle_exact_ground_energy(C.byref(spec), cap, C.byref(out), buf,
                                            C.c_size_t(bl)), buf)
    return out.value


def state(**kw):
    s = abi.BondState()
    for k, v in kw.items():
        if k == "history":
            for i, x in enumerate(v):
                s.history[i] = x
        else:
            setattr(s, k, v)
    return s
