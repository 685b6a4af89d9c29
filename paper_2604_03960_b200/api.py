"""Python front-end over the C-ABI (include/adaptchi_b200.h).

Names follow the reference API (proj/include/adaptchi/*.hpp): ``run_dmrg``,
``two_site_sweep`` (Chain.sweep), ``apply_effective_hamiltonian``,
``Environment.update_left/update_right``, ``svd_full``, ``eigs_lowest``,
``controller_update``.  Errors are raised as :class:`AchiError` carrying the
reference exception name (errors.hpp:8-59).  Every call runs on the GPU; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi


class AchiError(RuntimeError):
    def __init__(self, code, msg, residual=None):
        self.code = code
        self.name = abi.ERROR_NAMES.get(code, str(code))
        self.residual = residual
        super().__init__(f"{self.name}: {msg}")


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One device + one CUDA stream (achi_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = abi.load()
        self.h = C.c_void_p()
        rc = self.lib.achi_ctx_create(device, C.byref(self.h))
        if rc != 0:
            raise AchiError(rc, f"achi_ctx_create(device={device}) failed")

    def close(self):
        """Destroy the context; chains created on it are closed first."""
        if self.h:
            for ch in list(getattr(self, "_chains", ())):
                ch.close()
            self.lib.achi_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            buf = C.create_string_buffer(1024)
            self.lib.achi_last_error(self.h, buf, 1024)
            raise AchiError(rc, buf.value.decode(), self.lib.achi_last_residual(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.achi_launch_count(self.h))

    def synchronize(self):
        self._check(self.lib.achi_synchronize(self.h))

    def timer_start(self):
        self._check(self.lib.achi_timer_start(self.h))

    def timer_stop(self) -> float:
        """Device milliseconds since timer_start (CUDA events on the context stream)."""
        ms = C.c_double()
        self._check(self.lib.achi_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def device_times(self, enable=None, reset=False):
        """Per-phase CUDA-event device time: dict phase -> (ms, work, launches).
        enable: None (unchanged), False / True, or n > 1: a chain times one bond visit in n
        (timing events cost device time; the totals then cover the sampled visits)."""
        names = ("matvec", "svd", "env", "heff")
        n = len(names)
        out = np.zeros(3 * n)
        e = -1 if enable is None else int(enable)
        self._check(self.lib.achi_device_times_ex(self.h, e, int(bool(reset)), _dp(out), n))
        return {k: dict(ms=out[i], work=out[n + i], launches=int(out[2 * n + i]))
                for i, k in enumerate(names)}

    def svd_batched_device(self, d_a_ptr, batch, m, n, d_sigma_ptr):
        """Device-pointer batched SVD (inputs resident in HBM); returns Jacobi sweeps."""
        sw = C.c_int()
        self._check(self.lib.achi_svd_batched_device(self.h, batch, m, n, C.c_void_p(d_a_ptr),
                                                     C.c_void_p(d_sigma_ptr), C.byref(sw)))
        return sw.value

    def svd_device(self, d_a_ptr, m, n, d_sigma_ptr, d_u_ptr, d_vt_ptr):
        """Device-pointer svd_full with U and V^T (row-major); returns Jacobi sweeps."""
        sw = C.c_int()
        self._check(self.lib.achi_svd_device(self.h, m, n, C.c_void_p(d_a_ptr), C.c_void_p(d_sigma_ptr),
                                             C.c_void_p(d_u_ptr), C.c_void_p(d_vt_ptr), C.byref(sw)))
        return sw.value

    def set_lanczos_graph(self, mode):
        """1: Lanczos inner loop as a conditional CUDA graph (default); 0: stepped
        from the host (every kernel visible to ncu and to the per-matvec H_eff
        accounting, phase "heff" of device_times); -1: process default."""
        self._check(self.lib.achi_ctx_set_lanczos_graph(self.h, int(mode)))

    def flush_l2(self, nbytes=256 << 20):
        self._check(self.lib.achi_flush_l2(self.h, C.c_size_t(nbytes)))

    def set_grid_cap(self, max_ctas):
        """Cap this context's cooperative-kernel grids (0 = none): for several
        contexts sharing one GPU."""
        self._check(self.lib.achi_ctx_set_grid_cap(self.h, int(max_ctas)))

    # ---- local kernels (host buffers) ----
    def apply_effective_hamiltonian(self, L, W1, W2, R, theta):
        """dmrg.cpp:58-71; L (chl,D1,chl), W (D,d,d,D'), R (chr,D3,chr), theta (chl,d,d,chr)."""
        L, W1, W2, R, theta = map(_f64, (L, W1, W2, R, theta))
        chl, D1 = L.shape[0], L.shape[1]
        chr_, D3 = R.shape[0], R.shape[1]
        d, D2 = W1.shape[1], W1.shape[3]
        out = np.zeros((chl, d, d, chr_))
        self._check(self.lib.achi_heff_apply(self.h, chl, chr_, d, D1, D2, D3, _dp(L), _dp(W1),
                                             _dp(W2), _dp(R), _dp(theta), _dp(out)))
        return out

    def env_update_left(self, L, A, W):
        """Environment::update_left (dmrg.cpp:26-37)."""
        L, A, W = map(_f64, (L, A, W))
        chl, Dl = L.shape[0], L.shape[1]
        d, chn, Dr = A.shape[1], A.shape[2], W.shape[3]
        out = np.zeros((chn, Dr, chn))
        self._check(self.lib.achi_env_update_left(self.h, chl, chn, d, Dl, Dr, _dp(L), _dp(A),
                                                  _dp(W), _dp(out)))
        return out

    def env_update_right(self, R, B, W):
        """Environment::update_right (dmrg.cpp:39-49)."""
        R, B, W = map(_f64, (R, B, W))
        chr_, Dr = R.shape[0], R.shape[1]
        chn, d, Dl = B.shape[0], B.shape[1], W.shape[0]
        out = np.zeros((chn, Dl, chn))
        self._check(self.lib.achi_env_update_right(self.h, chr_, chn, d, Dl, Dr, _dp(R), _dp(B),
                                                   _dp(W), _dp(out)))
        return out

    def svd_full(self, a, out=None):
        """linalg.cpp:67-70 on the GPU Jacobi kernel: returns (u, sigma, vt, sweeps).

        out: optional caller-owned (u, sigma, vt) C-contiguous float64 arrays of
        shapes (m, k), (k,), (k, n) (e.g. pinned host memory) written in place."""
        a = _f64(a)
        m, n = a.shape
        k = min(m, n)
        if out is None:
            s, u, vt = np.zeros(k), np.zeros((m, k)), np.zeros((k, n))
        else:
            u, s, vt = out
            for arr, shp in ((u, (m, k)), (s, (k,)), (vt, (k, n))):
                if arr.dtype != np.float64 or arr.shape != shp or not arr.flags.c_contiguous:
                    raise ValueError(f"svd_full: out array must be C-contiguous float64 {shp}")
        sw = C.c_int()
        self._check(self.lib.achi_svd(self.h, m, n, _dp(a), _dp(s), _dp(u), _dp(vt), C.byref(sw)))
        return u, s, vt, sw.value

    def svd_complex(self, a):
        """Complex svd_full (linalg.cpp:67-70 on a MatrixXcd): returns (u, sigma, vdag)
        with A = u diag(sigma) vdag, fix_phases applied."""
        a = np.ascontiguousarray(a, dtype=np.complex128)
        if a.ndim != 2:
            raise AchiError(2, "svd: expected a matrix")
        m, n = a.shape
        r = min(m, n)
        s = np.zeros(r)
        u = np.zeros((m, r), np.complex128)
        vd = np.zeros((r, n), np.complex128)
        sw = C.c_int()
        self._check(self.lib.achi_svd_complex(self.h, m, n, a.view(np.float64).ctypes.data_as(
            C.POINTER(C.c_double)), _dp(s), u.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
            vd.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), C.byref(sw)))
        return u, s, vd

    def svd_complex_device(self, d_a_ptr, m, n, d_sigma_ptr, d_u_ptr, d_vdag_ptr):
        """Device-pointer complex svd_full (interleaved complex128); returns Jacobi sweeps."""
        sw = C.c_int()
        self._check(self.lib.achi_svd_complex_device(self.h, m, n, C.c_void_p(d_a_ptr),
                                                     C.c_void_p(d_sigma_ptr), C.c_void_p(d_u_ptr),
                                                     C.c_void_p(d_vdag_ptr), C.byref(sw)))
        return sw.value

    def svd_batched(self, a):
        a = _f64(a)
        b, m, n = a.shape
        s = np.zeros((b, min(m, n)))
        self._check(self.lib.achi_svd_batched(self.h, b, m, n, _dp(a), _dp(s)))
        return s

    def bond_select(self, cfg, sigma, state, sweep=0, bond=0):
        """Fused entropy / floor-rank / kept / controller_update kernel on one spectrum."""
        s = _f64(sigma)
        row, visit = abi.TraceRow(), abi.VisitRecord()
        self._check(self.lib.achi_bond_select(self.h, C.byref(cfg), len(s), _dp(s), C.byref(state),
                                              sweep, bond, C.byref(row), C.byref(visit)))
        return row, visit

    def spectrum_stats(self, sigma, kept=1, eps=0.0):
        """(entropy, truncation_error(kept), rank_for_discarded_weight(eps), significant)."""
        s = _f64(sigma)
        out = np.zeros(4)
        self._check(self.lib.achi_spectrum_stats(self.h, len(s), _dp(s), int(kept),
                                                 C.c_double(eps), _dp(out)))
        return float(out[0]), float(out[1]), int(out[2]), int(out[3])

    def eigs_lowest_dense(self, h, v0, tol=1e-10, max_iter=200):
        h, v0 = _f64(h), _f64(v0)
        dim = h.shape[0]
        ev, mv, res = C.c_double(), C.c_int(), C.c_double()
        vec = np.zeros(dim)
        self._check(self.lib.achi_eigs_lowest_dense(self.h, dim, _dp(h), _dp(v0), C.c_double(tol),
                                                    max_iter, C.byref(ev), _dp(vec), C.byref(mv),
                                                    C.byref(res)))
        return ev.value, vec, mv.value, res.value

    def eigs_lowest(self, matvec, v0, tol=1e-10, max_iter=200):
        """eigs_lowest(LinearMap, dim, v0, tol, max_iter) (linalg.hpp:64-78) with a host
        operator: matvec(x) -> H x for a real symmetric H (numpy in, numpy out).  The
        Lanczos runs on the device; each matvec round-trips through the host.
        Returns (eigenvalue, eigenvector, matvec_count, residual)."""
        v0 = _f64(v0).ravel()
        dim = v0.size
        err = []

        def cb(_user, pin, pout, n):
            try:
                x = np.ctypeslib.as_array(pin, shape=(n,)).copy()
                y = np.asarray(matvec(x), dtype=np.float64).ravel()
                np.ctypeslib.as_array(pout, shape=(n,))[:] = y
            except Exception as e:  # noqa: BLE001 - surfaced after the call
                err.append(e)
                np.ctypeslib.as_array(pout, shape=(n,))[:] = np.nan
        fn = abi.MATVEC_FN(cb)
        ev, mv, res = C.c_double(), C.c_int(), C.c_double()
        vec = np.zeros(dim)
        rc = self.lib.achi_eigs_lowest_callback(self.h, dim, fn, None, _dp(v0), tol, max_iter,
                                                C.byref(ev), _dp(vec), C.byref(mv), C.byref(res))
        if err:
            raise err[0]
        self._check(rc)
        return ev.value, vec, mv.value, res.value

    def dgemm_ozaki_device(self, M, N, K, d_a, lda, d_b, ldb, d_c, ldc, slices=8, a_trans=False,
                           b_kmajor=False):
        """Emulated-FP64 GEMM on the int8 tensor cores (device pointers): C = A B."""
        self._check(self.lib.achi_dgemm_ozaki_device(self.h, M, N, K, C.c_void_p(d_a), lda,
                                                     int(a_trans), C.c_void_p(d_b), ldb, int(b_kmajor),
                                                     C.c_void_p(d_c), ldc, int(slices)))

    def set_ozaki(self, slices, min_flops=1e9):
        """Emulated-FP64 contractions on the int8 tensor cores for GEMMs of at least
        min_flops (0 slices: off, the native DMMA engine)."""
        self._check(self.lib.achi_ctx_set_ozaki(self.h, int(slices), float(min_flops)))

    def dgemm_device(self, M, N, K, d_a, lda, d_b, ldb, d_c, ldc, a_kmajor=True, b_kmajor=False):
        """The DMMA GEMM engine on device pointers (queued, no sync): C = A B."""
        self._check(self.lib.achi_dgemm_device(self.h, M, N, K, int(a_kmajor), C.c_void_p(d_a), lda,
                                               int(b_kmajor), C.c_void_p(d_b), ldb, C.c_void_p(d_c), ldc))

    def dgemm(self, a, b, a_kmajor=True, b_kmajor=False):
        """C = A @ B on the TMA/DMMA engine.  a: (M,K) if a_kmajor else (K,M) stored;
        b: (N,K) if b_kmajor else (K,N) stored."""
        a, b = _f64(a), _f64(b)
        M, K = (a.shape[0], a.shape[1]) if a_kmajor else (a.shape[1], a.shape[0])
        N = b.shape[0] if b_kmajor else b.shape[1]
        c = np.zeros((M, N + (N & 1)))
        self._check(self.lib.achi_dgemm(self.h, M, N, K, int(a_kmajor), _dp(a), a.shape[1],
                                        int(b_kmajor), _dp(b), b.shape[1], _dp(c), c.shape[1]))
        return c[:, :N]

    # ---- DMRG ----
    def chain(self, spec, cfg) -> "Chain":
        return Chain(self, spec, cfg)

    def run_dmrg(self, spec, cfg):
        """run_dmrg (dmrg.cpp:216-282) on a device-resident chain."""
        ch = Chain(self, spec, cfg)
        try:
            return ch.run()
        finally:
            ch.close()


class Chain:
    """Device-resident MPS + environments + controller states (achi_chain)."""

    def __init__(self, ctx: Context, spec, cfg):
        self.ctx, self.spec, self.cfg = ctx, spec, cfg
        self.n = spec.n
        self.h = C.c_void_p()
        if not ctx.h:
            raise AchiError(21, "context is closed")
        ctx._check(ctx.lib.achi_chain_create(ctx.h, C.byref(spec), C.byref(cfg), C.byref(self.h)))
        if not hasattr(ctx, "_chains"):
            import weakref
            ctx._chains = weakref.WeakSet()
        ctx._chains.add(self)

    def close(self):
        if self.h and self.ctx.h:
            self.ctx.lib.achi_chain_destroy(self.h)
        self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sweep(self, index):
        """two_site_sweep (dmrg.cpp:175-214)."""
        n = self.n
        rec = abi.SweepRecord()
        chi = np.zeros(n - 1, np.int32)
        ent = np.zeros(n - 1)
        trace = (abi.TraceRow * (2 * (n - 1)))()
        visits = (abi.VisitRecord * (2 * (n - 1)))()
        self.ctx._check(self.ctx.lib.achi_chain_sweep(self.h, index, C.byref(rec), _ip(chi), _dp(ent),
                                                      trace, visits))
        return dict(record=rec, energy=rec.energy, chi_profile=chi, entropy_profile=ent,
                    trace=list(trace), visits=list(visits))

    def run(self):
        n, ms = self.n, self.cfg.max_sweeps
        res = abi.DmrgResult()
        recs = (abi.SweepRecord * ms)()
        chi = np.zeros(ms * (n - 1), np.int32)
        ent = np.zeros(ms * (n - 1))
        trace = (abi.TraceRow * (ms * 2 * (n - 1)))()
        visits = (abi.VisitRecord * (ms * 2 * (n - 1)))()
        self.ctx._check(self.ctx.lib.achi_chain_run(self.h, C.byref(res), recs, _ip(chi), _dp(ent),
                                                    trace, visits))
        ns = res.n_sweeps
        return dict(
            energy=res.energy, converged=bool(res.converged), max_chi_used=res.max_chi_used,
            max_monotonicity_violation=res.max_monotonicity_violation, n_sweeps=ns,
            records=[recs[i] for i in range(ns)], energies=[recs[i].energy for i in range(ns)],
            chi_profiles=chi[: ns * (n - 1)].reshape(ns, n - 1).copy(),
            entropy_profiles=ent[: ns * (n - 1)].reshape(ns, n - 1).copy(),
            trace=[trace[i] for i in range(ns * 2 * (n - 1))],
            visits=[visits[i] for i in range(ns * 2 * (n - 1))],
            bond_dims=self.bond_dims())

    def stats(self, profile=None):
        """Phase wall-clock split since creation; profile=True syncs per visit."""
        out = np.zeros(8)
        p = -1 if profile is None else int(bool(profile))
        if p < 0:
            p = 0
        self.ctx.lib.achi_chain_stats(self.h, p, _dp(out))
        keys = ("lanczos_s", "svd_s", "select_s", "absorb_env_s", "matvecs", "svd_sweeps", "visits")
        return dict(zip(keys, out[:7].tolist()))

    def bond_dims(self):
        d = np.zeros(self.n - 1, np.int32)
        self.ctx.lib.achi_chain_bond_dims(self.h, _ip(d))
        return d

    @property
    def is_complex(self):
        """True when the chain runs in complex128 (ARITH_COMPLEX or the complex random start)."""
        return bool(self.ctx.lib.achi_chain_is_complex(self.h))

    def site(self, k):
        """Site tensor k as a host (l, d, r) array (complex128 on a complex chain)."""
        dims = [1] + list(self.bond_dims()) + [1]
        if self.is_complex:
            out = np.zeros((dims[k], 2, dims[k + 1]), np.complex128)
            self.ctx._check(self.ctx.lib.achi_chain_get_site_complex(
                self.h, k, out.ctypes.data_as(C.POINTER(C.c_double)), 2 * out.size))
            return out
        out = np.zeros((dims[k], 2, dims[k + 1]))
        self.ctx._check(self.ctx.lib.achi_chain_get_site(self.h, k, _dp(out), out.size))
        return out

    def env(self, which, k):
        shape = (C.c_int64 * 3)()
        self.ctx._check(self.ctx.lib.achi_chain_get_env(self.h, which, k, shape, None, 0))
        out = np.zeros(tuple(shape))
        self.ctx._check(self.ctx.lib.achi_chain_get_env(self.h, which, k, shape, _dp(out), out.size))
        return out

    def states(self):
        arr = (abi.BondState * (self.n - 1))()
        self.ctx._check(self.ctx.lib.achi_chain_get_states(self.h, arr))
        return list(arr)

    def load_state(self, sites, canonicalize=False):
        """Load site tensors (l, d, r) and rebuild environments at centre 0;
        canonicalize=True first applies canonicalize(psi, 0) (mps.cpp:172-210)."""
        dims = np.array([s.shape[2] for s in sites[:-1]], np.int32)
        if self.is_complex:
            flat = [np.ascontiguousarray(s, dtype=np.complex128) for s in sites]
            ptrs = (C.POINTER(C.c_double) * len(flat))(
                *[a.ctypes.data_as(C.POINTER(C.c_double)) for a in flat])
            self.ctx._check(self.ctx.lib.achi_chain_load_mps_complex(self.h, _ip(dims), ptrs,
                                                                     int(canonicalize)))
            return
        flat = [np.ascontiguousarray(s, dtype=np.float64) for s in sites]
        ptrs = (C.POINTER(C.c_double) * len(flat))(*[_dp(a) for a in flat])
        self.ctx._check(self.ctx.lib.achi_chain_load_mps(self.h, _ip(dims), ptrs, int(canonicalize)))

    def sites(self):
        """The MPS as a list of host (l, d, r) arrays (MatrixProductState::sites)."""
        return [self.site(k) for k in range(self.n)]

    def energy(self):
        """expectation_energy (dmrg.cpp:284-298) of the current state, on the device."""
        e = C.c_double()
        self.ctx._check(self.ctx.lib.achi_chain_energy(self.h, C.byref(e)))
        return e.value


def heff_bench(ctx: Context, chi: int, reps: int = 20):
    """Device-resident H_eff timing at chl = chr = chi: (ms per matvec, TFLOP/s)."""
    ms, tf = C.c_double(), C.c_double()
    ctx._check(ctx.lib.achi_heff_bench(ctx.h, chi, reps, C.byref(ms), C.byref(tf)))
    return ms.value, tf.value
