"""ctypes mirror of include/adaptchi_b200.h (struct layouts, enums, loader).

The product library is ``paper_2604_03960_b200/_build/libadaptchi_b200.so``
(built by ``__graft_entry__.build()``).  There is no CPU fallback: if the
library is missing, :func:`load` raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libadaptchi_b200.so")

# ---- enums (adaptchi_b200.h) ----
HEISENBERG_XXZ, TRANSVERSE_ISING = 0, 1
SPIN_HALF, PAULI = 0, 1
MODE_FIXED, MODE_THRESHOLD, MODE_DIRECT, MODE_PID = 0, 1, 2, 3
PREDICT_OFF, PREDICT_LINEAR, PREDICT_QUADRATIC = 0, 1, 2
PID_ADDITIVE, PID_MULTIPLICATIVE = 0, 1
INIT_AUTOMATIC, INIT_NEEL, INIT_RANDOM, INIT_RANDOM_REAL = 0, 1, 2, 3
ARITH_REAL, ARITH_COMPLEX = 0, 1

ERROR_NAMES = {
    1: "Error", 2: "InvalidMatrix", 3: "NumericalFailure", 4: "InvalidRank",
    5: "EigenNonConvergence", 6: "InvalidBasisState", 7: "SizeGuard",
    8: "DegenerateSpectrum", 9: "UnsupportedModel", 10: "InvalidConfig",
    11: "InternalConsistency", 20: "CudaError", 21: "NoDevice",
}


# achi_matvec_fn: void (*)(void* user, const double* in, double* out, int64_t dim)
MATVEC_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)


class ModelSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("n", C.c_int32), ("jx", C.c_double),
                ("jy", C.c_double), ("jz", C.c_double), ("h", C.c_double),
                ("convention", C.c_int32), ("_pad", C.c_int32)]


class ControllerConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("predictor_order", C.c_int32),
                ("alpha_ema", C.c_double), ("gamma_margin", C.c_double),
                ("s_target", C.c_double), ("kp", C.c_double), ("ki", C.c_double),
                ("kd", C.c_double), ("beta_predict", C.c_double),
                ("chi_min", C.c_int32), ("chi_max", C.c_int32),
                ("pid_scale", C.c_int32), ("_pad", C.c_int32),
                ("eps_trunc", C.c_double)]


class DmrgConfig(C.Structure):
    _fields_ = [("max_sweeps", C.c_int32), ("eig_max_iter", C.c_int32),
                ("eps_conv", C.c_double), ("eig_tol", C.c_double),
                ("initial_state", C.c_int32), ("arithmetic", C.c_int32),
                ("seed", C.c_uint64), ("noise_floor", C.c_double),
                ("controller", ControllerConfig)]


class BondState(C.Structure):
    _fields_ = [("ema", C.c_double), ("prev_error", C.c_double),
                ("integral", C.c_double), ("history", C.c_double * 3),
                ("chi", C.c_int32), ("history_len", C.c_int32),
                ("initialized", C.c_int32), ("_pad", C.c_int32)]


class TraceRow(C.Structure):
    _fields_ = [("sweep", C.c_int32), ("bond", C.c_int32), ("chi", C.c_int32),
                ("clamped", C.c_int32), ("delta_chi", C.c_int64),
                ("s_raw", C.c_double), ("s_ema", C.c_double), ("s_pred", C.c_double),
                ("error", C.c_double), ("p_term", C.c_double), ("i_term", C.c_double),
                ("d_term", C.c_double)]


class VisitRecord(C.Structure):
    _fields_ = [("sweep", C.c_int32), ("bond", C.c_int32), ("moving_right", C.c_int32),
                ("kept", C.c_int32), ("floor_rank", C.c_int32), ("significant", C.c_int32),
                ("n_sigma", C.c_int32), ("matvecs", C.c_int32),
                ("degenerate_cut", C.c_int32), ("_pad", C.c_int32),
                ("energy", C.c_double), ("entropy", C.c_double),
                ("trunc_error", C.c_double), ("floor_margin", C.c_double),
                ("sigma_kept", C.c_double), ("sigma_next", C.c_double),
                ("lanczos_residual", C.c_double)]


class SweepRecord(C.Structure):
    _fields_ = [("sweep_index", C.c_int32), ("max_chi_used", C.c_int32),
                ("energy", C.c_double), ("delta_e_rel", C.c_double),
                ("max_trunc_error", C.c_double), ("wall_time", C.c_double),
                ("parameter_count", C.c_int64), ("average_chi", C.c_double)]


class DmrgResult(C.Structure):
    _fields_ = [("n_sweeps", C.c_int32), ("converged", C.c_int32),
                ("max_chi_used", C.c_int32), ("_pad", C.c_int32),
                ("energy", C.c_double), ("max_monotonicity_violation", C.c_double)]


def model_spec(n, family=HEISENBERG_XXZ, jx=1.0, jy=1.0, jz=1.0, h=0.0, convention=PAULI):
    """ModelSpec defaults (models.hpp:16-21)."""
    return ModelSpec(family, n, jx, jy, jz, h, convention, 0)


def controller_config(**kw):
    """ControllerConfig defaults (controller.hpp:17-39)."""
    c = ControllerConfig(MODE_PID, PREDICT_LINEAR, 0.3, 1.2, -1.0, 2.0, 0.1, 0.5, 0.4,
                         2, 64, PID_ADDITIVE, 0, 1e-10)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def dmrg_config(controller=None, **kw):
    """DmrgConfig defaults (dmrg.hpp:12-22)."""
    c = DmrgConfig(24, 200, 1e-8, 1e-10, INIT_AUTOMATIC, 0, 1234, 1e-14,
                   controller if controller is not None else controller_config())
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def fixed_config(chi, **kw):
    """test_dmrg.cpp:32-38 fixed_config."""
    return dmrg_config(controller_config(mode=MODE_FIXED, chi_max=chi, chi_min=min(2, chi)), **kw)


def adaptive_config(chi_max, eps=1e-10, **kw):
    """test_dmrg.cpp:40-46 adaptive_config (PID)."""
    return dmrg_config(controller_config(mode=MODE_PID, chi_max=chi_max, eps_trunc=eps), **kw)


_lib = None


def load():
    """Load the CUDA product library; raise if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libadaptchi_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    d, i32, vp, dp = C.c_double, C.c_int32, C.c_void_p, P(C.c_double)
    sig = {
        "achi_ctx_create": (C.c_int, [C.c_int, P(vp)]),
        "achi_ctx_destroy": (C.c_int, [vp]),
        "achi_last_error": (C.c_int, [vp, C.c_char_p, C.c_size_t]),
        "achi_last_residual": (d, [vp]),
        "achi_launch_count": (C.c_int64, [vp]),
        "achi_synchronize": (C.c_int, [vp]),
        "achi_timer_start": (C.c_int, [vp]),
        "achi_timer_stop": (C.c_int, [vp, dp]),
        "achi_flush_l2": (C.c_int, [vp, C.c_size_t]),
        "achi_ctx_set_grid_cap": (C.c_int, [vp, C.c_int]),
        "achi_chain_create": (C.c_int, [vp, P(ModelSpec), P(DmrgConfig), P(vp)]),
        "achi_chain_destroy": (C.c_int, [vp]),
        "achi_chain_sweep": (C.c_int, [vp, C.c_int, P(SweepRecord), P(i32), dp,
                                       P(TraceRow), P(VisitRecord)]),
        "achi_chain_run": (C.c_int, [vp, P(DmrgResult), P(SweepRecord), P(i32), dp,
                                     P(TraceRow), P(VisitRecord)]),
        "achi_chain_bond_dims": (C.c_int, [vp, P(i32)]),
        "achi_chain_stats": (C.c_int, [vp, C.c_int, dp]),
        "achi_chain_get_site": (C.c_int, [vp, C.c_int, dp, C.c_size_t]),
        "achi_chain_get_env": (C.c_int, [vp, C.c_int, C.c_int, P(C.c_int64), dp, C.c_size_t]),
        "achi_chain_get_states": (C.c_int, [vp, P(BondState)]),
        "achi_chain_set_states": (C.c_int, [vp, P(BondState)]),
        "achi_chain_load_state": (C.c_int, [vp, P(i32), P(dp)]),
        "achi_chain_load_mps": (C.c_int, [vp, P(i32), P(dp), C.c_int]),
        "achi_chain_energy": (C.c_int, [vp, dp]),
        "achi_chain_is_complex": (C.c_int, [vp]),
        "achi_chain_get_site_complex": (C.c_int, [vp, C.c_int, dp, C.c_size_t]),
        "achi_chain_load_mps_complex": (C.c_int, [vp, P(i32), P(dp), C.c_int]),
        "achi_heff_apply": (C.c_int, [vp] + [C.c_int] * 6 + [dp] * 6),
        "achi_env_update_left": (C.c_int, [vp] + [C.c_int] * 5 + [dp] * 4),
        "achi_env_update_right": (C.c_int, [vp] + [C.c_int] * 5 + [dp] * 4),
        "achi_svd": (C.c_int, [vp, C.c_int, C.c_int, dp, dp, dp, dp, P(C.c_int)]),
        "achi_svd_batched": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp, dp]),
        "achi_svd_batched_device": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                              C.c_void_p, P(C.c_int)]),
        "achi_device_times": (C.c_int, [vp, C.c_int, C.c_int, dp]),
        "achi_device_times_ex": (C.c_int, [vp, C.c_int, C.c_int, dp, C.c_int]),
        "achi_ctx_set_lanczos_graph": (C.c_int, [vp, C.c_int]),
        "achi_svd_complex": (C.c_int, [vp, C.c_int, C.c_int, dp, dp, dp, dp, P(C.c_int)]),
        "achi_ctx_set_ozaki": (C.c_int, [vp, C.c_int, d]),
        "achi_dgemm_device": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_long,
                                        C.c_int, C.c_void_p, C.c_long, C.c_void_p, C.c_long]),
        "achi_dgemm_ozaki_device": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_long,
                                              C.c_int, C.c_void_p, C.c_long, C.c_int, C.c_void_p,
                                              C.c_long, C.c_int]),
        "achi_eigs_lowest_callback": (C.c_int, [vp, C.c_int, MATVEC_FN, C.c_void_p, dp, d, C.c_int,
                                                dp, dp, P(C.c_int), dp]),
        "achi_svd_complex_device": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, P(C.c_int)]),
        "achi_bond_select": (C.c_int, [vp, P(DmrgConfig), C.c_int, dp, P(BondState),
                                       C.c_int, C.c_int, P(TraceRow), P(VisitRecord)]),
        "achi_eigs_lowest_dense": (C.c_int, [vp, C.c_int, dp, dp, d, C.c_int, dp, dp,
                                             P(C.c_int), dp]),
        "achi_dgemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp, C.c_long, C.c_int,
                                 dp, C.c_long, dp, C.c_long]),
        "achi_spectrum_stats": (C.c_int, [vp, C.c_int, dp, C.c_int, d, dp]),
        "achi_svd_device": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, P(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    _late_signatures(lib)
    _lib = lib
    return lib


def _late_signatures(lib):
    P = C.POINTER
    lib.achi_heff_bench.restype = C.c_int
    lib.achi_heff_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_double), P(C.c_double)]
