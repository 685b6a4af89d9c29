/*
 * adaptchi_b200.h — C-ABI of the B200-native two-site DMRG local update.
 *
 * This is the drop-in boundary for the hot path of arxiv/paper_2604_03960
 * ("adaptchi", /root/reference/proj).  Every entry point takes plain pointers
 * and sizes; no C++ or torch types cross it.  Each function names the
 * reference interface it replaces (file:line relative to /root/reference).
 *
 * Conventions
 *  - Return value: 0 (ACHI_OK) or one of the ACHI_E_* codes below, one per
 *    reference exception type (proj/include/adaptchi/errors.hpp:8-59) plus
 *    CUDA failures.  achi_last_error() returns the message of the last error
 *    on a context.  The C++ mirror (paper_2604_03960_b200/host) rethrows the
 *    matching typed exception.
 *  - Host arrays are caller-owned.  Device buffers are owned by the context or
 *    by a chain handle.  One context = one device + one CUDA stream; a context
 *    is used by one host thread at a time ("a DMRG run is
 *    strictly sequential; multiple runs may execute concurrently").
 *  - Arithmetic is real FP64 by default.  The reference stores complex128
 *    (tensor.hpp:14-17); for the XXZ/Heisenberg family with the Neel start all
 *    state data are real once the MPO's sigma^y channel is written in the real
 *    gauge (iY, -jy*iY): the dense Hamiltonian is identical.
 *    A chain with complex states (the complex random_mps start) runs in
 *    complex128 (achi_dmrg_config.arithmetic); its sites are read and loaded
 *    through the *_complex entry points as interleaved (re, im) pairs.
 *  - Tensor layouts are the reference's row-major layouts: site tensors
 *    (left, phys, right) (mps.hpp:28-29), environment blocks (bra, mpo, ket)
 *    (dmrg.hpp:38-39), MPO tensors (left, phys_out, phys_in, right)
 *    (models.hpp:25-26), two-site tensor theta (l, s1, s2, r) (dmrg.cpp:94).
 */
#ifndef ADAPTCHI_B200_H
#define ADAPTCHI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (errors.hpp:8-59) ---- */
enum {
  ACHI_OK = 0,
  ACHI_E_ERROR = 1,                 /* Error */
  ACHI_E_INVALID_MATRIX = 2,        /* InvalidMatrix */
  ACHI_E_NUMERICAL_FAILURE = 3,     /* NumericalFailure */
  ACHI_E_INVALID_RANK = 4,          /* InvalidRank */
  ACHI_E_EIGEN_NONCONVERGENCE = 5,  /* EigenNonConvergence{best_residual} */
  ACHI_E_INVALID_BASIS_STATE = 6,   /* InvalidBasisState */
  ACHI_E_SIZE_GUARD = 7,            /* SizeGuard */
  ACHI_E_DEGENERATE_SPECTRUM = 8,   /* DegenerateSpectrum */
  ACHI_E_UNSUPPORTED_MODEL = 9,     /* UnsupportedModel */
  ACHI_E_INVALID_CONFIG = 10,       /* InvalidConfig */
  ACHI_E_INTERNAL = 11,             /* InternalConsistency */
  ACHI_E_CUDA = 20,                 /* CUDA runtime / launch failure */
  ACHI_E_NO_DEVICE = 21             /* no sm_100 device or extension misuse */
};

/* ---- model / config (models.hpp:16-21, controller.hpp:17-42, dmrg.hpp:12-22) ---- */
enum { ACHI_HEISENBERG_XXZ = 0, ACHI_TRANSVERSE_ISING = 1 };
enum { ACHI_SPIN_HALF = 0, ACHI_PAULI = 1 };
enum { ACHI_MODE_FIXED = 0, ACHI_MODE_THRESHOLD = 1, ACHI_MODE_DIRECT = 2, ACHI_MODE_PID = 3 };
enum { ACHI_PREDICT_OFF = 0, ACHI_PREDICT_LINEAR = 1, ACHI_PREDICT_QUADRATIC = 2 };
enum { ACHI_PID_ADDITIVE = 0, ACHI_PID_MULTIPLICATIVE = 1 };
/* Initial state (dmrg.cpp:222-235).  ACHI_INIT_RANDOM is the reference's complex
 * random_mps (mps.cpp:75-95); it runs the chain in complex arithmetic.
 * ACHI_INIT_RANDOM_REAL draws the same mt19937_64(seed) normal sequence, one
 * real value per entry, on capped_bond_dims(n, 2, chi_min) (mps.cpp:60-73),
 * then canonicalize(psi, 0) and normalise as random_mps does.  On the real path
 * ACHI_INIT_AUTOMATIC resolves to RANDOM_REAL for the transverse-field Ising
 * family (its Hamiltonian is real, so its ground state is real). */
enum { ACHI_INIT_AUTOMATIC = 0, ACHI_INIT_NEEL = 1, ACHI_INIT_RANDOM = 2, ACHI_INIT_RANDOM_REAL = 3 };
/* Arithmetic of a chain.  ACHI_ARITH_REAL (default): real FP64 sites and
 * environments with the real-gauge MPO.  ACHI_ARITH_COMPLEX: complex128 sites
 * and environments as the reference stores them (tensor.hpp:14-21), computed
 * as 4M real DMMA contractions on planar [Re; Im] storage; AUTOMATIC then
 * resolves as the reference does (TFIM -> the complex random_mps start,
 * dmrg.cpp:222-235).  ACHI_INIT_RANDOM selects complex arithmetic by itself. */
enum { ACHI_ARITH_REAL = 0, ACHI_ARITH_COMPLEX = 1 };

typedef struct achi_model_spec {
  int32_t family;      /* ACHI_HEISENBERG_XXZ | ACHI_TRANSVERSE_ISING */
  int32_t n;           /* sites, >= 2 */
  double jx, jy, jz, h;
  int32_t convention;  /* ACHI_SPIN_HALF | ACHI_PAULI */
  int32_t _pad;
} achi_model_spec;

typedef struct achi_controller_config {
  int32_t mode;             /* ACHI_MODE_* (default pid) */
  int32_t predictor_order;  /* ACHI_PREDICT_* (default linear) */
  double alpha_ema;         /* 0.3 */
  double gamma_margin;      /* 1.2 */
  double s_target;          /* -1: resolve to ln(chi_max) - 0.5 */
  double kp, ki, kd;        /* 2.0, 0.1, 0.5 */
  double beta_predict;      /* 0.4 */
  int32_t chi_min;          /* 2 */
  int32_t chi_max;          /* 64 */
  int32_t pid_scale;        /* ACHI_PID_* */
  int32_t _pad;
  double eps_trunc;         /* 1e-10 */
} achi_controller_config;

typedef struct achi_dmrg_config {
  int32_t max_sweeps;       /* 24 */
  int32_t eig_max_iter;     /* 200 */
  double eps_conv;          /* 1e-8 */
  double eig_tol;           /* 1e-10 */
  int32_t initial_state;    /* ACHI_INIT_* */
  int32_t arithmetic;       /* ACHI_ARITH_* (0 = real) */
  uint64_t seed;            /* 1234 */
  double noise_floor;       /* 1e-14 */
  achi_controller_config controller;
} achi_dmrg_config;

/* BondControllerState (controller.hpp:45-56) */
typedef struct achi_bond_state {
  double ema, prev_error, integral;
  double history[3];
  int32_t chi, history_len, initialized, _pad;
} achi_bond_state;

/* ControllerDecision + TraceRow (controller.hpp:77-83,116-120) */
typedef struct achi_trace_row {
  int32_t sweep, bond, chi, clamped;
  int64_t delta_chi;
  double s_raw, s_ema, s_pred, error, p_term, i_term, d_term;
} achi_trace_row;

/* Per-visit record: everything needed to attribute a chi-profile divergence
 * to a threshold margin (north_star parity clause). */
typedef struct achi_visit_record {
  int32_t sweep, bond, moving_right, kept;
  int32_t floor_rank, significant, n_sigma, matvecs;
  int32_t degenerate_cut, _pad;
  double energy, entropy, trunc_error;
  double floor_margin;   /* min relative distance |tail - eps*total|/(eps*total) at the floor decision */
  double sigma_kept, sigma_next;  /* sigma[kept-1], sigma[kept] (0 when absent), normalised by sigma[0] */
  double lanczos_residual;
} achi_visit_record;

/* SweepRecord (dmrg.hpp:26-36); profiles are written to caller arrays of length n-1 */
typedef struct achi_sweep_record {
  int32_t sweep_index, max_chi_used;
  double energy, delta_e_rel, max_trunc_error, wall_time;
  int64_t parameter_count;
  double average_chi;
} achi_sweep_record;

/* DmrgResult scalars (dmrg.hpp:71-80) */
typedef struct achi_dmrg_result {
  int32_t n_sweeps, converged, max_chi_used, _pad;
  double energy, max_monotonicity_violation;
} achi_dmrg_result;

/* ---- context ---- */
typedef struct achi_ctx achi_ctx;
typedef struct achi_chain achi_chain;

int achi_ctx_create(int device, achi_ctx** out);
int achi_ctx_destroy(achi_ctx* ctx);
/* Cap the CTAs of the context's grid-wide (cooperative) kernels, 0 = none.  For
 * several contexts sharing one GPU (chains of an ensemble in flight): each
 * context's Lanczos orthogonalisation and fused H_eff then fit beside the
 * others' instead of serialising.  Reduction orders follow the grid, so results
 * are deterministic per cap and agree across caps to rounding. */
int achi_ctx_set_grid_cap(achi_ctx* ctx, int max_ctas);
/* copies the last error message (NUL-terminated, truncated to len) */
int achi_last_error(const achi_ctx* ctx, char* buf, size_t len);
/* EigenNonConvergence::best_residual of the last error (errors.hpp:302-306) */
double achi_last_residual(const achi_ctx* ctx);
/* number of device kernels this context launched so far (evidence counter) */
int64_t achi_launch_count(const achi_ctx* ctx);
int achi_synchronize(achi_ctx* ctx);
/* CUDA-event timer on the context's stream (device time between start and
 * stop, in ms, after a stream synchronize). */
int achi_timer_start(achi_ctx* ctx);
int achi_timer_stop(achi_ctx* ctx, double* ms);
/* write `bytes` through a scratch buffer on the context's stream (L2 flush) */
int achi_flush_l2(achi_ctx* ctx, size_t bytes);
/* Per-phase device time measured with CUDA events on the context stream
 * (phases: 0 H_eff matvec, 1 SVD, 2 environment update).  enable turns the
 * accounting on (1) or off (0), -1 leaves it; enable = n > 1 times one chain
 * bond visit in n (timing events cost device time; the totals and the work
 * then cover the sampled visits).  reset zeroes it.  out9 (may be NULL) =
 * {ms[3], algorithmic work[3] (flops, bytes, flops), launches[3]}. */
/* Lanczos inner loop of this context's chains: 1 = one conditional CUDA graph
 * per (bond, direction) (default), 0 = stepped from the host (same kernels and
 * arithmetic; every launch visible to profilers and to phase 3 of
 * achi_device_times_ex), -1 = the process default (ACHI_LANCZOS_GRAPH). */
int achi_ctx_set_lanczos_graph(achi_ctx* ctx, int mode);
int achi_device_times(achi_ctx* ctx, int enable, int reset, double* out9);
/* Same, for the first n_phases (<= 4) phases: 3 = H_eff applications alone
 * (recorded around each matvec outside graph capture, so they are seen with
 * ACHI_LANCZOS_GRAPH=0 or for the Lanczos matvecs issued from the host).
 * out = {ms[n], work[n] (flops, bytes, flops, flops), launches[n]}. */
int achi_device_times_ex(achi_ctx* ctx, int enable, int reset, double* out, int n_phases);

/* ---- DMRG (dmrg.hpp:40-90, dmrg.cpp:216-282) ---- */
/* run_dmrg setup: validate, build_mpo (real gauge), Neel product state,
 * canonicalize(psi,0), Environment::rebuild(psi,mpo,0), controller cold start
 * (dmrg.cpp:216-250).  Device-resident from here on. */
int achi_chain_create(achi_ctx* ctx, const achi_model_spec* spec,
                      const achi_dmrg_config* cfg, achi_chain** out);
int achi_chain_destroy(achi_chain* chain);
/* two_site_sweep (dmrg.cpp:175-214).  chi_profile/entropy_profile: n-1 each
 * (may be NULL).  trace: capacity 2(n-1) rows (may be NULL).  visits:
 * capacity 2(n-1) (may be NULL). */
int achi_chain_sweep(achi_chain* chain, int sweep_index, achi_sweep_record* rec,
                     int32_t* chi_profile, double* entropy_profile,
                     achi_trace_row* trace, achi_visit_record* visits);
/* run_dmrg sweep loop + convergence (dmrg.cpp:255-281) on an existing chain.
 * records: capacity cfg.max_sweeps; profiles: max_sweeps*(n-1); trace and
 * visits: max_sweeps*2(n-1) (each may be NULL). */
int achi_chain_run(achi_chain* chain, achi_dmrg_result* result,
                   achi_sweep_record* records, int32_t* chi_profiles,
                   double* entropy_profiles, achi_trace_row* trace,
                   achi_visit_record* visits);
/* bond dimensions chi_1..chi_{n-1} (MatrixProductState::bond_dims, mps.cpp:24-29) */
int achi_chain_bond_dims(const achi_chain* chain, int32_t* dims);
/* copy site tensor k (row-major (l,d,r)) to host; size = l*d*r doubles */
int achi_chain_get_site(const achi_chain* chain, int k, double* out, size_t capacity);
/* copy environment block (row-major (bra,mpo,ket)); which = 0 left, 1 right */
int achi_chain_get_env(const achi_chain* chain, int which, int k, int64_t* shape3,
                       double* out, size_t capacity);
/* per-bond controller states (n-1 entries) */
int achi_chain_get_states(const achi_chain* chain, achi_bond_state* out);
/* replace bond states (test hook for replaying the reference's states) */
int achi_chain_set_states(achi_chain* chain, const achi_bond_state* in);
/* load an MPS (host, row-major sites with the given bond dims) into the chain
 * and rebuild environments at centre 0 (Environment::rebuild, dmrg.cpp:51-56).
 * The state must be right-canonical with centre 0. */
int achi_chain_load_state(achi_chain* chain, const int32_t* bond_dims,
                          const double* const* sites);
/* Same, for any state: canonicalize != 0 first brings it to right-canonical
 * form with centre 0 (canonicalize(psi, 0), mps.cpp:172-210: Householder QR of
 * each site, host side, bond dimensions may shrink to min(chi, d * right)).
 * Replaces load_mps + canonicalize + Environment::rebuild for a resumed run. */
int achi_chain_load_mps(achi_chain* chain, const int32_t* bond_dims, const double* const* sites,
                        int canonicalize);
/* 1 when the chain runs in complex128 (ACHI_ARITH_COMPLEX or a complex start) */
int achi_chain_is_complex(const achi_chain* chain);
/* copy complex site tensor k (row-major (l,d,r), interleaved re/im: 2*l*d*r
 * doubles) of a complex chain (MatrixProductState::site, mps.hpp:28-29) */
int achi_chain_get_site_complex(const achi_chain* chain, int k, double* out, size_t capacity);
/* achi_chain_load_mps for a complex chain: sites interleaved re/im (mps.cpp:276-315
 * snapshots, resumed runs); canonicalize != 0 runs canonicalize(psi, 0) on the
 * device (complex SVD push_left) */
int achi_chain_load_mps_complex(achi_chain* chain, const int32_t* bond_dims,
                                const double* const* sites, int canonicalize);
/* expectation_energy (dmrg.cpp:284-298) of the chain's current state on the
 * device: left environments rebuilt from the boundary through every site
 * (independent of the cached environments); <psi|H|psi> (psi is normalised
 * after every visit). */
int achi_chain_energy(achi_chain* chain, double* energy);

/* Phase accounting since chain creation (host wall clock at sync points):
 * out[0..7] = {lanczos+merge s, svd s, bond-select s, absorb+env s, matvecs,
 * svd sweeps, visits, 0}.  profile != 0 adds a sync after each visit so the
 * phase split is exact (default off: the hot path keeps its own syncs only). */
int achi_chain_stats(achi_chain* chain, int profile, double* out8);

/* ---- local kernels, host buffers (for parity tests and API-level calls) ---- */
/* apply_effective_hamiltonian (dmrg.cpp:58-71): out(bl,s1',s2',br).
 * L: (chl, D1, chl) ; W1: (D1, d, d, D2); W2: (D2, d, d, D3); R: (chr, D3, chr);
 * theta/out: (chl, d, d, chr). */
int achi_heff_apply(achi_ctx* ctx, int chl, int chr, int d, int D1, int D2, int D3,
                    const double* L, const double* W1, const double* W2,
                    const double* R, const double* theta, double* out);
/* Environment::update_left (dmrg.cpp:26-37): Lnew(b',a',j') from L (chl,Dl,chl),
 * A (chl,d,chn), W (Dl,d,d,Dr) -> Lnew (chn, Dr, chn) */
int achi_env_update_left(achi_ctx* ctx, int chl, int chn, int d, int Dl, int Dr,
                         const double* L, const double* A, const double* W,
                         double* Lnew);
/* Environment::update_right (dmrg.cpp:39-49): Rnew(b',a,j) from R (chr,Dr,chr),
 * B (chn,d,chr), W (Dl,d,d,Dr) -> Rnew (chn, Dl, chn) */
int achi_env_update_right(achi_ctx* ctx, int chr, int chn, int d, int Dl, int Dr,
                          const double* R, const double* B, const double* W,
                          double* Rnew);

/* svd_full (linalg.cpp:67-70) + fix_phases (linalg.cpp:19-35) on the GPU
 * Jacobi kernel.  a: m x n ROW-major.  r = min(m,n).  Outputs (any may be
 * NULL): sigma[r] non-increasing; u: m x r row-major; vt: r x n row-major.
 * sweeps_out: Jacobi sweeps used.  Matrices too large for one cluster (the
 * streamed path) rotate only one factor and recover the other by GEMM
 * afterwards (svd_jacobi.cuh SvdWs::vrecover; decomposed again with both
 * accumulated when a singular value lies below 1e-5 sigma_1). */
int achi_svd(achi_ctx* ctx, int m, int n, const double* a, double* sigma,
             double* u, double* vt, int* sweeps_out);
/* Batched SVD of `batch` m x n row-major matrices stored back to back; only
 * singular values are returned (batch x r).  Device-resident timing hook for
 * config C2 (bench.cpp:635-668). */
int achi_svd_batched(achi_ctx* ctx, int batch, int m, int n, const double* a,
                     double* sigma);
/* Same on DEVICE pointers (inputs already resident in HBM; the benchmark's
 * device-time path).  d_sigma: batch x min(m,n) device buffer.  Values only:
 * no singular vectors are accumulated. */
int achi_svd_batched_device(achi_ctx* ctx, int batch, int m, int n, const double* d_a,
                            double* d_sigma, int* sweeps_out);
/* svd_full on DEVICE pointers with both factors (the truncated-SVD timing
 * path of bench.cpp:635-668: the reference computes U, sigma, V^dagger and
 * then truncates).  d_a: m x n row-major; d_sigma[r]; d_u: m x r row-major;
 * d_vt: r x n row-major (r = min(m, n)); fix_phases applied. */
int achi_svd_device(achi_ctx* ctx, int m, int n, const double* d_a, double* d_sigma,
                    double* d_u, double* d_vt, int* sweeps_out);

/* Complex svd_full (linalg.cpp:11-48, 67-70; DenseMatrix = Eigen::MatrixXcd,
 * tensor.hpp:15): a is m x n row-major complex128 as interleaved (re, im)
 * doubles.  Outputs sigma[r] (non-increasing), u (m x r) and vdag = V^dagger
 * (r x n), row-major interleaved, fix_phases applied (linalg.cpp:19-35: the
 * first largest-|u| entry of each U column real and positive).  Computed on
 * the real Jacobi engine through the realification [[Re, -Im], [Im, Re]]
 * (svd_complex.cu).  Non-finite input -> ACHI_E_INVALID_MATRIX.  Replaces
 * reference_svd for complex blocks, e.g. the cmd_svd_bench literal
 * (bench.cpp:646-648). */
int achi_svd_complex(achi_ctx* ctx, int m, int n, const double* a, double* sigma, double* u,
                     double* vdag, int* sweeps_out);
/* Same on device pointers (the caller guarantees finite input). */
int achi_svd_complex_device(achi_ctx* ctx, int m, int n, const double* d_a, double* d_sigma,
                            double* d_u, double* d_vdag, int* sweeps_out);

/* Fused bond-select kernel (K7) on a host spectrum: entropy_from_spectrum
 * (mps.cpp:97-113), rank_for_discarded_weight (controller.cpp:134-148),
 * kept-rank logic (dmrg.cpp:113-136), controller_update
 * (controller.cpp:150-190) and truncation_error (mps.cpp:115-122), executed
 * on the device.  state is updated in place. */
int achi_bond_select(achi_ctx* ctx, const achi_dmrg_config* cfg, int n_sigma,
                     const double* sigma, achi_bond_state* state, int sweep,
                     int bond, achi_trace_row* row, achi_visit_record* visit);

/* The contraction engine behind K1-K4 (TMA-fed DMMA GEMM), exposed for unit
 * tests: C (M x N, row-major, ldc) = A * B.  a_kmajor: A stored M x K
 * row-major (else K x M); b_kmajor: B stored N x K row-major (else K x N).
 * Leading dimensions must be even (16-byte TMA strides).  Replaces the GEMM
 * inside Tensor::contract (tensor.hpp:195-196). */
int achi_dgemm(achi_ctx* ctx, int M, int N, int K, int a_kmajor, const double* a, long lda,
               int b_kmajor, const double* b, long ldb, double* c, long ldc);

/* Route this context's contractions (H_eff, environments, theta merge) of at
 * least min_flops (2 M N K) through achi_dgemm_ozaki's engine with `slices`
 * digits (0 = off: the native DMMA engine, the default).  While on, the
 * context's Lanczos loops are stepped from the host. */
int achi_ctx_set_ozaki(achi_ctx* ctx, int slices, double min_flops);

/* achi_dgemm on device pointers (queued on the context stream, no sync). */
int achi_dgemm_device(achi_ctx* ctx, int M, int N, int K, int a_kmajor, const double* d_a, long lda,
                      int b_kmajor, const double* d_b, long ldb, double* d_c, long ldc);

/* Emulated-FP64 GEMM on the int8 tensor cores (Ozaki scheme, tcgen05.mma
 * kind::i8, the north_star's "optionally emulated-precision"
 * contraction): C (M x N row-major, ldc) = A B with every FP64 operand entry
 * cut into `slices` signed 7-bit digits against a power-of-two scale per row
 * of A / column of B, all digit products with p + q <= slices + 1 exact in
 * int32 TMEM accumulators.  slices = 8 carries 56 bits (FP64 level); fewer
 * trade accuracy for speed.  Device pointers.  A: M x K row-major (lda), or
 * K x M when a_trans; B: K x N row-major (ldb), or N x K when b_kmajor.
 * K <= 16384.  Queued on the context stream.  Replaces the GEMM inside
 * Tensor::contract (tensor.hpp:195-196) as an opt-in alternative to the DMMA engine. */
int achi_dgemm_ozaki_device(achi_ctx* ctx, int M, int N, int K, const double* d_a, long lda, int a_trans,
                            const double* d_b, long ldb, int b_kmajor, double* d_c, long ldc, int slices);

/* Device-resident timing hook for K1: `reps` applications of the effective
 * Hamiltonian at chl = chr = chi (XXZ bulk MPO, D = 5) on pseudo-random
 * device data; returns the average device ms per matvec and the achieved
 * algorithmic TFLOP/s (2 D d^2 chi^2 (2 chi) + 4 D^2 d^3 chi^2 flops). */
int achi_heff_bench(achi_ctx* ctx, int chi, int reps, double* ms_per_matvec, double* tflops);

/* Spectrum reductions on the device (one CTA, deterministic order):
 * out[0] = entropy_from_spectrum (mps.cpp:97-113), out[1] = truncation_error
 * at `kept` (mps.cpp:115-122), out[2] = rank_for_discarded_weight(eps)
 * (controller.cpp:134-148), out[3] = count of sigma > 1e-14 sigma_1.
 * Errors as the reference: empty/zero spectrum -> DegenerateSpectrum, kept
 * out of [1, n] -> InvalidRank. */
int achi_spectrum_stats(achi_ctx* ctx, int n_sigma, const double* sigma, int kept, double eps,
                        double* out4);

/* eigs_lowest (linalg.cpp:107-178) with a dense symmetric operator (test
 * hook for the device Lanczos): h is dim x dim row-major. */
int achi_eigs_lowest_dense(achi_ctx* ctx, int dim, const double* h,
                           const double* v0, double tol, int max_iter,
                           double* eigenvalue, double* eigenvector,
                           int* matvecs, double* residual);

/* eigs_lowest(const LinearMap&, dim, v0, tol, max_iter) (linalg.hpp:64-78,
 * linalg.cpp:107-178) for an operator given as a host callback:
 * fn(user, in, out, dim) must write out = H in for a real symmetric H (the
 * host mirror passes complex Hermitian LinearMaps through their real
 * 2 dim x 2 dim form).  The Lanczos iteration (basis, reorthogonalisation,
 * tridiagonal solve, restarts) runs on the device, stepped from the host;
 * every matvec copies the vector to the host, calls fn and copies the result
 * back.  Errors as achi_eigs_lowest_dense; a non-finite operator output ->
 * ACHI_E_INVALID_MATRIX. */
typedef void (*achi_matvec_fn)(void* user, const double* in, double* out, int64_t dim);
int achi_eigs_lowest_callback(achi_ctx* ctx, int dim, achi_matvec_fn fn, void* user, const double* v0,
                              double tol, int max_iter, double* eigenvalue, double* eigenvector,
                              int* matvecs, double* residual);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTCHI_B200_H */
