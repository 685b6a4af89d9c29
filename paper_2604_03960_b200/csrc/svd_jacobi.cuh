// Blocked one-sided Jacobi SVD (replaces reference_svd = Eigen BDCSVD +
// fix_phases, linalg.cpp:19-48, on the DMRG path svd_full at dmrg.cpp:117).
//
// The working matrix G (mg x ng, column-major) has its columns orthogonalised
// by cyclic block-pair rotations: columns are grouped in blocks of 16; each
// round pairs blocks by the circle method; one CTA per pair forms the 32x32
// Gram matrix with DMMA, diagonalises it by two-sided Jacobi in shared memory
// and applies the accumulated rotation to G and to V (ng x ng) with DMMA.
// After convergence sigma_c = ||G[:,c]||, columns are sorted non-increasing
// and the phase convention of fix_phases is applied to the kept vectors.
#pragma once

#include <vector>

#include "common.cuh"

namespace achi {

struct SvdWs {
  DevBuf G, Gw, V, sig, sorted, zero2;  // Gw: G * v_init (warm start)
  DevBuf Vq;                    // QR preconditioner factor (cold cluster-path SVDs)
  DevBuf jrec;                  // cluster mode: recorded block rotations (V replay)
  DevArr<unsigned char> jflag;
  DevArr<int> perm;
  DevArr<double> sign;
  DevArr<unsigned long long> conv;
  DevArr<double> gpart;         // stream mode, row split: partial Grams
  DevArr<unsigned> pcnt;        // stream mode: per-pair arrival and round-completion counters
  DevBuf blks;                  // stream mode: tracked diagonal block Grams (ACHI_JACOBI_TRACK)
  DevArr<int> sweeps;
  PinnedArr<int> sweeps_host;
  // defer_v (set by the chain): the cluster path's V replay runs on ctx.vstream
  // beside the caller's next steps (norms, sort, bond selection, the host round
  // trip); svd_wait_v joins it before V is read (svd_phase_signs and svd_gather
  // call it themselves)
  bool defer_v = false, v_pending = false;
  // skip_tol (set by the chain): cluster-path block pairs whose largest cosine is below
  // it are not rotated.  V stays exactly orthogonal and G = theta V exactly, so the
  // truncation U_k U_k^T theta is an exact projection; only the singular vectors carry
  // residual mixing of that size (sigma errors are its square).  0 = rotate to tol.
  double skip_tol = 0.0;
  // stop_tol: the iteration ends after a sweep whose weighted measure (the largest
  // cosine times the square root of its smaller column's relative norm, svd_jacobi.cu
  // finish_gram) is below it; the rotations of that sweep leave cosines ~ its square
  double stop_tol = 1e-7;
  // vrecover (set by the public SVD entries, not by the chain): on the stream path a cold,
  // single-matrix decomposition with vectors rotates only G (3 of the 5 matrix passes per
  // round) and recovers the accumulated factor afterwards as V = G0^T G Sigma^-2 by one
  // GEMM (G0 the loaded working matrix), corrected to first order for G's residual cosines
  // (two more GEMMs); column c is then accurate to ~eps sigma_1 / sigma_c; columns below
  // 1e-3 sigma_1 are projected off the others and re-orthonormalised (Newton-Schulz), and a
  // spectrum reaching below 1e-5 sigma_1 (rank-deficient or ill-conditioned input) is
  // decomposed again with V accumulated (svd_jacobi.cu v_recover)
  bool vrecover = false;
  DevBuf G0, vtail, vproj, vns;
  PinnedArr<int> vcounts;
};

void svd_wait_v(Ctx& ctx, SvdWs& ws);

// Orientation: kRows -> columns of G are the rows of theta (G = theta^T, V
// accumulates the left singular vectors U); kCols -> columns of G are the
// columns of theta (G = theta, V accumulates the right singular vectors).
enum class SvdSide { kRows = 0, kCols = 1 };

struct SvdResultDev {
  SvdSide side;
  int m, n;          // padded rows/cols of theta
  int m_true, n_true;
  int ng, mg;        // working matrix columns/rows (ng padded to a multiple of 32)
  int r_true;        // min(m_true, n_true)
  const int* sweeps_host;  // per cooperative launch; valid after the next stream sync
  int n_launches;
  int max_sweeps;    // the path's sweep cap (reaching it is a NumericalFailure)
  const double* G;   // mg x ng col-major (ld = mg, rows >= the true row count are zero)
  const double* V;   // ng x ng col-major (ld = ng)
  const double* sigma;  // sorted, r_true entries valid (device)
  const int* perm;      // perm[k] = working column of the k-th singular value
  // Jacobi sweeps used (max over launches); call after a stream sync.  Throws
  // NumericalFailure if the iteration hit its sweep cap (linalg.cpp:39-40).
  int sweeps() const;
};

// SVD of theta (m x n row-major, ld = n, padded; true dims m_true x n_true).
// Batched over `batch` matrices at stride `bstride` (sigma only for batch > 1).
// want_vectors = false skips the V accumulation (singular values only).
// v_init (batch 1 only, may be null): an orthogonal ng x ng matrix (col-major,
// ld ng) to start from: the iteration runs on G v_init and V accumulates from
// v_init.  Any orthogonal start gives the same decomposition; the chain passes
// the factor of the previous visit of the same bond and direction, which
// nearly diagonalises the new block once the state has converged (fewer
// sweeps).  v_init must keep pad columns fixed (it does when it comes from a
// decomposition of the same padded shape).
SvdResultDev svd_device(Ctx& ctx, SvdWs& ws, const double* theta, int m, int n, int m_true,
                        int n_true, SvdSide side, int batch = 1, long bstride = 0,
                        double* sigma_out = nullptr, bool want_vectors = true,
                        const double* v_init = nullptr);

// QR preconditioner (svd_precond.cu): G <- G Q in place and V0 <- Q (ng x ng,
// col-major, identity on entry) with G^T Pi = Q R over the real coordinates.
bool qr_precond_applicable(int mr, int nr);
void qr_precond(Ctx& ctx, double* G, long ldg, int mr, int ng, int nr, int pad_mod, int pad_lim,
                double* V0);

// working-matrix width (columns of G and order of V) for a theta of m x n
inline int svd_working_cols(int m, int n, SvdSide side) {
  const int c = side == SvdSide::kRows ? m : n;
  return ((c + 31) / 32) * 32;
}

// fix_phases signs for the first `kept` vectors on the accurate side (U for
// kRows, computed from G for kCols): writes ws.sign[0..kept).
void svd_phase_signs(Ctx& ctx, SvdWs& ws, const SvdResultDev& r, int kept);

// Gather thin factors to device row-major buffers: U (m_true x r) and VT (r x n_true).
void svd_gather(Ctx& ctx, SvdWs& ws, const SvdResultDev& r, int k, double* U, double* VT);

// Complex svd_full (svd_complex.cu): a (m x n row-major, interleaved re/im,
// device); sigma (r = min(m,n), device), U (m x r) and V^dagger (r x n),
// row-major interleaved, fix_phases applied.  Returns the Jacobi sweeps.
// side_pref: -1 by shape; 0 = U, 1 = V^dagger orthonormal to working precision
// across the whole spectrum (noise-level values included; the other factor's
// vectors of such values are only defined up to their sigma weight).
// Two-stage form for truncation (the complex chain): stage 1 decomposes, pairs the values and
// writes sigma (r, device); stage 2 forms only the first k complex singular vectors (the
// Gram-Schmidt of near-degenerate runs is the costly part, and only the kept vectors matter).
struct CsvdRun {
  int first, count;  // real members [first, first + count)
  int out;           // first complex output index
  int want;          // complex vectors to form (<= count / 2)
};
struct CsvdPlan {
  DevBuf E, UE, VTE, cand;
  DevArr<int> src_d, fail_d;
  DevArr<CsvdRun> runs_d;
  std::vector<double> s, sig;
  std::vector<int> src;
  std::vector<CsvdRun> runs, runs_k;
  int m = 0, n = 0, r = 0, r2 = 0, sweeps = 0;
  bool prim_u = true;
};
int svd_complex_stage1(Ctx& ctx, SvdWs& ws, CsvdPlan& plan, const double* a, int m, int n, double* sigma,
                       int side_pref = -1, const double* v_init = nullptr, double* v_keep = nullptr);
void svd_complex_stage2(Ctx& ctx, CsvdPlan& plan, int k, double* U, double* Vd);
// v_init / v_keep (optional, svd_working_cols(2m, 2n, side)^2 doubles): warm start of the
// realified decomposition and the buffer receiving its orthogonal factor (see svd_device).
int svd_complex_device(Ctx& ctx, SvdWs& ws, const double* a, int m, int n, double* sigma, double* U,
                       double* Vd, int side_pref = -1, const double* v_init = nullptr,
                       double* v_keep = nullptr);

}  // namespace achi
