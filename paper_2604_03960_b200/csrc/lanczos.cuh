// Restarted Lanczos with full reorthogonalisation, device-resident
// (eigs_lowest, linalg.cpp:107-178).  Vectors, basis, alpha/beta, the
// tridiagonal Ritz solve and the Ritz combination all live on the GPU; the
// host loop reads one small status record per step to take the reference's
// convergence / restart decisions.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "common.cuh"

namespace achi {
struct HeffOps;  // contract.cuh
}

namespace achi {

constexpr int LANCZOS_BLOCK = 48;  // linalg.cpp:113

// Device-side control of the Lanczos iteration (read/written by the
// orthogonalisation / decision kernels, see lanczos.cu).
struct LanczosCtl {
  int32_t j;         // current step: qcur = q_j is the next matvec input
  int32_t matvecs;   // matvecs of this eigs_lowest call so far
  int32_t block;     // min(dim, LANCZOS_BLOCK)
  int32_t max_iter;
  int32_t steps;     // inner steps executed (launch accounting)
  int32_t cycles;    // restart cycles executed
  int32_t flags;     // LZ_* below
  int32_t pad;
  double tol;
  double best;       // smallest explicit residual seen (EigenNonConvergence)
};
constexpr int32_t LZ_CONVERGED = 1, LZ_NONCONVERGED = 2, LZ_BAD_V0 = 4, LZ_BREAKDOWN = 8;

// What one eigensolve leaves for the host: copied to pinned memory on the
// stream at the end of eigs_lowest_async, read after the caller's next sync.
struct LanczosResult {
  LanczosCtl ctl;
  LanczosStatus st;
};

// One instantiated graph of the inner loop: WHILE { apply(qcur -> w);
// orthogonalise + decide }.  Cached per caller slot while its key (operator
// shape and buffers) is unchanged.
struct LanczosGraph {
  uint64_t key = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t body_launches = 0;   // kernels per inner loop iteration
  int64_t cycle_launches = 0;  // kernels per restart cycle outside the inner loop
  int64_t once_launches = 0;   // kernels per eigensolve outside the restart loop
  void reset();
};

struct LanczosWs {
  DevBuf basis;   // (LANCZOS_BLOCK + 1) x stride
  DevBuf w, ritz, tmp, qcur;
  DevBuf partials;
  DevBuf scal;    // alpha[64] beta[64] h1[64] h2[64] s[64] misc[64]
  DevArr<LanczosCtl> ctl;
  DevArr<unsigned> bar;  // sub-grid barrier counter of the fused small-chi step
  DevBuf pzd;            // persistent eigensolve: partials, eigenvector / result slots
  DevArr<int> pzi;       // persistent eigensolve: jobs, decisions, counters, barrier
  PinnedArr<LanczosCtl> ctl_h;
  PinnedArr<LanczosResult> res_h;  // result of the last eigs_lowest_async
  int64_t pend_body = 0, pend_cycle = 0, pend_once = 0;  // launch accounting of that call
  bool pend_graph = false;
  std::vector<LanczosGraph> graphs;
  long stride = 0;
  LanczosWs() = default;
  LanczosWs(const LanczosWs&) = delete;
  LanczosWs& operator=(const LanczosWs&) = delete;
  ~LanczosWs();
  // Buffers only grow here; a growth invalidates every cached graph.
  void reserve(long n);
  double* q(int i) { return basis.p + static_cast<long>(i) * stride; }
  double* alpha() { return scal.p; }
  double* beta() { return scal.p + 64; }
  double* h1() { return scal.p + 128; }
  double* h2() { return scal.p + 192; }
  double* s() { return scal.p + 256; }
  double* misc() { return scal.p + 320; }
};

struct EigsOut {
  double eigenvalue = 0;
  int matvecs = 0;
  double residual = 0;
};

using ApplyFn = std::function<void(const double* in, double* out)>;

// Lowest eigenpair of the operator `apply` on vectors of (padded) length n
// whose reference dimension is `dim` (block = min(dim, 48)).  v0 and out are
// device vectors of length n (out may alias v0).  Throws
// Error{ACHI_E_EIGEN_NONCONVERGENCE} with the best residual.
//
// Graph mode (default): the whole restarted iteration -- v0 normalisation,
// every restart cycle (the inner Lanczos loop, the Ritz vector, its explicit
// residual check and the restart decision of linalg.cpp:156-169) -- is ONE
// CUDA graph with nested conditional WHILE nodes, captured from `apply` on
// the context stream: `apply` must only enqueue kernels on ctx.stream and use
// buffers that stay allocated.  graph_slot >= 0 caches the instantiated graph
// under graph_key (the caller guarantees the key changes whenever apply's
// kernels, shapes or buffers do); -1 builds a one-off graph.
//
// eigs_lowest_async enqueues the eigensolve and returns without waiting on
// the device (graph mode); the outcome lands in ws.res_h, and eigs_finish
// reads it after the caller's next stream synchronisation (and throws the
// reference's exceptions).  eigs_lowest = async + sync + finish.
void eigs_lowest_async(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                       const double* v0, double tol, int max_iter, double* out,
                       int graph_slot = -1, uint64_t graph_key = 0,
                       const HeffOps* small_op = nullptr);
EigsOut eigs_finish(Ctx& ctx, LanczosWs& ws);
EigsOut eigs_lowest(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                    const double* v0, double tol, int max_iter, double* out,
                    int graph_slot = -1, uint64_t graph_key = 0,
                    const HeffOps* small_op = nullptr);

// Deterministic device reductions used across the hot path.
// sum_i x_i^2 -> *result (device)
// part: scratch of >= 2 * ceil(n / 1024) + 8 doubles, or null for the context's
void device_norm2(Ctx& ctx, const double* x, long n, double* result, double* part = nullptr);
// dst = src * (*scale) (scale device scalar), or src / (*scale) when invert
void device_scale(Ctx& ctx, double* dst, const double* src, long n, const double* scale, bool invert);

}  // namespace achi
