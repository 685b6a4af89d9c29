// Restarted Lanczos with full reorthogonalisation, device-resident
// (eigs_lowest, linalg.cpp:107-178).  Vectors, basis, alpha/beta, the
// tridiagonal Ritz solve and the Ritz combination all live on the GPU; the
// host loop reads one small status record per step to take the reference's
// convergence / restart decisions.
#pragma once

#include <functional>

#include "common.cuh"

namespace achi {

constexpr int LANCZOS_BLOCK = 48;  // linalg.cpp:113

struct LanczosWs {
  DevBuf basis;   // (LANCZOS_BLOCK + 1) x stride
  DevBuf w, ritz, tmp;
  DevBuf partials;
  DevBuf scal;    // alpha[64] beta[64] h1[64] h2[64] s[64] misc[64]
  long stride = 0;
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
EigsOut eigs_lowest(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                    const double* v0, double tol, int max_iter, double* out);

// Deterministic device reductions used across the hot path.
// sum_i x_i^2 -> *result (device)
void device_norm2(Ctx& ctx, const double* x, long n, double* result);
// dst = src * (*scale) (scale device scalar), or src / (*scale) when invert
void device_scale(Ctx& ctx, double* dst, const double* src, long n, const double* scale, bool invert);

}  // namespace achi
