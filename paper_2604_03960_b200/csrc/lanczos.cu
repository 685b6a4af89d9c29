// Device Lanczos (see lanczos.cuh).  All reductions are deterministic: each
// block owns a fixed contiguous chunk and partials are summed in fixed order.
#include <cooperative_groups.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "lanczos.cuh"
#include "heff_phases.cuh"

namespace cg = cooperative_groups;

namespace achi {

namespace {

constexpr int RED_THREADS = 256;
constexpr int DOT_GROUP = 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum in fixed order; result valid in thread 0
__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

constexpr int EPT = 4;                      // elements per thread
constexpr int CHUNK = RED_THREADS * EPT;    // elements per block (fixed: deterministic)

// partials[b * ld + v] = sum_{x in chunk b} Q_v[x] * w[x] for v < nv; plus w.w at v = nv if self.
// One warp-shuffle reduction per vector and a single __syncthreads per block.
__global__ void __launch_bounds__(RED_THREADS) multi_dot_kernel(const double* __restrict__ Q, long stride,
                                                                int nv, const double* __restrict__ w,
                                                                long n, double* __restrict__ partials,
                                                                int ld, int self) {
  __shared__ double sh[RED_THREADS / 32][65];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long base = static_cast<long>(blockIdx.x) * CHUNK + threadIdx.x;
  double wx[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const long x = base + e * RED_THREADS;
    wx[e] = x < n ? w[x] : 0.0;
  }
  const int nt = nv + self;
  for (int v0 = 0; v0 < nt; v0 += DOT_GROUP) {
    double acc[DOT_GROUP];
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) {
      const int v = v0 + g;
      double a = 0.0;
      if (v < nv) {
        const double* q = Q + v * stride;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const long x = base + e * RED_THREADS;
          if (x < n) a += q[x] * wx[e];
        }
      } else if (v == nv && self) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) a += wx[e] * wx[e];
      }
      acc[g] = warp_sum(a);
    }
    if (lane == 0)
#pragma unroll
      for (int g = 0; g < DOT_GROUP; ++g)
        if (v0 + g < nt) sh[warp][v0 + g] = acc[g];
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nt; v += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < RED_THREADS / 32; ++w8) s += sh[w8][v];
    partials[static_cast<long>(blockIdx.x) * ld + v] = s;
  }
}

// out[v] = sum_b partials[b * ld + v] (one block per v, fixed-order tree)
__global__ void __launch_bounds__(RED_THREADS) reduce_partials_kernel(
    const double* __restrict__ partials, int nblocks, int ld, int nv, double* __restrict__ out) {
  __shared__ double sh[32];
  const int v = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partials[static_cast<long>(b) * ld + v];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[v] = s;
}

// dst[x] = src[x] + sign * sum_v coef[v] * Q_v[x]; partials[b] = sum_chunk dst^2
// (nv_ctl non-null: nv = nv_ctl->j + 1, the basis size the device loop reached)
__global__ void __launch_bounds__(RED_THREADS) multi_axpy_kernel(
    const double* __restrict__ Q, long stride, int nv, const double* __restrict__ coef, double sign,
    const double* src, double* dst, long n, double* __restrict__ partials,
    const LanczosCtl* __restrict__ nv_ctl = nullptr) {
  __shared__ double c[64];
  __shared__ double sh[32];
  if (nv_ctl) nv = nv_ctl->j + 1;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) c[v] = sign * coef[v];
  __syncthreads();
  const long base = static_cast<long>(blockIdx.x) * CHUNK + threadIdx.x;
  double acc[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const long x = base + e * RED_THREADS;
    acc[e] = (src && x < n) ? src[x] : 0.0;
  }
  for (int i = 0; i < nv; ++i) {
    const double ci = c[i];
    const double* q = Q + i * stride;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const long x = base + e * RED_THREADS;
      if (x < n) acc[e] += ci * q[x];
    }
  }
  double nrm = 0.0;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const long x = base + e * RED_THREADS;
    if (x < n) {
      dst[x] = acc[e];
      nrm += acc[e] * acc[e];
    }
  }
  if (partials) {
    const double s = block_sum(nrm, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

__global__ void scale_kernel(double* __restrict__ dst, const double* __restrict__ src, long n,
                             const double* __restrict__ s, int invert) {
  const double f = invert ? 1.0 / *s : *s;
  for (long x = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<long>(gridDim.x) * blockDim.x)
    dst[x] = src[x] * f;
}

// ---- tridiagonal lowest eigenpair (Eigen computeFromTridiagonal, col 0) ----
// The Lanczos tridiagonal T (k <= 48, a = alpha, b = beta, bb = beta^2) is
// solved by block 0 of the fused step kernel: multisection on Sturm counts
// for the lowest eigenvalue (bracketed with the previous step's Ritz value),
// then a twisted factorization for the eigenvector.  Every sequential chain
// is a division-free FMA recurrence; divisions only happen in parallel across
// lanes.

// exact power of two 2^e (|e| < 1000)
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}
// binary exponent of |m| (m > 0, normal)
__device__ __forceinline__ int exponent_of(double m) {
  return static_cast<int>((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
}

// Sturm count (number of eigenvalues below x) from the characteristic-
// polynomial recurrence p_{i+1} = (a_i - x) p_i - bb_{i-1} p_{i-1}, p_0 = 1:
// the sign changes of p_0..p_k (a zero takes the sign +, counting a root of a
// leading minor once).  One dependent FMA per step, no division; operands
// are loaded 8 steps ahead and p is rescaled by an exact power of two, so it
// neither overflows nor underflows.
__device__ int sturm_count(const double* a, const double* bb, int k, double x) {
  double pm = 1.0, p = a[0] - x;
  int cnt = p < 0.0 ? 1 : 0;
  for (int i0 = 1; i0 < k; i0 += 8) {
    double da[8], db[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      da[u] = i < k ? a[i] - x : 0.0;
      db[u] = i < k ? bb[i - 1] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u < k) {
        const double pn = fma(da[u], p, -db[u] * pm);
        cnt += (pn < 0.0) != (p < 0.0) ? 1 : 0;
        pm = p;
        p = pn;
      }
    }
    const double m = fmax(fabs(p), fabs(pm));
    const int e = exponent_of(m);
    if (m > 0.0 && (e > 64 || e < -64)) {
      const double f = pow2(-e);
      p *= f;
      pm *= f;
    }
  }
  return cnt;
}

// Lowest eigenvalue by 32-point multisection on Sturm counts (one point per
// lane; all 32 lanes of one warp).  With a hint (the previous step's Ritz
// value theta_prev and residual bound r_prev) the first round searches
// [theta_prev - 2 r_prev, theta_prev]: by interlacing the new lowest value is
// not above theta_prev and the residual theorem puts an eigenvalue within
// r_prev of it; the count at the lower end verifies that it is the lowest
// (otherwise the Gershgorin interval is searched).  Returns the upper end of
// the final bracket; *scale_out = Gershgorin scale.
__device__ double tridiag_lowest_value(const double* sa, const double* sb, const double* sbb, int k,
                                       bool hinted, double theta_prev, double r_prev,
                                       double* scale_out) {
  const int lane = threadIdx.x & 31;
  double lo = INFINITY, hi = -INFINITY, scale = 0.0;
  for (int i = lane; i < k; i += 32) {
    const double r = (i > 0 ? fabs(sb[i - 1]) : 0.0) + (i + 1 < k ? fabs(sb[i]) : 0.0);
    lo = fmin(lo, sa[i] - r);
    hi = fmax(hi, sa[i] + r);
    scale = fmax(scale, fabs(sa[i]) + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  }
  *scale_out = scale;
  if (hinted) {
    const double pad = 4.0 * 2.3e-16 * scale;
    const double th = fmin(hi, theta_prev + pad);
    const double tl = fmax(lo, theta_prev - 2.0 * r_prev - pad);
    if (th > tl) {
      const double x = lane == 31 ? th : tl + lane * ((th - tl) / 31.0);
      const unsigned has = __ballot_sync(0xffffffffu, sturm_count(sa, sbb, k, x) >= 1);
      if ((has & 1u) == 0u && (has >> 31) != 0u) {  // count(tl) = 0 < count(th): valid bracket
        const int f = __ffs(has) - 1;
        lo = __shfl_sync(0xffffffffu, x, f - 1);
        hi = __shfl_sync(0xffffffffu, x, f);
      } else if ((has >> 31) != 0u) {
        hi = th;
      }
    }
  }
  for (int round = 0; round < 40; ++round) {
    const double w = hi - lo;
    if (!(w > 2.3e-16 * fmax(fabs(lo), fabs(hi)))) break;
    const double x = lo + (lane + 1) * (w / 33.0);
    const unsigned has = __ballot_sync(0xffffffffu, sturm_count(sa, sbb, k, x) >= 1);
    const double nlo = has == 0u ? __shfl_sync(0xffffffffu, x, 31)
                                 : (__ffs(has) >= 2 ? __shfl_sync(0xffffffffu, x, __ffs(has) - 2) : lo);
    const double nhi = has == 0u ? hi : __shfl_sync(0xffffffffu, x, __ffs(has) - 1);
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  return hi;
}

// Eigenvector for an eigenvalue theta at the bottom of the spectrum by a
// twisted factorization (the MRRR eigenvector kernel).  The top-down and
// bottom-up pivots d+_i = P_{i+1}/P_i and d-_i = Q_i/Q_{i+1} come from the
// polynomial recurrences P (top-down minors of T - theta) and Q (bottom-up
// minors), run as division-free FMA chains on thread 0 and thread 32 at the
// same time (stored as value and power-of-two exponent).  Both pivot
// sequences are positive away from the end they approach because every
// leading and trailing principal submatrix has its lowest eigenvalue above
// theta.  Twist r = argmin |gamma_r|, gamma_r = d+_r + d-_r - (a_r - theta);
// x_r = 1, x_i = -(b_i / d+_i) x_{i+1} (i < r), x_i = -(b_{i-1} / d-_i) x_{i-1}
// (i > r): the ratios are formed in parallel, the two products are again two
// concurrent chains.  Unit norm, first nonzero component positive.  Called by
// every thread of the block (>= 2 warps).
struct TwistScratch {
  double pv[LANCZOS_BLOCK + 1], qv[LANCZOS_BLOCK + 1], x[LANCZOS_BLOCK];
  int pe[LANCZOS_BLOCK + 1], qe[LANCZOS_BLOCK + 1];
  int r;
};

__device__ void tridiag_vector_twisted(const double* a, const double* b, const double* bb, int k,
                                       double theta, double scale, TwistScratch& w, double* s) {
  const int t = threadIdx.x, lane = t & 31;
  const double pivmin = (scale > 0 ? scale : 1.0) * 2.3e-16;
  if (t == 0 || t == 32) {
    // t == 0: P_0 = 1, P_1 = a_0 - theta, P_{i+1} = (a_i - theta) P_i - bb_{i-1} P_{i-1}
    // t == 32: Q_k = 1, Q_{k-1} = a_{k-1} - theta, Q_i = (a_i - theta) Q_{i+1} - bb_i Q_{i+2}
    const bool down = t == 0;
    double* v = down ? w.pv : w.qv;
    int* ex = down ? w.pe : w.qe;
    const int first = down ? 0 : k, second = down ? 1 : k - 1;
    double pm = 1.0, p = a[down ? 0 : k - 1] - theta;
    int e_acc = 0;
    v[first] = 1.0;
    ex[first] = 0;
    v[second] = p;
    ex[second] = 0;
    for (int step = 1; step < k; ++step) {
      const int i = down ? step : k - 1 - step;         // row being added
      const double c = down ? bb[i - 1] : bb[i];
      const double pn = fma(a[i] - theta, p, -c * pm);
      pm = p;
      p = pn;
      if ((step & 7) == 7) {
        const double m = fmax(fabs(p), fabs(pm));
        const int e = exponent_of(m);
        if (m > 0.0 && (e > 64 || e < -64)) {
          const double f = pow2(-e);
          p *= f;
          pm *= f;
          e_acc += e;
        }
      }
      const int slot = down ? step + 1 : k - 1 - step;
      v[slot] = p;
      ex[slot] = e_acc;
    }
  }
  __syncthreads();
  if (t < 32) {
    // pivots at r (parallel): d+_r = P_{r+1}/P_r, d-_r = Q_r/Q_{r+1}
    auto dplus = [&](int i) {
      const double d = (w.pv[i + 1] / w.pv[i]) * pow2(w.pe[i + 1] - w.pe[i]);
      return fabs(d) < pivmin || !(d == d) ? pivmin : d;
    };
    auto dminus = [&](int i) {
      const double d = (w.qv[i] / w.qv[i + 1]) * pow2(w.qe[i] - w.qe[i + 1]);
      return fabs(d) < pivmin || !(d == d) ? pivmin : d;
    };
    double best = INFINITY;
    int br = 0;
    for (int r = lane; r < k; r += 32) {
      const double g = fabs(dplus(r) + dminus(r) - (a[r] - theta));
      if (g < best) {
        best = g;
        br = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (ob < best || (ob == best && orr < br)) {
        best = ob;
        br = orr;
      }
    }
    if (lane == 0) w.r = br;
    for (int i = lane; i < k; i += 32)
      w.x[i] = i < br ? -b[i] / dplus(i) : (i > br ? -b[i - 1] / dminus(i) : 1.0);
  }
  __syncthreads();
  const int r = w.r;
  if (t == 0) {  // x_i = ratio_i x_{i+1}, i = r-1 .. 0
    double v = 1.0;
    for (int i = r - 1; i >= 0; --i) {
      v *= w.x[i];
      w.x[i] = v;
    }
  } else if (t == 32) {  // x_i = ratio_i x_{i-1}, i = r+1 .. k-1
    double v = 1.0;
    for (int i = r + 1; i < k; ++i) {
      v *= w.x[i];
      w.x[i] = v;
    }
  }
  __syncthreads();
  if (t < 32) {
    double s2 = 0.0;
    for (int i = lane; i < k; i += 32) s2 += w.x[i] * w.x[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    int first = k;  // deterministic sign: first nonzero component positive
    for (int i = lane; i < k; i += 32)
      if (w.x[i] != 0.0 && i < first) first = i;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    const double sg = (first < k && w.x[first] < 0.0) ? -1.0 : 1.0;
    const double inv = sg / sqrt(s2);
    for (int i = lane; i < k; i += 32) s[i] = w.x[i] * inv;
  }
}

// misc[0] = sqrt(sum partials) (a norm); used to normalise
__global__ void __launch_bounds__(RED_THREADS) norm_kernel(const double* __restrict__ partials,
                                                           int nblocks, double* out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = sqrt(v);
}

// residual of the explicit check: res = sqrt(sum partials); misc[1] = 1e-8/res
__global__ void __launch_bounds__(RED_THREADS) residual_kernel(const double* __restrict__ partials,
                                                               int nblocks, const double* ev,
                                                               double* misc, LanczosStatus* st) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    const double res = sqrt(v);
    st->ev = *ev;
    st->res = res;
    misc[1] = res > 0 ? 1e-8 / res : 0.0;
  }
}

// ---- the restart loop on the device (graph mode) ----
// Prologue of an eigensolve: misc[2] = ||v0||^2 (reduced before); misc[3] =
// ||v0||; control reset; the restart loop runs only for a valid v0
// (linalg.cpp:109-111: InvalidMatrix otherwise).
__global__ void eig_init_kernel(double* misc, LanczosCtl* ctl, int block, int max_iter, double tol,
                                cudaGraphConditionalHandle outer) {
  const double n2 = misc[2];
  const bool ok = n2 > 0;  // false for NaN too
  misc[3] = ok ? sqrt(n2) : 1.0;
  *ctl = LanczosCtl{0, 0, block, max_iter, 0, 0, ok ? 0 : LZ_BAD_V0, 0, tol, INFINITY};
  cudaGraphSetConditional(outer, ok && max_iter > 0 ? 1u : 0u);
}

// Start of a restart cycle (linalg.cpp:126): j = 0, the inner loop armed.
__global__ void eig_cycle_kernel(LanczosCtl* ctl, cudaGraphConditionalHandle inner) {
  ctl->j = 0;
  ctl->cycles += 1;
  ctl->flags &= ~LZ_BREAKDOWN;
  cudaGraphSetConditional(inner, 1u);
}

// Explicit residual check and restart decision (linalg.cpp:156-169), after
// w = H ritz, ev = ritz.w, tmp = w - ev ritz (its norm partials):
// converged -> stop; max_iter reached -> stop, EigenNonConvergence with the
// best residual; otherwise restart from the Ritz vector, on breakdown from
// ritz + 1e-8 tmp / ||tmp|| (misc[1] = that coefficient, else 0).
__global__ void __launch_bounds__(RED_THREADS) eig_decide_kernel(const double* __restrict__ partials,
                                                                 int nblocks, const double* ev,
                                                                 double* misc, LanczosStatus* st,
                                                                 LanczosCtl* ctl,
                                                                 cudaGraphConditionalHandle outer) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    const double res = sqrt(v), e = *ev;
    st->ev = e;
    st->res = res;
    LanczosCtl& c = *ctl;
    c.matvecs += 1;  // the Ritz vector's matvec
    c.best = fmin(c.best, res);
    const bool breakdown = st->bnorm <= 1e-14 * fmax(1.0, fabs(st->theta));
    const bool converged = res <= c.tol * fmax(1.0, fabs(e));
    misc[1] = (!converged && breakdown && res > 0) ? 1e-8 / res : 0.0;
    bool again = false;
    if (converged) {
      c.flags |= LZ_CONVERGED;
    } else {
      if (breakdown) c.flags |= LZ_BREAKDOWN;
      if (c.matvecs >= c.max_iter)
        c.flags |= LZ_NONCONVERGED;
      else
        again = true;
    }
    cudaGraphSetConditional(outer, again ? 1u : 0u);
  }
}

// Converged: out = ritz (when out is another buffer).  Restarting: q_0 =
// ritz, or on breakdown q_0 = (ritz + 1e-8 tmp/||tmp||) / ||.|| (q_0 holds the
// sum and *nrm its norm).
__global__ void eig_restart_kernel(double* __restrict__ q0, const double* __restrict__ ritz,
                                   double* out, long n, const double* __restrict__ nrm,
                                   const LanczosCtl* __restrict__ ctl) {
  const int flags = ctl->flags;
  const bool conv = flags & LZ_CONVERGED, brk = flags & LZ_BREAKDOWN;
  if (conv && out == ritz) return;
  const double f = brk ? 1.0 / *nrm : 0.0;
  for (long x = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<long>(gridDim.x) * blockDim.x) {
    if (conv)
      out[x] = ritz[x];
    else if (brk)
      q0[x] = q0[x] * f;
    else
      q0[x] = ritz[x];
  }
}

int red_blocks(const Ctx&, long n) { return std::max(1, cdiv(n, CHUNK)); }

// ---- fused Lanczos step (one cooperative launch) --------------------------
// After w = H q_j:  h1 = Q^T w (alpha_j = h1[j]);  w <- w - Q h1;  h2 = Q^T w;
// w <- w - Q h2;  beta_j = ||w||;  tridiagonal lowest pair (warp 0 of block 0);
// q_{j+1} = w / beta_j.  Classical Gram-Schmidt twice, equal to the reference's
// MGS (linalg.cpp:131-135) to rounding.  Each block owns a fixed contiguous
// chunk and every block reduces the per-block partials in the same fixed order,
// so all blocks see bit-identical coefficients (deterministic).
//
// The step index j lives on the device (ctl->j) so that one captured step
// (matvec on qcur + this kernel) can be replayed by a graph WHILE node: block 0
// takes the reference's per-step decision (linalg.cpp:141-148: converged
// residual bound, breakdown, end of block, max_iter) and either advances j
// (q_{j+1} also goes to qcur, the matvec input) or ends the loop through
// cudaGraphSetConditional.  The host only looks at the state when the loop ends.
struct OrthArgs {
  double* Q;
  long stride;
  double* w;
  long n;
  double* pa;  // [grid][64] partials of h1
  double* pb;  // [grid][64] partials of h2
  double* pc;  // [grid]     partials of ||w||^2
  double* alpha;
  double* beta;
  double* s;
  double* qcur;
  LanczosStatus* st;
  LanczosCtl* ctl;
  cudaGraphConditionalHandle loop;
  int in_graph;  // 0: host-stepped (profiling mode), the loop handle is not used
  unsigned long long* prof;  // optional clock64 phase totals (block 0), null in production
};

constexpr int ORTH_THREADS = 256;

template <int NT>
__device__ void orth_partials(const double* Q, long stride, int nv, const double* w, long b0,
                              long b1, double* part, double (*sh)[65]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v0 = 0; v0 < nv; v0 += DOT_GROUP) {
    double acc[DOT_GROUP];
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) acc[g] = 0.0;
    for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
      const double wx = w[x];
#pragma unroll
      for (int g = 0; g < DOT_GROUP; ++g)
        if (v0 + g < nv) acc[g] += Q[(v0 + g) * stride + x] * wx;
    }
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) {
      const double r = warp_sum(acc[g]);
      if (lane == 0 && v0 + g < nv) sh[warp][v0 + g] = r;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < NT / 32; ++w8) t += sh[w8][v];
    part[static_cast<long>(v) * gridDim.x + blockIdx.x] = t;  // [v][block]: coalesced reduce
  }
  __syncthreads();
}

// w[x] - sum_i coef[i] Q[i][x], i ascending; the loads of 8 basis vectors are
// issued together (the subtraction order, and so every bit, is unchanged)
__device__ __forceinline__ double project_out(const double* Q, long stride, int nv, const double* coef,
                                              double v, long x) {
  int i = 0;
  for (; i + 8 <= nv; i += 8) {
    double q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = Q[(i + u) * stride + x];
#pragma unroll
    for (int u = 0; u < 8; ++u) v -= coef[i + u] * q[u];
  }
  for (; i < nv; ++i) v -= coef[i] * Q[i * stride + x];
  return v;
}

// sum over blocks of part[v][0..grid) in a fixed order (lane-strided partial
// sums, then a fixed shuffle tree): identical in every block
__device__ __forceinline__ double grid_sum(const double* p, int lane) {
  double t = 0.0;
  for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) t += p[b];
  return warp_sum(t);
}

// every block: coef[v] = sum_b part[v][b]; one warp per coefficient
template <int NT>
__device__ void orth_reduce(const double* part, int nv, double* coef) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v = warp; v < nv; v += NT / 32) {
    const double t = grid_sum(part + static_cast<long>(v) * gridDim.x, lane);
    if (lane == 0) coef[v] = t;
  }
  __syncthreads();
}

// Orthogonalisation + tridiagonal + decision of step j (called by every CTA of
// a cooperative grid; block 0 writes the status and ctl, advancing ctl->j
// unless the loop ends).
// Step j, part 1 (every CTA of a cooperative grid): w <- w - Q (Q^T w) twice,
// beta_j = ||w||, q_{j+1} = w / beta_j into the basis and into qcur (the next
// matvec input); block 0 stores alpha_j, beta_j.
// NT threads per CTA of a cooperative grid.  (A one-cluster variant -- 8 or
// 16 CTAs, hardware cluster barriers, a C-way all-reduce -- measured slower on
// C3: 33k vs 25k cycles per step, the passes lose memory-level parallelism.)
template <int NT>
__device__ void orth_step_t(const OrthArgs& a) {
  __shared__ double sh[NT / 32][65];
  __shared__ double coef[64];
  __shared__ double red[32];
  auto gsync = [] { cg::this_grid().sync(); };
  const int j = a.ctl->j;  // advanced only by the tridiagonal kernel, after this one
  const bool prof = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long c0 = prof ? clock64() : 0;
  const int nv = j + 1;
  const long chunk = (a.n + gridDim.x - 1) / gridDim.x;
  const long b0 = static_cast<long>(blockIdx.x) * chunk, b1 = min(a.n, b0 + chunk);
  // pass 1: h1 = Q^T w
  orth_partials<NT>(a.Q, a.stride, nv, a.w, b0, b1, a.pa, sh);
  const unsigned long long c1 = prof ? clock64() : 0;
  gsync();
  const unsigned long long c2 = prof ? clock64() : 0;
  orth_reduce<NT>(a.pa, nv, coef);
  // pass 2: w <- w - Q h1 ; h2 partials
  double nrm1 = 0.0;  // ||w'||^2 partial, reduced with the second dots
  for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
    const double v = project_out(a.Q, a.stride, nv, coef, a.w[x], x);
    a.w[x] = v;
    nrm1 += v * v;
  }
  nrm1 = block_sum(nrm1, red);
  if (threadIdx.x == 0) a.pb[static_cast<long>(nv) * gridDim.x + blockIdx.x] = nrm1;
  __syncthreads();
  orth_partials<NT>(a.Q, a.stride, nv, a.w, b0, b1, a.pb, sh);
  const double alpha_j = coef[nv - 1];
  gsync();
  orth_reduce<NT>(a.pb, nv + 1, coef);
  // beta_j = ||w' - Q h2|| = sqrt(||w'||^2 - ||h2||^2) (Q orthonormal) when the
  // second projection is small against w' (always, short of an invariant
  // subspace); otherwise the norm is formed explicitly after one more barrier.
  // Every block evaluates the same reduced values: the branch is grid-uniform.
  double h2sq = 0.0;
  for (int i = 0; i < nv; ++i) h2sq = fma(coef[i], coef[i], h2sq);
  const double wn2 = coef[nv];
  const bool pyth = h2sq <= 0.25 * wn2;
  __shared__ double bn_s;
  double nrm = 0.0;
  // pass 3: w <- w - Q h2 (and ||w||^2 partials on the explicit path)
  for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
    const double v = project_out(a.Q, a.stride, nv, coef, a.w[x], x);
    a.w[x] = v;
    nrm += v * v;
  }
  if (!pyth) {
    nrm = block_sum(nrm, red);
    if (threadIdx.x == 0) a.pc[blockIdx.x] = nrm;
    gsync();
    if (threadIdx.x < 32) {
      const double t = grid_sum(a.pc, threadIdx.x);
      if (threadIdx.x == 0) bn_s = sqrt(t);
    }
  } else if (threadIdx.x == 0) {
    bn_s = sqrt(fmax(wn2 - h2sq, 0.0));
  }
  const unsigned long long c3 = prof ? clock64() : 0;
  __syncthreads();
  const double bn = bn_s;
  // q_{j+1} = w / beta_j (unused when the step converges or breaks down)
  if (j + 1 <= LANCZOS_BLOCK && bn > 0) {
    const double inv = 1.0 / bn;
    double* qn = a.Q + (j + 1) * a.stride;
    for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
      const double v = a.w[x] * inv;
      qn[x] = v;
      a.qcur[x] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.alpha[j] = alpha_j;
    a.beta[j] = bn;
    if (prof) {
      a.prof[0] += c1 - c0;  // pass 1 (dots)
      a.prof[1] += c2 - c1;  // grid barrier 1
      a.prof[2] += c3 - c2;  // reduce, pass 2, barrier 2, reduce, pass 3, barrier 3
      a.prof[3] += clock64() - c3;  // ||w||, q_{j+1}
    }
  }
}

// Step j, part 2 (one CTA): lowest eigenpair of T_{j+1}, residual bound and
// the reference's step decision (linalg.cpp:141-148), which advances ctl->j or
// ends the loop.  In the graph it runs concurrently with the speculative
// matvec of q_{j+1} (wasted only on the last step of a cycle).
__device__ void orth_step(const OrthArgs& a) { orth_step_t<ORTH_THREADS>(a); }
__global__ void __launch_bounds__(ORTH_THREADS) lanczos_orth_kernel(OrthArgs a) { orth_step(a); }

__device__ void tridiag_step(const OrthArgs& a) {
  __shared__ double sa[LANCZOS_BLOCK], sb[LANCZOS_BLOCK], sbb[LANCZOS_BLOCK];
  __shared__ double th_s, sc_s;
  __shared__ TwistScratch tw;
  const int j = a.ctl->j;
  const bool prof = a.prof && threadIdx.x == 0;
  const unsigned long long c4 = prof ? clock64() : 0;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    const double bi = a.beta[i];
    sa[i] = a.alpha[i];
    sb[i] = bi;
    sbb[i] = bi * bi;
  }
  __syncthreads();
  const int k = j + 1;
  const double alpha_j = sa[j], bn = sb[j];
  if (threadIdx.x < 32) {
    double theta = sa[0], scale = fabs(sa[0]);
    if (k > 1) {
      // the previous step's Ritz value / residual bound (this cycle's step j-1)
      const double theta_prev = a.st->theta, r_prev = a.st->res_bound;
      __syncwarp();
      theta = tridiag_lowest_value(sa, sb, sbb, k, true, theta_prev, r_prev, &scale);
    }
    if (threadIdx.x == 0) {
      th_s = theta;
      sc_s = scale;
    }
  }
  __syncthreads();
  const double theta = th_s, scale = sc_s;
  const unsigned long long c45 = prof ? clock64() : 0;
  if (k > 1)
    tridiag_vector_twisted(sa, sb, sbb, k, theta, scale, tw, a.s);
  else if (threadIdx.x == 0)
    a.s[0] = 1.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (prof) {
      const unsigned long long c5 = clock64();
      a.prof[7] += c5 - c45;  // eigenvector
      a.prof[4] += c5 - c4;   // tridiagonal eigenpair
      a.prof[5] += 1;
      a.prof[6] += static_cast<unsigned long long>(k);
    }
    const double res_bound = bn * fabs(a.s[j]);
    a.st->theta = theta;
    a.st->bnorm = bn;
    a.st->alpha = alpha_j;
    a.st->res_bound = res_bound;
    LanczosCtl& c = *a.ctl;
    const int matvecs = c.matvecs + 1;
    const double tscale = fmax(1.0, fabs(theta));
    const bool breakdown = bn <= 1e-14 * tscale;
    const bool stop = res_bound <= c.tol * tscale || breakdown || j + 1 == c.block ||
                      matvecs >= c.max_iter;
    c.matvecs = matvecs;
    c.steps += 1;
    if (!stop) c.j = j + 1;
    if (a.in_graph) cudaGraphSetConditional(a.loop, stop ? 0u : 1u);
  }
}

__global__ void __launch_bounds__(ORTH_THREADS) lanczos_tridiag_kernel(OrthArgs a) { tridiag_step(a); }

// One Lanczos step for chi <= 128 as ONE cooperative launch (the graph body):
// the orthogonalisation on every CTA, one grid barrier, then CTA 0 solves the
// tridiagonal problem and takes the step decision while the other CTAs run
// the fused H_eff matvec of q_{j+1} (heff_phases.cuh) with barriers over
// themselves only.  Replaces orth -> fork(tridiag || heff) -> join: two
// cooperative launches and the fork/join edges per step.
struct FusedStepArgs {
  OrthArgs o;
  hs::HsArgs h;
  unsigned* bar;  // arrival counter of the matvec CTAs (reset by CTA 0 each launch)
};

__device__ __forceinline__ void sub_grid_sync(unsigned* ctr, unsigned n, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += n;
    __threadfence();
    atomicAdd(ctr, 1u);
    while (*reinterpret_cast<volatile unsigned*>(ctr) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(ORTH_THREADS) lanczos_step_small_kernel(FusedStepArgs f) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ hs::MixSmem w;
  cg::grid_group grid = cg::this_grid();
  orth_step(f.o);
  if (blockIdx.x == 0 && threadIdx.x == 0) *f.bar = 0u;
  grid.sync();
  if (blockIdx.x == 0) {
    tridiag_step(f.o);
    return;
  }
  double* As = reinterpret_cast<double*>(dyn);
  double* Bs = As + hs::HS_TM * hs::hs_ld<hs::HS_KMAX>();
  hs::load_mix(f.h.mix, w);
  __syncthreads();
  const int blk = blockIdx.x - 1, nblk = gridDim.x - 1;
  unsigned target = 0;
  hs::phase_a<hs::HS_KMAX>(f.h, w, f.h.theta, As, Bs, blk, nblk);
  sub_grid_sync(f.bar, static_cast<unsigned>(nblk), target);
  hs::phase_b<hs::HS_KMAX>(f.h, As, Bs, blk, nblk);
  sub_grid_sync(f.bar, static_cast<unsigned>(nblk), target);
  hs::phase_c(f.h, f.h.out, blk, nblk);
}

// ---- persistent eigensolve for small blocks (chi <= 128) -----------------
// The whole restarted Lanczos of one eigs_lowest call as ONE cooperative
// launch: W worker CTAs run every phase of every step -- the fused H_eff
// matvec (heff_phases.cuh phases A and B; phase C is folded into the first
// orthogonalisation pass), the CGS2 orthogonalisation, the Ritz vector, the
// explicit residual check and the restart -- separated by a barrier among the
// workers; one more CTA (the "tridiagonal CTA") solves the tridiagonal
// eigenproblem of each step concurrently and posts the reference's step
// decision (linalg.cpp:141-148).  The workers run the next step
// speculatively and read the decision of step j at the end of step j+1 (a
// step later), so the tridiagonal solve is off their critical path; a step
// computed after the loop should have stopped is discarded (its matvec is not
// counted).  Deterministic stops (end of block, max_iter) are known without
// the decision.  This replaces per-step kernel launches, the graph's
// conditional loop and the fork/join to the tridiagonal stream with barriers.
constexpr int PZ_THREADS = hs::HS_THREADS;  // 256, = ORTH_THREADS

struct PzArgs {
  hs::HsArgs h;          // L, R, mix, dims; theta/out unused (set per matvec)
  double* Q;             // basis, LANCZOS_BLOCK + 1 vectors at stride
  long stride;
  double* w;             // matvec output / orthogonalised vector
  double* ritz;
  double* tmp;
  const double* v0;
  double* out;
  long n;                // padded two-site length
  double* pa;            // [64][W] partials
  double* pb;            // [65][W]
  double* pc;            // [W]
  double* alpha;         // [64]
  double* beta;          // [64]
  double* sbuf;          // [2][64] tridiagonal eigenvectors by job parity
  double* tres;          // [2][4] theta, res_bound, bnorm, alpha by job parity
  int* dec;              // [2] stop decision by job parity
  int* job;              // [2][2] (j, matvecs before the cycle) by job parity
  unsigned* posted;      // jobs posted (seq)
  unsigned* done;        // jobs finished by the tridiagonal CTA
  unsigned* bar;         // [2] worker barrier: arrivals, generation
  LanczosCtl* ctl;
  LanczosStatus* st;
  double tol;
  int block, max_iter;
  int W;                 // worker CTAs; CTA W is the tridiagonal CTA
  unsigned long long* prof;  // optional clock64 phase totals of worker 0 (ACHI_LANCZOS_PROF)
  LanczosResult* res_host;   // pinned: the outcome for the host, written by the kernel itself
  int lazy;                  // next matvec from w'/beta (see the step loop), no q_{j+1} barrier
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// barrier among the W worker CTAs: one monotonic arrival counter (zeroed per
// launch); arrival is a release reduction, the wait an acquire poll for
// W * (barriers passed so far)
__device__ __forceinline__ void pz_sync(const PzArgs& a, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (gen + 1u) * static_cast<unsigned>(a.W);
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.bar), "r"(1u) : "memory");
    while (ld_acquire(a.bar) < target) {
    }
  }
  ++gen;
  __syncthreads();
}

// every worker: sum over workers of part[v][0..W) for v < nv (fixed order)
__device__ void pz_reduce(const double* part, int nv, int W, double* coef) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v = warp; v < nv; v += PZ_THREADS / 32) {
    double t = 0.0;
    for (int b = lane; b < W; b += 32) t += __ldcg(part + static_cast<long>(v) * W + b);
    t = warp_sum(t);
    if (lane == 0) coef[v] = t;
  }
  __syncthreads();
}

// block partial of sum_x f(x) over [b0, b1) -> part[rank] (thread 0 writes)
__device__ __forceinline__ void pz_put(double v, double* part, int rank, double* red) {
  v = block_sum(v, red);
  if (threadIdx.x == 0) part[rank] = v;
}

// partial dots of w against q_0..q_{nv-1} over [b0, b1) -> part[v][rank];
// also self-dot w.w -> part[nv][rank] when self
__device__ void pz_dots(const PzArgs& a, int nv, long b0, long b1, int rank, double* part, bool self,
                        double (*sh)[65]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = nv + (self ? 1 : 0);
  for (int v0 = 0; v0 < nt; v0 += DOT_GROUP) {
    double acc[DOT_GROUP];
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) acc[g] = 0.0;
    for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
      const double wx = a.w[x];
#pragma unroll
      for (int g = 0; g < DOT_GROUP; ++g) {
        const int v = v0 + g;
        if (v < nv)
          acc[g] += a.Q[v * a.stride + x] * wx;
        else if (v == nv && self)
          acc[g] += wx * wx;
      }
    }
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) {
      const double r = warp_sum(acc[g]);
      if (lane == 0 && v0 + g < nt) sh[warp][v0 + g] = r;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nt; v += PZ_THREADS) {
    double t = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < PZ_THREADS / 32; ++w8) t += sh[w8][v];
    part[static_cast<long>(v) * a.W + rank] = t;
  }
  __syncthreads();
}

// One pass over the worker's chunk for nv <= PZ_FUSE basis vectors, every Q
// value loaded once and held in registers: the vector is either formed from
// the matvec partials (first = true: w = sum_e P_e, phase C) or projected
// (w <- w - Q coef, ||w'||^2 -> part[nv][rank]); then the partial dots
// Q^T w -> part[v][rank].  Same per-element operation order as pz_w /
// project_out + pz_dots.
constexpr int PZ_FUSE = 16;
__device__ __forceinline__ double pz_w(const hs::HsArgs& h, long tot, long x) {
  double v = 0.0;
  for (int e = 0; e < h.D3; ++e) v += h.part[e * tot + x];
  return v;
}
__device__ void pz_fused_pass(const PzArgs& a, const hs::HsArgs& h, long tot, int nv, bool first,
                              const double* coef, long b0, long b1, int rank, double* part,
                              double (*sh)[65], double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[PZ_FUSE];
#pragma unroll
  for (int i = 0; i < PZ_FUSE; ++i) acc[i] = 0.0;
  double nrm = 0.0;
  for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
    double q[PZ_FUSE];
#pragma unroll
    for (int i = 0; i < PZ_FUSE; ++i) q[i] = i < nv ? a.Q[i * a.stride + x] : 0.0;
    double v;
    if (first) {
      v = pz_w(h, tot, x);
    } else {
      v = a.w[x];
#pragma unroll
      for (int i = 0; i < PZ_FUSE; ++i)
        if (i < nv) v -= coef[i] * q[i];
      nrm += v * v;
    }
    a.w[x] = v;
#pragma unroll
    for (int i = 0; i < PZ_FUSE; ++i) acc[i] += q[i] * v;
  }
#pragma unroll
  for (int i = 0; i < PZ_FUSE; ++i) {
    const double r = warp_sum(acc[i]);
    if (lane == 0 && i < nv) sh[warp][i] = r;
  }
  if (!first) {
    nrm = block_sum(nrm, red);  // (block_sum synchronises the CTA)
    if (threadIdx.x == 0) part[static_cast<long>(nv) * a.W + rank] = nrm;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += PZ_THREADS) {
    double t = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < PZ_THREADS / 32; ++w8) t += sh[w8][v];
    part[static_cast<long>(v) * a.W + rank] = t;
  }
  __syncthreads();
}

// matvec w = H theta over the workers: phases A and B of heff_phases.cuh with
// a barrier after each; the caller folds phase C (sum over e) into its next
// elementwise pass via pz_w().
__device__ void pz_matvec(const PzArgs& a, hs::HsArgs& h, const hs::MixSmem& mw, const double* theta,
                          double* As, double* Bs, int rank, unsigned& gen, double* Lc, double* Rc) {
  hs::phase_a<hs::HS_KMAX>(h, mw, theta, As, Bs, rank, a.W, nullptr, Lc, false);
  pz_sync(a, gen);
  hs::phase_b<hs::HS_KMAX>(h, As, Bs, rank, a.W, Rc, false);
  pz_sync(a, gen);
}

// the tridiagonal CTA: one job per step (j, matvecs before the cycle); the
// lowest pair of T_{j+1} (hinted by the previous step of the same cycle), the
// residual bound and the stop decision, posted by job parity.
__device__ void pz_tridiag_cta(const PzArgs& a) {
  __shared__ double sa[LANCZOS_BLOCK], sb[LANCZOS_BLOCK], sbb[LANCZOS_BLOCK];
  __shared__ double th_s, sc_s;
  __shared__ int jj_s, mv_s;
  __shared__ TwistScratch tw;
  unsigned seq = 0;
  double theta_prev = 0.0, r_prev = 0.0;
  for (;;) {
    if (threadIdx.x == 0) {
      while (ld_acquire(a.posted) <= seq) __nanosleep(32);
      const int p = (seq + 1) & 1;
      jj_s = *reinterpret_cast<volatile int*>(&a.job[2 * p]);
      mv_s = *reinterpret_cast<volatile int*>(&a.job[2 * p + 1]);
    }
    __syncthreads();
    ++seq;
    const int j = jj_s, mv0 = mv_s;
    if (j < 0) return;  // the workers are done
    const int p = seq & 1;
    for (int i = threadIdx.x; i <= j; i += blockDim.x) {
      const double bi = __ldcg(a.beta + i);
      sa[i] = __ldcg(a.alpha + i);
      sb[i] = bi;
      sbb[i] = bi * bi;
    }
    __syncthreads();
    const int k = j + 1;
    double* s = a.sbuf + 64 * p;
    if (threadIdx.x < 32) {
      double theta = sa[0], scale = fabs(sa[0]);
      if (k > 1) theta = tridiag_lowest_value(sa, sb, sbb, k, true, theta_prev, r_prev, &scale);
      if (threadIdx.x == 0) {
        th_s = theta;
        sc_s = scale;
      }
    }
    __syncthreads();
    const double theta = th_s, scale = sc_s;
    if (k > 1)
      tridiag_vector_twisted(sa, sb, sbb, k, theta, scale, tw, s);
    else if (threadIdx.x == 0)
      s[0] = 1.0;
    __syncthreads();
    const double bn = sb[j];
    const double res_bound = bn * fabs(s[j]);
    theta_prev = theta;
    r_prev = res_bound;
    if (threadIdx.x == 0) {
      const double tscale = fmax(1.0, fabs(theta));
      const bool breakdown = bn <= 1e-14 * tscale;
      const bool stop = res_bound <= a.tol * tscale || breakdown || j + 1 == a.block ||
                        mv0 + j + 1 >= a.max_iter;
      double* r = a.tres + 4 * p;
      r[0] = theta;
      r[1] = res_bound;
      r[2] = bn;
      r[3] = sa[j];
      a.dec[p] = stop ? 1 : 0;
      __threadfence();
      st_release(a.done, seq);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PZ_THREADS) lanczos_persistent_kernel(PzArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ hs::MixSmem mw;
  __shared__ double sh[PZ_THREADS / 32][65];
  __shared__ double coef[66];
  __shared__ double red[32];
  __shared__ double scal[8];
  const int rank = blockIdx.x;
  if (rank == a.W) {
    pz_tridiag_cta(a);
    return;
  }
  double* As = reinterpret_cast<double*>(dyn);
  double* Bs = As + hs::HS_TM * hs::hs_ld<hs::HS_KMAX>();
  // L and R tiles of this worker's first items, kept for the whole eigensolve
  double* Lc = Bs + hs::HS_TN * hs::hs_ld<hs::HS_KMAX>();
  double* Rc = Lc + hs::HS_TM * hs::hs_ld<hs::HS_KMAX>();
  bool cfill = true;
  hs::load_mix(a.h.mix, mw);
  hs::HsArgs h = a.h;
  const long n = a.n, tot = n;
  const long chunk = (n + a.W - 1) / a.W;
  const long b0 = static_cast<long>(rank) * chunk, b1 = min(n, b0 + chunk);
  unsigned gen = 0, seq = 0;
  auto post = [&](int j, int mv0) {  // worker 0 posts step j to the tridiagonal CTA
    if (rank == 0 && threadIdx.x == 0) {
      const int p = (seq + 1) & 1;
      a.job[2 * p] = j;
      a.job[2 * p + 1] = mv0;
      __threadfence();
      st_release(a.posted, seq + 1);
    }
    ++seq;
  };
  auto wait_done = [&](unsigned s) {
    if (threadIdx.x == 0)
      while (ld_acquire(a.done) < s) __nanosleep(32);
    __syncthreads();
  };
  auto finish = [&](int flags, int matvecs, int steps, int cycles, double best, double ev, double res,
                    const double* tr) {
    if (rank == 0 && threadIdx.x == 0) {
      LanczosCtl& c = *a.ctl;
      c.flags = flags;
      c.matvecs = matvecs;
      c.steps = steps;
      c.cycles = cycles;
      c.best = best;
      c.tol = a.tol;
      c.block = a.block;
      c.max_iter = a.max_iter;
      a.st->ev = ev;
      a.st->res = res;
      if (tr) {
        a.st->theta = __ldcg(tr);
        a.st->res_bound = __ldcg(tr + 1);
        a.st->bnorm = __ldcg(tr + 2);
        a.st->alpha = __ldcg(tr + 3);
      }
      a.res_host->ctl = c;
      a.res_host->st = *a.st;
    }
    post(-1, 0);  // release the tridiagonal CTA
  };
  // ---- prologue: q_0 = v0 / ||v0|| (linalg.cpp:109-115) ----
  {
    double v = 0.0;
    for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) v += a.v0[x] * a.v0[x];
    pz_put(v, a.pc, rank, red);
    pz_sync(a, gen);
    pz_reduce(a.pc, 1, a.W, coef);
    const double n2 = coef[0];
    if (!(n2 > 0)) {
      finish(LZ_BAD_V0, 0, 0, 0, INFINITY, 0.0, 0.0, nullptr);
      return;
    }
    const double inv = 1.0 / sqrt(n2);
    for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.Q[x] = a.v0[x] * inv;
    pz_sync(a, gen);
  }
  int matvecs = 0, steps = 0, cycles = 0;
  double best = INFINITY;
  for (;;) {  // restart cycles (linalg.cpp:126-170)
    ++cycles;
    const int mv0 = matvecs;
    int j = 0, k = 0;
    unsigned seq_last = 0;  // job of the final step
    double inv_prev = 1.0;  // 1 / beta_{j-1} (lazy matvec input)
    for (;; ++j) {
      // ---- step j: w = H q_j, orthogonalise, q_{j+1} ----
      const bool pf = a.prof && rank == 0 && threadIdx.x == 0;
      unsigned long long t0 = pf ? clock64() : 0, t1 = 0;
      auto mark = [&](int slot) {
        if (pf) {
          t1 = clock64();
          a.prof[slot] += t1 - t0;
          t0 = t1;
        }
      };
      // lazy: the matvec input of step j >= 1 is w'/beta_{j-1} (w' = w after the first
      // projection, complete since the previous step's last barrier) instead of the stored
      // q_j = (w' - Q c2) / beta_{j-1}; they differ by the second projection (rounding-level
      // components along the basis, which the full reorthogonalisation removes from the
      // next w anyway), and q_j itself is written by each worker into its own slice of Q
      const bool from_w = a.lazy && j > 0;
      hs::phase_a<hs::HS_KMAX>(h, mw, from_w ? a.w : a.Q + j * a.stride, As, Bs, rank, a.W,
                               pf ? a.prof + 12 : nullptr, Lc, cfill, from_w ? inv_prev : 1.0);
      mark(0);
      pz_sync(a, gen);
      mark(1);
      hs::phase_b<hs::HS_KMAX>(h, As, Bs, rank, a.W, Rc, cfill);
      cfill = false;
      mark(2);
      pz_sync(a, gen);
      mark(3);
      const int nv = j + 1;
      if (nv <= PZ_FUSE) {
        pz_fused_pass(a, h, tot, nv, true, coef, b0, b1, rank, a.pa, sh, red);
      } else {
        for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.w[x] = pz_w(h, tot, x);
        // (each thread reads back only the w[x] it wrote)
        pz_dots(a, nv, b0, b1, rank, a.pa, false, sh);
      }
      mark(4);
      pz_sync(a, gen);
      mark(5);
      pz_reduce(a.pa, nv, a.W, coef);
      const double alpha_j = coef[nv - 1];
      if (nv <= PZ_FUSE) {
        pz_fused_pass(a, h, tot, nv, false, coef, b0, b1, rank, a.pb, sh, red);
      } else {
        double nrm1 = 0.0;
        for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
          const double v = project_out(a.Q, a.stride, nv, coef, a.w[x], x);
          a.w[x] = v;
          nrm1 += v * v;
        }
        nrm1 = block_sum(nrm1, red);
        if (threadIdx.x == 0) a.pb[static_cast<long>(nv) * a.W + rank] = nrm1;
        __syncthreads();
        pz_dots(a, nv, b0, b1, rank, a.pb, false, sh);
      }
      mark(6);
      pz_sync(a, gen);
      mark(7);
      pz_reduce(a.pb, nv + 1, a.W, coef);
      double h2sq = 0.0;
      for (int i = 0; i < nv; ++i) h2sq = fma(coef[i], coef[i], h2sq);
      const double wn2 = coef[nv];
      const bool pyth = h2sq <= 0.25 * wn2;
      double nrm = 0.0;
      double* w2 = a.lazy ? a.tmp : a.w;  // lazy: w' stays in w for the next matvec
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
        const double v = project_out(a.Q, a.stride, nv, coef, a.w[x], x);
        w2[x] = v;
        nrm += v * v;
      }
      double bn;
      if (!pyth) {
        pz_put(nrm, a.pc, rank, red);
        pz_sync(a, gen);
        pz_reduce(a.pc, 1, a.W, scal);
        bn = sqrt(scal[0]);
      } else {
        bn = sqrt(fmax(wn2 - h2sq, 0.0));
      }
      inv_prev = bn > 0 ? 1.0 / bn : 0.0;
      if (j + 1 <= LANCZOS_BLOCK && bn > 0) {
        const double inv = 1.0 / bn;
        double* qn = a.Q + (j + 1) * a.stride;
        for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) qn[x] = w2[x] * inv;
      }
      if (rank == 0 && threadIdx.x == 0) {
        a.alpha[j] = alpha_j;
        a.beta[j] = bn;
      }
      __syncthreads();
      mark(8);
      post(j, mv0);
      const unsigned seq_j = seq;
      if (!a.lazy) pz_sync(a, gen);  // q_{j+1} complete (lazy: w' was, at the last barrier)
      else __syncthreads();
      mark(9);
      ++steps;
      // the decision of step j-1 (posted one step ago)
      if (j >= 1) {
        wait_done(seq_j - 1);
        mark(10);
        if (pf) a.prof[11] += 1;
        if (__ldcg(a.dec + ((seq_j - 1) & 1))) {  // stopped at j-1: this step is discarded
          k = j;
          seq_last = seq_j - 1;
          --steps;
          break;
        }
      }
      if (j + 1 == a.block || mv0 + j + 1 >= a.max_iter) {  // stops at j regardless
        wait_done(seq_j);
        k = j + 1;
        seq_last = seq_j;
        break;
      }
    }
    matvecs = mv0 + k;
    // ---- Ritz vector r = normalize(Q s), s from step k-1 (linalg.cpp:154-155) ----
    const double* s = a.sbuf + 64 * (seq_last & 1);
    const double* tr = a.tres + 4 * (seq_last & 1);
    for (int i = threadIdx.x; i < k; i += PZ_THREADS) coef[i] = __ldcg(s + i);
    __syncthreads();
    {
      double v = 0.0;
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
        double r = 0.0;
        for (int i = 0; i < k; ++i) r += coef[i] * a.Q[i * a.stride + x];
        a.ritz[x] = r;
        v += r * r;
      }
      pz_put(v, a.pc, rank, red);
      pz_sync(a, gen);
      pz_reduce(a.pc, 1, a.W, scal);
      const double inv = 1.0 / sqrt(scal[0]);
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.ritz[x] *= inv;
      pz_sync(a, gen);
    }
    // ---- explicit residual (linalg.cpp:156-162): w = H r, ev = r.w, ||w - ev r|| ----
    pz_matvec(a, h, mw, a.ritz, As, Bs, rank, gen, Lc, Rc);
    ++matvecs;
    {
      double v = 0.0;
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
        const double wx = pz_w(h, tot, x);
        a.w[x] = wx;
        v += a.ritz[x] * wx;
      }
      pz_put(v, a.pc, rank, red);
      pz_sync(a, gen);
      pz_reduce(a.pc, 1, a.W, scal);
    }
    const double ev = scal[0];
    {
      double v = 0.0;
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
        const double t = a.w[x] - ev * a.ritz[x];
        a.tmp[x] = t;
        v += t * t;
      }
      pz_put(v, a.pa, rank, red);
      pz_sync(a, gen);
      pz_reduce(a.pa, 1, a.W, scal + 1);
    }
    const double res = sqrt(scal[1]);
    best = fmin(best, res);
    if (res <= a.tol * fmax(1.0, fabs(ev))) {
      if (a.out != a.ritz)
        for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.out[x] = a.ritz[x];
      finish(LZ_CONVERGED, matvecs, steps, cycles, best, ev, res, tr);
      return;
    }
    if (matvecs >= a.max_iter) {
      finish(LZ_NONCONVERGED, matvecs, steps, cycles, best, ev, res, tr);
      return;
    }
    // ---- restart (linalg.cpp:163-169) ----
    const bool breakdown = __ldcg(tr + 2) <= 1e-14 * fmax(1.0, fabs(__ldcg(tr)));
    if (breakdown) {
      const double f = res > 0 ? 1e-8 / res : 0.0;
      double v = 0.0;
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) {
        const double q = a.ritz[x] + f * a.tmp[x];
        a.Q[x] = q;
        v += q * q;
      }
      pz_put(v, a.pb, rank, red);
      pz_sync(a, gen);
      pz_reduce(a.pb, 1, a.W, scal + 2);
      const double inv = 1.0 / sqrt(scal[2]);
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.Q[x] *= inv;
    } else {
      for (long x = b0 + threadIdx.x; x < b1; x += PZ_THREADS) a.Q[x] = a.ritz[x];
    }
    pz_sync(a, gen);
  }
}

struct Kernels {
  Ctx& ctx;
  LanczosWs& ws;
  long n;
  int nb;
  // h[0..nv) = Q[0..nv)^T w
  void dots(const double* Q, int nv, const double* w, double* h) {
    multi_dot_kernel<<<nb, RED_THREADS, 0, ctx.stream>>>(Q, ws.stride, nv, w, n, ws.partials.p, 64, 0);
    ACHI_LAUNCHED(ctx);
    reduce_partials_kernel<<<nv, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, nb, 64, nv, h);
    ACHI_LAUNCHED(ctx);
  }
  // dst = src + sign * Q c ; norm partials -> ws.partials (first nb entries)
  void axpy(const double* Q, int nv, const double* c, double sign, const double* src, double* dst,
            bool norm, const LanczosCtl* nv_ctl = nullptr) {
    multi_axpy_kernel<<<nb, RED_THREADS, 0, ctx.stream>>>(Q, ws.stride, nv, c, sign, src, dst, n,
                                                          norm ? ws.partials.p : nullptr, nv_ctl);
    ACHI_LAUNCHED(ctx);
  }
  void scale(double* dst, const double* src, const double* s, bool invert) {
    const int blocks = static_cast<int>(std::min<long>(cdiv(n, 256), 4L * ctx.num_sms));
    scale_kernel<<<blocks, 256, 0, ctx.stream>>>(dst, src, n, s, invert ? 1 : 0);
    ACHI_LAUNCHED(ctx);
  }
  void norm_from_partials(double* out) {
    norm_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, nb, out);
    ACHI_LAUNCHED(ctx);
  }
  LanczosStatus read_status() {
    LanczosStatus* hst = ctx.status.reserve(1);
    ACHI_CUDA(cudaMemcpyAsync(hst, ws.misc() + 8, sizeof(LanczosStatus), cudaMemcpyDeviceToHost,
                              ctx.stream));
    ctx.sync();
    return *hst;
  }
  LanczosStatus* dev_status() { return reinterpret_cast<LanczosStatus*>(ws.misc() + 8); }
};

}  // namespace

void LanczosGraph::reset() {
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  exec = nullptr;
  graph = nullptr;
  key = 0;
  body_launches = 0;
}

LanczosWs::~LanczosWs() {
  for (auto& g : graphs) g.reset();
}

void LanczosWs::reserve(long n) {
  const long s = (n + 31) & ~31L;  // 256-byte aligned vectors
  if (s > stride || basis.p == nullptr) {
    for (auto& g : graphs) g.reset();  // captured pointers would dangle
    stride = s;
    basis.reserve(static_cast<size_t>(LANCZOS_BLOCK + 1) * s);
    w.reserve(s);
    ritz.reserve(s);
    tmp.reserve(s);
    qcur.reserve(s);
    // reduction partials: multi-dot (64 per CHUNK block) and the fused
    // orthogonalisation (129 per block, at most 2 blocks per SM)
    partials.reserve(std::max<size_t>(64L * cdiv(s, CHUNK) + 1024, 129L * 2 * 160 + 64));
    scal.reserve(512);
    ctl.reserve(1);
    ctl_h.reserve(1);
    res_h.reserve(1);
  }
}

void device_norm2(Ctx& ctx, const double* x, long n, double* result, double* part) {
  const int nb = red_blocks(ctx, n);
  if (!part) part = ctx.red.reserve(static_cast<size_t>(nb) * 2 + 8);
  multi_dot_kernel<<<nb, RED_THREADS, 0, ctx.stream>>>(x, 0, 0, x, n, part, 1, 1);
  ACHI_LAUNCHED(ctx);
  reduce_partials_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(part, nb, 1, 1, result);
  ACHI_LAUNCHED(ctx);
}

void device_scale(Ctx& ctx, double* dst, const double* src, long n, const double* scale, bool invert) {
  const int blocks = static_cast<int>(std::min<long>(cdiv(n, 256), 4L * ctx.num_sms));
  scale_kernel<<<blocks, 256, 0, ctx.stream>>>(dst, src, n, scale, invert ? 1 : 0);
  ACHI_LAUNCHED(ctx);
}

void eigs_lowest_async(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                       const double* v0, double tol, int max_iter, double* out, int graph_slot,
                       uint64_t graph_key, const HeffOps* small_op) {
  ws.reserve(n);
  Kernels K{ctx, ws, n, red_blocks(ctx, n)};
  double* misc = ws.misc();
  const int block = static_cast<int>(std::min<long>(dim, LANCZOS_BLOCK));
  const int orth_max = per_device_once("lanczos_orth_kernel", ctx.device, [&] {
    int per_sm = 0;
    ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lanczos_orth_kernel,
                                                            ORTH_THREADS, 0));
    return std::max(1, std::min(per_sm, 2)) * ctx.num_sms;
  });
  // fixed for a given n: the chunking (and so every reduction order) is deterministic
  // (about one element per thread up to two CTAs per SM: the passes are latency-bound)
  static const bool graph_default = [] {
    const char* e = std::getenv("ACHI_LANCZOS_GRAPH");
    return !(e && e[0] == '0');
  }();
  // (the emulated-FP64 engine sizes its digit workspace per call: no graph capture)
  const bool use_graph = ctx.ozaki_slices == 0 &&
                         (ctx.lanczos_graph >= 0 ? ctx.lanczos_graph != 0 : graph_default);
  ws.pend_graph = use_graph;
  // ACHI_LANCZOS_FUSED=1 (opt-in): for chi <= 128 in graph mode the whole step is
  // one cooperative launch (lanczos_step_small_kernel) over max(orthogonalisation
  // grid, matvec items + 1) CTAs.  Measured slower on C3 (Lanczos 0.134 vs 0.122
  // s/sweep at sweep 7): one CTA per SM for the combined kernel and a smaller
  // matvec grid cost more than the launch and fork/join it saves.
  static const bool fused_on = [] {
    const char* e = std::getenv("ACHI_LANCZOS_FUSED");
    return e && e[0] == '1';
  }();
  hs::HsArgs fused_h{};
  long fused_items = 0;
  const bool fused = use_graph && fused_on && small_op &&
                     heff_small_fusable(ctx, *small_op, ws.qcur.p, ws.w.p, &fused_h, &fused_items);
  const int fused_max = !fused ? 0 : per_device_once("lanczos_step_small_kernel", ctx.device, [&] {
    const size_t fsm = hs::smem_bytes<hs::HS_KMAX>();
    ACHI_CUDA(cudaFuncSetAttribute(lanczos_step_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(fsm)));
    int per_sm = 0;
    ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lanczos_step_small_kernel,
                                                            ORTH_THREADS, fsm));
    return std::max(1, per_sm) * ctx.num_sms;
  });
  const int orth_grid =
      fused ? std::max(2, ctx.cap_grid(std::min<long>(
                              std::max<long>(cdiv(n, ORTH_THREADS), fused_items + 1), fused_max)))
            : std::max(1, ctx.cap_grid(std::min<long>(cdiv(n, ORTH_THREADS), orth_max)));
  if (fused) ws.bar.reserve(1);
  const size_t need_part = static_cast<size_t>(129) * orth_grid + 64;
  if (ws.partials.cap < need_part) {
    for (auto& g : ws.graphs) g.reset();
    ws.partials.reserve(need_part);
  }

  // ---- the inner loop as a graph: WHILE { apply(qcur -> w); orth + decide } ----
  // ACHI_LANCZOS_GRAPH=0 steps the same kernels from the host instead (ncu cannot
  // profile kernel nodes of graphs with conditional nodes).
  // ACHI_LANCZOS_PROF=1: clock64 phase split of the fused step, printed every 200 calls
  static const bool prof_on = std::getenv("ACHI_LANCZOS_PROF") != nullptr;
  static DevArr<unsigned long long> prof_buf;
  static PinnedArr<unsigned long long> prof_h;
  static thread_local long prof_calls = 0;
  if (prof_on && !prof_buf.p) {
    prof_buf.reserve(16);
    prof_h.reserve(8);
    ACHI_CUDA(cudaMemsetAsync(prof_buf.p, 0, 16 * sizeof(unsigned long long), ctx.stream));
  }
  if (prof_on && ++prof_calls % 200 == 0) {
    ACHI_CUDA(cudaMemcpyAsync(prof_h.p, prof_buf.p, 8 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const double s = prof_h.p[5] ? static_cast<double>(prof_h.p[5]) : 1.0;
    std::fprintf(stderr,
                 "[lanczos] steps=%llu avg_k=%.1f grid=%d cycles/step: dots %.0f bar1 %.0f "
                 "rest %.0f norm+q %.0f tridiag %.0f (of which inverse iteration %.0f)\n",
                 prof_h.p[5], prof_h.p[6] / s, orth_grid, prof_h.p[0] / s, prof_h.p[1] / s,
                 prof_h.p[2] / s, prof_h.p[3] / s, prof_h.p[4] / s, prof_h.p[7] / s);
  }
  auto orth_args = [&](cudaGraphConditionalHandle handle, int in_graph) {
    return OrthArgs{ws.q(0), ws.stride, ws.w.p, n,
                    ws.partials.p, ws.partials.p + 64L * orth_grid, ws.partials.p + 128L * orth_grid,
                    ws.alpha(), ws.beta(), ws.s(), ws.qcur.p, K.dev_status(), ws.ctl.p, handle, in_graph,
                    prof_on ? prof_buf.p : nullptr};
  };
  auto launch_orth = [&](cudaGraphConditionalHandle handle, int in_graph) {
    const OrthArgs oa = orth_args(handle, in_graph);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(orth_grid);
    lc.blockDim = dim3(ORTH_THREADS);
    lc.stream = ctx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    ACHI_CUDA(cudaLaunchKernelEx(&lc, lanczos_orth_kernel, oa));
    ACHI_LAUNCHED(ctx);
    return oa;
  };
  auto launch_tridiag = [&](const OrthArgs& oa, cudaStream_t s) {
    lanczos_tridiag_kernel<<<1, ORTH_THREADS, 0, s>>>(oa);
    ACHI_LAUNCHED(ctx);
  };
  LanczosGraph local;
  struct LocalGuard {
    LanczosGraph& g;
    ~LocalGuard() { g.reset(); }
  } local_guard{local};
  if (graph_slot >= 0 && static_cast<size_t>(graph_slot) >= ws.graphs.size())
    ws.graphs.resize(static_cast<size_t>(graph_slot) + 1);
  LanczosGraph& lg = graph_slot >= 0 ? ws.graphs[static_cast<size_t>(graph_slot)] : local;
  const uint64_t key = graph_key ^ (static_cast<uint64_t>(n) << 40) ^ static_cast<uint64_t>(orth_grid) ^
                       (fused ? 0x5a5a000000000000ull : 0ull) ^
                       (reinterpret_cast<uint64_t>(v0) * 0x9E3779B97F4A7C15ull) ^
                       (reinterpret_cast<uint64_t>(out) * 0xC2B2AE3D27D4EB4Full) ^
                       (static_cast<uint64_t>(block) << 32) ^ (static_cast<uint64_t>(max_iter) << 48) ^
                       static_cast<uint64_t>(std::llround(-std::log10(std::max(tol, 1e-300)) * 1000.0)) << 20;
  static thread_local long builds = 0, updates = 0;
  static thread_local double build_s = 0.0;
  if (prof_on && prof_calls % 200 == 0)
    std::fprintf(stderr, "[lanczos] graph builds %ld (%ld by exec update), %.3f ms each\n", builds,
                 updates, builds ? 1e3 * build_s / builds : 0.0);

  if (!use_graph) {
    // host-stepped (profiling mode): the same kernels, each decision read back
    ws.pend_body = ws.pend_cycle = ws.pend_once = 0;
    LanczosResult& R = *ws.res_h.p;
    R = LanczosResult{};
    R.ctl.best = std::numeric_limits<double>::infinity();
    device_norm2(ctx, v0, n, misc + 2, ws.partials.p);
    double h_n2;
    ACHI_CUDA(cudaMemcpyAsync(&h_n2, misc + 2, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (!(h_n2 > 0)) {
      R.ctl.flags = LZ_BAD_V0;
      return;
    }
    {
      const double nrm = std::sqrt(h_n2);
      ACHI_CUDA(cudaMemcpyAsync(misc + 3, &nrm, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
    }
    K.scale(ws.q(0), v0, misc + 3, true);
    double best = std::numeric_limits<double>::infinity();
    int matvecs = 0;
    while (matvecs < max_iter) {
      ACHI_CUDA(cudaMemcpyAsync(ws.qcur.p, ws.q(0), sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                ctx.stream));
      LanczosCtl* ch = ws.ctl_h.p;
      *ch = LanczosCtl{0, matvecs, block, max_iter, 0, 0, 0, 0, tol, best};
      ACHI_CUDA(cudaMemcpyAsync(ws.ctl.p, ch, sizeof(LanczosCtl), cudaMemcpyHostToDevice, ctx.stream));
      apply(ws.qcur.p, ws.w.p);
      for (int j = 0;;) {
        launch_tridiag(launch_orth(0, 0), ctx.stream);
        ACHI_CUDA(cudaMemcpyAsync(ch, ws.ctl.p, sizeof(LanczosCtl), cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        if (ch->j == j) break;
        j = ch->j;
        apply(ws.qcur.p, ws.w.p);
      }
      const LanczosStatus st = K.read_status();  // syncs the stream
      const LanczosCtl cs = *ch;
      matvecs = cs.matvecs;
      const int k = cs.j + 1;
      const bool breakdown = st.bnorm <= 1e-14 * std::max(1.0, std::fabs(st.theta));
      K.axpy(ws.q(0), k, ws.s(), 1.0, nullptr, ws.ritz.p, true);
      K.norm_from_partials(misc + 4);
      K.scale(ws.ritz.p, ws.ritz.p, misc + 4, true);
      apply(ws.ritz.p, ws.w.p);
      ++matvecs;
      K.dots(ws.ritz.p, 1, ws.w.p, misc + 5);
      K.axpy(ws.ritz.p, 1, misc + 5, -1.0, ws.w.p, ws.tmp.p, true);
      residual_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, K.nb, misc + 5, misc,
                                                         K.dev_status());
      ACHI_LAUNCHED(ctx);
      const LanczosStatus rs = K.read_status();
      best = std::min(best, rs.res);
      R.st = rs;
      R.ctl = cs;
      R.ctl.matvecs = matvecs;
      R.ctl.best = best;
      if (rs.res <= tol * std::max(1.0, std::fabs(rs.ev))) {
        if (out != ws.ritz.p)
          ACHI_CUDA(cudaMemcpyAsync(out, ws.ritz.p, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                    ctx.stream));
        R.ctl.flags = LZ_CONVERGED;
        return;
      }
      if (breakdown) {
        // q = normalize(ritz + 1e-8 * tmp / ||tmp||)
        K.axpy(ws.tmp.p, 1, misc + 1, 1.0, ws.ritz.p, ws.q(0), true);
        K.norm_from_partials(misc + 4);
        K.scale(ws.q(0), ws.q(0), misc + 4, true);
      } else {
        ACHI_CUDA(cudaMemcpyAsync(ws.q(0), ws.ritz.p, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                  ctx.stream));
      }
    }
    R.ctl.matvecs = matvecs;
    R.ctl.best = best;
    R.ctl.flags = LZ_NONCONVERGED;
    return;
  }

  // ---- small blocks: the whole eigensolve as one persistent cooperative kernel ----
  static const bool persist_on = [] {
    const char* e = std::getenv("ACHI_LANCZOS_PERSIST");
    return !(e && e[0] == '0');
  }();
  hs::HsArgs pz_h{};
  long pz_items = 0;
  if (persist_on && small_op && heff_small_fusable(ctx, *small_op, ws.qcur.p, ws.w.p, &pz_h, &pz_items)) {
    const size_t smem = 2 * hs::smem_bytes<hs::HS_KMAX>();  // As, Bs + the L / R tile caches
    const int maxres = per_device_once("lanczos_persistent_kernel", ctx.device, [&] {
      ACHI_CUDA(cudaFuncSetAttribute(lanczos_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      int per_sm = 0;
      ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lanczos_persistent_kernel, PZ_THREADS,
                                                              smem));
      return std::max(1, per_sm) * ctx.num_sms;
    });
    // workers: at least one per matvec work item, and few enough vector elements per
    // thread that the orthogonalisation passes keep their loads in flight
    static const int pz_elems = [] {
      const char* e = std::getenv("ACHI_PZ_ELEMS");
      return e ? std::max(1, std::atoi(e)) : 1;
    }();
    const int W = static_cast<int>(std::max<long>(1, std::min<long>(
        std::max<long>(pz_items, cdiv(n, static_cast<long>(pz_elems) * PZ_THREADS)), ctx.cap_grid(maxres) - 1)));
    static const int pz_lazy = [] {  // ACHI_PZ_LAZY=0: the stored q_j as matvec input (+1 barrier)
      const char* e = std::getenv("ACHI_PZ_LAZY");
      return e ? std::atoi(e) : 1;
    }();
    double* pzd = ws.pzd.reserve(static_cast<size_t>(130) * W + 256);
    int* pzi = ws.pzi.reserve(16);
    ACHI_CUDA(cudaMemsetAsync(pzi, 0, 16 * sizeof(int), ctx.stream));
    PzArgs pa{pz_h, ws.q(0), ws.stride, ws.w.p, ws.ritz.p, ws.tmp.p, v0, out, n,
              pzd, pzd + 64L * W, pzd + 129L * W, ws.alpha(), ws.beta(),
              pzd + 130L * W, pzd + 130L * W + 128, pzi, pzi + 2,
              reinterpret_cast<unsigned*>(pzi + 6), reinterpret_cast<unsigned*>(pzi + 7),
              reinterpret_cast<unsigned*>(pzi + 8), ws.ctl.p, K.dev_status(), tol, block, max_iter, W,
              prof_on ? prof_buf.p : nullptr, ws.res_h.p, pz_lazy};
    if (prof_on && prof_calls % 200 == 0) {
      static PinnedArr<unsigned long long> ph;
      ph.reserve(16);
      ACHI_CUDA(cudaMemcpyAsync(ph.p, prof_buf.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                ctx.stream));
      ctx.sync();
      const double st = ph.p[11] ? static_cast<double>(ph.p[11]) : 1.0;
      std::fprintf(stderr,
                   "[lanczos-persist] W=%d steps=%llu cycles/step: A %.0f bar %.0f B %.0f bar %.0f C+dots %.0f "
                   "bar %.0f proj+dots %.0f bar %.0f proj+q %.0f bar %.0f wait %.0f | A: loads %.0f mma %.0f mix %.0f\n",
                   W, ph.p[11], ph.p[0] / st, ph.p[1] / st, ph.p[2] / st, ph.p[3] / st, ph.p[4] / st,
                   ph.p[5] / st, ph.p[6] / st, ph.p[7] / st, ph.p[8] / st, ph.p[9] / st, ph.p[10] / st,
                   ph.p[12] / st, ph.p[13] / st, ph.p[14] / st);
    }
    void* kargs[] = {&pa};
    ACHI_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lanczos_persistent_kernel), dim3(W + 1),
                                          dim3(PZ_THREADS), kargs, smem, ctx.stream));
    ACHI_LAUNCHED(ctx);
    ws.pend_graph = false;  // (the kernel writes ws.res_h itself: no copies on the stream)
    return;
  }

  // ---- graph mode: the whole eigensolve as one graph ----
  //   norm2(v0); init (decides whether the restart loop runs); q_0 = v0 / ||v0||
  //   WHILE restart {
  //     qcur = q_0; cycle init; w = H q_0
  //     WHILE step { orthogonalise + (aux stream) tridiagonal/decision || w = H q_{j+1} }
  //     ritz = normalize(Q s); w = H ritz; ev = ritz.w; tmp = w - ev ritz; decide;
  //     q_0 = ritz or the breakdown restart vector; out = ritz once converged
  //   }
  if (!lg.exec || lg.key != key) {
    const auto tb = std::chrono::steady_clock::now();
    ++builds;
    // every buffer a captured kernel uses is sized before capture and owned by
    // ws (growth resets the cached graphs); the v0 norm reduces into ws.partials,
    // not the context's shared scratch, whose growth another solver could trigger
    // keep the executable graph: a graph of the same topology (another shape
    // of this bond) is applied to it by cudaGraphExecUpdate, much cheaper than
    // a new instantiation; anything else re-instantiates
    cudaGraphExec_t old_exec = lg.exec;
    lg.exec = nullptr;
    lg.reset();
    ACHI_CUDA(cudaGraphCreate(&lg.graph, 0));
    int64_t l0 = ctx.launches;
    std::vector<cudaGraphNode_t> leaves;
    auto begin = [&](cudaGraph_t g, const cudaGraphNode_t* deps, size_t nd) {
      ACHI_CUDA(cudaStreamBeginCaptureToGraph(ctx.stream, g, deps, nullptr, nd,
                                              cudaStreamCaptureModeRelaxed));
      ctx.acc.in_capture = true;
    };
    auto finish = [&](bool want_leaves) {
      if (want_leaves) {
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        ACHI_CUDA(cudaStreamGetCaptureInfo(ctx.stream, &cs, nullptr, nullptr, &deps, &nd));
        leaves.assign(deps, deps + nd);
      }
      cudaGraph_t captured;
      ctx.acc.in_capture = false;
      ACHI_CUDA(cudaStreamEndCapture(ctx.stream, &captured));
    };
    auto add_while = [&](cudaGraph_t parent, cudaGraphConditionalHandle h) {
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      ACHI_CUDA(cudaGraphAddNode(&node, parent, leaves.data(), leaves.size(), &cp));
      return std::make_pair(node, cp.conditional.phGraph_out[0]);
    };
    try {
      cudaGraphConditionalHandle outer, inner;
      ACHI_CUDA(cudaGraphConditionalHandleCreate(&outer, lg.graph, 0, 0));
      // prologue
      begin(lg.graph, nullptr, 0);
      device_norm2(ctx, v0, n, misc + 2, ws.partials.p);
      eig_init_kernel<<<1, 1, 0, ctx.stream>>>(misc, ws.ctl.p, block, max_iter, tol, outer);
      ACHI_LAUNCHED(ctx);
      K.scale(ws.q(0), v0, misc + 3, true);
      finish(true);
      lg.once_launches = ctx.launches - l0;
      auto [onode, obody] = add_while(lg.graph, outer);
      (void)onode;
      ACHI_CUDA(cudaGraphConditionalHandleCreate(&inner, obody, 0, 0));
      // restart cycle, part 1
      l0 = ctx.launches;
      begin(obody, nullptr, 0);
      ACHI_CUDA(cudaMemcpyAsync(ws.qcur.p, ws.q(0), sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                ctx.stream));
      eig_cycle_kernel<<<1, 1, 0, ctx.stream>>>(ws.ctl.p, inner);
      ACHI_LAUNCHED(ctx);
      apply(ws.qcur.p, ws.w.p);  // w = H q_0; every later step's matvec runs inside the loop
      finish(true);
      auto [inode, ibody] = add_while(obody, inner);
      // inner loop body
      const int64_t l1 = ctx.launches;
      begin(ibody, nullptr, 0);
      if (fused) {
        FusedStepArgs fa{orth_args(inner, 1), fused_h, ws.bar.p};
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(orth_grid);
        lc.blockDim = dim3(ORTH_THREADS);
        lc.dynamicSmemBytes = hs::smem_bytes<hs::HS_KMAX>();
        lc.stream = ctx.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        ACHI_CUDA(cudaLaunchKernelEx(&lc, lanczos_step_small_kernel, fa));
        ACHI_LAUNCHED(ctx);
      } else {
        // orthogonalise step j; then the tridiagonal/decision kernel on the aux
        // stream runs concurrently with the (speculative) matvec of q_{j+1}
        const OrthArgs oa = launch_orth(inner, 1);
        ACHI_CUDA(cudaEventRecord(ctx.ev_fork, ctx.stream));
        ACHI_CUDA(cudaStreamWaitEvent(ctx.aux, ctx.ev_fork, 0));
        launch_tridiag(oa, ctx.aux);
        ACHI_CUDA(cudaEventRecord(ctx.ev_join, ctx.aux));
        apply(ws.qcur.p, ws.w.p);
        ACHI_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_join, 0));
      }
      finish(false);
      lg.body_launches = ctx.launches - l1;
      // restart cycle, part 2: Ritz vector, explicit residual, restart decision
      const int64_t l2 = ctx.launches;
      begin(obody, &inode, 1);
      K.axpy(ws.q(0), LANCZOS_BLOCK, ws.s(), 1.0, nullptr, ws.ritz.p, true, ws.ctl.p);
      K.norm_from_partials(misc + 4);
      K.scale(ws.ritz.p, ws.ritz.p, misc + 4, true);
      apply(ws.ritz.p, ws.w.p);
      K.dots(ws.ritz.p, 1, ws.w.p, misc + 5);
      K.axpy(ws.ritz.p, 1, misc + 5, -1.0, ws.w.p, ws.tmp.p, true);
      eig_decide_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, K.nb, misc + 5, misc,
                                                           K.dev_status(), ws.ctl.p, outer);
      ACHI_LAUNCHED(ctx);
      K.axpy(ws.tmp.p, 1, misc + 1, 1.0, ws.ritz.p, ws.q(0), true);
      K.norm_from_partials(misc + 4);
      {
        const int blocks = static_cast<int>(std::min<long>(cdiv(n, 256), 4L * ctx.num_sms));
        eig_restart_kernel<<<blocks, 256, 0, ctx.stream>>>(ws.q(0), ws.ritz.p, out, n, misc + 4,
                                                           ws.ctl.p);
        ACHI_LAUNCHED(ctx);
      }
      finish(false);
      lg.cycle_launches = (l1 - l0) + (ctx.launches - l2);
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(ctx.stream, &cs);
      if (cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(ctx.stream, &dummy);
      ctx.acc.in_capture = false;
      cudaGetLastError();
      lg.reset();
      if (old_exec) cudaGraphExecDestroy(old_exec);
      throw;
    }
    ctx.launches -= lg.once_launches + lg.cycle_launches + lg.body_launches;  // counted per execution
    static const bool exec_update = [] {
      const char* e = std::getenv("ACHI_GRAPH_UPDATE");
      return !(e && e[0] == '0');
    }();
    bool updated = false;
    if (old_exec && exec_update) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(old_exec, lg.graph, &info) == cudaSuccess) {
        lg.exec = old_exec;
        updated = true;
        ++updates;
      } else {
        cudaGetLastError();  // clear the failed update
      }
    }
    if (!updated) {
      if (old_exec) cudaGraphExecDestroy(old_exec);
      ACHI_CUDA(cudaGraphInstantiate(&lg.exec, lg.graph, 0));
    }
    lg.key = key;
    build_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
  }
  ACHI_CUDA(cudaGraphLaunch(lg.exec, ctx.stream));
  LanczosResult* R = ws.res_h.p;
  ACHI_CUDA(cudaMemcpyAsync(&R->ctl, ws.ctl.p, sizeof(LanczosCtl), cudaMemcpyDeviceToHost, ctx.stream));
  ACHI_CUDA(cudaMemcpyAsync(&R->st, K.dev_status(), sizeof(LanczosStatus), cudaMemcpyDeviceToHost,
                            ctx.stream));
  ws.pend_body = lg.body_launches;
  ws.pend_cycle = lg.cycle_launches;
  ws.pend_once = lg.once_launches;
  if (&lg == &local) {
    // a one-off graph must outlive its execution
    ctx.sync();
  }
}

EigsOut eigs_finish(Ctx& ctx, LanczosWs& ws) {
  const LanczosResult& R = *ws.res_h.p;
  if (ws.pend_graph)
    ctx.launches += ws.pend_once + ws.pend_cycle * R.ctl.cycles + ws.pend_body * R.ctl.steps;
  ws.pend_graph = false;
  if (R.ctl.flags & LZ_BAD_V0) fail(ACHI_E_INVALID_MATRIX, "eigs_lowest: v0 must have norm > 0");
  if (!(R.ctl.flags & LZ_CONVERGED)) {
    Error e(ACHI_E_EIGEN_NONCONVERGENCE, "eigs_lowest: no convergence within max_iter");
    e.residual = R.ctl.best;
    throw e;
  }
  return EigsOut{R.st.ev, R.ctl.matvecs, R.st.res};
}

EigsOut eigs_lowest(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                    const double* v0, double tol, int max_iter, double* out, int graph_slot,
                    uint64_t graph_key, const HeffOps* small_op) {
  eigs_lowest_async(ctx, ws, apply, n, dim, v0, tol, max_iter, out, graph_slot, graph_key, small_op);
  ctx.sync();
  return eigs_finish(ctx, ws);
}

}  // namespace achi
