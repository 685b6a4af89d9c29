// Device Lanczos (see lanczos.cuh).  All reductions are deterministic: each
// block owns a fixed contiguous chunk and partials are summed in fixed order.
#include <cooperative_groups.h>

#include <cmath>
#include <limits>

#include "lanczos.cuh"

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
__global__ void __launch_bounds__(RED_THREADS) multi_axpy_kernel(
    const double* __restrict__ Q, long stride, int nv, const double* __restrict__ coef, double sign,
    const double* src, double* dst, long n, double* __restrict__ partials) {
  __shared__ double c[64];
  __shared__ double sh[32];
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
// Bisection on Sturm counts for the smallest eigenvalue, then inverse
// iteration with partially pivoted tridiagonal elimination (dgtsv scheme).
__device__ int sturm_count(const double* a, const double* b, int k, double x) {
  int cnt = 0;
  double q = a[0] - x;
  const double tiny = 1e-300;
  if (q < 0) ++cnt;
  for (int i = 1; i < k; ++i) {
    if (fabs(q) < tiny) q = -tiny;
    q = (a[i] - x) - b[i - 1] * b[i - 1] / q;
    if (q < 0) ++cnt;
  }
  return cnt;
}

// Eigenvector of the k x k tridiagonal for the eigenvalue theta by inverse
// iteration (partially pivoted elimination, dgtsv scheme), unit norm, first
// nonzero component positive.
__device__ void tridiag_vector_from_theta(const double* a, const double* b, int k, double theta,
                                          double scale, double* s) {
  double dd[LANCZOS_BLOCK], du[LANCZOS_BLOCK], dl[LANCZOS_BLOCK], x[LANCZOS_BLOCK];
  const double tiny = (scale > 0 ? scale : 1.0) * 1e-300 + 1e-300;
  const double pivmin = (scale > 0 ? scale : 1.0) * 2.3e-16;
  // generic deterministic start (a symmetric start can be an exact eigenvector)
  for (int i = 0; i < k; ++i) x[i] = 1.0 + 0.5 * sin(1.0 + 2.3 * i);
  for (int iter = 0; iter < 2; ++iter) {
    for (int i = 0; i < k; ++i) dd[i] = a[i] - theta;
    for (int i = 0; i + 1 < k; ++i) dl[i] = du[i] = b[i];
    for (int i = 0; i + 1 < k; ++i) {
      if (fabs(dd[i]) >= fabs(dl[i])) {
        if (fabs(dd[i]) < pivmin) dd[i] = dd[i] >= 0 ? pivmin : -pivmin;
        const double f = dl[i] / dd[i];
        dd[i + 1] -= f * du[i];
        x[i + 1] -= f * x[i];
        dl[i] = 0.0;
      } else {
        const double f = dd[i] / dl[i];
        dd[i] = dl[i];
        const double t = dd[i + 1];
        dd[i + 1] = du[i] - f * t;
        if (i + 2 < k) {
          dl[i] = du[i + 1];
          du[i + 1] = -f * dl[i];
        } else {
          dl[i] = 0.0;
        }
        du[i] = t;
        const double tx = x[i];
        x[i] = x[i + 1];
        x[i + 1] = tx - f * x[i + 1];
      }
    }
    if (fabs(dd[k - 1]) < pivmin) dd[k - 1] = dd[k - 1] >= 0 ? pivmin : -pivmin;
    x[k - 1] /= dd[k - 1];
    x[k - 2] = (x[k - 2] - du[k - 2] * x[k - 1]) / dd[k - 2];
    for (int i = k - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - dl[i] * x[i + 2]) / dd[i];
    double nrm = 0;
    for (int i = 0; i < k; ++i) nrm += x[i] * x[i];
    nrm = sqrt(nrm);
    if (!(nrm > tiny)) nrm = 1.0;
    for (int i = 0; i < k; ++i) x[i] /= nrm;
  }
  // deterministic sign: first nonzero component positive
  double sg = 1.0;
  for (int i = 0; i < k; ++i)
    if (x[i] != 0.0) { sg = x[i] > 0 ? 1.0 : -1.0; break; }
  for (int i = 0; i < k; ++i) s[i] = sg * x[i];
}

// Warp version: 32-point multisection on Sturm counts (one point per lane,
// ~11 rounds to machine precision instead of ~60 serial bisection steps),
// then inverse iteration on lane 0.  Called by all 32 lanes of one warp.
__device__ void tridiag_lowest_warp(const double* a, const double* b, int k, double* theta_out,
                                    double* s) {
  const int lane = threadIdx.x & 31;
  if (k == 1) {
    if (lane == 0) {
      *theta_out = a[0];
      s[0] = 1.0;
    }
    return;
  }
  double lo = INFINITY, hi = -INFINITY, scale = 0.0;
  for (int i = lane; i < k; i += 32) {
    const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < k ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
    scale = fmax(scale, fabs(a[i]) + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  }
  for (int round = 0; round < 40; ++round) {
    const double w = hi - lo;
    if (!(w > 2.3e-16 * fmax(fabs(lo), fabs(hi)))) break;
    const double x = lo + (lane + 1) * (w / 33.0);
    const unsigned has = __ballot_sync(0xffffffffu, sturm_count(a, b, k, x) >= 1);
    const double nlo = has == 0u ? __shfl_sync(0xffffffffu, x, 31)
                                 : (__ffs(has) >= 2 ? __shfl_sync(0xffffffffu, x, __ffs(has) - 2) : lo);
    const double nhi = has == 0u ? hi : __shfl_sync(0xffffffffu, x, __ffs(has) - 1);
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) {
    tridiag_vector_from_theta(a, b, k, hi, scale, s);
    *theta_out = hi;
  }
}

// After CGS2: alpha[j] = h1[j]; beta[j] = sqrt(sum partials); tridiagonal solve.
__global__ void __launch_bounds__(RED_THREADS) finish_step_kernel(
    const double* __restrict__ partials, int nblocks, double* alpha, double* beta,
    const double* h1, double* s, int j, LanczosStatus* st) {
  __shared__ double sh[32];
  __shared__ double bn_s;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    bn_s = sqrt(v);
    alpha[j] = h1[j];
    beta[j] = bn_s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double theta;
    tridiag_lowest_warp(alpha, beta, j + 1, &theta, s);
    if (threadIdx.x == 0) {
      st->theta = theta;
      st->bnorm = bn_s;
      st->alpha = alpha[j];
      st->res_bound = bn_s * fabs(s[j]);
    }
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

int red_blocks(const Ctx&, long n) { return std::max(1, cdiv(n, CHUNK)); }

// ---- fused Lanczos step (one cooperative launch) --------------------------
// After w = H q_j:  h1 = Q^T w (alpha_j = h1[j]);  w <- w - Q h1;  h2 = Q^T w;
// w <- w - Q h2;  beta_j = ||w||;  tridiagonal lowest pair (warp 0 of block 0);
// q_{j+1} = w / beta_j.  Classical Gram-Schmidt twice, equal to the reference's
// MGS (linalg.cpp:131-135) to rounding.  Each block owns a fixed contiguous
// chunk and every block reduces the per-block partials in the same fixed order,
// so all blocks see bit-identical coefficients (deterministic).
struct OrthArgs {
  const double* Q;
  long stride;
  int nv;  // j + 1
  double* w;
  long n;
  double* pa;  // [grid][64] partials of h1
  double* pb;  // [grid][64] partials of h2
  double* pc;  // [grid]     partials of ||w||^2
  double* alpha;
  double* beta;
  double* s;
  double* qnext;
  LanczosStatus* st;
  int j;
};

constexpr int ORTH_THREADS = 256;

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
    for (int w8 = 0; w8 < ORTH_THREADS / 32; ++w8) t += sh[w8][v];
    part[static_cast<long>(blockIdx.x) * 64 + v] = t;
  }
  __syncthreads();
}

// every block: coef[v] = sum_b part[b][v] in fixed order
__device__ void orth_reduce(const double* part, int nv, double* coef) {
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) t += part[static_cast<long>(b) * 64 + v];
    coef[v] = t;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(ORTH_THREADS) lanczos_orth_kernel(OrthArgs a) {
  __shared__ double sh[ORTH_THREADS / 32][65];
  __shared__ double coef[64];
  __shared__ double red[32];
  cg::grid_group grid = cg::this_grid();
  const long chunk = (a.n + gridDim.x - 1) / gridDim.x;
  const long b0 = static_cast<long>(blockIdx.x) * chunk, b1 = min(a.n, b0 + chunk);
  // pass 1: h1 = Q^T w
  orth_partials(a.Q, a.stride, a.nv, a.w, b0, b1, a.pa, sh);
  grid.sync();
  orth_reduce(a.pa, a.nv, coef);
  // pass 2: w <- w - Q h1 ; h2 partials
  for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
    double v = a.w[x];
    for (int i = 0; i < a.nv; ++i) v -= coef[i] * a.Q[i * a.stride + x];
    a.w[x] = v;
  }
  __syncthreads();
  orth_partials(a.Q, a.stride, a.nv, a.w, b0, b1, a.pb, sh);
  const double alpha_j = coef[a.nv - 1];
  grid.sync();
  orth_reduce(a.pb, a.nv, coef);
  // pass 3: w <- w - Q h2 ; ||w||^2 partials
  double nrm = 0.0;
  for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
    double v = a.w[x];
    for (int i = 0; i < a.nv; ++i) v -= coef[i] * a.Q[i * a.stride + x];
    a.w[x] = v;
    nrm += v * v;
  }
  nrm = block_sum(nrm, red);
  if (threadIdx.x == 0) a.pc[blockIdx.x] = nrm;
  grid.sync();
  __shared__ double bn_s;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) t += a.pc[b];
    bn_s = sqrt(t);
  }
  __syncthreads();
  const double bn = bn_s;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      a.alpha[a.j] = alpha_j;
      a.beta[a.j] = bn;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double theta;
      tridiag_lowest_warp(a.alpha, a.beta, a.j + 1, &theta, a.s);
      if (threadIdx.x == 0) {
        a.st->theta = theta;
        a.st->bnorm = bn;
        a.st->alpha = alpha_j;
        a.st->res_bound = bn * fabs(a.s[a.j]);
      }
    }
  }
  // q_{j+1} = w / beta_j (unused when the step converges or breaks down)
  if (a.qnext && bn > 0) {
    const double inv = 1.0 / bn;
    for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) a.qnext[x] = a.w[x] * inv;
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
            bool norm) {
    multi_axpy_kernel<<<nb, RED_THREADS, 0, ctx.stream>>>(Q, ws.stride, nv, c, sign, src, dst, n,
                                                          norm ? ws.partials.p : nullptr);
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

void LanczosWs::reserve(long n) {
  const long s = (n + 31) & ~31L;  // 256-byte aligned vectors
  if (s > stride || basis.p == nullptr) {
    stride = s;
    basis.reserve(static_cast<size_t>(LANCZOS_BLOCK + 1) * s);
    w.reserve(s);
    ritz.reserve(s);
    tmp.reserve(s);
  }
  partials.reserve(64L * cdiv(s, CHUNK) + 1024);
  scal.reserve(512);
}

void device_norm2(Ctx& ctx, const double* x, long n, double* result) {
  const int nb = red_blocks(ctx, n);
  double* part = ctx.red.reserve(static_cast<size_t>(nb) * 2 + 8);
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

EigsOut eigs_lowest(Ctx& ctx, LanczosWs& ws, const ApplyFn& apply, long n, long dim,
                    const double* v0, double tol, int max_iter, double* out) {
  ws.reserve(n);
  Kernels K{ctx, ws, n, red_blocks(ctx, n)};
  double* misc = ws.misc();
  // n0 = ||v0||; q = v0 / n0
  device_norm2(ctx, v0, n, misc + 2);
  double h_n2;
  ACHI_CUDA(cudaMemcpyAsync(&h_n2, misc + 2, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (!(h_n2 > 0)) fail(ACHI_E_INVALID_MATRIX, "eigs_lowest: v0 must have norm > 0");
  {
    // misc[3] = sqrt(misc[2]) computed on device for bitwise consistency
    const double nrm = std::sqrt(h_n2);
    ACHI_CUDA(cudaMemcpyAsync(misc + 3, &nrm, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  }
  K.scale(ws.q(0), v0, misc + 3, true);

  const int block = static_cast<int>(std::min<long>(dim, LANCZOS_BLOCK));
  static int orth_max = 0;
  if (orth_max == 0) {
    int per_sm = 0;
    ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lanczos_orth_kernel,
                                                            ORTH_THREADS, 0));
    orth_max = std::max(1, std::min(per_sm, 2)) * ctx.num_sms;
  }
  // fixed for a given n: the chunking (and so every reduction order) is deterministic
  // (about one element per thread up to two CTAs per SM: the passes are latency-bound)
  const int orth_grid = static_cast<int>(std::max<long>(1, std::min<long>(cdiv(n, ORTH_THREADS), orth_max)));
  ws.partials.reserve(static_cast<size_t>(129) * orth_grid + 64);
  double best = std::numeric_limits<double>::infinity();
  int matvecs = 0;
  while (matvecs < max_iter) {
    for (int j = 0; j < block && matvecs < max_iter; ++j) {
      apply(ws.q(j), ws.w.p);
      ++matvecs;
      // classical Gram-Schmidt twice + tridiagonal Ritz pair + q_{j+1}, one launch
      {
        OrthArgs oa{ws.q(0), ws.stride, j + 1, ws.w.p, n,
                    ws.partials.p, ws.partials.p + 64L * orth_grid,
                    ws.partials.p + 128L * orth_grid, ws.alpha(), ws.beta(), ws.s(),
                    j + 1 <= LANCZOS_BLOCK ? ws.q(j + 1) : nullptr, K.dev_status(), j};
        void* args[] = {&oa};
        ACHI_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lanczos_orth_kernel),
                                              dim3(orth_grid), dim3(ORTH_THREADS), args, 0,
                                              ctx.stream));
        ACHI_LAUNCHED(ctx);
      }
      const LanczosStatus st = K.read_status();
      const int k = j + 1;
      const double theta = st.theta, bnorm = st.bnorm;
      const bool breakdown = bnorm <= 1e-14 * std::max(1.0, std::fabs(theta));
      if (st.res_bound <= tol * std::max(1.0, std::fabs(theta)) || breakdown || k == block ||
          matvecs >= max_iter) {
        // ritz = normalize(sum_i s_i q_i)
        K.axpy(ws.q(0), k, ws.s(), 1.0, nullptr, ws.ritz.p, true);
        K.norm_from_partials(misc + 4);
        K.scale(ws.ritz.p, ws.ritz.p, misc + 4, true);
        apply(ws.ritz.p, ws.w.p);
        ++matvecs;
        // ev = ritz . w ; tmp = w - ev ritz ; res = ||tmp||
        K.dots(ws.ritz.p, 1, ws.w.p, misc + 5);
        K.axpy(ws.ritz.p, 1, misc + 5, -1.0, ws.w.p, ws.tmp.p, true);
        residual_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, K.nb, misc + 5, misc,
                                                           K.dev_status());
        ACHI_LAUNCHED(ctx);
        const LanczosStatus rs = K.read_status();
        best = std::min(best, rs.res);
        if (rs.res <= tol * std::max(1.0, std::fabs(rs.ev))) {
          if (out != ws.ritz.p)
            ACHI_CUDA(cudaMemcpyAsync(out, ws.ritz.p, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                      ctx.stream));
          return EigsOut{rs.ev, matvecs, rs.res};
        }
        if (breakdown) {
          // q = normalize(ritz + 1e-8 * tmp / ||tmp||)
          K.axpy(ws.tmp.p, 1, misc + 1, 1.0, ws.ritz.p, ws.q(0), true);
          K.norm_from_partials(misc + 4);
          K.scale(ws.q(0), ws.q(0), misc + 4, true);
        } else {
          ACHI_CUDA(cudaMemcpyAsync(ws.q(0), ws.ritz.p, sizeof(double) * n,
                                    cudaMemcpyDeviceToDevice, ctx.stream));
        }
        break;
      }
    }
  }
  Error e(ACHI_E_EIGEN_NONCONVERGENCE, "eigs_lowest: no convergence within max_iter");
  e.residual = best;
  throw e;
}

}  // namespace achi
