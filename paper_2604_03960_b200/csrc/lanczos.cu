// Device Lanczos (see lanczos.cuh).  All reductions are deterministic: each
// block owns a fixed contiguous chunk and partials are summed in fixed order.
#include <cmath>
#include <limits>

#include "lanczos.cuh"

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

__device__ __forceinline__ void chunk_of(long n, long& begin, long& end) {
  const long chunk = (n + gridDim.x - 1) / gridDim.x;
  begin = blockIdx.x * chunk;
  end = min(n, begin + chunk);
}

// partials[b * ld + v] = sum_{x in chunk b} Q_v[x] * w[x] for v < nv; plus w.w at v = nv if self
__global__ void __launch_bounds__(RED_THREADS) multi_dot_kernel(const double* __restrict__ Q, long stride,
                                                                int nv, const double* __restrict__ w,
                                                                long n, double* __restrict__ partials,
                                                                int ld, int self) {
  __shared__ double sh[32];
  long b0, b1;
  chunk_of(n, b0, b1);
  for (int v0 = 0; v0 < nv + self; v0 += DOT_GROUP) {
    double acc[DOT_GROUP];
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) acc[g] = 0.0;
    for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
      const double wx = w[x];
#pragma unroll
      for (int g = 0; g < DOT_GROUP; ++g) {
        const int v = v0 + g;
        if (v < nv) acc[g] += Q[v * stride + x] * wx;
        else if (v == nv && self) acc[g] += wx * wx;
      }
    }
#pragma unroll
    for (int g = 0; g < DOT_GROUP; ++g) {
      const int v = v0 + g;
      if (v >= nv + self) break;
      const double s = block_sum(acc[g], sh);
      if (threadIdx.x == 0) partials[static_cast<long>(blockIdx.x) * ld + v] = s;
    }
  }
}

// out[v] = sum_b partials[b * ld + v], fixed order, for v < nv
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nblocks, int ld,
                                       int nv, double* __restrict__ out) {
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partials[static_cast<long>(b) * ld + v];
    out[v] = s;
  }
}

// dst[x] = src[x] + sign * sum_v coef[v] * Q_v[x]; partials[b] = sum_chunk dst^2
__global__ void __launch_bounds__(RED_THREADS) multi_axpy_kernel(
    const double* __restrict__ Q, long stride, int nv, const double* __restrict__ coef, double sign,
    const double* src, double* dst, long n, double* __restrict__ partials) {
  __shared__ double c[64];
  __shared__ double sh[32];
  for (int v = threadIdx.x; v < nv; v += blockDim.x) c[v] = sign * coef[v];
  __syncthreads();
  long b0, b1;
  chunk_of(n, b0, b1);
  double nrm = 0.0;
  for (long x = b0 + threadIdx.x; x < b1; x += blockDim.x) {
    double v = src ? src[x] : 0.0;
    for (int i = 0; i < nv; ++i) v += c[i] * Q[i * stride + x];
    dst[x] = v;
    nrm += v * v;
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

__device__ void tridiag_lowest_dev(const double* a, const double* b, int k, double* theta_out,
                                   double* s) {
  if (k == 1) {
    *theta_out = a[0];
    s[0] = 1.0;
    return;
  }
  double lo = a[0], hi = a[0], scale = 0;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < k ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
    scale = fmax(scale, fabs(a[i]) + r);
  }
  for (int it = 0; it < 256; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(a, b, k, mid) >= 1) hi = mid; else lo = mid;
  }
  const double theta = hi;
  *theta_out = theta;
  // inverse iteration
  double dd[LANCZOS_BLOCK], du[LANCZOS_BLOCK], dl[LANCZOS_BLOCK], x[LANCZOS_BLOCK];
  const double tiny = (scale > 0 ? scale : 1.0) * 1e-300 + 1e-300;
  const double pivmin = (scale > 0 ? scale : 1.0) * 2.3e-16;
  // generic deterministic start (a symmetric start can be an exact eigenvector)
  for (int i = 0; i < k; ++i) x[i] = 1.0 + 0.5 * sin(1.0 + 2.3 * i);
  for (int iter = 0; iter < 3; ++iter) {
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

// After CGS2: alpha[j] = h1[j]; beta[j] = sqrt(sum partials); tridiagonal solve.
__global__ void __launch_bounds__(RED_THREADS) finish_step_kernel(
    const double* __restrict__ partials, int nblocks, double* alpha, double* beta,
    const double* h1, double* s, int j, LanczosStatus* st) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += partials[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    const double bn = sqrt(v);
    alpha[j] = h1[j];
    beta[j] = bn;
    double theta;
    tridiag_lowest_dev(alpha, beta, j + 1, &theta, s);
    st->theta = theta;
    st->bnorm = bn;
    st->alpha = alpha[j];
    st->res_bound = bn * fabs(s[j]);
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

int red_blocks(const Ctx& ctx, long n) {
  return static_cast<int>(std::max<long>(1, std::min<long>(cdiv(n, RED_THREADS * 4), 2L * ctx.num_sms)));
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
    reduce_partials_kernel<<<1, 64, 0, ctx.stream>>>(ws.partials.p, nb, 64, nv, h);
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
  partials.reserve(64L * 2 * 148 * 4 + 1024);
  scal.reserve(512);
}

void device_norm2(Ctx& ctx, const double* x, long n, double* result) {
  const int nb = red_blocks(ctx, n);
  double* part = ctx.red.reserve(static_cast<size_t>(nb) * 2 + 8);
  multi_dot_kernel<<<nb, RED_THREADS, 0, ctx.stream>>>(x, 0, 0, x, n, part, 1, 1);
  ACHI_LAUNCHED(ctx);
  reduce_partials_kernel<<<1, 32, 0, ctx.stream>>>(part, nb, 1, 1, result);
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
  double best = std::numeric_limits<double>::infinity();
  int matvecs = 0;
  while (matvecs < max_iter) {
    for (int j = 0; j < block && matvecs < max_iter; ++j) {
      apply(ws.q(j), ws.w.p);
      ++matvecs;
      // classical Gram-Schmidt, twice (h1[j] = alpha_j = q_j . H q_j)
      K.dots(ws.q(0), j + 1, ws.w.p, ws.h1());
      K.axpy(ws.q(0), j + 1, ws.h1(), -1.0, ws.w.p, ws.w.p, false);
      K.dots(ws.q(0), j + 1, ws.w.p, ws.h2());
      K.axpy(ws.q(0), j + 1, ws.h2(), -1.0, ws.w.p, ws.w.p, true);
      finish_step_kernel<<<1, RED_THREADS, 0, ctx.stream>>>(ws.partials.p, K.nb, ws.alpha(),
                                                            ws.beta(), ws.h1(), ws.s(), j,
                                                            K.dev_status());
      ACHI_LAUNCHED(ctx);
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
      // q_{j+1} = w / beta_j
      K.scale(ws.q(j + 1), ws.w.p, ws.beta() + j, true);
    }
  }
  Error e(ACHI_E_EIGEN_NONCONVERGENCE, "eigs_lowest: no convergence within max_iter");
  e.residual = best;
  throw e;
}

}  // namespace achi
