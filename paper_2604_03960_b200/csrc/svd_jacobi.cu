// Blocked one-sided Jacobi SVD on sm_100a (see svd_jacobi.cuh).
#include <cmath>
#include <cstring>

#include "gemm_dmma.cuh"
#include "svd_jacobi.cuh"

namespace achi {

namespace {

constexpr int JB = 16;       // columns per block
constexpr int JW = 32;       // columns per block pair
constexpr int JT = 256;      // threads per CTA
constexpr int JCH = 64;      // rows per streamed chunk
constexpr int JLD = JCH + 4; // conflict-free DMMA fragment loads
constexpr int SLD = JW + 4;
constexpr double EPS = 2.220446049250313e-16;

__device__ __forceinline__ void mma16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// circle-method round robin: pair p of round r among n (even) players
__device__ __forceinline__ void circle_pair(int n, int r, int p, int& a, int& b) {
  if (p == 0) {
    a = r;
    b = n - 1;
  } else {
    a = (r + p) % (n - 1);
    b = (r - p + n - 1) % (n - 1);
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

struct RoundArgs {
  double* G;
  long ldg, gstride;
  int mg;
  double* V;
  long ldv, vstride;
  int vrows;
  int nb, round;
  double tol;
  const double* zero2;  // per batch: columns with ||g||^2 <= zero2 are numerically zero
  unsigned long long* conv;
};

struct JacobiSmem {
  double X[JW][JLD];
  double S[JW][SLD];
  double J[JW][SLD];
  double cs[16][2];
  double red[JT / 32];
  double ath;
  int changed;
};

// rows [r0, r0+JCH) of the 32 pair columns -> X[col][row]
__device__ __forceinline__ void load_chunk(JacobiSmem& sm, const double* M, long ld, int rows,
                                           int r0, int ca, int cb) {
  for (int idx = threadIdx.x; idx < JW * JCH; idx += JT) {
    const int c = idx / JCH, r = idx - c * JCH;
    const int col = c < JB ? ca + c : cb + c - JB;
    sm.X[c][r] = (r0 + r < rows) ? M[col * ld + r0 + r] : 0.0;
  }
}

// M[:, pair cols] <- M[:, pair cols] * J, streamed in row chunks (DMMA)
__device__ void apply_rotation(JacobiSmem& sm, double* M, long ld, int rows, int ca, int cb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int mt = warp >> 1;
  for (int r0 = 0; r0 < rows; r0 += JCH) {
    load_chunk(sm, M, ld, rows, r0, ca, cb);
    __syncthreads();
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int k4 = 0; k4 < JW / 4; ++k4) {
      const int k = k4 * 4 + tig;
      const double a0 = sm.X[k][mt * 16 + gid], a1 = sm.X[k][mt * 16 + gid + 8];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int nt = (warp & 1) * 2 + q;
        mma16x8x4(acc[q], a0, a1, sm.J[k][nt * 8 + gid]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int nt = (warp & 1) * 2 + q;
      const int r = mt * 16 + gid, j = nt * 8 + 2 * tig;
      sm.X[j][r] = acc[q][0];
      sm.X[j + 1][r] = acc[q][1];
      sm.X[j][r + 8] = acc[q][2];
      sm.X[j + 1][r + 8] = acc[q][3];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < JW * JCH; idx += JT) {
      const int c = idx / JCH, r = idx - c * JCH;
      const int col = c < JB ? ca + c : cb + c - JB;
      if (r0 + r < rows) M[col * ld + r0 + r] = sm.X[c][r];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(JT) jacobi_round_kernel(RoundArgs a) {
  __shared__ JacobiSmem sm;
  double* G = a.G + blockIdx.y * a.gstride;
  double* V = a.V + blockIdx.y * a.vstride;
  const double z2 = a.zero2[blockIdx.y];
  int ba, bb;
  circle_pair(a.nb, a.round, blockIdx.x, ba, bb);
  const int ca = ba * JB, cb = bb * JB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;

  // ---- 32x32 Gram matrix S = X^T X (DMMA, one 16x8 tile per warp) ----
  {
    const int mt = warp >> 2, nt = warp & 3;
    double acc[4] = {0, 0, 0, 0};
    for (int r0 = 0; r0 < a.mg; r0 += JCH) {
      load_chunk(sm, G, a.ldg, a.mg, r0, ca, cb);
      __syncthreads();
#pragma unroll
      for (int k4 = 0; k4 < JCH / 4; ++k4) {
        const int k = k4 * 4 + tig;
        mma16x8x4(acc, sm.X[mt * 16 + gid][k], sm.X[mt * 16 + gid + 8][k], sm.X[nt * 8 + gid][k]);
      }
      __syncthreads();
    }
    const int r = mt * 16 + gid, c = nt * 8 + 2 * tig;
    sm.S[r][c] = acc[0];
    sm.S[r][c + 1] = acc[1];
    sm.S[r + 8][c] = acc[2];
    sm.S[r + 8][c + 1] = acc[3];
  }
  for (int idx = threadIdx.x; idx < JW * JW; idx += JT) {
    const int r = idx / JW, c = idx - r * JW;
    sm.J[r][c] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();

  // ---- off-diagonal measure max |s_ij| / sqrt(s_ii s_jj) ----
  double meas = 0.0;
  for (int idx = threadIdx.x; idx < JW * JW; idx += JT) {
    const int i = idx / JW, j = idx - i * JW;
    if (i < j && sm.S[i][i] > z2 && sm.S[j][j] > z2)
      meas = fmax(meas, fabs(sm.S[i][j]) / sqrt(sm.S[i][i] * sm.S[j][j]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) meas = fmax(meas, __shfl_xor_sync(0xffffffffu, meas, o));
  if (lane == 0) sm.red[warp] = meas;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0;
    for (int w = 0; w < JT / 32; ++w) m = fmax(m, sm.red[w]);
    sm.red[0] = m;
    atomicMax(a.conv, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
  __syncthreads();
  if (!(sm.red[0] > a.tol)) return;  // pair already orthogonal

  // ---- two-sided cyclic Jacobi on S, accumulating J ----
  for (int sweep = 0; sweep < 6; ++sweep) {
    if (threadIdx.x == 0) sm.changed = 0;
    __syncthreads();
    for (int step = 0; step < JW - 1; ++step) {
      if (threadIdx.x < JW / 2) {
        int i, j;
        circle_pair(JW, step, threadIdx.x, i, j);
        const double app = sm.S[i][i], aqq = sm.S[j][j], apq = sm.S[i][j];
        double c = 1.0, s = 0.0;
        if (app > z2 && aqq > z2 && fabs(apq) > a.tol * sqrt(app * aqq)) {
          const double tau = (aqq - app) / (2.0 * apq);
          const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          sm.changed = 1;
        }
        sm.cs[threadIdx.x][0] = c;
        sm.cs[threadIdx.x][1] = s;
      }
      __syncthreads();
      // columns of S and J
      for (int it = threadIdx.x; it < 2 * (JW / 2) * JW; it += JT) {
        const int mat = it / ((JW / 2) * JW), rem = it - mat * (JW / 2) * JW;
        const int p = rem / JW, r = rem - p * JW;
        const double s = sm.cs[p][1];
        if (s != 0.0) {
          int i, j;
          circle_pair(JW, step, p, i, j);
          const double c = sm.cs[p][0];
          double (*M)[SLD] = mat ? sm.J : sm.S;
          const double x = M[r][i], y = M[r][j];
          M[r][i] = c * x - s * y;
          M[r][j] = s * x + c * y;
        }
      }
      __syncthreads();
      // rows of S
      for (int it = threadIdx.x; it < (JW / 2) * JW; it += JT) {
        const int p = it / JW, col = it - p * JW;
        const double s = sm.cs[p][1];
        if (s != 0.0) {
          int i, j;
          circle_pair(JW, step, p, i, j);
          const double c = sm.cs[p][0];
          const double x = sm.S[i][col], y = sm.S[j][col];
          sm.S[i][col] = c * x - s * y;
          sm.S[j][col] = s * x + c * y;
        }
      }
      __syncthreads();
    }
    if (!sm.changed) break;
    __syncthreads();
  }
  apply_rotation(sm, G, a.ldg, a.mg, ca, cb);
  apply_rotation(sm, V, a.ldv, a.vrows, ca, cb);
}

// ---- setup / finalisation kernels ----
__global__ void identity_kernel(double* V, long ld, int n, long bstride) {
  double* Vb = V + blockIdx.y * bstride;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
       idx < static_cast<long>(n) * n; idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long c = idx / n, r = idx - c * n;
    Vb[c * ld + r] = r == c ? 1.0 : 0.0;
  }
}

// G (col-major, ld = mg, ng cols) from theta row-major (m x n):
//   rows side: G[c][r] = theta[c][r] (c < m, r < n), zero for c >= m
//   cols side: G[c][r] = theta[r][c] (c < n, r < m), zero for c >= n
__global__ void load_g_kernel(const double* __restrict__ theta, long tstride, int m, int n,
                              double* __restrict__ G, long gstride, int mg, int ng, int rows_side) {
  __shared__ double tile[32][33];
  const double* T = theta + blockIdx.z * tstride;
  double* Gb = G + blockIdx.z * gstride;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;  // G column / row tile
  if (rows_side) {
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int c = c0 + dy, r = r0 + threadIdx.x;
      if (c < ng && r < mg) Gb[static_cast<long>(c) * mg + r] = c < m ? T[static_cast<long>(c) * n + r] : 0.0;
    }
  } else {
    // read theta rows r (G rows) x cols c coalesced along c, write G coalesced along r
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int r = r0 + dy, c = c0 + threadIdx.x;
      tile[dy][threadIdx.x] = (r < m && c < n) ? T[static_cast<long>(r) * n + c] : 0.0;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int c = c0 + dy, r = r0 + threadIdx.x;
      if (c < ng && r < mg) Gb[static_cast<long>(c) * mg + r] = tile[threadIdx.x][dy];
    }
  }
}

// zero2[b] = (sqrt(mg) * eps * ||G_b||_F)^2: the rounding floor of a column norm
__global__ void zero_floor_kernel(const double* __restrict__ G, long gstride, long len, int mg,
                                  double* __restrict__ zero2) {
  __shared__ double sh[32];
  const double* g = G + blockIdx.x * gstride;
  double s = 0.0;
  for (long i = threadIdx.x; i < len; i += blockDim.x) s += g[i] * g[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) t += sh[w];
    // columns below 64 sqrt(mg) eps ||G||_F are rounding noise (a rank-deficient
    // theta leaves such columns; their direction is undefined and their norm is
    // below the reference's own normwise accuracy): they are not rotated
    const double f = 64.0 * sqrt(static_cast<double>(mg)) * EPS;
    zero2[blockIdx.x] = f * f * t;
  }
}

// sigma_c = ||G[:,c]|| for real columns, -1 for pad columns (sorted last)
__global__ void col_norm_kernel(const double* __restrict__ G, long gstride, int mg, int ng,
                                int ng_real, int pad_mod, int pad_lim, double* __restrict__ sig,
                                long sstride) {
  const int warps = blockDim.x >> 5;
  const int c = blockIdx.x * warps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= ng) return;
  const double* col = G + blockIdx.y * gstride + static_cast<long>(c) * mg;
  double s = 0.0;
  for (int r = lane; r < mg; r += 32) s += col[r] * col[r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const bool pad = c >= ng_real || (c % pad_mod) >= pad_lim;
    sig[blockIdx.y * sstride + c] = pad ? -1.0 : sqrt(s);
  }
}

// rank sort (descending, ties by index): sorted[rank] = sig[c], perm[rank] = c
__global__ void __launch_bounds__(1024) sort_kernel(const double* __restrict__ sig, long sstride,
                                                    int ng, double* __restrict__ sorted,
                                                    int* __restrict__ perm) {
  extern __shared__ double keys[];
  const double* s = sig + blockIdx.x * sstride;
  for (int i = threadIdx.x; i < ng; i += blockDim.x) keys[i] = s[i];
  __syncthreads();
  for (int c = threadIdx.x; c < ng; c += blockDim.x) {
    const double k = keys[c];
    int rank = 0;
    for (int o = 0; o < ng; ++o) {
      const double ko = keys[o];
      rank += (ko > k) || (ko == k && o < c);
    }
    sorted[blockIdx.x * sstride + rank] = k;
    perm[blockIdx.x * sstride + rank] = c;
  }
}

// fix_phases (linalg.cpp:19-35): first largest-|u| entry of each kept U column positive
__global__ void phase_kernel(const double* __restrict__ base, long ld, int len,
                             const int* __restrict__ perm, int kept, double* __restrict__ sign) {
  const int warps = blockDim.x >> 5;
  const int k = blockIdx.x * warps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= kept) return;
  const double* u = base + static_cast<long>(perm[k]) * ld;
  double best = 0.0, val = 0.0;
  int idx = 0x7fffffff;
  for (int r = lane; r < len; r += 32) {
    const double a = fabs(u[r]);
    if (a > best) { best = a; idx = r; val = u[r]; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    const double ov = __shfl_xor_sync(0xffffffffu, val, o);
    if (ob > best || (ob == best && oi < idx)) { best = ob; idx = oi; val = ov; }
  }
  if (lane == 0) sign[k] = (best > 0 && val < 0) ? -1.0 : 1.0;
}

// U (m_true x k) and VT (k x n_true) row-major from the Jacobi factors
__global__ void gather_kernel(const double* __restrict__ G, int mg, const double* __restrict__ V,
                              int ng, const double* __restrict__ sorted, const int* __restrict__ perm,
                              const double* __restrict__ sign, int k, int rows_side, int m_true,
                              int n_true, int n_pad_mod, double* __restrict__ U,
                              double* __restrict__ VT) {
  // rows side: U[i][q] = V[perm q][i] * sg ; VT[q][j] = G[perm q][j] * sg / sigma
  // cols side: U[i][q] = G[perm q][i] * sg / sigma ; VT[q][j] = V[perm q][j] * sg
  const long tot_u = static_cast<long>(m_true) * k, tot_v = static_cast<long>(k) * n_true;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot_u + tot_v;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    if (t < tot_u) {
      const int i = static_cast<int>(t / k), q = static_cast<int>(t % k);
      const double sg = sign[q], s = sorted[q];
      U[t] = rows_side ? V[static_cast<long>(perm[q]) * ng + i] * sg
                       : (s > 0 ? G[static_cast<long>(perm[q]) * mg + i] * sg / s : 0.0);
    } else {
      const long u = t - tot_u;
      const int q = static_cast<int>(u / n_true), j = static_cast<int>(u % n_true);
      const double sg = sign[q], s = sorted[q];
      VT[u] = rows_side ? (s > 0 ? G[static_cast<long>(perm[q]) * mg + j] * sg / s : 0.0)
                        : V[static_cast<long>(perm[q]) * ng + j] * sg;
    }
  }
  (void)n_pad_mod;
}

}  // namespace

SvdResultDev svd_device(Ctx& ctx, SvdWs& ws, const double* theta, int m, int n, int m_true,
                        int n_true, SvdSide side, int batch, long bstride, double* sigma_out) {
  const bool rows = side == SvdSide::kRows;
  const int ng_real = rows ? m : n;
  const int mg = rows ? n : m;
  const int ng = ((ng_real + JW - 1) / JW) * JW;
  const long gstride = static_cast<long>(mg) * ng, vstride = static_cast<long>(ng) * ng;
  double* G = ws.G.reserve(static_cast<size_t>(gstride) * batch);
  double* V = ws.V.reserve(static_cast<size_t>(vstride) * batch);
  double* sig = ws.sig.reserve(static_cast<size_t>(ng) * batch);
  double* sorted = ws.sorted.reserve(static_cast<size_t>(ng) * batch);
  int* perm = ws.perm.reserve(static_cast<size_t>(ng) * batch);
  unsigned long long* conv = ws.conv.reserve(4);
  double* zero2 = ws.zero2.reserve(static_cast<size_t>(batch));
  unsigned long long* conv_h = ws.conv_host.reserve(4);

  {
    dim3 grid(cdiv(ng, 32), cdiv(mg, 32), batch), blk(32, 8);
    load_g_kernel<<<grid, blk, 0, ctx.stream>>>(theta, bstride, m, n, G, gstride, mg, ng, rows ? 1 : 0);
    ACHI_LAUNCHED(ctx);
    dim3 g2(static_cast<unsigned>(std::min<long>(cdiv(vstride, 256), 4L * ctx.num_sms)), batch);
    identity_kernel<<<g2, 256, 0, ctx.stream>>>(V, ng, ng, vstride);
    ACHI_LAUNCHED(ctx);
    zero_floor_kernel<<<batch, 1024, 0, ctx.stream>>>(G, gstride, gstride, mg, zero2);
    ACHI_LAUNCHED(ctx);
  }
  const int nb = ng / JB;  // even (ng multiple of 32)
  const double tol = std::max(1e-15, 2.0 * std::sqrt(static_cast<double>(mg)) * EPS);
  int sweeps = 0;
  for (; sweeps < 40; ++sweeps) {
    ACHI_CUDA(cudaMemsetAsync(conv, 0, sizeof(unsigned long long), ctx.stream));
    for (int r = 0; r < nb - 1; ++r) {
      RoundArgs a{G, mg, gstride, mg, V, ng, vstride, ng, nb, r, tol, zero2, conv};
      jacobi_round_kernel<<<dim3(nb / 2, batch), JT, 0, ctx.stream>>>(a);
      ACHI_LAUNCHED(ctx);
    }
    ACHI_CUDA(cudaMemcpyAsync(conv_h, conv, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              ctx.stream));
    ctx.sync();
    double meas;
    std::memcpy(&meas, conv_h, sizeof(double));
    if (!(meas >= 0)) fail(ACHI_E_NUMERICAL_FAILURE, "svd: non-finite Jacobi measure");
    if (meas < 1e-9) {
      ++sweeps;
      break;
    }
  }
  if (sweeps >= 40) fail(ACHI_E_NUMERICAL_FAILURE, "svd: decomposition did not converge");
  // pad columns: rows side -> columns >= m_true (theta rows (l,s1) with padded l last);
  // cols side -> columns (s2, jr) with jr >= chr_true, i.e. c % (n / d) >= n_true / d is
  // encoded by the caller through m_true/n_true with the modulus rule below.
  int pad_mod = ng, pad_lim = rows ? m_true : n_true;
  if (!rows && n != n_true) {
    // theta columns are (s2, jr) with jr padded: n = d * chr~, n_true = d * chr
    // (d = 2 on every path that pads); c % chr~ >= chr marks a pad column.
    pad_mod = n / 2;
    pad_lim = n_true / 2;
  }
  {
    dim3 grid(cdiv(ng, 8), batch);
    col_norm_kernel<<<grid, 256, 0, ctx.stream>>>(G, gstride, mg, ng, ng_real, pad_mod, pad_lim, sig, ng);
    ACHI_LAUNCHED(ctx);
    sort_kernel<<<batch, 1024, sizeof(double) * ng, ctx.stream>>>(sig, ng, ng, sorted, perm);
    ACHI_LAUNCHED(ctx);
  }
  const int r_true = std::min(m_true, n_true);
  if (sigma_out) {
    ACHI_CUDA(cudaMemcpy2DAsync(sigma_out, sizeof(double) * r_true, sorted, sizeof(double) * ng,
                                sizeof(double) * r_true, batch, cudaMemcpyDeviceToDevice, ctx.stream));
  }
  SvdResultDev r;
  r.side = side;
  r.m = m;
  r.n = n;
  r.m_true = m_true;
  r.n_true = n_true;
  r.ng = ng;
  r.mg = mg;
  r.r_true = r_true;
  r.sweeps = sweeps;
  r.G = G;
  r.V = V;
  r.sigma = sorted;
  r.perm = perm;
  return r;
}

void svd_phase_signs(Ctx& ctx, SvdWs& ws, const SvdResultDev& r, int kept) {
  double* sign = ws.sign.reserve(static_cast<size_t>(std::max(kept, 1)));
  if (kept <= 0) return;
  const bool rows = r.side == SvdSide::kRows;
  // U columns: rows side -> V[:, perm k] (length m); cols side -> G[:, perm k] (length mg = m)
  const double* base = rows ? r.V : r.G;
  const long ld = rows ? r.ng : r.mg;
  phase_kernel<<<cdiv(kept, 8), 256, 0, ctx.stream>>>(base, ld, r.m, r.perm, kept, sign);
  ACHI_LAUNCHED(ctx);
}

void svd_gather(Ctx& ctx, SvdWs& ws, const SvdResultDev& r, int k, double* U, double* VT) {
  const long tot = static_cast<long>(r.m_true) * k + static_cast<long>(k) * r.n_true;
  const int blocks = static_cast<int>(std::min<long>(cdiv(tot, 256), 4L * ctx.num_sms));
  gather_kernel<<<blocks, 256, 0, ctx.stream>>>(r.G, r.mg, r.V, r.ng, r.sigma, r.perm, ws.sign.p, k,
                                                r.side == SvdSide::kRows ? 1 : 0, r.m_true,
                                                r.n_true, 0, U, VT);
  ACHI_LAUNCHED(ctx);
}

}  // namespace achi
