// Blocked one-sided Jacobi SVD on sm_100a (see svd_jacobi.cuh).
//
// One cooperative launch runs every sweep and every round of the Jacobi
// iteration: CTA p owns block pair p of the current round (circle-method
// ordering of 16-column blocks), forms the 32x32 Gram matrix of its columns
// with DMMA, diagonalises it by two-sided Jacobi in shared memory and applies
// the accumulated rotation to its columns of G and V with DMMA; a grid-wide
// barrier separates rounds.  Small problems (<= 256 rows) keep the pair's
// columns resident in shared memory for the whole round; large ones stream
// 64-row chunks with double-buffered cp.async.  Convergence is decided on the
// device (max off-diagonal measure of a sweep), so the host never waits
// inside the iteration.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "svd_jacobi.cuh"

namespace cg = cooperative_groups;

namespace achi {

namespace {

constexpr int JB = 16;        // columns per block
constexpr int JW = 32;        // columns per block pair
constexpr int JT = 256;       // threads per CTA
constexpr int JCH = 64;       // rows per chunk
constexpr int JLD = JCH + 4;  // conflict-free DMMA fragment loads
constexpr int SLD = JW + 4;
constexpr int RES_CHUNKS = 4; // resident mode: up to 256 rows of G and of V
constexpr int MAX_SWEEPS = 40;
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

typedef double Chunk[JW][JLD];

struct PersArgs {
  double* G;
  long ldg, gstride;
  int mg;
  double* V;
  long ldv, vstride;
  int vrows;
  int nb, npairs, batch0;
  int max_inner;
  double tol, stop_tol;
  const double* zero2;
  unsigned long long* conv;  // [MAX_SWEEPS] per-sweep max measure (whole launch)
  int* sweeps_out;
  long long* prof;  // optional clock64 phase accounting (CTA 0), null in production
};

struct Small {
  double S[JW][SLD];
  double J[JW][SLD];
  double cs[16][2];
  double red[JT / 32];
  unsigned char pi[JW - 1][JW / 2], pj[JW - 1][JW / 2];
  int changed;
};

// ---- cp.async chunk loads: rows [r0, r0+64) of the 32 pair columns -> X[col][row] ----
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void load_chunk_async(Chunk& X, const double* M, long ld, int rows, int r0,
                                                 int ca, int cb) {
  // 32 columns x 32 segments of 16 B
  for (int idx = threadIdx.x; idx < JW * (JCH / 2); idx += JT) {
    const int c = idx / (JCH / 2), seg = idx - c * (JCH / 2);
    const int col = c < JB ? ca + c : cb + c - JB;
    const int r = r0 + 2 * seg;
    const int valid = rows - r;  // rows (elements) available from r
    const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
    const double* src = M + col * ld + (bytes ? r : 0);
    cp_async16(&X[c][2 * seg], src, bytes);
  }
}

__device__ __forceinline__ void store_chunk(const Chunk& X, double* M, long ld, int rows, int r0,
                                            int ca, int cb) {
  for (int idx = threadIdx.x; idx < JW * JCH; idx += JT) {
    const int c = idx / JCH, r = idx - c * JCH;
    const int col = c < JB ? ca + c : cb + c - JB;
    if (r0 + r < rows) M[col * ld + r0 + r] = X[c][r];
  }
}

// acc += (32 x 64)^T-tile Gram contribution of chunk X (one 16x8 tile per warp)
__device__ __forceinline__ void gram_chunk(const Chunk& X, double (&acc)[4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3, mt = warp >> 2, nt = warp & 3;
#pragma unroll
  for (int k4 = 0; k4 < JCH / 4; ++k4) {
    const int k = k4 * 4 + tig;
    mma16x8x4(acc, X[mt * 16 + gid][k], X[mt * 16 + gid + 8][k], X[nt * 8 + gid][k]);
  }
}

// X <- X * J in place (rows of the chunk times the 32x32 rotation)
__device__ __forceinline__ void rotate_chunk(Chunk& X, const Small& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3, mt = warp >> 1;
  double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
  for (int k4 = 0; k4 < JW / 4; ++k4) {
    const int k = k4 * 4 + tig;
    const double a0 = X[k][mt * 16 + gid], a1 = X[k][mt * 16 + gid + 8];
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
    X[j][r] = acc[q][0];
    X[j + 1][r] = acc[q][1];
    X[j][r + 8] = acc[q][2];
    X[j + 1][r + 8] = acc[q][3];
  }
  __syncthreads();
}

// two-sided cyclic Jacobi on S (32x32 in smem), accumulating J (starts at I).
// Each parallel step rotates 16 disjoint pairs; the two-sided update splits
// into 16x16 independent 2x2 blocks S[{ip,jp},{iq,jq}] <- Rp^T S Rq, one per
// thread, so a step costs two barriers.  Pair tables are precomputed.
__device__ void inner_jacobi(Small& sm, double z2, double inv_f2, double tol, int max_inner) {
  const int t = threadIdx.x;
  const int bp = t >> 4, bq = t & 15;  // this thread's 2x2 block of S
  for (int sweep = 0; sweep < max_inner; ++sweep) {
    if (t == 0) sm.changed = 0;
    __syncthreads();
    for (int step = 0; step < JW - 1; ++step) {
      if (t < JW / 2) {
        const int i = sm.pi[step][t], j = sm.pj[step][t];
        const double app = sm.S[i][i], aqq = sm.S[j][j], apq = sm.S[i][j];
        double c = 1.0, s = 0.0;
        // rotate iff |apq| > tol sqrt(app aqq).  The angle t = tan(theta) of the
        // classical Jacobi rotation is computed in FP32 from the scale-free
        // tau = (aqq - app) / (2 apq) (an approximate angle still gives an exactly
        // orthogonal rotation; its error only leaves a ~1e-7 relative residue
        // that later sweeps remove, preserving superlinear convergence); c and
        // s = t c are then made orthonormal to FP64 precision by two Newton steps
        // on rsqrt(1 + t^2).  Cuts the serial FP64 sqrt/div chain of every step.
        if (app > z2 && aqq > z2 && apq * apq > tol * tol * (app * aqq)) {
          const float zf = static_cast<float>((aqq - app) * inv_f2);
          const float qf = static_cast<float>(2.0 * apq * inv_f2);
          const float tau = __fdividef(zf, qf);
          const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
          const double td = tf;
          const double x = fma(td, td, 1.0);
          double y = rsqrtf(static_cast<float>(x));
          y = y * (1.5 - 0.5 * x * y * y);
          y = y * (1.5 - 0.5 * x * y * y);
          c = y;
          s = td * y;
          sm.changed = 1;
        }
        sm.cs[t][0] = c;
        sm.cs[t][1] = s;
      }
      __syncthreads();
      {
        const int ip = sm.pi[step][bp], jp = sm.pj[step][bp];
        const int iq = sm.pi[step][bq], jq = sm.pj[step][bq];
        const double cp = sm.cs[bp][0], sp = sm.cs[bp][1], cq = sm.cs[bq][0], sq = sm.cs[bq][1];
        if (sp != 0.0 || sq != 0.0) {
          const double a = sm.S[ip][iq], b = sm.S[ip][jq], c = sm.S[jp][iq], d = sm.S[jp][jq];
          // columns: (x, y) -> (cq x - sq y, sq x + cq y)
          const double a1 = cq * a - sq * b, b1 = sq * a + cq * b;
          const double c1 = cq * c - sq * d, d1 = sq * c + cq * d;
          // rows: (u, v) -> (cp u - sp v, sp u + cp v)
          sm.S[ip][iq] = cp * a1 - sp * c1;
          sm.S[jp][iq] = sp * a1 + cp * c1;
          sm.S[ip][jq] = cp * b1 - sp * d1;
          sm.S[jp][jq] = sp * b1 + cp * d1;
          if (bp == bq && sp != 0.0) {  // the annihilated element (exact zero)
            sm.S[ip][jq] = 0.0;
            sm.S[jp][iq] = 0.0;
          }
        }
        // J <- J * R: 32 rows x 16 pairs, two items per thread
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int item = t + h * JT, p = item >> 5, r = item & 31;
          const double s = sm.cs[p][1];
          if (s != 0.0) {
            const int i = sm.pi[step][p], j = sm.pj[step][p];
            const double c = sm.cs[p][0];
            const double x = sm.J[r][i], y = sm.J[r][j];
            sm.J[r][i] = c * x - s * y;
            sm.J[r][j] = s * x + c * y;
          }
        }
      }
      __syncthreads();
    }
    if (!sm.changed) break;
    __syncthreads();
  }
}

__device__ void init_pair_tables(Small& sm) {
  for (int idx = threadIdx.x; idx < (JW - 1) * (JW / 2); idx += JT) {
    const int step = idx / (JW / 2), p = idx - step * (JW / 2);
    int i, j;
    circle_pair(JW, step, p, i, j);
    sm.pi[step][p] = static_cast<unsigned char>(i);
    sm.pj[step][p] = static_cast<unsigned char>(j);
  }
}

// Gram -> measure -> (inner Jacobi).  Returns true when the pair must be rotated.
__device__ bool finish_gram(Small& sm, const double (&acc)[4], double z2, double inv_f2, const PersArgs& a,
                            int sweep) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3, mt = warp >> 2, nt = warp & 3;
  {
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
    atomicMax(&a.conv[sweep], static_cast<unsigned long long>(__double_as_longlong(m)));
  }
  __syncthreads();
  const bool rotate = sm.red[0] > a.tol;
  if (rotate) inner_jacobi(sm, z2, inv_f2, a.tol, a.max_inner);
  return rotate;
}

// RESIDENT: the pair's G columns (<= 256 rows) and V columns (<= 256 rows)
// stay in shared memory for the whole round.
__global__ void __launch_bounds__(JT, 1) jacobi_resident_kernel(PersArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  Chunk* XG = reinterpret_cast<Chunk*>(dyn);
  Chunk* XV = XG + RES_CHUNKS;
  Small& sm = *reinterpret_cast<Small*>(XV + RES_CHUNKS);
  init_pair_tables(sm);
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const int p = blockIdx.x % a.npairs, b = a.batch0 + blockIdx.x / a.npairs;
  double* G = a.G + b * a.gstride;
  double* V = a.V + b * a.vstride;
  const double z2 = a.zero2[2 * b], inv_f2 = a.zero2[2 * b + 1];
  const int ncg = (a.mg + JCH - 1) / JCH, ncv = (a.vrows + JCH - 1) / JCH;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int round = 0; round < a.nb - 1; ++round) {
      int ba, bb;
      circle_pair(a.nb, round, p, ba, bb);
      const int ca = ba * JB, cb = bb * JB;
      const bool prof = a.prof && blockIdx.x == 0 && threadIdx.x == 0;
      long long t0 = prof ? clock64() : 0;
      for (int k = 0; k < ncg; ++k) load_chunk_async(XG[k], G, a.ldg, a.mg, k * JCH, ca, cb);
      for (int k = 0; k < ncv; ++k) load_chunk_async(XV[k], V, a.ldv, a.vrows, k * JCH, ca, cb);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      long long t1 = prof ? clock64() : 0;
      double acc[4] = {0, 0, 0, 0};
      for (int k = 0; k < ncg; ++k) gram_chunk(XG[k], acc);
      __syncthreads();
      long long t2 = prof ? clock64() : 0, t3 = 0;
      if (finish_gram(sm, acc, z2, inv_f2, a, sweep)) {
        t3 = prof ? clock64() : 0;
        for (int k = 0; k < ncg; ++k) {
          rotate_chunk(XG[k], sm);
          store_chunk(XG[k], G, a.ldg, a.mg, k * JCH, ca, cb);
        }
        for (int k = 0; k < ncv; ++k) {
          rotate_chunk(XV[k], sm);
          store_chunk(XV[k], V, a.ldv, a.vrows, k * JCH, ca, cb);
        }
      } else {
        t3 = prof ? clock64() : 0;
      }
      long long t4 = prof ? clock64() : 0;
      grid.sync();
      if (prof) {
        const long long t5 = clock64();
        a.prof[0] += t1 - t0;  // load
        a.prof[1] += t2 - t1;  // gram
        a.prof[2] += t3 - t2;  // measure + inner Jacobi
        a.prof[3] += t4 - t3;  // rotate + store
        a.prof[4] += t5 - t4;  // grid barrier
        a.prof[5] += 1;
      }
    }
    const double meas = __longlong_as_double(
        static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&a.conv[sweep])));
    if (meas < a.stop_tol) {
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_out = sweep;
}

// STREAM: 64-row chunks double-buffered through shared memory.
__device__ void stream_rotate(Chunk* X, double* M, long ld, int rows, int ca, int cb, const Small& sm) {
  const int nch = (rows + JCH - 1) / JCH;
  load_chunk_async(X[0], M, ld, rows, 0, ca, cb);
  cp_commit();
  for (int k = 0; k < nch; ++k) {
    if (k + 1 < nch) load_chunk_async(X[(k + 1) & 1], M, ld, rows, (k + 1) * JCH, ca, cb);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    rotate_chunk(X[k & 1], sm);
    store_chunk(X[k & 1], M, ld, rows, k * JCH, ca, cb);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(JT, 2) jacobi_stream_kernel(PersArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  Chunk* X = reinterpret_cast<Chunk*>(dyn);
  Small& sm = *reinterpret_cast<Small*>(X + 2);
  init_pair_tables(sm);
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const int p = blockIdx.x % a.npairs, b = a.batch0 + blockIdx.x / a.npairs;
  double* G = a.G + b * a.gstride;
  double* V = a.V + b * a.vstride;
  const double z2 = a.zero2[2 * b], inv_f2 = a.zero2[2 * b + 1];
  const int nch = (a.mg + JCH - 1) / JCH;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int round = 0; round < a.nb - 1; ++round) {
      int ba, bb;
      circle_pair(a.nb, round, p, ba, bb);
      const int ca = ba * JB, cb = bb * JB;
      double acc[4] = {0, 0, 0, 0};
      load_chunk_async(X[0], G, a.ldg, a.mg, 0, ca, cb);
      cp_commit();
      for (int k = 0; k < nch; ++k) {
        if (k + 1 < nch) load_chunk_async(X[(k + 1) & 1], G, a.ldg, a.mg, (k + 1) * JCH, ca, cb);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        gram_chunk(X[k & 1], acc);
        __syncthreads();
      }
      if (finish_gram(sm, acc, z2, inv_f2, a, sweep)) {
        stream_rotate(X, G, a.ldg, a.mg, ca, cb, sm);
        stream_rotate(X, V, a.ldv, a.vrows, ca, cb, sm);
      }
      grid.sync();
    }
    const double meas = __longlong_as_double(
        static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&a.conv[sweep])));
    if (meas < a.stop_tol) {
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_out = sweep;
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

// G (col-major, ld = ldg >= mg, ng cols) from theta row-major (m x n):
//   rows side: G[c][r] = theta[c][r] (c < m, r < n), zero for c >= m
//   cols side: G[c][r] = theta[r][c] (c < n, r < m), zero for c >= n
// rows mg..ldg-1 are zero.
__global__ void load_g_kernel(const double* __restrict__ theta, long tstride, int m, int n,
                              double* __restrict__ G, long gstride, long ldg, int mg, int ng,
                              int rows_side) {
  __shared__ double tile[32][33];
  const double* T = theta + blockIdx.z * tstride;
  double* Gb = G + blockIdx.z * gstride;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;  // G column / row tile
  if (rows_side) {
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int c = c0 + dy, r = r0 + threadIdx.x;
      if (c < ng && r < ldg)
        Gb[static_cast<long>(c) * ldg + r] = (c < m && r < mg) ? T[static_cast<long>(c) * n + r] : 0.0;
    }
  } else {
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int r = r0 + dy, c = c0 + threadIdx.x;
      tile[dy][threadIdx.x] = (r < m && c < n) ? T[static_cast<long>(r) * n + c] : 0.0;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
      const int c = c0 + dy, r = r0 + threadIdx.x;
      if (c < ng && r < ldg) Gb[static_cast<long>(c) * ldg + r] = tile[threadIdx.x][dy];
    }
  }
}

// zero2[b] = (64 sqrt(mg) eps ||G_b||_F)^2.  Columns below this norm are
// rounding noise (a rank-deficient theta leaves such columns; their direction
// is undefined and their norm is below the reference's own normwise accuracy):
// they are not rotated and do not enter the convergence measure.
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
    const double f = 64.0 * sqrt(static_cast<double>(mg)) * EPS;
    zero2[2 * blockIdx.x] = f * f * t;
    zero2[2 * blockIdx.x + 1] = t > 0 ? 1.0 / t : 1.0;  // 1 / ||G||_F^2 (scale-free angles)
  }
}

// sigma_c = ||G[:,c]|| for real columns, -1 for pad columns (sorted last)
__global__ void col_norm_kernel(const double* __restrict__ G, long gstride, long ldg, int ng,
                                int ng_real, int pad_mod, int pad_lim, double* __restrict__ sig,
                                long sstride) {
  const int warps = blockDim.x >> 5;
  const int c = blockIdx.x * warps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= ng) return;
  const double* col = G + blockIdx.y * gstride + static_cast<long>(c) * ldg;
  double s = 0.0;
  for (int r = lane; r < ldg; r += 32) s += col[r] * col[r];
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
    const double av = fabs(u[r]);
    if (av > best) { best = av; idx = r; val = u[r]; }
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
__global__ void gather_kernel(const double* __restrict__ G, long ldg, const double* __restrict__ V,
                              int ng, const double* __restrict__ sorted, const int* __restrict__ perm,
                              const double* __restrict__ sign, int k, int rows_side, int m_true,
                              int n_true, double* __restrict__ U, double* __restrict__ VT) {
  // rows side: U[i][q] = V[perm q][i] * sg ; VT[q][j] = G[perm q][j] * sg / sigma
  // cols side: U[i][q] = G[perm q][i] * sg / sigma ; VT[q][j] = V[perm q][j] * sg
  const long tot_u = static_cast<long>(m_true) * k, tot_v = static_cast<long>(k) * n_true;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot_u + tot_v;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    if (t < tot_u) {
      const int i = static_cast<int>(t / k), q = static_cast<int>(t % k);
      const double sg = sign[q], s = sorted[q];
      U[t] = rows_side ? V[static_cast<long>(perm[q]) * ng + i] * sg
                       : (s > 0 ? G[static_cast<long>(perm[q]) * ldg + i] * sg / s : 0.0);
    } else {
      const long u = t - tot_u;
      const int q = static_cast<int>(u / n_true), j = static_cast<int>(u % n_true);
      const double sg = sign[q], s = sorted[q];
      VT[u] = rows_side ? (s > 0 ? G[static_cast<long>(perm[q]) * ldg + j] * sg / s : 0.0)
                        : V[static_cast<long>(perm[q]) * ng + j] * sg;
    }
  }
}

size_t resident_smem() { return sizeof(Chunk) * 2 * RES_CHUNKS + sizeof(Small) + 16; }
size_t stream_smem() { return sizeof(Chunk) * 2 + sizeof(Small) + 16; }

}  // namespace

SvdResultDev svd_device(Ctx& ctx, SvdWs& ws, const double* theta, int m, int n, int m_true,
                        int n_true, SvdSide side, int batch, long bstride, double* sigma_out) {
  const bool rows = side == SvdSide::kRows;
  const int ng_real = rows ? m : n;
  const int mg = rows ? n : m;
  const long ldg = mg + (mg & 1);  // 16-byte aligned columns for cp.async
  const int ng = ((ng_real + JW - 1) / JW) * JW;
  const long gstride = ldg * ng, vstride = static_cast<long>(ng) * ng;
  double* G = ws.G.reserve(static_cast<size_t>(gstride) * batch);
  double* V = ws.V.reserve(static_cast<size_t>(vstride) * batch);
  double* sig = ws.sig.reserve(static_cast<size_t>(ng) * batch);
  double* sorted = ws.sorted.reserve(static_cast<size_t>(ng) * batch);
  int* perm = ws.perm.reserve(static_cast<size_t>(ng) * batch);
  unsigned long long* conv = ws.conv.reserve(MAX_SWEEPS * 8);
  double* zero2 = ws.zero2.reserve(2 * static_cast<size_t>(batch));
  int* sweeps_dev = ws.sweeps.reserve(64);
  int* sweeps_host = ws.sweeps_host.reserve(64);
  {
    dim3 grid(cdiv(ng, 32), cdiv(ldg, 32), batch), blk(32, 8);
    load_g_kernel<<<grid, blk, 0, ctx.stream>>>(theta, bstride, m, n, G, gstride, ldg, mg, ng,
                                                rows ? 1 : 0);
    ACHI_LAUNCHED(ctx);
    dim3 g2(static_cast<unsigned>(std::min<long>(cdiv(vstride, 256), 4L * ctx.num_sms)), batch);
    identity_kernel<<<g2, 256, 0, ctx.stream>>>(V, ng, ng, vstride);
    ACHI_LAUNCHED(ctx);
    zero_floor_kernel<<<batch, 1024, 0, ctx.stream>>>(G, gstride, gstride, mg, zero2);
    ACHI_LAUNCHED(ctx);
  }
  const int nb = ng / JB;  // even (ng multiple of 32)
  const int npairs = nb / 2;
  const bool resident = ldg <= RES_CHUNKS * JCH && ng <= RES_CHUNKS * JCH;
  const size_t smem = resident ? resident_smem() : stream_smem();
  void* kern = resident ? reinterpret_cast<void*>(jacobi_resident_kernel)
                        : reinterpret_cast<void*>(jacobi_stream_kernel);
  static int max_blocks[2] = {0, 0};
  int& mb = max_blocks[resident ? 0 : 1];
  if (mb == 0) {
    ACHI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    int per_sm = 0;
    ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, JT, smem));
    mb = per_sm * ctx.num_sms;
    if (mb < 1) fail(ACHI_E_CUDA, "svd: Jacobi kernel cannot be resident");
  }
  if (npairs > mb) fail(ACHI_E_SIZE_GUARD, "svd: matrix too wide for one cooperative launch");
  const int per_launch = std::max(1, mb / npairs);
  const double tol = std::max(1e-15, 2.0 * std::sqrt(static_cast<double>(mg)) * EPS);
  // inner sweeps per block pair and the outer stop threshold (measure of the
  // last sweep; off-diagonals after it are ~measure^2).  Tunable for studies.
  static const int max_inner = [] {
    const char* e = std::getenv("ACHI_JACOBI_INNER");
    return e ? std::max(1, std::atoi(e)) : 1;  // 1 measured fastest (profiles/svd_inner_study_r01.txt)
  }();
  static const double stop_tol = [] {
    const char* e = std::getenv("ACHI_JACOBI_STOP");
    return e ? std::atof(e) : 1e-7;
  }();
  int launches = 0;
  for (int b0 = 0; b0 < batch; b0 += per_launch, ++launches) {
    const int nbat = std::min(per_launch, batch - b0);
    ACHI_CUDA(cudaMemsetAsync(conv, 0, sizeof(unsigned long long) * MAX_SWEEPS, ctx.stream));
    PersArgs a{G, ldg, gstride, mg, V, ng, vstride, ng, nb, npairs, b0,
               max_inner, tol, stop_tol, zero2, conv, sweeps_dev + (launches % 64), nullptr};
    static const bool prof_on = std::getenv("ACHI_JACOBI_PROF") != nullptr;
    static DevArr<long long> profbuf;
    if (prof_on) {
      a.prof = profbuf.reserve(8);
      ACHI_CUDA(cudaMemsetAsync(a.prof, 0, 8 * sizeof(long long), ctx.stream));
    }
    void* args[] = {&a};
    ACHI_CUDA(cudaLaunchCooperativeKernel(kern, dim3(npairs * nbat), dim3(JT), args, smem, ctx.stream));
    ACHI_LAUNCHED(ctx);
    if (prof_on) {
      long long h[8];
      ACHI_CUDA(cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
      const double r = h[5] > 0 ? static_cast<double>(h[5]) : 1.0;
      std::fprintf(stderr,
                   "[jacobi] n=%d rounds=%lld cycles/round: load %.0f gram %.0f inner %.0f rotate %.0f "
                   "barrier %.0f\n",
                   ng, h[5], h[0] / r, h[1] / r, h[2] / r, h[3] / r, h[4] / r);
    }
  }
  // pad columns: rows side -> columns >= m_true (theta rows (l,s1), padded l last);
  // cols side with padding -> columns (s2, jr) with jr >= chr_true (d = 2 on the padded path)
  int pad_mod = ng, pad_lim = rows ? m_true : n_true;
  if (!rows && n != n_true) {
    pad_mod = n / 2;
    pad_lim = n_true / 2;
  }
  {
    dim3 grid(cdiv(ng, 8), batch);
    col_norm_kernel<<<grid, 256, 0, ctx.stream>>>(G, gstride, ldg, ng, ng_real, pad_mod, pad_lim,
                                                  sig, ng);
    ACHI_LAUNCHED(ctx);
    sort_kernel<<<batch, 1024, sizeof(double) * ng, ctx.stream>>>(sig, ng, ng, sorted, perm);
    ACHI_LAUNCHED(ctx);
  }
  ACHI_CUDA(cudaMemcpyAsync(sweeps_host, sweeps_dev, sizeof(int) * std::min(launches, 64),
                            cudaMemcpyDeviceToHost, ctx.stream));
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
  r.mg = static_cast<int>(ldg);
  r.r_true = r_true;
  r.sweeps_host = sweeps_host;
  r.n_launches = std::min(launches, 64);
  r.G = G;
  r.V = V;
  r.sigma = sorted;
  r.perm = perm;
  return r;
}

int SvdResultDev::sweeps() const {
  int s = 0;
  for (int i = 0; i < n_launches; ++i) s = std::max(s, sweeps_host[i]);
  if (s >= MAX_SWEEPS) fail(ACHI_E_NUMERICAL_FAILURE, "svd: decomposition did not converge");
  return s;
}

void svd_phase_signs(Ctx& ctx, SvdWs& ws, const SvdResultDev& r, int kept) {
  double* sign = ws.sign.reserve(static_cast<size_t>(std::max(kept, 1)));
  if (kept <= 0) return;
  const bool rows = r.side == SvdSide::kRows;
  // U columns: rows side -> V[:, perm k] (length m); cols side -> G[:, perm k] (length m)
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
                                                r.n_true, U, VT);
  ACHI_LAUNCHED(ctx);
}

}  // namespace achi
