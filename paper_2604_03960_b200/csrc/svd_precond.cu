// QR preconditioner for the cluster-resident Jacobi SVD (svd_jacobi.cu).
//
// One-sided Jacobi on G converges in far fewer sweeps when it runs on R^T from
// a QR factorisation instead of on G itself (Drmac & Veselic's preconditioned
// Jacobi): with G^T Pi = Q R (Pi sorting G's rows by decreasing norm, Q
// orthogonal), G Q = Pi R^T, whose column Gram R R^T is strongly graded and
// nearly diagonal.  Measured on C3 thetas (tools/precond_study.py): 11-12 ->
// 5 Jacobi sweeps.  Q is exactly orthogonal (Householder), so it is a valid
// start factor: the Jacobi runs on G Q and V accumulates from Q, which is how
// svd_device already treats a warm start.  Only G's real columns (coordinates)
// take part; pad coordinates keep the identity, so pads stay exactly zero.
//
// qr_precond_kernel: one thread-block cluster, CTA t owns 32 columns of A =
// (G^T Pi restricted to real coordinates, nr x mr) and 32 columns of Q.
// Panel p (32 reflectors) is factored by CTA p (unblocked Householder with
// LAPACK dlarfg signs, one warp forms each reflector), its compact-WY factor
// T is built in place, one cluster barrier publishes it, and every later CTA
// applies I - V T^T V^T to its block after staging V from CTA p's shared
// memory.  Q = H_1 ... H_k is then formed block by block.  Outputs: G <- G Q
// (= Pi R^T, written from R), V0 <- Q embedded at the real coordinates.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "svd_jacobi.cuh"

namespace cg = cooperative_groups;

namespace achi {

namespace {

constexpr int PQ_T = 256;    // threads per CTA
constexpr int PQ_B = 32;     // columns per CTA / panel width
constexpr int PQ_MAX = 256;  // max real coordinates (nr) and rows (mr)
constexpr int PQ_LD = PQ_MAX + 4;  // = 4 mod 16 doubles: conflict-free DMMA fragments
constexpr int PQ_WLD = PQ_B + 4;

struct PqSmem {
  double A[PQ_B][PQ_LD];   // this CTA's columns of A (column c at A[c][row])
  double Vs[PQ_B][PQ_LD];  // staged reflectors of the panel being applied
  double Qr[PQ_B][PQ_LD];  // this CTA's rows of Q (row r at Qr[r][col])
  double T[PQ_B][PQ_B + 1];
  double W[PQ_B][PQ_WLD];
  double Ts[PQ_B][PQ_B + 1];  // staged T of a remote panel
  double tau[PQ_B];
  double key[PQ_MAX];
  int P[PQ_MAX];
  int Pown[PQ_B];  // Pi entries of this CTA's columns
};

struct PqArgs {
  double* G;
  long ldg;
  int mr;        // rows of G that take part (= working rows mg)
  int ng;        // columns of G / order of V0
  int nr;        // real coordinates
  int pad_mod, pad_lim;  // real coordinate i -> column (i / pad_lim) * pad_mod + i % pad_lim
  int k;         // reflectors = min(nr, mr)
  double* V0;    // ng x ng col-major, identity on entry
  long long* prof;  // ACHI_QR_PROF: cycles of CTA 1 {sort, load, stage, columns, factor, qrows, out}
};

__device__ __forceinline__ int coord(const PqArgs& a, int i) {
  return (i / a.pad_lim) * a.pad_mod + (i % a.pad_lim);
}

// 1/x from the FP64 reciprocal estimate and two Newton steps (to rounding;
// the reflector stays orthogonal to working precision), off the DDIV slow path
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// stage panel p's reflectors (unit diagonal, zeros above) and T from CTA p
__device__ void stage_panel(cg::cluster_group& cl, PqSmem& sm, const PqArgs& a, int p, int bw) {
  PqSmem* rs = cl.map_shared_rank(&sm, p);
  const int j0 = p * PQ_B;
  const int nrp = (a.nr + 15) & ~15;
  for (int idx = threadIdx.x; idx < PQ_B * nrp; idx += PQ_T) {
    const int c = idx / nrp, i = idx - c * nrp;
    double v = 0.0;
    if (c < bw && i < a.nr) v = i < j0 + c ? 0.0 : (i == j0 + c ? 1.0 : rs->A[c][i]);
    sm.Vs[c][i] = v;
  }
  for (int idx = threadIdx.x; idx < PQ_B * PQ_B; idx += PQ_T) {
    const int r = idx / PQ_B, c = idx - r * PQ_B;
    sm.Ts[r][c] = rs->T[r][c];
  }
  __syncthreads();
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Fragments of m16n8k4 (row.col): a0 = A[g][t], a1 = A[g+8][t], b0 = B[t][g],
// c = {C[g][2t], C[g][2t+1], C[g+8][2t], C[g+8][2t+1]} with g = lane/4, t = lane%4.

// W (32 x 32) = Vs (32 x K rows-major) . X^T, X stored as X[c][i] (columns), K = nrp
__device__ __forceinline__ void dmma_vtx(const double (*Vr)[PQ_LD], const double (*X)[PQ_LD], int nrp,
                                         double (*W)[PQ_WLD]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int m0 = (warp >> 2) * 16, n0 = (warp & 3) * 8;
  double acc[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < nrp; k0 += 4)
    dmma(acc, Vr[m0 + g][k0 + tq], Vr[m0 + g + 8][k0 + tq], X[n0 + g][k0 + tq]);
  W[m0 + g][n0 + 2 * tq] = acc[0];
  W[m0 + g][n0 + 2 * tq + 1] = acc[1];
  W[m0 + g + 8][n0 + 2 * tq] = acc[2];
  W[m0 + g + 8][n0 + 2 * tq + 1] = acc[3];
}

// A block (columns) <- (I - V T^T V^T) A  (QR trailing update, H^T from the left)
__device__ void update_columns(PqSmem& sm, int nr, int bw) {
  const int nrp = (nr + 15) & ~15;
  dmma_vtx(sm.Vs, sm.A, nrp, sm.W);  // W = V^T A
  __syncthreads();
  {
    constexpr int Q = PQ_B * PQ_B / PQ_T;  // W2 = T^T W: W2[r][c] = sum_{b <= r} T[b][r] W[b][c]
    const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    double s[Q] = {};
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int r = r0 + 8 * q;
      if (r < bw)
        for (int b = 0; b <= r; ++b) s[q] = fma(sm.Ts[b][r], sm.W[b][c], s[q]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < Q; ++q) sm.W[r0 + 8 * q][c] = s[q];
  }
  __syncthreads();
  // A[c][i] -= sum_r V[i][r] W2[r][c]: C tile rows i (16), columns c (8), K = r (32)
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int ntile = (nrp / 16) * 4;
    for (int tile = warp; tile < ntile; tile += PQ_T / 32) {
      const int m0 = (tile >> 2) * 16, n0 = (tile & 3) * 8;
      double acc[4] = {sm.A[n0 + 2 * tq][m0 + g], sm.A[n0 + 2 * tq + 1][m0 + g],
                       sm.A[n0 + 2 * tq][m0 + g + 8], sm.A[n0 + 2 * tq + 1][m0 + g + 8]};
#pragma unroll
      for (int k0 = 0; k0 < PQ_B; k0 += 4)
        dmma(acc, -sm.Vs[k0 + tq][m0 + g], -sm.Vs[k0 + tq][m0 + g + 8], sm.W[k0 + tq][n0 + g]);
      sm.A[n0 + 2 * tq][m0 + g] = acc[0];
      sm.A[n0 + 2 * tq + 1][m0 + g] = acc[1];
      sm.A[n0 + 2 * tq][m0 + g + 8] = acc[2];
      sm.A[n0 + 2 * tq + 1][m0 + g + 8] = acc[3];
    }
  }
  __syncthreads();
}

// Q rows <- Q rows (I - V T V^T)  (forward accumulation of Q = H_1 ... H_k)
__device__ void update_qrows(PqSmem& sm, int nr, int bw) {
  const int nrp = (nr + 15) & ~15;
  dmma_vtx(sm.Qr, sm.Vs, nrp, sm.W);  // W = Qr V  (W[r][a] = sum_i Qr[r][i] Vs[a][i])
  __syncthreads();
  {
    constexpr int Q = PQ_B * PQ_B / PQ_T;  // W2 = W T: W2[r][a] = sum_{b <= a} W[r][b] T[b][a]
    const int a = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    double s[Q] = {};
    if (a < bw)
      for (int b = 0; b <= a; ++b) {
        const double tb = sm.Ts[b][a];
#pragma unroll
        for (int q = 0; q < Q; ++q) s[q] = fma(sm.W[r0 + 8 * q][b], tb, s[q]);
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < Q; ++q) sm.W[r0 + 8 * q][a] = s[q];
  }
  __syncthreads();
  // Qr[r][i] -= sum_a W2[r][a] Vs[a][i]: C tile rows r (16), columns i (8), K = a (32)
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int ntile = 2 * (nrp / 8);
    for (int tile = warp; tile < ntile; tile += PQ_T / 32) {
      const int m0 = (tile & 1) * 16, n0 = (tile >> 1) * 8;
      double acc[4] = {sm.Qr[m0 + g][n0 + 2 * tq], sm.Qr[m0 + g][n0 + 2 * tq + 1],
                       sm.Qr[m0 + g + 8][n0 + 2 * tq], sm.Qr[m0 + g + 8][n0 + 2 * tq + 1]};
#pragma unroll
      for (int k0 = 0; k0 < PQ_B; k0 += 4)
        dmma(acc, -sm.W[m0 + g][k0 + tq], -sm.W[m0 + g + 8][k0 + tq], sm.Vs[k0 + tq][n0 + g]);
      sm.Qr[m0 + g][n0 + 2 * tq] = acc[0];
      sm.Qr[m0 + g][n0 + 2 * tq + 1] = acc[1];
      sm.Qr[m0 + g + 8][n0 + 2 * tq] = acc[2];
      sm.Qr[m0 + g + 8][n0 + 2 * tq + 1] = acc[3];
    }
  }
  __syncthreads();
}

// Householder factorisation of panel p (owner CTA), register resident: warp w
// holds panel columns w, w+8, w+16, w+24 (lane l: rows l + 32 q).  Step c: the
// owner of column c has published it to shared memory; every warp reads it,
// forms the reflector (same bits in every warp: dlarfg signs), and applies it
// to its own columns in registers (the reflector is used unscaled with its
// scale factor); the owner of column c + 1 then publishes that column.  One
// block barrier per column.  Finally the columns (R above, v below the
// diagonal) go back to shared memory and T of the compact WY form is built.
constexpr int PQ_NQ = PQ_MAX / 32;  // rows per lane

__device__ void factor_panel(PqSmem& sm, const PqArgs& a, int p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool prof = a.prof && threadIdx.x == 0 && p == 1;
  const long long tstart = prof ? clock64() : 0;
  const int j0 = p * PQ_B, bw = min(PQ_B, a.k - j0), wcols = min(PQ_B, a.mr - j0);
  const int nr = a.nr;
  double col[4][PQ_NQ];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int cc = warp + 8 * m;
#pragma unroll
    for (int q = 0; q < PQ_NQ; ++q) {
      const int i = lane + 32 * q;
      col[m][q] = (cc < wcols && i < nr) ? sm.A[cc][i] : 0.0;
    }
  }
  for (int c = 0; c < bw; ++c) {
    const int j = j0 + c;
    double piv[PQ_NQ];
    double xn = 0.0;
#pragma unroll
    for (int q = 0; q < PQ_NQ; ++q) {
      const int i = lane + 32 * q;
      piv[q] = (i > j && i < nr) ? sm.A[c][i] : 0.0;
      xn = fma(piv[q], piv[q], xn);
    }
    const long long pc0 = prof ? clock64() : 0;
    const double alpha = sm.A[c][j];
    xn = warp_sum(xn);
    const long long pc1 = prof ? clock64() : 0;
    double tau = 0.0, sc = 0.0, beta = alpha;
    if (xn > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, xn));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) * rcp_nr(beta);
      sc = rcp_nr(alpha - beta);
    }
    const long long pc2 = prof ? clock64() : 0;
    if (threadIdx.x == 0) sm.tau[c] = tau;
    // v = (1 at row j, sc * x below), zero above; a <- a - tau (v^T a) v
    double v[PQ_NQ];
#pragma unroll
    for (int q = 0; q < PQ_NQ; ++q) {
      const int i = lane + 32 * q;
      v[q] = i > j ? piv[q] * sc : (i == j ? 1.0 : 0.0);
    }
    if (tau != 0.0) {
      double d[4] = {0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < PQ_NQ; ++q)
#pragma unroll
        for (int m = 0; m < 4; ++m) d[m] = fma(v[q], col[m][q], d[m]);
#pragma unroll
      for (int m = 0; m < 4; ++m) d[m] = warp_sum(d[m]);
      if (prof) a.prof[11] += clock64() - pc2;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int cc = warp + 8 * m;
        if (cc > c && cc < wcols) {
          const double f = tau * d[m];
#pragma unroll
          for (int q = 0; q < PQ_NQ; ++q) col[m][q] = fma(-f, v[q], col[m][q]);
        }
      }
    }
    // the owner finishes column c in registers: v below the diagonal, beta on it
    if ((c & 7) == warp) {
      const int m = c >> 3;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
        if (mm == m) {
#pragma unroll
          for (int q = 0; q < PQ_NQ; ++q) {
            const int i = lane + 32 * q;
            col[mm][q] = i > j ? (tau != 0.0 ? v[q] : col[mm][q]) : (i == j ? beta : col[mm][q]);
          }
        }
    }
    // the owner of column c + 1 publishes it for the next step
    if (c + 1 < bw && ((c + 1) & 7) == warp) {
      const int m = (c + 1) >> 3;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
        if (mm == m) {
#pragma unroll
          for (int q = 0; q < PQ_NQ; ++q) {
            const int i = lane + 32 * q;
            if (i < nr) sm.A[c + 1][i] = col[mm][q];
          }
        }
    }
    const long long pc3 = prof ? clock64() : 0;
    __syncthreads();
    if (prof) {
      const long long pc4 = clock64();
      a.prof[9] += pc1 - pc0;   // alpha load + norm warp reduction
      a.prof[10] += pc2 - pc1;  // sqrt / divisions
      a.prof[12] += pc3 - pc2;  // dots, reductions, updates, publish (warp 0)
      a.prof[13] += pc4 - pc3;  // barrier
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int cc = warp + 8 * m;
    if (cc < wcols)
#pragma unroll
      for (int q = 0; q < PQ_NQ; ++q) {
        const int i = lane + 32 * q;
        if (i < nr) sm.A[cc][i] = col[m][q];
      }
  }
  __syncthreads();
  if (prof) a.prof[6] += clock64() - tstart;
  // compact WY: T upper triangular, T[c][c] = tau_c,
  // T[0:c, c] = -tau_c T[0:c, 0:c] Y[0:c, c],  Y = V^T V (strict upper part).
  // Y: lane = column c, warp = rows r0 + 8 q; the reflector entries are
  // selected branch-free (unit on the diagonal, zero above, v below).
  {
    // Y = Vm^T Vm with the reflector masks applied on the fragments
    const int g = lane >> 2, tq = lane & 3;
    const int m0 = (warp >> 2) * 16, n0 = (warp & 3) * 8;
    const int nrp = (nr + 15) & ~15;
    auto vm = [&](int r, int i) -> double {  // reflector r, row i
      const int jr = j0 + r;
      const double x = sm.A[r][i];
      return i > jr ? x : (i == jr ? 1.0 : 0.0);
    };
    double acc[4] = {0, 0, 0, 0};
    for (int k0 = j0 & ~3; k0 < nrp; k0 += 4)
      dmma(acc, vm(m0 + g, k0 + tq), vm(m0 + g + 8, k0 + tq), vm(n0 + g, k0 + tq));
    const int r = m0 + g, c = n0 + 2 * tq;
    sm.W[r][c] = (r < c && c < bw) ? acc[0] : 0.0;
    sm.W[r][c + 1] = (r < c + 1 && c + 1 < bw) ? acc[1] : 0.0;
    sm.W[r + 8][c] = (r + 8 < c && c < bw) ? acc[2] : 0.0;
    sm.W[r + 8][c + 1] = (r + 8 < c + 1 && c + 1 < bw) ? acc[3] : 0.0;
  }
  __syncthreads();
  if (prof) a.prof[8] += clock64() - tstart;
  if (warp == 0) {  // lane r holds row r of T in registers; T[r][b] = 0 for b < r
    double trow[PQ_B];
#pragma unroll
    for (int b = 0; b < PQ_B; ++b) trow[b] = 0.0;
#pragma unroll
    for (int c = 0; c < PQ_B; ++c) {
      if (c < bw) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int b = 0; b < c; ++b) {
          if (b & 1) s1 = fma(trow[b], sm.W[b][c], s1);
          else s0 = fma(trow[b], sm.W[b][c], s0);
        }
        const double tc = sm.tau[c];
        trow[c] = lane < c ? -tc * (s0 + s1) : (lane == c ? tc : 0.0);
      }
    }
#pragma unroll
    for (int b = 0; b < PQ_B; ++b) sm.T[lane][b] = trow[b];
  }
  __syncthreads();
  if (prof) a.prof[7] += clock64() - tstart;
}

__global__ void __launch_bounds__(PQ_T, 1) qr_precond_kernel(PqArgs a) {
  pdl_wait();  // launched with launch_pdl / the PDL attribute (common.cuh)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PqSmem& sm = *reinterpret_cast<PqSmem*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int t = static_cast<int>(cl.block_rank());

  // 1. CTA 0: rows of G by decreasing norm (ties by index), bitonic sort
  if (t == 0) {
    for (int r = threadIdx.x; r < PQ_MAX; r += PQ_T) {
      double s = -1.0;
      if (r < a.mr) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int c = 0;
        for (; c + 8 <= a.ng; c += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double g = a.G[static_cast<long>(c + u) * a.ldg + r];
            acc[u] = fma(g, g, acc[u]);
          }
        }
        for (; c < a.ng; ++c) {
          const double g = a.G[static_cast<long>(c) * a.ldg + r];
          acc[0] = fma(g, g, acc[0]);
        }
        s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      }
      sm.key[r] = s;
      sm.P[r] = r;
    }
    __syncthreads();
    for (int size = 2; size <= PQ_MAX; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < PQ_MAX; i += PQ_T) {
          const int j = i ^ stride;
          if (j > i) {
            const bool desc = (i & size) == 0;  // descending runs first
            const double ki = sm.key[i], kj = sm.key[j];
            const int pi = sm.P[i], pj = sm.P[j];
            // "i before j" in descending order: larger key, or equal key and smaller index
            const bool i_first = ki > kj || (ki == kj && pi < pj);
            if (desc != i_first) {
              sm.key[i] = kj;
              sm.key[j] = ki;
              sm.P[i] = pj;
              sm.P[j] = pi;
            }
          }
        }
        __syncthreads();
      }
  }
  cl.sync();

  // 2. this CTA's columns of A = G^T Pi (real coordinates), its rows of Q = I
  if (threadIdx.x < PQ_B) {
    const int* P0 = cl.map_shared_rank(sm.P, 0);
    const int col = t * PQ_B + threadIdx.x;
    sm.Pown[threadIdx.x] = col < a.mr ? P0[col] : -1;
  }
  __syncthreads();
  const int nrp = (a.nr + 15) & ~15;
  for (int idx = threadIdx.x; idx < PQ_B * nrp; idx += PQ_T) {
    const int c = idx / nrp, i = idx - c * nrp;
    const int row = sm.Pown[c];
    sm.A[c][i] = (row >= 0 && i < a.nr) ? a.G[static_cast<long>(coord(a, i)) * a.ldg + row] : 0.0;
    sm.Qr[c][i] = (t * PQ_B + c == i && i < a.nr) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npan = (a.k + PQ_B - 1) / PQ_B;

  // 3. panels: CTA p factors panel p; after the barrier every later CTA applies
  // it to its columns and every CTA folds it into its rows of Q.  The next
  // panel's owner factors before its own Q update (critical path first).
  const bool prof = a.prof && t == 1 && threadIdx.x == 0;
  long long tp = prof ? clock64() : 0;
  auto tick = [&](int slot) {
    if (prof) {
      const long long now = clock64();
      a.prof[slot] += now - tp;
      tp = now;
    }
  };
  if (t == 0 && npan > 0) factor_panel(sm, a, 0);
  for (int p = 0; p < npan; ++p) {
    const int bw = min(PQ_B, a.k - p * PQ_B);
    cl.sync();
    tick(0);
    stage_panel(cl, sm, a, p, bw);
    tick(1);
    if (t > p && t * PQ_B < a.mr) update_columns(sm, a.nr, bw);
    tick(2);
    if (t == p + 1 && p + 1 < npan) factor_panel(sm, a, p + 1);
    tick(3);
    if (t * PQ_B < a.nr) update_qrows(sm, a.nr, bw);
    tick(4);
  }
  cl.sync();  // no CTA leaves while its shared memory may still be read
  tick(5);

  // 4. outputs: G <- Pi R^T (row Pi(c) of G = column c of R), V0 <- Q at real coordinates
  for (int idx = threadIdx.x; idx < PQ_B * a.nr; idx += PQ_T) {
    const int c = idx / a.nr, i = idx - c * a.nr;
    const int col = t * PQ_B + c;
    if (col < a.mr) {
      const int row = sm.Pown[c];
      a.G[static_cast<long>(coord(a, i)) * a.ldg + row] = (i <= col && i < a.k) ? sm.A[c][i] : 0.0;
    }
    if (col < a.nr) a.V0[static_cast<long>(coord(a, i)) * a.ng + coord(a, col)] = sm.Qr[c][i];
  }
}

}  // namespace

bool qr_precond_applicable(int mr, int nr) { return mr <= PQ_MAX && nr <= PQ_MAX && nr >= 1 && mr >= 1; }

void qr_precond(Ctx& ctx, double* G, long ldg, int mr, int ng, int nr, int pad_mod, int pad_lim,
                double* V0) {
  if (!qr_precond_applicable(mr, nr)) fail(ACHI_E_INTERNAL, "qr_precond: shape beyond the cluster kernel");
  per_device_once("qr_precond_kernel", ctx.device, [] {
    ACHI_CUDA(cudaFuncSetAttribute(qr_precond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sizeof(PqSmem))));
    return 1;
  });
  static const bool prof_on = std::getenv("ACHI_QR_PROF") != nullptr;
  static DevArr<long long> profbuf;
  PqArgs a{G, ldg, mr, ng, nr, pad_mod, pad_lim, std::min(nr, mr), V0, nullptr};
  if (prof_on) {
    a.prof = profbuf.reserve(16);
    ACHI_CUDA(cudaMemsetAsync(a.prof, 0, 16 * sizeof(long long), ctx.stream));
  }
  const int ncta = (std::max(mr, nr) + PQ_B - 1) / PQ_B;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ncta);
  lc.blockDim = dim3(PQ_T);
  lc.dynamicSmemBytes = sizeof(PqSmem);
  lc.stream = ctx.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  lc.numAttrs = pdl_allowed(lc.stream) ? 2 : 1;
  ACHI_CUDA(cudaLaunchKernelEx(&lc, qr_precond_kernel, a));
  ACHI_LAUNCHED(ctx);
  if (prof_on) {
    long long h[16];
    ACHI_CUDA(cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    std::fprintf(stderr, "[qr-precond] mr=%d nr=%d ctas=%d cycles(CTA1): wait %lld stage %lld columns %lld "
                 "factor %lld qrows %lld tail %lld | panel1 loop %lld loop+Y %lld loop+T %lld | per panel-1 loop: norm %lld sqrtdiv %lld dots %lld work %lld bar %lld\n", mr, nr, ncta, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[8], h[7], h[9], h[10], h[11], h[12], h[13]);
  }
}

}  // namespace achi
