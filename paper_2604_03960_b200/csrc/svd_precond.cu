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

#include "svd_jacobi.cuh"

namespace cg = cooperative_groups;

namespace achi {

namespace {

constexpr int PQ_T = 256;    // threads per CTA
constexpr int PQ_B = 32;     // columns per CTA / panel width
constexpr int PQ_MAX = 256;  // max real coordinates (nr) and rows (mr)
constexpr int PQ_LD = PQ_MAX + 1;

struct PqSmem {
  double A[PQ_B][PQ_LD];   // this CTA's columns of A (column c at A[c][row])
  double Vs[PQ_B][PQ_LD];  // staged reflectors of the panel being applied
  double Qb[PQ_B][PQ_LD];  // this CTA's columns of Q
  double T[PQ_B][PQ_B + 1];
  double W[PQ_B][PQ_B + 1];
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
};

__device__ __forceinline__ int coord(const PqArgs& a, int i) {
  return (i / a.pad_lim) * a.pad_mod + (i % a.pad_lim);
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
  for (int idx = threadIdx.x; idx < PQ_B * a.nr; idx += PQ_T) {
    const int c = idx / a.nr, i = idx - c * a.nr;
    double v = 0.0;
    if (c < bw) v = i < j0 + c ? 0.0 : (i == j0 + c ? 1.0 : rs->A[c][i]);
    sm.Vs[c][i] = v;
  }
  for (int idx = threadIdx.x; idx < PQ_B * PQ_B; idx += PQ_T) {
    const int r = idx / PQ_B, c = idx - r * PQ_B;
    sm.Ts[r][c] = rs->T[r][c];
  }
  __syncthreads();
}

// X (this CTA's 32 columns, nr rows) <- (I - V op(T) V^T) X; op = T^T (trans) or T
__device__ void apply_block_reflector(PqSmem& sm, double (*X)[PQ_LD], int nr, int bw, bool trans) {
  // W = V^T X (bw x 32)
  for (int idx = threadIdx.x; idx < PQ_B * PQ_B; idx += PQ_T) {
    const int r = idx / PQ_B, c = idx - r * PQ_B;
    double s = 0.0;
    if (r < bw)
      for (int i = 0; i < nr; ++i) s = fma(sm.Vs[r][i], X[c][i], s);
    sm.W[r][c] = s;
  }
  __syncthreads();
  // W2 = op(T) W, written over T-staging-free storage: compute into registers then store
  double w2[PQ_B * PQ_B / PQ_T];
  for (int q = 0; q < PQ_B * PQ_B / PQ_T; ++q) {
    const int idx = threadIdx.x + q * PQ_T;
    const int r = idx / PQ_B, c = idx - r * PQ_B;
    double s = 0.0;
    if (r < bw) {
      if (trans) {
        for (int b = 0; b <= r; ++b) s = fma(sm.Ts[b][r], sm.W[b][c], s);  // (T^T)[r][b] = T[b][r]
      } else {
        for (int b = r; b < bw; ++b) s = fma(sm.Ts[r][b], sm.W[b][c], s);
      }
    }
    w2[q] = s;
  }
  __syncthreads();
  for (int q = 0; q < PQ_B * PQ_B / PQ_T; ++q) {
    const int idx = threadIdx.x + q * PQ_T;
    sm.W[idx / PQ_B][idx % PQ_B] = w2[q];
  }
  __syncthreads();
  // X -= V W2: thread per row i, all 32 columns
  for (int i = threadIdx.x; i < nr; i += PQ_T) {
    double v[PQ_B];
#pragma unroll
    for (int r = 0; r < PQ_B; ++r) v[r] = r < bw ? sm.Vs[r][i] : 0.0;
    for (int c = 0; c < PQ_B; ++c) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < PQ_B; ++r) s = fma(v[r], sm.W[r][c], s);
      X[c][i] -= s;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(PQ_T, 1) qr_precond_kernel(PqArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PqSmem& sm = *reinterpret_cast<PqSmem*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int t = static_cast<int>(cl.block_rank());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // 1. CTA 0: rows of G by decreasing norm (ties by index), bitonic sort
  if (t == 0) {
    for (int r = threadIdx.x; r < PQ_MAX; r += PQ_T) {
      double s = -1.0;
      if (r < a.mr) {
        s = 0.0;
        for (int c = 0; c < a.ng; ++c) {
          const double g = a.G[static_cast<long>(c) * a.ldg + r];
          s = fma(g, g, s);
        }
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

  // 2. load this CTA's columns of A = G^T Pi (real coordinates) and Q = I
  {
    const int* P0 = cl.map_shared_rank(sm.P, 0);
    for (int idx = threadIdx.x; idx < PQ_B * a.nr; idx += PQ_T) {
      const int c = idx / a.nr, i = idx - c * a.nr;
      const int col = t * PQ_B + c;
      sm.A[c][i] = col < a.mr ? a.G[static_cast<long>(coord(a, i)) * a.ldg + P0[col]] : 0.0;
      sm.Qb[c][i] = (t * PQ_B + c == i) ? 1.0 : 0.0;
    }
    if (threadIdx.x < PQ_B) {
      const int col = t * PQ_B + threadIdx.x;
      sm.Pown[threadIdx.x] = col < a.mr ? P0[col] : -1;
    }
  }
  cl.sync();
  const int npan = (a.k + PQ_B - 1) / PQ_B;

  // 3. panels
  for (int p = 0; p < npan; ++p) {
    const int j0 = p * PQ_B, bw = min(PQ_B, a.k - j0);
    if (t == p) {
      const int wcols = min(PQ_B, a.mr - j0);  // columns of this block (reflectors + trailing)
      for (int c = 0; c < bw; ++c) {
        const int j = j0 + c;
        if (warp == 0) {
          double xn = 0.0;
          for (int i = j + 1 + lane; i < a.nr; i += 32) xn = fma(sm.A[c][i], sm.A[c][i], xn);
          xn = warp_sum(xn);
          const double alpha = sm.A[c][j];
          double tau = 0.0;
          if (xn > 0.0) {
            const double nrm = sqrt(fma(alpha, alpha, xn));
            const double beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            const double sc = 1.0 / (alpha - beta);
            for (int i = j + 1 + lane; i < a.nr; i += 32) sm.A[c][i] *= sc;
            __syncwarp();
            if (lane == 0) sm.A[c][j] = beta;
          }
          if (lane == 0) sm.tau[c] = tau;
        }
        __syncthreads();
        const double tau = sm.tau[c];
        if (tau != 0.0)
          for (int c2 = c + 1 + warp; c2 < wcols; c2 += PQ_T / 32) {
            double s = 0.0;
            for (int i = j + 1 + lane; i < a.nr; i += 32) s = fma(sm.A[c][i], sm.A[c2][i], s);
            s = warp_sum(s) + sm.A[c2][j];
            const double f = tau * s;
            for (int i = j + 1 + lane; i < a.nr; i += 32) sm.A[c2][i] = fma(-f, sm.A[c][i], sm.A[c2][i]);
            __syncwarp();
            if (lane == 0) sm.A[c2][j] -= f;
          }
        __syncthreads();
      }
      // compact WY: T upper triangular, T[c][c] = tau_c,
      // T[0:c, c] = -tau_c T[0:c, 0:c] (V[:, 0:c]^T v_c); Y = V^T V into W
      for (int idx = threadIdx.x; idx < PQ_B * PQ_B; idx += PQ_T) {
        const int r = idx / PQ_B, c = idx - r * PQ_B;
        double s = 0.0;
        if (r < c && c < bw) {
          // v_r has unit at j0 + r, zeros above; v_c unit at j0 + c
          s = sm.A[r][j0 + c];
          for (int i = j0 + c + 1; i < a.nr; ++i) s = fma(sm.A[r][i], sm.A[c][i], s);
        }
        sm.W[r][c] = s;
        sm.T[r][c] = 0.0;
      }
      __syncthreads();
      for (int c = 0; c < bw; ++c) {
        if (threadIdx.x < c) {
          const int r = threadIdx.x;
          double s = 0.0;
          for (int b = r; b < c; ++b) s = fma(sm.T[r][b], sm.W[b][c], s);
          sm.T[r][c] = -sm.tau[c] * s;
        }
        if (threadIdx.x == c) sm.T[c][c] = sm.tau[c];
        __syncthreads();
      }
    }
    cl.sync();
    if (t > p && t * PQ_B < a.mr) {
      stage_panel(cl, sm, a, p, bw);
      apply_block_reflector(sm, sm.A, a.nr, bw, true);
    }
  }

  // 4. Q = H_1 ... H_k, this CTA's columns: X <- (I - V_p T_p V_p^T) X for p = last .. 0
  if (t * PQ_B < a.nr)
    for (int p = npan - 1; p >= 0; --p) {
      const int bw = min(PQ_B, a.k - p * PQ_B);
      stage_panel(cl, sm, a, p, bw);
      apply_block_reflector(sm, sm.Qb, a.nr, bw, false);
    }
  cl.sync();  // no CTA leaves while its shared memory may still be read

  // 5. outputs: G <- Pi R^T (row Pi(c) of G = column c of R), V0 <- Q at real coordinates
  for (int idx = threadIdx.x; idx < PQ_B * a.nr; idx += PQ_T) {
    const int c = idx / a.nr, i = idx - c * a.nr;
    const int col = t * PQ_B + c;
    if (col < a.mr) {
      const int row = sm.Pown[c];
      a.G[static_cast<long>(coord(a, i)) * a.ldg + row] = (i <= col && i < a.k) ? sm.A[c][i] : 0.0;
    }
    if (col < a.nr) a.V0[static_cast<long>(coord(a, col)) * a.ng + coord(a, i)] = sm.Qb[c][i];
  }
}

}  // namespace

bool qr_precond_applicable(int mr, int nr) { return mr <= PQ_MAX && nr <= PQ_MAX && nr >= 1 && mr >= 1; }

void qr_precond(Ctx& ctx, double* G, long ldg, int mr, int ng, int nr, int pad_mod, int pad_lim,
                double* V0) {
  if (!qr_precond_applicable(mr, nr)) fail(ACHI_E_INTERNAL, "qr_precond: shape beyond the cluster kernel");
  static bool attr = false;
  if (!attr) {
    ACHI_CUDA(cudaFuncSetAttribute(qr_precond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sizeof(PqSmem))));
    attr = true;
  }
  PqArgs a{G, ldg, mr, ng, nr, pad_mod, pad_lim, std::min(nr, mr), V0};
  const int ncta = (std::max(mr, nr) + PQ_B - 1) / PQ_B;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ncta);
  lc.blockDim = dim3(PQ_T);
  lc.dynamicSmemBytes = sizeof(PqSmem);
  lc.stream = ctx.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  ACHI_CUDA(cudaLaunchKernelEx(&lc, qr_precond_kernel, a));
  ACHI_LAUNCHED(ctx);
}

}  // namespace achi
