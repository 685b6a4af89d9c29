// Device phases of the fused small-chi H_eff matvec (heff_small.cu).  See
// heff_small.cu for the contraction; each phase loops its work items over the
// CTAs [blk, blk + nblk) of a cooperative grid, and the caller puts a grid
// barrier between phases.
#pragma once

#include "contract.cuh"

namespace achi {
namespace hs {

constexpr int HS_THREADS = 256;
constexpr int HS_TM = 32;        // tile rows
constexpr int HS_TN = 64;        // tile cols
constexpr int HS_KMAX = 128;     // contraction length bound of the small instantiation
constexpr int HS_KMAX_WIDE = 256; // ... and of the wide one (chi 129..256)
template <int K>
__host__ __device__ constexpr int hs_ld() { return K + 4; }
constexpr int HS_MAXW = 64;      // max MPO mixing inputs/outputs (D d^2)
constexpr int HS_MAXNNZ = 512;

struct HsArgs {
  const double* L;
  const double* R;
  const double* theta;
  double* out;
  double* X;     // Y, the mixed first contraction: [chl*d*d][D3][chr]
  double* part;  // [D3][chl*d*d][chr]
  DevMix mix;
  int chl, chr, d, D1, D3;
};

__device__ __forceinline__ void mma16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// C (32 x 64) = As (32 x K, row-major, ld HS_LD) * Bs^T (Bs: 64 x K, ld HS_LD);
// warp w: rows 16 (w / 4), cols 16 (w % 4) = two n8 tiles.  Returns the
// warp's accumulators for the store.
template <int KM>
__device__ __forceinline__ void tile_mma(const double* As, const double* Bs, int K, double (&acc)[2][4]) {
  constexpr int HS_LD = hs_ld<KM>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int mr = (warp >> 2) * 16, nc = (warp & 3) * 16;
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[q][i] = 0.0;
  // every lane runs the same number of mma.sync; K tails are zero-padded by the loaders
  const int K4 = (K + 3) & ~3;
  for (int k = tig; k < K4; k += 4) {
    const double a0 = As[(mr + gid) * HS_LD + k], a1 = As[(mr + gid + 8) * HS_LD + k];
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16x8x4(acc[q], a0, a1, Bs[(nc + q * 8 + gid) * HS_LD + k]);
  }
}

__device__ __forceinline__ void tile_store(const double (&acc)[2][4], double* C, long ldc, int m0,
                                           int n0, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int mr = m0 + (warp >> 2) * 16 + gid, nc0 = n0 + (warp & 3) * 16;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = nc0 + q * 8 + 2 * tig;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = mr + 8 * h;
      if (r < M) {
        if (c < N) C[static_cast<long>(r) * ldc + c] = acc[q][2 * h];
        if (c + 1 < N) C[static_cast<long>(r) * ldc + c + 1] = acc[q][2 * h + 1];
      }
    }
  }
}


// Mixing coefficients of the bond (CSR) staged once per CTA, plus a dense
// copy (HS_MIXD x HS_MIXD, zero-filled) for the register-blocked mixing of
// phase A when nout, nin <= HS_MIXD (every XXZ bulk bond: D = 5, d = 2 -> 20 x 20).
constexpr int HS_MIXD = 20;
struct MixSmem {
  double wv[HS_MAXNNZ];
  int wc[HS_MAXNNZ], wr[HS_MAXW + 1];
  double wd[HS_MIXD * HS_MIXD];  // wd[j * HS_MIXD + i]
};
__device__ __forceinline__ void load_mix(const DevMix& m, MixSmem& w) {
  for (int i = threadIdx.x; i < m.nnz; i += blockDim.x) {
    w.wv[i] = m.val[i];
    w.wc[i] = m.col[i];
  }
  for (int i = threadIdx.x; i <= m.nout; i += blockDim.x) w.wr[i] = m.rowptr[i];
  for (int i = threadIdx.x; i < HS_MIXD * HS_MIXD; i += blockDim.x) w.wd[i] = 0.0;
  __syncthreads();
  if (m.nout <= HS_MIXD && m.nin <= HS_MIXD)
    for (int j = threadIdx.x; j < m.nout; j += blockDim.x)
      for (int p = m.rowptr[j]; p < m.rowptr[j + 1]; ++p) w.wd[j * HS_MIXD + m.col[p]] = m.val[p];
}

// Tile shape of phase A: rows = a block of `blb` left indices bl with all D1
// MPO rows a (blb * D1 <= 32), columns = a block of 16 right indices jr for
// all d^2 physical pairs s (d^2 * 16 = 64), so the MPO mixing of the tile's
// outputs only needs the tile itself.
__device__ __forceinline__ int phase_a_blb(const HsArgs& a) { return HS_TM / a.D1; }
constexpr int HS_JRB = 16;  // jr per phase-A tile (d = 2)
constexpr int HS_SSTR = 20; // column stride of the s blocks in the staged tile (4 x 20 <= HS_LD)

// A: Y[((bl,s'),e), jr] = sum_{(a,s)} W12[(s',e),(a,s)] sum_jl L[(bl,a),jl] theta[jl,(s,jr)]
// The GEMM tile is staged in shared memory and mixed there (no X buffer).
template <int KM>
// Lc (optional, persistent callers): a shared-memory cache of the L tile of the
// CTA's first item, filled when lfill (the first matvec of an eigensolve) and
// read instead of global memory afterwards (L is constant within an eigensolve)
__device__ __forceinline__ void phase_a(const HsArgs& a, const MixSmem& w, const double* theta,
                                        double* As, double* Bs, int blk, int nblk,
                                        unsigned long long* prof = nullptr, double* Lc = nullptr,
                                        bool lfill = false, double tscale = 1.0) {
  // prof (optional, thread 0 of the caller's CTA): cycles in [0] loads, [1] MMA, [2] mixing
  const bool pf = prof && threadIdx.x == 0;
  unsigned long long pt = pf ? clock64() : 0;
  auto pmark = [&](int i) {
    if (pf) {
      const unsigned long long n = clock64();
      prof[i] += n - pt;
      pt = n;
    }
  };
  constexpr int HS_LD = hs_ld<KM>(), RG = HS_THREADS / KM;  // row groups of the K-major loads
  const int t = threadIdx.x;
  const int chl = a.chl, chr = a.chr, dd = a.d * a.d, D1 = a.D1, D3 = a.D3;
  const int N1 = dd * chr, blb = phase_a_blb(a), rows = blb * D1;
  const int tm = (chl + blb - 1) / blb, tn = (chr + HS_JRB - 1) / HS_JRB;
  const int K4 = (chl + 3) & ~3;  // zero-padded K tail
  for (int item = blk; item < tm * tn; item += nblk) {
    const int bl0 = (item / tn) * blb, jr0 = (item % tn) * HS_JRB;
    __syncthreads();
    const bool cached = Lc && item == blk;
    double* At = cached ? Lc : As;  // A operand of this item's GEMM
    if (!cached || lfill) {
      // At[m][k] = L[bl0*D1 + m][k] (m < blb*D1): thread -> (k = t % KM, rows t / KM + RG u);
      // every load of a thread is issued before its stores
      const int k = t % KM, r0 = t / KM;
      double v[HS_TM / RG];
#pragma unroll
      for (int u = 0; u < HS_TM / RG; ++u) {
        const int m = r0 + RG * u;
        v[u] = (m < rows && bl0 * D1 + m < chl * D1 && k < chl)
                   ? a.L[static_cast<long>(bl0 * D1 + m) * chl + k]
                   : 0.0;
      }
      if (k < K4)
#pragma unroll
        for (int u = 0; u < HS_TM / RG; ++u) At[(r0 + RG * u) * HS_LD + k] = v[u];
    }
    {
      // Bs[n][k] = theta[k][s*chr + jr0 + q], n = s*16 + q: thread -> (n = t % 64, k = t / 64 + 4u),
      // in chunks of 32 loads
      const int n = t & (HS_TN - 1), kq = t >> 6;
      const int s = n / HS_JRB, jr = jr0 + (n % HS_JRB);
      const bool ok = s < dd && jr < chr;
#pragma unroll
      for (int h = 0; h < KM / 128; ++h) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int k = kq + 4 * (32 * h + u);
          v[u] = (ok && k < chl) ? theta[static_cast<long>(k) * N1 + s * chr + jr] * tscale : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int k = kq + 4 * (32 * h + u);
          if (k < K4) Bs[n * HS_LD + k] = v[u];
        }
      }
    }
    __syncthreads();
    pmark(0);
    double acc[2][4];
    tile_mma<KM>(At, Bs, chl, acc);
    __syncthreads();
    pmark(1);
    // stage the 32 x 64 tile (rows (bl, a), cols (s, q)) into As, then mix; the s blocks
    // sit HS_SSTR apart so the mixing's fragment loads (4 s values x 8 q per warp
    // request) hit every bank exactly twice
    {
      const int warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
      const int mr = (warp >> 2) * 16 + gid, nc0 = (warp & 3) * 16;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = nc0 + q * 8 + 2 * tig, cs = (c / HS_JRB) * HS_SSTR + c % HS_JRB;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          As[(mr + 8 * h) * HS_LD + cs] = acc[q][2 * h];
          As[(mr + 8 * h) * HS_LD + cs + 1] = acc[q][2 * h + 1];
        }
      }
    }
    __syncthreads();
    if (dd * D3 <= HS_MIXD && D1 * dd <= HS_MIXD) {
      // MPO mixing on the tensor cores: Y (njo x pairs) = W12 (njo x nin) . X (nin x pairs),
      // X[(a, s)][(bll, q)] = As[(bll D1 + a) LD + s 16 + q] (the staged GEMM tile), one
      // m16n8k4 DMMA chain of K = 20 per 16 x 8 output tile; warp w keeps the W12 rows of
      // m-tile w & 1 in registers for all its tiles
      const int nin = D1 * dd, njo = dd * D3, pairs = blb * HS_JRB;
      const int warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
      const int mt = warp & 1, tiles = 2 * (pairs / 8);
      constexpr int KS = (HS_MIXD + 3) / 4;
      double wa0[KS], wa1[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int i = ks * 4 + tig, ja = mt * 16 + gid;
        wa0[ks] = (ja < njo && i < nin) ? w.wd[ja * HS_MIXD + i] : 0.0;
        wa1[ks] = (ja + 8 < njo && i < nin) ? w.wd[(ja + 8) * HS_MIXD + i] : 0.0;
      }
      for (int tile = warp; tile < tiles; tile += HS_THREADS / 32) {
        const int nt = tile >> 1;
        const int nb = nt * 8 + gid, bllb = nb / HS_JRB, qb = nb % HS_JRB;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int i = ks * 4 + tig;
          const int aa = i / dd, ss = i - aa * dd;
          const double bv = i < nin ? As[(bllb * D1 + aa) * HS_LD + ss * HS_SSTR + qb] : 0.0;
          mma16x8x4(acc, wa0[ks], wa1[ks], bv);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = mt * 16 + gid + 8 * h;
          if (j >= njo) continue;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int n2 = nt * 8 + 2 * tig + cc, bll = n2 / HS_JRB, q = n2 % HS_JRB;
            const int bl = bl0 + bll, jr = jr0 + q;
            if (bl < chl && jr < chr) a.X[(static_cast<long>(bl) * njo + j) * chr + jr] = acc[2 * h + cc];
          }
        }
      }
      pmark(2);
      continue;
    }
    const int nout = blb * dd * D3 * HS_JRB;  // outputs (bl, s', e, q)
    for (int o = t; o < nout; o += HS_THREADS) {
      const int q = o % HS_JRB, rest = o / HS_JRB;
      const int e = rest % D3, r2 = rest / D3;
      const int sp = r2 % dd, bll = r2 / dd;
      const int bl = bl0 + bll, jr = jr0 + q;
      if (bl >= chl || jr >= chr) continue;
      const int j = sp * D3 + e;
      double v = 0.0;
      for (int p = w.wr[j]; p < w.wr[j + 1]; ++p) {
        const int in = w.wc[p], aa = in / dd, s = in - aa * dd;  // input (a, s)
        v += w.wv[p] * As[(bll * D1 + aa) * HS_LD + s * HS_SSTR + q];
      }
      a.X[((static_cast<long>(bl) * dd + sp) * D3 + e) * chr + jr] = v;  // Y[(bl s') (e jr)]
    }
    pmark(2);
  }
}

// B: P_e[(bl,s'), br] = sum_jr Y[(bl,s'),(e,jr)] R[br,(e,jr)]  (one item per e: split-K)
// Rc (optional): shared-memory cache of the R tile of the CTA's first item, as Lc
template <int KM>
__device__ __forceinline__ void phase_b(const HsArgs& a, double* As, double* Bs, int blk, int nblk,
                                        double* Rc = nullptr, bool rfill = false) {
  constexpr int HS_LD = hs_ld<KM>(), RG = HS_THREADS / KM;
  const int t = threadIdx.x;
  const int chl = a.chl, chr = a.chr, dd = a.d * a.d, D3 = a.D3;
  const int M2 = chl * dd, N2 = chr;
  const int tm = (M2 + HS_TM - 1) / HS_TM, tn = (N2 + HS_TN - 1) / HS_TN;
  const int items = tm * tn * D3;
  const int K4 = (chr + 3) & ~3;  // zero-padded K tail
  for (int item = blk; item < items; item += nblk) {
    const int e = item / (tm * tn), rest = item - e * tm * tn;
    const int m0 = (rest / tn) * HS_TM, n0 = (rest % tn) * HS_TN;
    __syncthreads();
    {
      // As[m][jr] = Y[(m0+m), e, jr]: thread -> (jr = t % KM, rows t / KM + RG u)
      const int jr = t % KM, r0 = t / KM;
      double v[HS_TM / RG];
#pragma unroll
      for (int u = 0; u < HS_TM / RG; ++u) {
        const int row = m0 + r0 + RG * u;
        v[u] = (row < M2 && jr < chr) ? a.X[(static_cast<long>(row) * D3 + e) * chr + jr] : 0.0;
      }
      if (jr < K4)
#pragma unroll
        for (int u = 0; u < HS_TM / RG; ++u) As[(r0 + RG * u) * HS_LD + jr] = v[u];
    }
    const bool cached = Rc && item == blk;
    double* Bt = cached ? Rc : Bs;  // B operand of this item's GEMM
    if (!cached || rfill) {
      // Bt[n][jr] = R[n0+n][e][jr]: thread -> (jr = t % KM, n = t / KM + RG u), chunks of 32
      const int jr = t % KM, q0 = t / KM;
#pragma unroll
      for (int h = 0; h < HS_TN / RG / 32; ++h) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int n = q0 + RG * (32 * h + u);
          v[u] = (n0 + n < N2 && jr < chr) ? a.R[(static_cast<long>(n0 + n) * D3 + e) * chr + jr] : 0.0;
        }
        if (jr < K4)
#pragma unroll
          for (int u = 0; u < 32; ++u) Bt[(q0 + RG * (32 * h + u)) * HS_LD + jr] = v[u];
      }
    }
    __syncthreads();
    double acc[2][4];
    tile_mma<KM>(As, Bt, chr, acc);
    tile_store(acc, a.part + static_cast<long>(e) * M2 * N2, N2, m0, n0, M2, N2);
  }
}

// C: out = sum_e P_e (fixed order)
__device__ __forceinline__ void phase_c(const HsArgs& a, double* out, int blk, int nblk) {
  const int t = threadIdx.x;
  const int M2 = a.chl * a.d * a.d, N2 = a.chr;
  const long tot = static_cast<long>(M2) * N2;
  for (long i = blk * static_cast<long>(HS_THREADS) + t; i < tot;
       i += static_cast<long>(nblk) * HS_THREADS) {
    double v = 0.0;
    for (int e = 0; e < a.D3; ++e) v += a.part[e * tot + i];
    out[i] = v;
  }
}

template <int KM>
inline size_t smem_bytes() { return sizeof(double) * (HS_TM + HS_TN) * hs_ld<KM>(); }

}  // namespace hs

// Arguments of the fused small-chi matvec (KM = 128) for theta -> out, with its
// workspaces reserved; false when the op takes another path (heff_small.cu).
// items = max(phase-A, phase-B work items).
bool heff_small_fusable(Ctx& ctx, const HeffOps& op, const double* theta, double* out, hs::HsArgs* args,
                        long* items);

}  // namespace achi
