// FP64 tensor-core GEMM for sm_100a: TMA (cp.async.bulk.tensor) stages
// operand tiles into 128B-swizzled shared memory behind an mbarrier
// full/empty ring (thread 0 doubles as the TMA producer); all warps issue mma.sync.m16n8k4.f64 (SASS
// DMMA.8x8x4, the only FP64 MMA on Blackwell: tcgen05 has no kind::f64).
//
// This is the contraction engine behind every chi^3 step of the hot path:
// the two GEMMs of the effective-Hamiltonian matvec (dmrg.cpp:58-71), the
// two GEMMs of each environment update (dmrg.cpp:26-49) and the theta merge
// (dmrg.cpp:94).  The reference does all of them through Tensor::contract
// (tensor.hpp:152-198: permute + Eigen GEMM); here every contraction is laid
// out so that no permutation copy is needed, only operand-major flags.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace achi {

// Operand storage: kK = the stored rows run over the M (or N) index with K
// contiguous; kMN = the stored rows run over K with M (or N) contiguous.
enum class Major : int { kK = 0, kMN = 1 };

struct Operand {
  const double* ptr;
  long ld;      // elements between consecutive stored rows (must be even)
  Major major;
};

namespace gemm_detail {

constexpr int BK = 16;           // 16 doubles = one 128-byte swizzle row
constexpr int ROW_BYTES = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// byte offset of element (r, k) in a K-major 128B-swizzled tile (rows of 16 k)
__device__ __forceinline__ uint32_t off_kmajor(int r, int k) {
  return static_cast<uint32_t>(r * ROW_BYTES + ((((k >> 1) ^ (r & 7)) << 4) | ((k & 1) << 3)));
}
// byte offset of element (k, c) in an MN-major tile built from 16x16 boxes
__device__ __forceinline__ uint32_t off_mnmajor(int k, int c) {
  return static_cast<uint32_t>((c >> 4) * (16 * ROW_BYTES) + k * ROW_BYTES +
                               (((((c & 15) >> 1) ^ (k & 7)) << 4) | ((c & 1) << 3)));
}

template <Major MJ>
__device__ __forceinline__ double lds_op(const unsigned char* tile, int mn, int k) {
  uint32_t off = MJ == Major::kK ? off_kmajor(mn, k) : off_mnmajor(k, mn);
  return *reinterpret_cast<const double*>(tile + off);
}

__device__ __forceinline__ void mma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// CTA tile BM x BN, warp tile WTM x WTN, STAGES-deep TMA ring.  C (or the split-K slab z) = A[:, kslice] * B[kslice, :].
template <int BM, int BN, int WTM, int WTN, int STAGES, Major AM, Major BMJ>
struct Cfg {
  static constexpr int WM = BM / WTM, WN = BN / WTN;
  static constexpr int CONSUMERS = WM * WN;
  static constexpr int THREADS = CONSUMERS * 32;
  static constexpr int MT = WTM / 16, NT = WTN / 8;
  static constexpr int A_BYTES = BM * ROW_BYTES, B_BYTES = BN * ROW_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8 + 64;
};

template <int BM, int BN, int WTM, int WTN, int STAGES, Major AM, Major BMJ>
__global__ void __launch_bounds__(Cfg<BM, BN, WTM, WTN, STAGES, AM, BMJ>::THREADS, 1)
    dmma_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, double* __restrict__ C, long ldc,
                     long split_stride, int M, int N, int K, int kt_per_split) {
  pdl_wait();  // launched with launch_pdl / the PDL attribute (common.cuh)
  using G = Cfg<BM, BN, WTM, WTN, STAGES, AM, BMJ>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kt_total = (K + BK - 1) / BK;
  const int kt_begin = blockIdx.z * kt_per_split;
  const int kt_end = min(kt_total, kt_begin + kt_per_split);
  const int nk = max(0, kt_end - kt_begin);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // TMA issue for k-tile i into stage i % STAGES (thread 0 of warp 0 doubles
  // as the producer; the stage's previous use must be released first).
  auto issue = [&](int i) {
    const int s = i % STAGES;
    if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
    mbar_expect_tx(&full[s], G::STAGE_BYTES);
    unsigned char* sa = smem + s * G::STAGE_BYTES;
    unsigned char* sb = sa + G::A_BYTES;
    const int k0 = (kt_begin + i) * BK;
    if constexpr (AM == Major::kK) {
      tma_load_2d(sa, &mapA, &full[s], k0, m0);
    } else {
#pragma unroll
      for (int j = 0; j < BM / 16; ++j)
        tma_load_2d(sa + j * 16 * ROW_BYTES, &mapA, &full[s], m0 + 16 * j, k0);
    }
    if constexpr (BMJ == Major::kK) {
      tma_load_2d(sb, &mapB, &full[s], k0, n0);
    } else {
#pragma unroll
      for (int j = 0; j < BN / 16; ++j)
        tma_load_2d(sb + j * 16 * ROW_BYTES, &mapB, &full[s], n0 + 16 * j, k0);
    }
  };
  if (threadIdx.x == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    for (int i = 0; i < STAGES - 1 && i < nk; ++i) issue(i);
  }

  // ---- consumer warps ----
  const int wm0 = (warp / G::WN) * WTM, wn0 = (warp % G::WN) * WTN;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[G::MT][G::NT][4];
#pragma unroll
  for (int i = 0; i < G::MT; ++i)
#pragma unroll
    for (int j = 0; j < G::NT; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.0;

  for (int i = 0; i < nk; ++i) {
    if (threadIdx.x == 0 && i + STAGES - 1 < nk) issue(i + STAGES - 1);
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const unsigned char* sa = smem + s * G::STAGE_BYTES;
    const unsigned char* sb = sa + G::A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + tig;
      double a0[G::MT], a1[G::MT], b[G::NT];
#pragma unroll
      for (int mt = 0; mt < G::MT; ++mt) {
        a0[mt] = lds_op<AM>(sa, wm0 + mt * 16 + gid, k);
        a1[mt] = lds_op<AM>(sa, wm0 + mt * 16 + gid + 8, k);
      }
#pragma unroll
      for (int nt = 0; nt < G::NT; ++nt) b[nt] = lds_op<BMJ>(sb, wn0 + nt * 8 + gid, k);
#pragma unroll
      for (int mt = 0; mt < G::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < G::NT; ++nt) mma_16x8x4(acc[mt][nt], a0[mt], a1[mt], b[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- epilogue: registers -> global (row-major, split slab z) ----
  double* Cz = C + static_cast<long>(blockIdx.z) * split_stride;
  const bool vec_ok = (ldc & 1) == 0;
#pragma unroll
  for (int mt = 0; mt < G::MT; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = m0 + wm0 + mt * 16 + gid + 8 * h;
      if (row >= M) continue;
      double* crow = Cz + static_cast<long>(row) * ldc;
#pragma unroll
      for (int nt = 0; nt < G::NT; ++nt) {
        const int col = n0 + wn0 + nt * 8 + 2 * tig;
        const double v0 = acc[mt][nt][2 * h], v1 = acc[mt][nt][2 * h + 1];
        if (vec_ok && col + 1 < N) {
          *reinterpret_cast<double2*>(crow + col) = make_double2(v0, v1);
        } else {
          if (col < N) crow[col] = v0;
          if (col + 1 < N) crow[col + 1] = v1;
        }
      }
    }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ ws, long split_stride, int splits,
                                     double* __restrict__ C, long ldc, long ldw, int M, int N);

}  // namespace gemm_detail

// C[M x N] (row-major, ldc) = A * B; see Operand for the storage conventions.
// Deterministic: split-K partials are summed in fixed order by a second kernel.
void gemm(Ctx& ctx, int M, int N, int K, const Operand& A, const Operand& B, double* C, long ldc);

}  // namespace achi
