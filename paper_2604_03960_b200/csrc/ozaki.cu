// Emulated-FP64 GEMM on the int8 tensor cores (Ozaki scheme; tcgen05.mma kind::i8).
//
// The north_star's "optionally emulated-precision" contraction for K1-K4
// (SURVEY.md §8 f5).  Blackwell has no FP64 tcgen05 kind; its int8 tensor
// cores (UTCIMMA) are exact on integers, so an FP64 product can be rebuilt
// from int8 products (Ozaki, Ogita, Oishi, Rump 2012):
//
//   every row i of A gets a power-of-two scale 2^ea_i >= max_k |a_ik|, every
//   column j of B one 2^eb_j; the scaled entries (in (-1, 1)) are cut into s
//   signed 7-bit digits:  a_ik = 2^ea_i sum_p A_p[i,k] 2^-7p  (+ a remainder
//   below 2^(ea_i - 7s)), each digit an int8 in [-127, 127], exact (the
//   digits come from trunc(128 r), r <- 128 r - trunc(128 r), all exact in
//   FP64);
//   C_ij = 2^(ea_i + eb_j) sum_{p+q <= s+1} 2^-7(p+q) (A_p B_q)_ij, every
//   A_p B_q an exact int32 GEMM (|sum| <= K 127^2 (s) < 2^31 for K <= 2^14).
//
// The kernel: one CTA per 128 x 64 output tile; warp 0 is the TMA producer
// (int8 digit tiles, 128-byte rows, 128B swizzle), warp 1 issues
// tcgen05.mma.cta_group::1.kind::i8 (M=128, N=64, K=32 per instruction) into
// a TMEM int32 accumulator, one accumulation group per digit weight w = p+q
// (all pairs of that weight summed in TMEM), two TMEM buffers so the MMAs of
// weight w-1 run while four epilogue warps read weight w with tcgen05.ld and
// add 2^-7w times it to their FP64 registers (one output row per thread).
// Weights are summed from the smallest up.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "ozaki.cuh"

namespace achi {

namespace {

constexpr int TM = 128, TN = 64;   // output tile
constexpr int TKB = 128;           // K bytes (int8 entries) per stage: one 128B swizzle row
constexpr int UMMA_K = 32;         // kind::i8: K per instruction
constexpr int STAGES = 6;
constexpr int A_BYTES = TM * TKB, B_BYTES = TN * TKB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int OZ_THREADS = 192;    // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int OZ_SMEM = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// K-major operand tile with 128-byte rows and 128B swizzle: 8-row swizzle
// atoms 1024 bytes apart (SBO), LBO 1 (unused for swizzled K-major),
// descriptor version 1 (tcgen05)
__device__ __forceinline__ uint64_t smem_desc(const void* tile, int k_bytes) {
  const uint32_t addr = smem_u32(tile) + static_cast<uint32_t>(k_bytes);
  return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024u >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// kind::i8: D s32 (bits 4-5 = 2), A and B signed int8 (bits 7-9, 10-12 = 1),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(TN >> 3) << 17) |
                           (static_cast<uint32_t>(TM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
                   static_cast<uint64_t>(smem_u32(bar)))
               : "memory");
}

// digit weights w = p + q run from s+1 down to 2; pairs (p, q = w - p), 1 <= p, q <= s
__device__ __forceinline__ int w_of(int g, int s) { return s + 1 - g; }

__global__ void __launch_bounds__(OZ_THREADS, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C,
                      long ldc, int M, int N, int K, int s) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int nk = (K + TKB - 1) / TKB;
  const int groups = s;  // weights s+1 .. 2
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: two 64-column int32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int g = 0; g < groups; ++g) {
        const int w = w_of(g, s);
        for (int p = max(1, w - s); p <= min(s, w - 1); ++p) {
          const int q = w - p;
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1);
            unsigned char* st = smem + stage * STAGE_BYTES;
            mbar_expect_tx(&full[stage], STAGE_BYTES);
            tma_load_3d(st, &mapA, &full[stage], kc * TKB, m0, p - 1);
            tma_load_3d(st + A_BYTES, &mapB, &full[stage], kc * TKB, n0, q - 1);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      for (int g = 0; g < groups; ++g) {
        const int w = w_of(g, s), ab = g & 1;
        mbar_wait(&tempty[ab], ((g >> 1) & 1) ^ 1);  // the epilogue has drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + static_cast<uint32_t>(ab * TN);
        uint32_t acc = 0;
        for (int p = max(1, w - s); p <= min(s, w - 1); ++p) {
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&full[stage], phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned char* st = smem + stage * STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < TKB / UMMA_K; ++kk) {
              mma_i8(d, smem_desc(st, kk * UMMA_K), smem_desc(st + A_BYTES, kk * UMMA_K), acc);
              acc = 1;
            }
            umma_commit(&empty[stage]);  // frees the stage once these MMAs have read it
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        umma_commit(&tfull[ab]);  // weight w complete in TMEM buffer ab
      }
    }
  } else {
    // epilogue: warp e (2..5) owns TMEM lanes 32 (e % 4) ... (the row of the tile)
    const int lg = warp & 3;
    const int row = m0 + 32 * lg + lane;
    double c[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) c[j] = 0.0;
    for (int g = 0; g < groups; ++g) {
      const int w = w_of(g, s), ab = g & 1;
      mbar_wait(&tfull[ab], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * lg) << 16) + static_cast<uint32_t>(ab * TN);
      uint32_t v[TN];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
          "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63},"
          " [%64];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]),
            "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]),
            "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
            "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
            "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      const double f = ldexp(1.0, -7 * w);
#pragma unroll
      for (int j = 0; j < TN; ++j) c[j] = fma(static_cast<double>(static_cast<int32_t>(v[j])), f, c[j]);
    }
    if (row < M) {
      const int er = ea[row];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int col = n0 + j;
        if (col < N) C[static_cast<long>(row) * ldc + col] = ldexp(c[j], er + eb[col]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

// ---- staged variant: every digit tile of a K chunk is loaded once ----
// For each 64-byte K chunk all s digit tiles of A (128 rows) and of B (64 rows)
// are staged (SWIZZLE_64B), then every digit pair with p + q <= s + 1 is issued
// into the TMEM accumulator of its weight (s accumulators x 64 columns <= 512):
// each digit tile is read from L2 once per chunk instead of once per pair (the
// pair loop of ozaki_gemm_kernel re-streams it ~s/2 times).  Two stages.
constexpr int SKB = 64;  // K bytes per stage row (64B swizzle)
constexpr int S_STAGES = 2;
__host__ __device__ constexpr int staged_stage_bytes(int s) { return s * (TM + TN) * SKB; }
__host__ __device__ constexpr int staged_smem(int s) { return S_STAGES * staged_stage_bytes(s) + 1024 + 256; }

__device__ __forceinline__ uint64_t smem_desc64(const void* tile, int k_bytes) {
  const uint32_t addr = smem_u32(tile) + static_cast<uint32_t>(k_bytes);
  return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (static_cast<uint64_t>(512u >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}

__global__ void __launch_bounds__(OZ_THREADS, 1)
    ozaki_staged_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                        const int* __restrict__ ea, const int* __restrict__ eb, double* __restrict__ C,
                        long ldc, int M, int N, int K, int s) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int SB = staged_stage_bytes(s);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_STAGES * SB);
  uint64_t* empty = full + S_STAGES;
  uint64_t* tfull = empty + S_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int nk = (K + SKB - 1) / SKB;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: one 64-column int32 accumulator per digit weight
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer: all digits of A and B for chunk kc
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* st = smem + stage * SB;
        mbar_expect_tx(&full[stage], SB);
        for (int p = 0; p < s; ++p) {
          tma_load_3d(st + p * TM * SKB, &mapA, &full[stage], kc * SKB, m0, p);
          tma_load_3d(st + s * TM * SKB + p * TN * SKB, &mapB, &full[stage], kc * SKB, n0, p);
        }
        if (++stage == S_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: pairs (p, q), p + q <= s + 1, into accumulator w - 2
      int stage = 0;
      uint32_t phase = 0;
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&full[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned char* st = smem + stage * SB;
        for (int w = 2; w <= s + 1; ++w) {
          const uint32_t d = tmem + static_cast<uint32_t>((w - 2) * TN);
          for (int p = max(1, w - s); p <= min(s, w - 1); ++p) {
            const int q = w - p;
            const unsigned char* ta = st + (p - 1) * TM * SKB;
            const unsigned char* tb = st + s * TM * SKB + (q - 1) * TN * SKB;
#pragma unroll
            for (int kk = 0; kk < SKB / UMMA_K; ++kk) {
              const bool first = kc == 0 && p == max(1, w - s) && kk == 0;
              mma_i8(d, smem_desc64(ta, kk * UMMA_K), smem_desc64(tb, kk * UMMA_K), first ? 0u : 1u);
            }
          }
        }
        umma_commit(&empty[stage]);
        if (++stage == S_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(tfull);
    }
  } else {
    const int lg = warp & 3;
    const int row = m0 + 32 * lg + lane;
    double c[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) c[j] = 0.0;
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int w = s + 1; w >= 2; --w) {  // smallest weight first
      const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * lg) << 16) + static_cast<uint32_t>((w - 2) * TN);
      uint32_t v[TN];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
          "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63},"
          " [%64];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]),
            "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]),
            "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
            "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
            "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const double f = ldexp(1.0, -7 * w);
#pragma unroll
      for (int j = 0; j < TN; ++j) c[j] = fma(static_cast<double>(static_cast<int32_t>(v[j])), f, c[j]);
    }
    if (row < M) {
      const int er = ea[row];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int col = n0 + j;
        if (col < N) C[static_cast<long>(row) * ldc + col] = ldexp(c[j], er + eb[col]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

// Digits of the rows of X (R x K): row r = X[r][k] (ld, !trans) or X[k][r] (trans).
// ex[r]: 2^ex[r] > max_k |x|; D[p][r][k] (int8, row stride Kp) for p < s.
__global__ void rowexp_kernel(const double* __restrict__ X, long ld, int R, int K, int trans,
                              int* __restrict__ ex) {
  if (!trans) {  // one warp per row
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= R) return;
    double m = 0.0;
    for (int k = lane; k < K; k += 32) m = fmax(m, fabs(X[static_cast<long>(r) * ld + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) ex[r] = m > 0 ? ilogb(m) + 1 : 0;
  } else {  // one thread per column of X (coalesced over r)
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    double m = 0.0;
    for (int k = 0; k < K; ++k) m = fmax(m, fabs(X[static_cast<long>(k) * ld + r]));
    ex[r] = m > 0 ? ilogb(m) + 1 : 0;
  }
}

// 32 x 32 (r, k) tiles through shared memory: coalesced reads in either
// layout, digit rows written k-contiguous
__global__ void digits_kernel(const double* __restrict__ X, long ld, int R, int K, int Kp, int trans, int s,
                              const int* __restrict__ ex, int8_t* __restrict__ D) {
  __shared__ double t[32][33];
  const int r0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    if (!trans) {
      const int r = r0 + i, k = k0 + tx;
      t[i][tx] = (r < R && k < K) ? X[static_cast<long>(r) * ld + k] : 0.0;
    } else {
      const int k = k0 + i, r = r0 + tx;
      t[tx][i] = (r < R && k < K) ? X[static_cast<long>(k) * ld + r] : 0.0;
    }
  }
  __syncthreads();
  const long plane = static_cast<long>(R) * Kp;
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, k = k0 + tx;
    if (r >= R || k >= Kp) continue;
    double v = ldexp(t[i][tx], -ex[r]);  // |v| < 1
    for (int p = 0; p < s; ++p) {
      const double dd = v * 128.0;
      const double tr = trunc(dd);
      D[p * plane + static_cast<long>(r) * Kp + k] = static_cast<int8_t>(tr);
      v = dd - tr;
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      fail(ACHI_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// int8 digit planes [s][rows][Kp] as a 3-D tensor (K bytes, rows, plane), box TKB x box_rows x 1
CUtensorMap digit_map(const int8_t* base, int rows, int Kp, int s, int box_rows, int box_k = TKB,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(s)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp) * rows};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_k), static_cast<cuuint32_t>(box_rows), 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ACHI_E_CUDA, "cuTensorMapEncodeTiled (digits) failed: " + std::to_string(r));
  return m;
}

}  // namespace

void dgemm_ozaki(Ctx& ctx, int M, int N, int K, const double* A, long lda, bool a_trans,
                 const double* B, long ldb, bool b_kmajor, double* C, long ldc, int slices) {
  if (slices < 2 || slices > OZ_MAX_SLICES) fail(ACHI_E_INVALID_CONFIG, "ozaki: slices must be in [2, 9]");
  if (K > (1 << 14)) fail(ACHI_E_SIZE_GUARD, "ozaki: K too long for exact int32 digit products");
  const int Kp = ((K + 15) / 16) * 16;  // 16-byte digit rows for TMA
  const size_t planeA = static_cast<size_t>(M) * Kp, planeB = static_cast<size_t>(N) * Kp;
  int8_t* DA = reinterpret_cast<int8_t*>(ctx.oz_digits.reserve((slices * (planeA + planeB) + 7) / 8));
  int8_t* DB = DA + slices * planeA;
  int* ea = ctx.oz_ex.reserve(static_cast<size_t>(M) + N);
  int* eb = ea + M;
  // A's rows are its M rows (A stored M x K, or K x M when a_trans); B's rows are its
  // N columns (B stored K x N row-major, or N x K when b_kmajor)
  rowexp_kernel<<<a_trans ? cdiv(M, 256) : cdiv(M, 8), 256, 0, ctx.stream>>>(A, lda, M, K, a_trans ? 1 : 0, ea);
  ACHI_LAUNCHED(ctx);
  rowexp_kernel<<<b_kmajor ? cdiv(N, 8) : cdiv(N, 256), 256, 0, ctx.stream>>>(B, ldb, N, K, b_kmajor ? 0 : 1, eb);
  ACHI_LAUNCHED(ctx);
  digits_kernel<<<dim3(cdiv(Kp, 32), cdiv(M, 32)), dim3(32, 8), 0, ctx.stream>>>(A, lda, M, K, Kp,
                                                                                   a_trans ? 1 : 0, slices, ea, DA);
  ACHI_LAUNCHED(ctx);
  digits_kernel<<<dim3(cdiv(Kp, 32), cdiv(N, 32)), dim3(32, 8), 0, ctx.stream>>>(B, ldb, N, K, Kp,
                                                                                   b_kmajor ? 0 : 1, slices, eb, DB);
  ACHI_LAUNCHED(ctx);
  static const int staged_env = [] {  // ACHI_OZAKI_STAGED=0: the pair-streaming kernel
    const char* e = std::getenv("ACHI_OZAKI_STAGED");
    return e ? std::atoi(e) : 1;
  }();
  if (staged_env && slices <= 8) {
    per_device_once("ozaki_staged_kernel", ctx.device, [] {
      ACHI_CUDA(cudaFuncSetAttribute(ozaki_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     staged_smem(8)));
      return 1;
    });
    const CUtensorMap ma = digit_map(DA, M, Kp, slices, TM, SKB, CU_TENSOR_MAP_SWIZZLE_64B);
    const CUtensorMap mb = digit_map(DB, N, Kp, slices, TN, SKB, CU_TENSOR_MAP_SWIZZLE_64B);
    ozaki_staged_kernel<<<dim3(cdiv(N, TN), cdiv(M, TM)), OZ_THREADS, staged_smem(slices), ctx.stream>>>(
        ma, mb, ea, eb, C, ldc, M, N, Kp, slices);
    ACHI_LAUNCHED(ctx);
    return;
  }
  per_device_once("ozaki_gemm_kernel", ctx.device, [] {
    ACHI_CUDA(cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM));
    return 1;
  });
  const CUtensorMap ma = digit_map(DA, M, Kp, slices, TM);
  const CUtensorMap mb = digit_map(DB, N, Kp, slices, TN);
  ozaki_gemm_kernel<<<dim3(cdiv(N, TN), cdiv(M, TM)), OZ_THREADS, OZ_SMEM, ctx.stream>>>(ma, mb, ea, eb, C, ldc, M,
                                                                                        N, Kp, slices);
  ACHI_LAUNCHED(ctx);
}

}  // namespace achi
