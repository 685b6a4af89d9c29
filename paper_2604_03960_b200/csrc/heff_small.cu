// Fused small-chi effective-Hamiltonian matvec (dmrg.cpp:58-71) for
// chl, chr <= 128 -- every bond of config C3.  At these sizes the TMA path
// (GEMM -> MPO mixing -> split-K GEMM -> reduce, four launches) is bound by
// launch and pipeline latency (~37 us per matvec at chi = 110); here one
// cooperative launch runs the contraction in three phases separated by grid
// barriers, every operand tile staged once in shared memory and multiplied
// with mma.sync.m16n8k4.f64 (DMMA), ~25 us:
//
//   A: tiles of X[(bl,a),(s jr)] = L[(bl,a), jl] theta[jl, (s jr)] covering all
//      MPO rows a of a block of bl and all s of a block of jr, so the MPO
//      mixing Y[((bl,s'),e), jr] = sum W12[(s',e),(a,s)] X[(bl,a),(s,jr)] is
//      done on the tile in shared memory (X is never written)
//   B: P_e[(bl,s'), br] = sum_jr Y[(bl,s'),(e,jr)] R[br,(e,jr)]   (split over e)
//   C: out = sum_e P_e (fixed order)
//
// Every sum runs in a fixed order: the result is deterministic.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "heff_phases.cuh"

namespace cg = cooperative_groups;

namespace achi {

namespace {

using namespace hs;

template <int KM>
__global__ void __launch_bounds__(HS_THREADS) heff_small_kernel(HsArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  double* As = reinterpret_cast<double*>(dyn);  // [32][LD]
  double* Bs = As + HS_TM * hs_ld<KM>();        // [64][LD]
  __shared__ MixSmem w;
  cg::grid_group grid = cg::this_grid();
  load_mix(a.mix, w);
  __syncthreads();
  phase_a<KM>(a, w, a.theta, As, Bs, blockIdx.x, gridDim.x);
  grid.sync();
  phase_b<KM>(a, As, Bs, blockIdx.x, gridDim.x);
  grid.sync();
  phase_c(a, a.out, blockIdx.x, gridDim.x);
}

template <int KM>
void launch_small(Ctx& ctx, const HeffOps& op, const double* theta, double* out, double* X, double* part) {
  const int dd = op.d * op.d;
  const long M2 = static_cast<long>(op.chl) * dd, N2 = op.chr;
  const size_t smem = smem_bytes<KM>();
  const int max_blocks = per_device_once("heff_small_kernel:" + std::to_string(KM), ctx.device, [&] {
    ACHI_CUDA(cudaFuncSetAttribute(heff_small_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    int per_sm = 0;
    ACHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, heff_small_kernel<KM>, HS_THREADS, smem));
    return std::max(1, per_sm) * ctx.num_sms;
  });
  const long itemsA = cdiv(op.chl, HS_TM / op.D1) * cdiv(op.chr, HS_JRB);
  const long itemsB = cdiv(M2, HS_TM) * cdiv(N2, HS_TN) * op.D3;
  const int grid = std::max(1, ctx.cap_grid(std::min<long>(std::max(itemsA, itemsB), max_blocks)));
  HsArgs a{op.L, op.R, theta, out, X, part, op.mix, op.chl, op.chr, op.d, op.D1, op.D3};
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(HS_THREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  ACHI_CUDA(cudaLaunchKernelEx(&lc, heff_small_kernel<KM>, a));
  ACHI_LAUNCHED(ctx);
}

}  // namespace

bool heff_small_applicable(const HeffOps& op) {
  return op.d == 2 && op.D1 >= 1 && op.D1 <= HS_TM && op.chl <= HS_KMAX_WIDE &&
         op.chr <= HS_KMAX_WIDE && op.mix.nin <= HS_MAXW && op.mix.nout <= HS_MAXW &&
         op.mix.nnz <= HS_MAXNNZ;
}

bool heff_small_fusable(Ctx& ctx, const HeffOps& op, const double* theta, double* out, HsArgs* args,
                        long* items) {
  static const bool small_on = [] {
    const char* e = std::getenv("ACHI_HEFF_SMALL");
    return !(e && e[0] == '0');
  }();
  if (!small_on || std::max(op.chl, op.chr) > HS_KMAX || !heff_small_applicable(op)) return false;
  const int dd = op.d * op.d;
  const long M2 = static_cast<long>(op.chl) * dd, N2 = op.chr;
  double* X = ctx.ws_a.reserve(static_cast<size_t>(M2 * op.D3 * N2));
  double* part = ctx.ws_b.reserve(static_cast<size_t>(op.D3 * M2 * N2));
  *args = HsArgs{op.L, op.R, theta, out, X, part, op.mix, op.chl, op.chr, op.d, op.D1, op.D3};
  const long itemsA = cdiv(op.chl, HS_TM / op.D1) * cdiv(op.chr, HS_JRB);
  const long itemsB = cdiv(M2, HS_TM) * cdiv(N2, HS_TN) * op.D3;
  *items = std::max(itemsA, itemsB);
  return true;
}

void heff_apply_small(Ctx& ctx, const HeffOps& op, const double* theta, double* out) {
  const int dd = op.d * op.d;
  const long M2 = static_cast<long>(op.chl) * dd, N2 = op.chr;
  double* X = ctx.ws_a.reserve(static_cast<size_t>(M2 * op.D3 * N2));  // Y
  double* part = ctx.ws_b.reserve(static_cast<size_t>(op.D3 * M2 * N2));
  if (op.chl <= HS_KMAX && op.chr <= HS_KMAX)
    launch_small<HS_KMAX>(ctx, op, theta, out, X, part);
  else
    launch_small<HS_KMAX_WIDE>(ctx, op, theta, out, X, part);
}

}  // namespace achi
