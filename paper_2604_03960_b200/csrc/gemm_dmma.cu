// Host side of the TMA-fed DMMA GEMM: tensor-map encoding, tile-config and
// split-K selection, deterministic split-K reduction.
#include "gemm_dmma.cuh"
#include "ozaki.cuh"

namespace achi {
namespace gemm_detail {

__global__ void splitk_reduce_kernel(const double* __restrict__ ws, long split_stride, int splits,
                                     double* __restrict__ C, long ldc, long ldw, int M, int N) {
  pdl_wait();  // launched with launch_pdl / the PDL attribute (common.cuh)
  const long total = static_cast<long>(M) * N;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long r = i / N, c = i % N;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[z * split_stride + r * ldw + c];
    C[r * ldc + c] = s;
  }
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ACHI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      fail(ACHI_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D map over a row-major (rows x cols, ld) FP64 matrix, 16 x box_rows boxes,
// 128B swizzle, zero fill out of bounds.
CUtensorMap make_map(const double* ptr, long rows, long cols, long ld, int box_rows) {
  if ((ld & 1) != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    fail(ACHI_E_INTERNAL, "gemm: operand stride/base not 16-byte aligned (bond dims must be padded)");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  cuuint32_t box[2] = {16u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ACHI_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

template <int BM, int BN, int WTM, int WTN, int STAGES, Major AM, Major BMJ>
void launch(Ctx& ctx, int M, int N, int K, const Operand& A, const Operand& B, double* C,
            long ldc, int splits) {
  using G = Cfg<BM, BN, WTM, WTN, STAGES, AM, BMJ>;
  auto kern = dmma_gemm_kernel<BM, BN, WTM, WTN, STAGES, AM, BMJ>;
  per_device_once(std::string("dmma_gemm_kernel:") + std::to_string(reinterpret_cast<uintptr_t>(
                      reinterpret_cast<const void*>(kern))), ctx.device, [&] {
    ACHI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    return 1;
  });
  CUtensorMap ma = AM == Major::kK ? make_map(A.ptr, M, K, A.ld, BM) : make_map(A.ptr, K, M, A.ld, 16);
  CUtensorMap mb = BMJ == Major::kK ? make_map(B.ptr, N, K, B.ld, BN) : make_map(B.ptr, K, N, B.ld, 16);
  const int kt_total = cdiv(K, BK);
  const int kt_per = cdiv(kt_total, splits);
  splits = cdiv(kt_total, kt_per);
  dim3 grid(cdiv(N, BN), cdiv(M, BM), splits);
  if (splits == 1) {
    ACHI_CUDA(launch_pdl(kern, grid, G::THREADS, G::SMEM, ctx.stream, ma, mb, C, ldc, 0L, M, N, K, kt_per));
    ACHI_LAUNCHED(ctx);
    return;
  }
  const long slab = static_cast<long>(M) * N;
  // slab * splits <= 4096 (296 + tiles) < 4096 * 592 on this path (dispatch
  // below): reserving that bound once keeps the buffer (and every captured
  // graph that uses it) stable
  double* ws = ctx.ws_split.reserve(std::max<size_t>(static_cast<size_t>(slab) * splits, 4096UL * 592));
  ACHI_CUDA(launch_pdl(kern, grid, G::THREADS, G::SMEM, ctx.stream, ma, mb, ws, static_cast<long>(N), slab, M, N, K,
                       kt_per));
  ACHI_LAUNCHED(ctx);
  const int blocks = std::min<long>(cdiv(slab, 256), 4L * ctx.num_sms);
  ACHI_CUDA(launch_pdl(splitk_reduce_kernel, blocks, 256, 0, ctx.stream, ws, slab, splits, C, ldc,
                       static_cast<long>(N), M, N));
  ACHI_LAUNCHED(ctx);
}

template <Major AM, Major BMJ>
void dispatch(Ctx& ctx, int M, int N, int K, const Operand& A, const Operand& B, double* C,
              long ldc) {
  const long big_tiles = static_cast<long>(cdiv(M, 128)) * cdiv(N, 128);
  if (big_tiles >= 3L * ctx.num_sms) {
    launch<128, 128, 64, 32, 4, AM, BMJ>(ctx, M, N, K, A, B, C, ldc, 1);
    return;
  }
  const long tiles = static_cast<long>(cdiv(M, 64)) * cdiv(N, 64);
  const int kt = cdiv(K, BK);
  int splits = 1;
  if (tiles < 2L * ctx.num_sms && kt >= 16) {
    splits = static_cast<int>(std::min<long>(cdiv(2L * ctx.num_sms, tiles), kt / 8));
    splits = std::max(1, std::min(splits, 16));
  }
  launch<64, 64, 32, 32, 6, AM, BMJ>(ctx, M, N, K, A, B, C, ldc, splits);
}

}  // namespace
}  // namespace gemm_detail

void gemm(Ctx& ctx, int M, int N, int K, const Operand& A, const Operand& B, double* C, long ldc) {
  using namespace gemm_detail;
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    for (int r = 0; r < M; ++r)
      ACHI_CUDA(cudaMemsetAsync(C + static_cast<long>(r) * ldc, 0, sizeof(double) * N, ctx.stream));
    return;
  }
  if (ctx.ozaki_slices > 0 && 2.0 * M * N * K >= ctx.ozaki_min_flops && K <= (1 << 14)) {
    // opt-in emulated FP64 on the int8 tensor cores (ozaki.cu)
    dgemm_ozaki(ctx, M, N, K, A.ptr, A.ld, A.major == Major::kMN, B.ptr, B.ld, B.major == Major::kK, C, ldc,
                ctx.ozaki_slices);
    return;
  }
  if (A.major == Major::kK && B.major == Major::kMN)
    dispatch<Major::kK, Major::kMN>(ctx, M, N, K, A, B, C, ldc);
  else if (A.major == Major::kK && B.major == Major::kK)
    dispatch<Major::kK, Major::kK>(ctx, M, N, K, A, B, C, ldc);
  else if (A.major == Major::kMN && B.major == Major::kMN)
    dispatch<Major::kMN, Major::kMN>(ctx, M, N, K, A, B, C, ldc);
  else
    dispatch<Major::kMN, Major::kK>(ctx, M, N, K, A, B, C, ldc);
}

}  // namespace achi
