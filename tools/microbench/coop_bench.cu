// Launch cost of cooperative kernels with grid barriers, large vs small dynamic
// shared memory, and the cost of alternating shared-memory configurations.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coop_bench coop_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)
namespace cg = cooperative_groups;

__global__ void coop_k(int syncs, double* out) {
  __shared__ double s0;  // the dynamic allocation is only reserved, never touched
  cg::grid_group g = cg::this_grid();
  if (threadIdx.x == 0) s0 = blockIdx.x;
  for (int i = 0; i < syncs; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = s0;
}
__global__ void plain_k(double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] += 1.0;
}

float run(int grid, size_t smem, int syncs, bool alternate, int reps) {
  double* out;
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(out, 0, 64));
  CK(cudaFuncSetAttribute(coop_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  void* args[] = {&syncs, &out};
  for (int w = 0; w < 10; ++w) CK(cudaLaunchCooperativeKernel((void*)coop_k, grid, 256, args, smem, 0));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) {
    cudaLaunchCooperativeKernel((void*)coop_k, grid, 256, args, smem, 0);
    if (alternate) plain_k<<<148, 256>>>(out);
  }
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms * 1000.f / reps;
}

int main() {
  const int reps = 2000;
  printf("grid 140, smem   0 KB, 0 syncs: %.2f us\n", run(140, 0, 0, false, reps));
  printf("grid 140, smem   0 KB, 2 syncs: %.2f us\n", run(140, 0, 2, false, reps));
  printf("grid 140, smem 100 KB, 0 syncs: %.2f us\n", run(140, 100 * 1024, 0, false, reps));
  printf("grid 140, smem 100 KB, 2 syncs: %.2f us\n", run(140, 100 * 1024, 2, false, reps));
  printf("grid 140, smem 100 KB, 2 syncs + plain kernel (alternating): %.2f us\n",
         run(140, 100 * 1024, 2, true, reps));
  printf("grid 140, smem   0 KB, 2 syncs + plain kernel (alternating): %.2f us\n",
         run(140, 0, 2, true, reps));
  printf("grid  16, smem 100 KB, 2 syncs: %.2f us\n", run(16, 100 * 1024, 2, false, reps));
  return 0;
}
