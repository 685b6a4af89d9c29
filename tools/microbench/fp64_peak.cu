// FP64 pipe microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA throughput.
// Used once to establish the FP64 roofline denominator (no FP64 entry in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, b0 = 1.0 - a0;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 - a0;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - a * 1e-3;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double run(K kernel, int blocks, int threads, int iters, double flop_per_thread_iter, double* buf) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kernel<<<blocks, threads>>>(buf, iters / 10);
  cudaEventRecord(e0);
  kernel<<<blocks, threads>>>(buf, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = double(blocks) * threads * iters * flop_per_thread_iter;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * 148 * 64 * 1024);
  // m16n8k4: 16*8*4 FMA = 512 FMA = 1024 flop per warp per instr -> 32 flop/thread
  for (int wpb : {4, 8, 16}) {
    printf("dmma m16n8k4 chains=4 warps/SM=%d : %.2f TFLOP/s\n", wpb,
           run(dmma_m16n8k4<4>, sms, 32 * wpb, 20000, 4 * 32.0, buf));
    printf("dmma m16n8k4 chains=8 warps/SM=%d : %.2f TFLOP/s\n", wpb,
           run(dmma_m16n8k4<8>, sms, 32 * wpb, 20000, 8 * 32.0, buf));
    printf("dmma m8n8k4  chains=8 warps/SM=%d : %.2f TFLOP/s\n", wpb,
           run(dmma_m8n8k4<8>, sms, 32 * wpb, 20000, 8 * 16.0, buf));
    printf("dfma chains=8 warps/SM=%d : %.2f TFLOP/s\n", wpb,
           run(dfma_peak<8>, sms, 32 * wpb, 20000, 8 * 2.0, buf));
  }
  printf("dmma m16n8k4 chains=8 2 blocks x 16 warps/SM: %.2f TFLOP/s\n",
         run(dmma_m16n8k4<8>, 2 * sms, 512, 20000, 8 * 32.0, buf));
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
