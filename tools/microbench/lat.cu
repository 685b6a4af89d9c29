// Dependent-chain latency of the instructions on the inner-Jacobi critical path
// (DFMA, DMUL, DADD, MUFU.RCP64H, F2F, FFMA, MUFU, LDS.64, BAR) on sm_100a.
// One warp, clock64 around 256 dependent ops; prints cycles per op.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>

#define N 256

__global__ void k_dfma(double* out, long long* cyc, double a) {
  double x = a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, a, 0.5);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dadd(double* out, long long* cyc, double a) {
  double x = a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x + a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ffma(double* out, long long* cyc, double a) {
  float x = (float)a, fa = (float)a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fmaf(x, fa, 0.5f);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_rcp64(double* out, long long* cyc, double a) {
  double x = a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_rcp32(double* out, long long* cyc, double a) {
  float x = (float)a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x));
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_f2f(double* out, long long* cyc, double a) {
  double x = a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    float f = __double2float_rn(x);
    asm volatile("" : "+f"(f));
    x = (double)f;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc, double a) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = idx[x];
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dsqrt(double* out, long long* cyc, double a) {
  double x = a + 1.0;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = sqrt(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ddiv(double* out, long long* cyc, double a) {
  double x = a + 1.0;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = 1.0 / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_bar(double* out, long long* cyc, double a) {
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

typedef void (*K)(double*, long long*, double);

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  struct { const char* name; K k; int threads; double per; } ks[] = {
      {"DFMA", k_dfma, 32, N},        {"DADD", k_dadd, 32, N},     {"FFMA", k_ffma, 32, N},
      {"MUFU.RCP64H", k_rcp64, 32, N}, {"MUFU.RCP", k_rcp32, 32, N}, {"F2F d->f->d (pair)", k_f2f, 32, N / 2},
      {"LDS.32 chain", k_lds, 32, N}, {"DSQRT+DADD", k_dsqrt, 32, N}, {"DDIV+DADD", k_ddiv, 32, N},
      {"SHFL.f64+DADD", k_shfl, 32, N},  {"BAR.SYNC 256 thr", k_bar, 256, N}, {"BAR.SYNC 32 thr", k_bar, 32, N}};
  for (auto& k : ks) {
    long long best = 1LL << 60;
    for (int rep = 0; rep < 5; ++rep) {
      k.k<<<1, k.threads>>>(out, cyc, 0.999);
      long long h;
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      if (h < best) best = h;
    }
    printf("%-22s %6.1f cycles/op\n", k.name, best / k.per);
  }
  return 0;
}
