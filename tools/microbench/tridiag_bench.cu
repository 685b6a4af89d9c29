
#include <cstdio>
#include <cmath>
#define LANCZOS_BLOCK 48
// exact power of two 2^e (|e| < 1000)
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}
// binary exponent of |m| (m > 0, normal)
__device__ __forceinline__ int exponent_of(double m) {
  return static_cast<int>((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
}

// Characteristic-polynomial recurrence at x with its x-derivative:
//   p_{i+1} = (a_i - x) p_i - bb_{i-1} p_{i-1},
//   p'_{i+1} = (a_i - x) p'_i - bb_{i-1} p'_{i-1} - p_i,  p_0 = 1, p'_0 = 0.
// Returns the Sturm count (sign changes of p_0..p_k = number of eigenvalues
// below x; a zero takes the sign +, counting a root of a leading minor once)
// and *ratio = p_k / p'_k (the Newton correction).  p and p' are rescaled by
// an exact power of two every 8 steps, so neither overflows nor underflows.
__device__ int char_poly(const double* a, const double* bb, int k, double x, double* ratio) {
  double pm = 1.0, p = a[0] - x, qm = 0.0, q = -1.0;
  int cnt = p < 0.0 ? 1 : 0;
  for (int i0 = 1; i0 < k; i0 += 8) {
    double da[8], db[8];  // operands loaded up front: shared-memory latency off the chain
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      da[u] = i < k ? a[i] - x : 0.0;
      db[u] = i < k ? bb[i - 1] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u < k) {
        const double pn = fma(da[u], p, -db[u] * pm);
        const double qn = fma(da[u], q, -db[u] * qm) - p;
        cnt += (pn < 0.0) != (p < 0.0) ? 1 : 0;
        pm = p;
        p = pn;
        qm = q;
        q = qn;
      }
    }
    const double m = fmax(fmax(fabs(p), fabs(pm)), fmax(fabs(q), fabs(qm)));
    const int e = exponent_of(m);
    if (m > 0.0 && (e > 64 || e < -64)) {
      const double f = pow2(-e);
      p *= f;
      pm *= f;
      q *= f;
      qm *= f;
    }
  }
  *ratio = p / q;
  return cnt;
}

// Lowest eigenvalue by safeguarded Newton (one thread).  The bracket [lo, hi]
// keeps count(lo) = 0 and count(hi) >= 1: lo starts at the Gershgorin bound,
// hi at the previous step's Ritz value (interlacing: the new lowest value is
// not above it; Gershgorin when there is none).  Newton from above overshoots
// at most once and then converges monotonically from below; steps leaving the
// bracket are replaced by bisection.  Stops when the Newton correction is
// below 4 ulp.  *scale_out = Gershgorin scale.
__device__ double tridiag_lowest_newton(const double* a, const double* b, const double* bb, int k,
                                        bool hinted, double theta_prev, double* scale_out) {
  double lo = INFINITY, hi = -INFINITY, scale = 0.0;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < k ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
    scale = fmax(scale, fabs(a[i]) + r);
  }
  *scale_out = scale;
  const double pad = 4.0 * 2.3e-16 * scale;
  lo -= pad;
  hi += pad;
  double ratio;
  double x = hinted ? fmin(hi, theta_prev + pad) : hi;
  if (char_poly(a, bb, k, x, &ratio) < 1) {
    x = hi;
    char_poly(a, bb, k, x, &ratio);
  }
  hi = x;
  for (int it = 0; it < 200; ++it) {
    double xn = x - ratio;
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    if (fabs(xn - x) <= 4.0 * 2.3e-16 * fabs(x) || !(hi - lo > 2.3e-16 * fmax(fabs(lo), fabs(hi))))
      return xn;
    x = xn;
    if (char_poly(a, bb, k, x, &ratio) >= 1)
      hi = x;
    else
      lo = x;
  }
  return x;
}


__device__ int sturm_only(const double* a, const double* bb, int k, double x) {
  double pm = 1.0, p = a[0] - x;
  int cnt = p < 0.0 ? 1 : 0;
  for (int i = 1; i < k; ++i) {
    const double pn = fma(a[i] - x, p, -bb[i - 1] * pm);
    cnt += (pn < 0.0) != (p < 0.0) ? 1 : 0;
    pm = p; p = pn;
  }
  return cnt;
}
__global__ void kern(const double* ag, const double* bg, int k, long long* out, double* res) {
  __shared__ double a[48], b[48], bb[48];
  for (int i = threadIdx.x; i < k; i += 32) { a[i] = ag[i]; b[i] = bg[i]; bb[i] = bg[i]*bg[i]; }
  __syncwarp();
  if (threadIdx.x) return;
  double r, acc = 0; int c = 0;
  long long t0 = clock64();
  for (int it = 0; it < 100; ++it) { c += char_poly(a, bb, k, -1.0 + 1e-3 * it, &r); acc += r; }
  long long t1 = clock64();
  for (int it = 0; it < 100; ++it) { c += sturm_only(a, bb, k, -1.0 + 1e-3 * it); }
  long long t2 = clock64();
  double sc;
  double th = 0;
  for (int it = 0; it < 10; ++it) th += tridiag_lowest_newton(a, b, bb, k, it > 0, -1.5 + 0.01*it, &sc);
  long long t3 = clock64();
  out[0] = (t1 - t0) / 100; out[1] = (t2 - t1) / 100; out[2] = (t3 - t2) / 10;
  res[0] = acc + c + th;
}
int main() {
  const int k = 15;
  double ha[48], hb[48];
  for (int i = 0; i < k; ++i) { ha[i] = -0.5 + 0.1 * (i % 7); hb[i] = 0.3 + 0.05 * (i % 5); }
  double *da, *db, *dr; long long* dout;
  cudaMalloc(&da, 48*8); cudaMalloc(&db, 48*8); cudaMalloc(&dr, 8); cudaMalloc(&dout, 3*8);
  cudaMemcpy(da, ha, 48*8, cudaMemcpyHostToDevice); cudaMemcpy(db, hb, 48*8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) kern<<<1, 32>>>(da, db, k, dout, dr);
  long long h[3]; cudaMemcpy(h, dout, 24, cudaMemcpyDeviceToHost);
  printf("k=%d char_poly %lld cycles, sturm_only %lld cycles, newton solve %lld cycles\n", k, h[0], h[1], h[2]);
}
