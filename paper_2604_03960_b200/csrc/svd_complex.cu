// Complex svd_full (linalg.cpp:11-48, 67-70: DenseMatrix = Eigen::MatrixXcd) on
// the real one-sided Jacobi engine.
//
// A complex m x n matrix A = Ar + i Ai acts on z = x + i y as the real
// 2m x 2n matrix E = [[Ar, -Ai], [Ai, Ar]] on [x; y].  E has every singular
// value of A twice: for a right singular pair (z, w) of A (A z = s w) both
// [x; y] and [-y; x] (i.e. z and i z) are right singular vectors of E with
// value s.  So the real SVD of E (svd_jacobi.cu) gives A's decomposition:
//   * the sorted values of E come in equal pairs; each pair is one value of A;
//   * a run of values closer than 1e-6 sigma_1 (a pair, or a complex multiplet
//     of k values = 2k real ones) spans a k-dimensional complex subspace; its
//     complex basis is the real vectors read as complex ones, orthonormalised
//     by complex Gram-Schmidt (keeping k of the 2k candidates: a vector and
//     its i-multiple are dependent), the left vectors combined identically;
//   * a lone pair needs no Gram-Schmidt: its first real vector is the complex
//     singular vector (unit norm, the phase is fixed next).
// Then fix_phases (linalg.cpp:19-35): the first largest-|u| entry of every U
// column is made real and positive, the conjugate factor goes into V^dagger.
// E costs 8x the real flops of an m x n matrix; runs of near-equal values
// are separated from the rest by >= 1e-6 sigma_1, so the complex vectors are
// orthonormal to ~eps/1e-6 even where the real vectors of neighbouring values
// mix.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "svd_jacobi.cuh"

namespace achi {

namespace {

// E (2m x 2n row-major) from A (m x n row-major, interleaved re/im)
__global__ void embed_kernel(const double2* __restrict__ a, int m, int n, double* __restrict__ e) {
  const long tot = static_cast<long>(m) * n;
  const long ld = 2L * n;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const long i = t / n, j = t - i * n;
    const double2 v = a[t];
    e[i * ld + j] = v.x;
    e[i * ld + n + j] = -v.y;
    e[(i + m) * ld + j] = v.y;
    e[(i + m) * ld + n + j] = v.x;
  }
}

// lone pairs: complex index q takes real index src[q] (src < 0: Gram-Schmidt run)
//   U[i][q] = p_i + i q_i from UE[:, src], Vd[q][j] = conj(x_j + i y_j) from VTE[src, :]
__global__ void pick_kernel(const double* __restrict__ ue, const double* __restrict__ vte, int m,
                            int n, int r2, const int* __restrict__ src, int r, int k,
                            double2* __restrict__ U, double2* __restrict__ Vd) {
  const long tu = static_cast<long>(m) * k, tv = static_cast<long>(k) * n;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tu + tv;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    if (t < tu) {
      const int i = static_cast<int>(t / k), q = static_cast<int>(t % k);
      const int s = src[q];
      if (s >= 0)
        U[static_cast<long>(i) * r + q] =
            make_double2(ue[static_cast<long>(i) * r2 + s], ue[static_cast<long>(i + m) * r2 + s]);
    } else {
      const long u = t - tu;
      const int q = static_cast<int>(u / n), j = static_cast<int>(u % n);
      const int s = src[q];
      if (s >= 0) Vd[u] = make_double2(vte[static_cast<long>(s) * 2 * n + j],
                                       -vte[static_cast<long>(s) * 2 * n + n + j]);
    }
  }
}

__device__ double2 block_sum2(double2 v, double2* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) {
    r.x += sh[k].x;
    r.y += sh[k].y;
  }
  return r;  // every thread, same order
}


// Complex Gram-Schmidt of one run (one CTA): candidate t (real index) read as
// z = x + i y (length n) with its left vector w (length m); projected (twice)
// against the vectors already kept for this run, kept when at least half of its norm
// remains, until count / 2 are kept.  The inner products and norms are taken
// on the side whose real vectors are orthonormal by construction (prim_u: the
// left side; the other side is normalised Jacobi columns, zero for zero
// values), the other side gets the same combination.  cand: scratch (n + m)
// complex per run.
__global__ void gs_kernel(const double* __restrict__ ue, const double* __restrict__ vte, int m, int n,
                          int r2, const CsvdRun* __restrict__ runs, int r, double2* __restrict__ U,
                          double2* __restrict__ Vd, double2* __restrict__ cand, int prim_u,
                          int* __restrict__ fail) {
  __shared__ double2 sh[32];
  const CsvdRun g = runs[blockIdx.x];
  double2* cz = cand + static_cast<long>(blockIdx.x) * (n + m);
  double2* cw = cz + n;
  const int want = g.want;
  // primary side: length lp, entry i of kept vector k and of the candidate
  const int lp = prim_u ? m : n;
  auto kept_p = [&](int k, int i) -> double2 {
    if (prim_u) return U[static_cast<long>(i) * r + g.out + k];
    const double2 v = Vd[static_cast<long>(g.out + k) * n + i];
    return make_double2(v.x, -v.y);
  };
  double2* cp = prim_u ? cw : cz;
  int kept = 0;
  for (int t = g.first; t < g.first + g.count && kept < want; ++t) {
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      cz[j] = make_double2(vte[static_cast<long>(t) * 2 * n + j], vte[static_cast<long>(t) * 2 * n + n + j]);
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      cw[i] = make_double2(ue[static_cast<long>(i) * r2 + t], ue[static_cast<long>(i + m) * r2 + t]);
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass)  // projected twice (CGS2-style reorthogonalisation)
    for (int k = 0; k < kept; ++k) {
      double2 c = make_double2(0.0, 0.0);  // c = <p_k, cand_p> = sum conj(p_k) cand_p
      for (int i = threadIdx.x; i < lp; i += blockDim.x) {
        const double2 pk = kept_p(k, i), v = cp[i];
        c.x += pk.x * v.x + pk.y * v.y;
        c.y += pk.x * v.y - pk.y * v.x;
      }
      c = block_sum2(c, sh);
      const double2* vk = Vd + static_cast<long>(g.out + k) * n;  // z_k = conj(vk)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double2 zk = make_double2(vk[j].x, -vk[j].y);
        cz[j].x -= c.x * zk.x - c.y * zk.y;
        cz[j].y -= c.x * zk.y + c.y * zk.x;
      }
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double2 wk = U[static_cast<long>(i) * r + g.out + k];
        cw[i].x -= c.x * wk.x - c.y * wk.y;
        cw[i].y -= c.x * wk.y + c.y * wk.x;
      }
      __syncthreads();
    }
    double2 nn = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < lp; i += blockDim.x) nn.x += cp[i].x * cp[i].x + cp[i].y * cp[i].y;
    nn = block_sum2(nn, sh);
    if (nn.x > 0.25) {
      const double inv = 1.0 / sqrt(nn.x);
      const int q = g.out + kept;
      for (int j = threadIdx.x; j < n; j += blockDim.x)
        Vd[static_cast<long>(q) * n + j] = make_double2(cz[j].x * inv, -cz[j].y * inv);
      for (int i = threadIdx.x; i < m; i += blockDim.x)
        U[static_cast<long>(i) * r + q] = make_double2(cw[i].x * inv, cw[i].y * inv);
      ++kept;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && kept < want) atomicAdd(fail, 1);
}

// fix_phases (linalg.cpp:19-35), one warp per column q: f = conj(u_imax) / |u_imax|
// for the first index of the largest |u|; U[:, q] *= f, Vd[q, :] *= conj(f)
__global__ void cphase_kernel(double2* __restrict__ U, double2* __restrict__ Vd, int m, int n, int r,
                              int k) {
  const int warps = blockDim.x >> 5;
  const int q = blockIdx.x * warps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (q >= k) return;
  double best = 0.0;
  int idx = 0x7fffffff;
  for (int i = lane; i < m; i += 32) {
    const double2 v = U[static_cast<long>(i) * r + q];
    const double a = hypot(v.x, v.y);
    if (a > best) {
      best = a;
      idx = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  if (!(best > 0)) return;
  const double2 um = U[static_cast<long>(idx) * r + q];
  const double fx = um.x / best, fy = -um.y / best;  // f = conj(u) / |u|
  for (int i = lane; i < m; i += 32) {
    double2& v = U[static_cast<long>(i) * r + q];
    v = make_double2(v.x * fx - v.y * fy, v.x * fy + v.y * fx);
  }
  for (int j = lane; j < n; j += 32) {
    double2& v = Vd[static_cast<long>(q) * n + j];  // * conj(f)
    v = make_double2(v.x * fx + v.y * fy, v.y * fx - v.x * fy);
  }
}

}  // namespace

int svd_complex_stage1(Ctx& c, SvdWs& ws, CsvdPlan& P, const double* a, int m, int n, double* sigma,
                       int side_pref, const double* v_init, double* v_keep) {
  const int r = std::min(m, n), r2 = 2 * r, m2 = 2 * m, n2 = 2 * n;
  P.m = m;
  P.n = n;
  P.r = r;
  P.r2 = r2;
  P.E.reserve(static_cast<size_t>(m2) * n2);
  embed_kernel<<<std::max(1, std::min(cdiv(static_cast<long>(m) * n, 256), 8 * c.num_sms)), 256, 0, c.stream>>>(
      reinterpret_cast<const double2*>(a), m, n, P.E.p);
  ACHI_LAUNCHED(c);
  const SvdSide side = side_pref < 0 ? (m2 <= n2 ? SvdSide::kRows : SvdSide::kCols)
                                     : (side_pref == 0 ? SvdSide::kRows : SvdSide::kCols);
  P.prim_u = side == SvdSide::kRows;
  SvdResultDev res = svd_device(c, ws, P.E.p, m2, n2, m2, n2, side, 1, 0, nullptr, true, v_init);
  svd_wait_v(c, ws);
  if (v_keep)  // the real factor of E, a warm start for the next decomposition of this shape
    ACHI_CUDA(cudaMemcpyAsync(v_keep, res.V, sizeof(double) * res.ng * res.ng, cudaMemcpyDeviceToDevice,
                              c.stream));
  svd_phase_signs(c, ws, res, r2);
  P.UE.reserve(static_cast<size_t>(m2) * r2);
  P.VTE.reserve(static_cast<size_t>(r2) * n2);
  svd_gather(c, ws, res, r2, P.UE.p, P.VTE.p);
  std::vector<double>& s = P.s;
  s.resize(r2);
  ACHI_CUDA(cudaMemcpyAsync(s.data(), res.sigma, sizeof(double) * r2, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  P.sweeps = res.sweeps();
  // runs: values closer than 1e-4 sigma_1 to the next one (or than the Jacobi
  // noise floor 64 sqrt(mg) eps ||E||_F, svd_jacobi.cu zero_floor_kernel); the
  // values at or below the floor join the run above them (the vectors of values
  // near the floor are as undetermined as the noise subspace, so the two are
  // orthonormalised together).  Real vectors of values a gap g apart mix by
  // ~eps sigma_1 / g, so a lone pair's first real vector is its complex vector
  // to ~2e-12; inside a run the complex Gram-Schmidt visits the candidates in
  // sigma order and keeps one vector per pair, so each kept vector stays with
  // its own value unless the values are degenerate to that level.  (A gap
  // relative to the values themselves is not enough: measured 1e-6..1e-8
  // non-orthogonality on graded spectra, tools/csvd_study.py.)
  double fro2 = 0.0;
  for (int t = 0; t < r2; ++t) fro2 += s[t] * s[t];
  const double floor_v = 64.0 * std::sqrt(static_cast<double>(res.mg)) * 2.220446049250313e-16 *
                         std::sqrt(fro2);
  P.src.assign(r, -1);
  P.runs.clear();
  P.sig.assign(r, 0.0);
  int q = 0;
  for (int t = 0; t < r2;) {
    int e = t + 1;
    while (e < r2 && (s[e] <= floor_v || s[e - 1] - s[e] <= std::max(1e-4 * s[0], floor_v))) ++e;
    int cnt = e - t;
    if (cnt % 2) {  // a run must hold whole pairs: extend by the next value
      if (e >= r2) fail(ACHI_E_NUMERICAL_FAILURE, "svd (complex): unpaired singular value");
      ++e;
      ++cnt;
    }
    if (q + cnt / 2 > r) fail(ACHI_E_NUMERICAL_FAILURE, "svd (complex): singular value pairing");
    for (int k = 0; k < cnt / 2; ++k) P.sig[q + k] = s[t + 2 * k];
    if (cnt == 2)
      P.src[q] = t;
    else
      P.runs.push_back(CsvdRun{t, cnt, q, cnt / 2});
    q += cnt / 2;
    t = e;
  }
  if (q != r) fail(ACHI_E_NUMERICAL_FAILURE, "svd (complex): singular value pairing");
  // (P.sig and P.src stay alive until the next stage 1, which synchronises first)
  ACHI_CUDA(cudaMemcpyAsync(sigma, P.sig.data(), sizeof(double) * r, cudaMemcpyHostToDevice, c.stream));
  ACHI_CUDA(cudaMemcpyAsync(P.src_d.reserve(r), P.src.data(), sizeof(int) * r, cudaMemcpyHostToDevice,
                            c.stream));
  return P.sweeps;
}

void svd_complex_stage2(Ctx& c, CsvdPlan& P, int k, double* U, double* Vd) {
  const int m = P.m, n = P.n, r = P.r, r2 = P.r2;
  k = std::max(0, std::min(k, r));
  double2* U2 = reinterpret_cast<double2*>(U);
  double2* V2 = reinterpret_cast<double2*>(Vd);
  {
    const long tot = static_cast<long>(m) * k + static_cast<long>(k) * n;
    pick_kernel<<<std::max(1, std::min(cdiv(tot, 256), 8 * c.num_sms)), 256, 0, c.stream>>>(
        P.UE.p, P.VTE.p, m, n, r2, P.src_d.p, r, k, U2, V2);
    ACHI_LAUNCHED(c);
  }
  // only the runs that hold one of the first k values, each up to value k
  P.runs_k.clear();
  for (const CsvdRun& g : P.runs)
    if (g.out < k) P.runs_k.push_back(CsvdRun{g.first, g.count, g.out, std::min(g.want, k - g.out)});
  if (!P.runs_k.empty()) {
    const size_t nr = P.runs_k.size();
    CsvdRun* pr = P.runs_d.reserve(nr);
    int* pf = P.fail_d.reserve(1);
    P.cand.reserve(2 * nr * static_cast<size_t>(n + m));
    ACHI_CUDA(cudaMemcpyAsync(pr, P.runs_k.data(), sizeof(CsvdRun) * nr, cudaMemcpyHostToDevice, c.stream));
    ACHI_CUDA(cudaMemsetAsync(pf, 0, sizeof(int), c.stream));
    gs_kernel<<<static_cast<unsigned>(nr), 256, 0, c.stream>>>(
        P.UE.p, P.VTE.p, m, n, r2, pr, r, U2, V2, reinterpret_cast<double2*>(P.cand.p), P.prim_u ? 1 : 0, pf);
    ACHI_LAUNCHED(c);
    int hf = 0;
    ACHI_CUDA(cudaMemcpyAsync(&hf, pf, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (hf) fail(ACHI_E_NUMERICAL_FAILURE, "svd (complex): multiplet basis");
  }
  if (k > 0) {
    cphase_kernel<<<cdiv(k, 8), 256, 0, c.stream>>>(U2, V2, m, n, r, k);
    ACHI_LAUNCHED(c);
  }
}

int svd_complex_device(Ctx& c, SvdWs& ws, const double* a, int m, int n, double* sigma, double* U,
                       double* Vd, int side_pref, const double* v_init, double* v_keep) {
  CsvdPlan P;
  const int sweeps = svd_complex_stage1(c, ws, P, a, m, n, sigma, side_pref, v_init, v_keep);
  svd_complex_stage2(c, P, P.r, U, Vd);
  c.sync();  // the plan's host vectors must outlive their copies
  return sweeps;
}

}  // namespace achi
