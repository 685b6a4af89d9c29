// DMRG chain driver on device-resident state (see chain.cuh).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <random>

#include "chain.cuh"

namespace achi {

void validate_spec(const achi_model_spec& s) {  // models.cpp:11-17
  if (s.n < 2) fail(ACHI_E_INVALID_CONFIG, "model: n must be >= 2");
  if (!std::isfinite(s.jx) || !std::isfinite(s.jy) || !std::isfinite(s.jz) || !std::isfinite(s.h))
    fail(ACHI_E_INVALID_CONFIG, "model: couplings must be finite");
  if (s.family != ACHI_HEISENBERG_XXZ && s.family != ACHI_TRANSVERSE_ISING)
    fail(ACHI_E_UNSUPPORTED_MODEL, "build_mpo: unknown model family");
}

void validate_config(const achi_dmrg_config& g) {  // dmrg.cpp:8-16, controller.cpp:17-33
  const auto& c = g.controller;
  if (g.max_sweeps < 1) fail(ACHI_E_INVALID_CONFIG, "dmrg: max_sweeps must be >= 1");
  if (!(g.eps_conv > 0)) fail(ACHI_E_INVALID_CONFIG, "dmrg: eps_conv must be > 0");
  if (!(g.eig_tol > 0)) fail(ACHI_E_INVALID_CONFIG, "dmrg: eig_tol must be > 0");
  if (g.eig_max_iter < 1) fail(ACHI_E_INVALID_CONFIG, "dmrg: eig_max_iter must be >= 1");
  if (c.chi_min < 1) fail(ACHI_E_INVALID_CONFIG, "controller: chi_min must be >= 1");
  if (c.chi_min > c.chi_max) fail(ACHI_E_INVALID_CONFIG, "controller: chi_min must be <= chi_max");
  if (!(c.alpha_ema > 0.0) || c.alpha_ema > 1.0)
    fail(ACHI_E_INVALID_CONFIG, "controller: alpha_ema must lie in (0, 1]");
  if (c.gamma_margin < 1.0) fail(ACHI_E_INVALID_CONFIG, "controller: gamma_margin must be >= 1");
  if (c.beta_predict < 0.0) fail(ACHI_E_INVALID_CONFIG, "controller: beta_predict must be >= 0");
  if (!(c.eps_trunc >= 0.0)) fail(ACHI_E_INVALID_CONFIG, "controller: eps_trunc must be >= 0");
  if (c.kp < 0 || c.ki < 0 || c.kd < 0 || !std::isfinite(c.kp) || !std::isfinite(c.ki) ||
      !std::isfinite(c.kd))
    fail(ACHI_E_INVALID_CONFIG, "controller: gains must be finite and >= 0");
}

std::vector<HostMpo> build_mpo_real(const achi_model_spec& s) {
  validate_spec(s);
  const double sc = s.convention == ACHI_SPIN_HALF ? 0.5 : 1.0;
  const double id[4] = {1, 0, 0, 1}, x[4] = {0, sc, sc, 0}, z[4] = {sc, 0, 0, -sc};
  const double iy[4] = {0, sc, -sc, 0};  // i*sigma^y (scaled): real
  int w;
  HostMpo bulk;
  auto put = [&](int row, int col, const double* op, double f) {
    for (int so = 0; so < 2; ++so)
      for (int si = 0; si < 2; ++si)
        bulk.w[((static_cast<size_t>(row) * 2 + so) * 2 + si) * w + col] = f * op[so * 2 + si];
  };
  if (s.family == ACHI_HEISENBERG_XXZ) {
    w = 5;
    bulk = HostMpo{w, 2, w, std::vector<double>(static_cast<size_t>(w) * 4 * w, 0.0)};
    put(0, 0, id, 1.0);
    put(1, 0, x, 1.0);
    put(2, 0, iy, 1.0);
    put(3, 0, z, 1.0);
    put(4, 0, z, -s.h);
    put(4, 1, x, s.jx);
    put(4, 2, iy, -s.jy);
    put(4, 3, z, s.jz);
    put(4, 4, id, 1.0);
  } else {
    w = 3;
    bulk = HostMpo{w, 2, w, std::vector<double>(static_cast<size_t>(w) * 4 * w, 0.0)};
    put(0, 0, id, 1.0);
    put(1, 0, z, 1.0);
    put(2, 0, x, -s.h);
    put(2, 1, z, -s.jz);
    put(2, 2, id, 1.0);
  }
  HostMpo first{1, 2, w, std::vector<double>(4 * w, 0.0)}, last{w, 2, 1, std::vector<double>(4 * w, 0.0)};
  for (int so = 0; so < 2; ++so)
    for (int si = 0; si < 2; ++si) {
      for (int c = 0; c < w; ++c) first.w[(so * 2 + si) * w + c] = bulk.at(w - 1, so, si, c);
      for (int r = 0; r < w; ++r) last.w[(static_cast<size_t>(r) * 2 + so) * 2 + si] = bulk.at(r, so, si, 0);
    }
  std::vector<HostMpo> out;
  out.push_back(first);
  for (int i = 1; i < s.n - 1; ++i) out.push_back(bulk);
  out.push_back(last);
  return out;
}

namespace {

// Neel product state (dmrg.cpp:222-232) followed by canonicalize(psi, 0)
// (mps.cpp:186-210): Householder QR of each 2x1 column, signs as dlarfg.
std::vector<std::vector<double>> neel_canonical(int n, int d) {
  std::vector<std::vector<double>> s(n, std::vector<double>(d, 0.0));
  for (int i = 0; i < n; ++i) s[i][i % 2] = 1.0;
  for (int i = n - 1; i >= 1; --i) {
    const double alpha = s[i][0], xnorm = std::fabs(s[i][1]);
    double beta, q0, q1;
    if (xnorm == 0.0) {
      beta = alpha;
      q0 = 1.0;
      q1 = 0.0;
    } else {
      const double nrm = std::hypot(alpha, xnorm);
      beta = alpha >= 0 ? -nrm : nrm;
      const double tau = (beta - alpha) / beta;
      const double v1 = s[i][1] / (alpha - beta);
      q0 = 1.0 - tau;
      q1 = -tau * v1;
    }
    s[i][0] = q0;
    s[i][1] = q1;
    for (double& v : s[i - 1]) v *= beta;
  }
  return s;
}

}  // namespace

// capped_bond_dims (mps.cpp:60-73): min(chi, d^k, d^(n-k)) per bond
std::vector<int> capped_bond_dims(int n, int d, int chi) {
  std::vector<int> dims(n - 1, chi);
  long grow = 1;
  for (int i = 0; i < n - 1; ++i) {
    grow = std::min<long>(grow * d, chi);
    dims[i] = static_cast<int>(std::min<long>(dims[i], grow));
  }
  grow = 1;
  for (int i = n - 2; i >= 0; --i) {
    grow = std::min<long>(grow * d, chi);
    dims[i] = static_cast<int>(std::min<long>(dims[i], grow));
  }
  return dims;
}

namespace {

// C (M x N) = A (M x K) * B (K x N), row-major, any shapes (setup-sized
// products of canonicalisation; 16 x 16 shared-memory tiles, FP64 FMA)
__global__ void matmul_kernel(const double* __restrict__ A, const double* __restrict__ B,
                              double* __restrict__ C, int M, int N, int K) {
  __shared__ double As[16][17], Bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    As[ty][tx] = (row < M && k0 + tx < K) ? A[static_cast<long>(row) * K + k0 + tx] : 0.0;
    Bs[ty][tx] = (k0 + ty < K && col < N) ? B[static_cast<long>(k0 + ty) * N + col] : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fma(As[ty][k], Bs[k][tx], acc);
    __syncthreads();
  }
  if (row < M && col < N) C[static_cast<long>(row) * N + col] = acc;
}

// U (m x k row-major) <- U * diag(sigma)
__global__ void scale_cols_kernel(double* __restrict__ U, int m, int k, const double* __restrict__ sigma) {
  const long tot = static_cast<long>(m) * k;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot;
       t += static_cast<long>(gridDim.x) * blockDim.x)
    U[t] *= sigma[t % k];
}

__global__ void scale_all_kernel(double* __restrict__ x, long n, const double* __restrict__ nrm2,
                                 int* __restrict__ bad) {
  const double n2 = *nrm2;
  if (!(n2 > 0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *bad = 1;
    return;
  }
  const double inv = 1.0 / sqrt(n2);
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long>(gridDim.x) * blockDim.x)
    x[t] *= inv;
}

}  // namespace

// canonicalize(psi, 0) (mps.cpp:172-210: push_left on sites n-1..1) on the
// device.  Site i as M (l x d r, row-major) is factored M = (U S) V^T by the
// Jacobi SVD with V accumulated (orthonormal also across zero and noise-level
// values); site i <- V^T (k x d r, rows orthonormal), site i-1 <- site i-1 *
// (U S).  This is push_left with an SVD instead of Householder QR: the same
// bond dimensions k = min(l, d r) and the same state, in another gauge of
// bond i (a k x k rotation), which every later step is covariant under
// (energies and kept ranks agree with the QR gauge to rounding).
void device_canonicalize_left(Ctx& c, std::vector<DevBuf>& s, std::vector<int>& dims, int d) {
  const int n = static_cast<int>(s.size());
  SvdWs ws;
  for (int i = n - 1; i >= 1; --i) {
    const int l = dims[i], r = dims[i + 1], cols = d * r, k = std::min(l, cols), ll = dims[i - 1];
    SvdResultDev res = svd_device(c, ws, s[i].p, l, cols, l, cols, SvdSide::kCols);
    svd_phase_signs(c, ws, res, k);
    DevBuf U, VT, nb;
    U.reserve(static_cast<size_t>(l) * k);
    VT.reserve(static_cast<size_t>(k) * cols);
    svd_gather(c, ws, res, k, U.p, VT.p);
    scale_cols_kernel<<<std::max(1, std::min(cdiv(static_cast<long>(l) * k, 256), 4 * c.num_sms)), 256, 0,
                        c.stream>>>(U.p, l, k, res.sigma);
    ACHI_LAUNCHED(c);
    nb.reserve(static_cast<size_t>(ll) * d * k);
    matmul_kernel<<<dim3(cdiv(k, 16), cdiv(static_cast<long>(ll) * d, 16)), dim3(16, 16), 0, c.stream>>>(
        s[i - 1].p, U.p, nb.p, ll * d, k, l);
    ACHI_LAUNCHED(c);
    c.sync();
    res.sweeps();  // NumericalFailure if the Jacobi iteration hit its cap
    s[i] = std::move(VT);
    s[i - 1] = std::move(nb);
    dims[i] = k;
  }
}

// host sites -> device (unpadded), canonicalize(psi, 0) on the device
std::vector<DevBuf> canonical_on_device(Ctx& c, const std::vector<std::vector<double>>& hs,
                                        std::vector<int>& dims, int d, int times) {
  std::vector<DevBuf> ds(hs.size());
  for (size_t k = 0; k < hs.size(); ++k) {
    ds[k].reserve(hs[k].size());
    ACHI_CUDA(cudaMemcpyAsync(ds[k].p, hs[k].data(), sizeof(double) * hs[k].size(),
                              cudaMemcpyHostToDevice, c.stream));
  }
  for (int t = 0; t < times; ++t) {
    device_canonicalize_left(c, ds, dims, d);
    if (t + 1 < times) {
      // normalise the centre site between the two canonicalisations (random_mps, mps.cpp:93-95)
      const long n0 = static_cast<long>(dims[0]) * d * dims[1];
      DevBuf nrm;
      DevArr<int> bad;
      nrm.reserve(1);
      int* pb = bad.reserve(1);
      ACHI_CUDA(cudaMemsetAsync(pb, 0, sizeof(int), c.stream));
      device_norm2(c, ds[0].p, n0, nrm.p);
      scale_all_kernel<<<std::max(1, std::min(cdiv(n0, 256), 4 * c.num_sms)), 256, 0, c.stream>>>(
          ds[0].p, n0, nrm.p, pb);
      ACHI_LAUNCHED(c);
      int hb = 0;
      ACHI_CUDA(cudaMemcpyAsync(&hb, pb, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (hb) fail(ACHI_E_NUMERICAL_FAILURE, "random_mps: zero-norm state");
    }
  }
  return ds;
}

namespace {

// random_mps (mps.cpp:75-95) with one real normal draw per entry (host
// generator: the reference's mt19937_64 sequence), canonicalize + normalise,
// then the second canonicalize of run_dmrg (dmrg.cpp:236) -- on the device.
std::vector<std::vector<double>> random_real_sites(int n, int d, int chi, uint64_t seed,
                                                   std::vector<int>& dims_out) {
  if (chi < 1) fail(ACHI_E_INVALID_RANK, "random_mps: chi must be >= 1");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  const auto cd = capped_bond_dims(n, d, chi);
  std::vector<int> dims(n + 1, 1);
  for (int k = 1; k < n; ++k) dims[k] = cd[k - 1];
  std::vector<std::vector<double>> s(n);
  for (int i = 0; i < n; ++i) {
    s[i].resize(static_cast<size_t>(dims[i]) * d * dims[i + 1]);
    for (double& x : s[i]) x = gauss(rng);
  }
  dims_out = dims;
  return s;
}

__global__ void set_boundary_kernel(double* p) { p[0] = 1.0; }

}  // namespace

// Jacobi stop threshold of the chain's SVDs (svd_jacobi.cuh SvdWs::stop_tol): after the
// last sweep the remaining cosines are ~its square, far below what the truncation and the
// energy see (kept ranks, entropies and energies are checked against the oracle in tests)
constexpr double CHAIN_SVD_STOP = 1e-5;

void Chain::create(Ctx& c, const achi_model_spec& s, const achi_dmrg_config& g) {
  ctx = &c;
  spec = s;
  cfg = g;
  validate_spec(s);
  validate_config(g);
  n = s.n;
  mpo = build_mpo_real(s);
  if (g.arithmetic != ACHI_ARITH_REAL && g.arithmetic != ACHI_ARITH_COMPLEX)
    fail(ACHI_E_INVALID_CONFIG, "dmrg: arithmetic must be ACHI_ARITH_REAL or ACHI_ARITH_COMPLEX");
  int init = g.initial_state;
  if (init == ACHI_INIT_AUTOMATIC)  // dmrg.cpp:222-235 (complex: TFIM -> random_mps)
    init = s.family == ACHI_HEISENBERG_XXZ
               ? ACHI_INIT_NEEL
               : (g.arithmetic == ACHI_ARITH_COMPLEX ? ACHI_INIT_RANDOM : ACHI_INIT_RANDOM_REAL);
  if (init != ACHI_INIT_NEEL && init != ACHI_INIT_RANDOM_REAL && init != ACHI_INIT_RANDOM)
    fail(ACHI_E_INVALID_CONFIG, "dmrg: unknown initial state");
  cplx = g.arithmetic == ACHI_ARITH_COMPLEX || init == ACHI_INIT_RANDOM;
  svd.defer_v = !cplx;  // the real visit joins the replay at svd_phase_signs
  // the real truncation needs the kept subspace, not 1e-15 vectors; the complex pairing
  // of svd_complex.cu reads the real vectors themselves, so it keeps the full rotation
  svd.skip_tol = cplx ? 0.0 : 1e-9;
  svd.stop_tol = cplx ? 1e-7 : CHAIN_SVD_STOP;
  const size_t planes = cplx ? 2 : 1;
  // mixing matrices
  std::vector<MixMatrix> all;
  for (int b = 0; b + 1 < n; ++b) all.push_back(mix_heff(mpo[b], mpo[b + 1]));
  for (int k = 0; k < n; ++k) all.push_back(mix_env_left(mpo[k]));
  for (int k = 0; k < n; ++k) all.push_back(mix_env_right(mpo[k]));
  auto dm = mixes.upload(c, all);
  mheff.assign(dm.begin(), dm.begin() + (n - 1));
  mleft.assign(dm.begin() + (n - 1), dm.begin() + (2 * n - 1));
  mright.assign(dm.begin() + (2 * n - 1), dm.end());
  // capacities chi_k <= min(chi_max, d^k, d^(n-k))
  cap.assign(n + 1, 1);
  chi.assign(n + 1, 1);
  for (int k = 1; k < n; ++k) {
    long v = g.controller.chi_max;
    long gl = 1, gr = 1;
    for (int i = 0; i < k && gl < v; ++i) gl *= d;
    for (int i = 0; i < n - k && gr < v; ++i) gr *= d;
    cap[k] = static_cast<int>(std::min({v, gl, gr}));
  }
  site.resize(n);
  L.resize(n);
  R.resize(n);
  vkeep.resize(2 * static_cast<size_t>(n - 1));
  {
    const char* e = std::getenv("ACHI_SVD_WARM");
    warm_svd = !(e && e[0] == '0');
  }
  size_t max_vec = 0, max_ws = 0, max_lhat = 0, max_rhat = 0, max_scr = 0;
  for (int k = 0; k < n; ++k) {
    const size_t cl = pad2i(cap[k]), cr = pad2i(cap[k + 1]);
    site[k].reserve(planes * cl * d * cr);
    L[k].reserve(planes * cl * cl * mpo[k].l);
    R[k].reserve(planes * cr * cr * mpo[k].r);
    max_lhat = std::max(max_lhat, 4 * cl * cl * mpo[k].l);
    max_rhat = std::max(max_rhat, 4 * cr * cr * mpo[k].r);
    // realified operands of the merge / environment updates + a transposed site
    max_scr = std::max(max_scr, std::max({4 * cl * cl * mpo[k].l, 4 * cr * cr * mpo[k].r, 4 * cl * d * cr}) +
                                    2 * cl * d * cr);
    ACHI_CUDA(cudaMemsetAsync(L[k].p, 0, sizeof(double) * L[k].cap, c.stream));
    ACHI_CUDA(cudaMemsetAsync(R[k].p, 0, sizeof(double) * R[k].cap, c.stream));
    if (k + 1 < n) {
      const size_t c2 = pad2i(cap[k + 2]);
      max_vec = std::max(max_vec, cl * d * d * c2);
      max_ws = std::max(max_ws, cl * d * d * c2 * std::max(mpo[k].l, mpo[k + 1].r));
    }
    max_ws = std::max(max_ws, cl * cr * d * std::max(mpo[k].l, mpo[k].r));
  }
  theta.reserve(planes * max_vec);
  vec.reserve(planes * max_vec);
  c.ws_a.reserve(planes * max_ws);
  c.ws_b.reserve(planes * max_ws);
  lz.reserve(static_cast<long>(planes * max_vec));
  if (cplx) {
    lhat.reserve(max_lhat);
    rhat.reserve(max_rhat);
    scr.reserve(max_scr);
    cth.reserve(2 * max_vec);
    cu.reserve(2 * max_vec);
    cv.reserve(2 * max_vec);
    csig.reserve(max_vec);
  }
  states.reserve(n);
  trace.reserve(2 * (n - 1));
  visits.reserve(2 * (n - 1));
  bout.reserve(1);
  bout_h.reserve(1);
  vh.assign(2 * (n - 1), VisitHost{0, 0, 0});
  // boundary environments (dmrg.cpp:18-24)
  set_boundary_kernel<<<1, 1, 0, c.stream>>>(L[0].p);
  ACHI_LAUNCHED(c);
  set_boundary_kernel<<<1, 1, 0, c.stream>>>(R[n - 1].p);
  ACHI_LAUNCHED(c);
  // initial state + canonicalize, environments, controller cold start (dmrg.cpp:222-250)
  if (init == ACHI_INIT_NEEL) {
    auto hs = neel_canonical(n, d);
    if (cplx) {  // real values, zero imaginary parts
      for (auto& v : hs) {
        std::vector<double> z(2 * v.size(), 0.0);
        for (size_t t = 0; t < v.size(); ++t) z[2 * t] = v[t];
        v.swap(z);
      }
      upload_sites_c(hs);
    } else {
      upload_sites(hs);
    }
  } else if (init == ACHI_INIT_RANDOM) {
    std::vector<int> dims;
    auto hs = random_complex_sites(n, d, g.controller.chi_min, g.seed, dims);
    auto ds = canonical_on_device_c(c, hs, dims, d, 2);
    for (int k = 1; k < n; ++k) chi[k] = dims[k];
    copy_sites_device_c(ds);
  } else if (cplx) {  // the real random start in complex storage
    std::vector<int> dims;
    auto hs = random_real_sites(n, d, g.controller.chi_min, g.seed, dims);
    for (auto& v : hs) {
      std::vector<double> z(2 * v.size(), 0.0);
      for (size_t t = 0; t < v.size(); ++t) z[2 * t] = v[t];
      v.swap(z);
    }
    auto ds = canonical_on_device_c(c, hs, dims, d, 2);
    for (int k = 1; k < n; ++k) chi[k] = dims[k];
    copy_sites_device_c(ds);
  } else {
    std::vector<int> dims;
    auto hs = random_real_sites(n, d, g.controller.chi_min, g.seed, dims);
    auto ds = canonical_on_device(c, hs, dims, d, 2);
    for (int k = 1; k < n; ++k) chi[k] = dims[k];
    copy_sites_device(ds);
  }
  std::vector<achi_bond_state> st(n - 1);
  for (auto& b : st) {
    b = achi_bond_state{};
    b.chi = g.controller.chi_min;
    b.ema = 0.0;
    b.initialized = 1;
    b.history[0] = 0.0;
    b.history_len = 1;
  }
  ACHI_CUDA(cudaMemcpyAsync(states.p, st.data(), sizeof(achi_bond_state) * (n - 1),
                            cudaMemcpyHostToDevice, c.stream));
  rebuild_envs();
  c.sync();
}

void Chain::upload_sites(const std::vector<std::vector<double>>& hs) {
  for (int k = 0; k < n; ++k) {
    const int l = chi[k], r = chi[k + 1];
    if (static_cast<long>(hs[k].size()) != static_cast<long>(l) * d * r)
      fail(ACHI_E_INTERNAL, "upload_sites: size mismatch");
    upload_padded3(*ctx, hs[k].data(), l, d, r, site[k].p);
  }
  ctx->sync();
}

// unpadded device sites (l, d, r) -> the chain's padded storage
void Chain::copy_sites_device(const std::vector<DevBuf>& ds) {
  for (int k = 0; k < n; ++k) {
    const int l = chi[k], r = chi[k + 1], lp = pad2i(l), rp = pad2i(r);
    ACHI_CUDA(cudaMemsetAsync(site[k].p, 0, sizeof(double) * lp * d * rp, ctx->stream));
    ACHI_CUDA(cudaMemcpy2DAsync(site[k].p, sizeof(double) * rp, ds[k].p, sizeof(double) * r,
                                sizeof(double) * r, static_cast<size_t>(l) * d, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  }
  ctx->sync();
}

// expectation_energy (dmrg.cpp:284-298): left environments from the boundary
// through every site into two scratch buffers; L_n (1 x 1 x 1, stored padded)
// is <psi|H|psi>.  Independent of the cached environments.
double Chain::expectation_energy() {
  Ctx& c = *ctx;
  size_t mx = 1;
  for (int k = 0; k <= n; ++k) {
    const size_t cp = pad2i(chi[k]);
    const int D = k < n ? mpo[k].l : 1;
    mx = std::max(mx, cp * cp * static_cast<size_t>(D));
  }
  if (cplx) mx *= 2;
  DevBuf e[2];
  for (auto& b : e) {
    b.reserve(mx);
    ACHI_CUDA(cudaMemsetAsync(b.p, 0, sizeof(double) * mx, c.stream));
  }
  set_boundary_kernel<<<1, 1, 0, c.stream>>>(e[0].p);
  ACHI_LAUNCHED(c);
  int cur = 0;
  for (int k = 0; k < n; ++k) {
    ACHI_CUDA(cudaMemsetAsync(e[cur ^ 1].p, 0, sizeof(double) * mx, c.stream));
    if (cplx)  // planar: the real part of L_n is plane 0
      env_left_c(c, e[cur].p, site[k].p, pad2i(chi[k]), pad2i(chi[k + 1]), d, mpo[k].l, mpo[k].r,
                 mleft[k], scr.p, e[cur ^ 1].p);
    else
      env_left(c, e[cur].p, site[k].p, pad2i(chi[k]), pad2i(chi[k + 1]), d, mpo[k].l, mpo[k].r,
               mleft[k], e[cur ^ 1].p);
    cur ^= 1;
  }
  double h = 0.0;
  ACHI_CUDA(cudaMemcpyAsync(&h, e[cur].p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return h;
}

void Chain::rebuild_envs() {  // Environment::rebuild(psi, mpo, 0), dmrg.cpp:51-56
  for (int k = n - 2; k >= 0; --k) {
    if (cplx)
      env_right_c(*ctx, R[k + 1].p, site[k + 1].p, pad2i(chi[k + 2]), pad2i(chi[k + 1]), d,
                  mpo[k + 1].l, mpo[k + 1].r, mright[k + 1], scr.p, R[k].p);
    else
      env_right(*ctx, R[k + 1].p, site[k + 1].p, pad2i(chi[k + 2]), pad2i(chi[k + 1]), d,
                mpo[k + 1].l, mpo[k + 1].r, mright[k + 1], R[k].p);
  }
}

// visit_bond (dmrg.cpp:84-171)
void Chain::visit(int b, bool right, int sweep_index, int slot) {
  Ctx& c = *ctx;
  EventAccPause untimed(c.acc, c.acc.enabled && !c.acc.visit_timed());
  if (cplx) {
    visit_complex(b, right, sweep_index, slot);
    return;
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int chl = chi[b], chm = chi[b + 1], chr = chi[b + 2];
  const int chlp = pad2i(chl), chmp = pad2i(chm), chrp = pad2i(chr);
  const long nvec = static_cast<long>(chlp) * d * d * chrp;
  const long dim = static_cast<long>(chl) * d * d * chr;
  theta_merge(c, site[b].p, site[b + 1].p, chlp, chmp, chrp, d, theta.p);
  HeffOps op{L[b].p, R[b + 1].p, chlp, chrp, d, mpo[b].l, mpo[b + 1].r, mheff[b]};
  // algorithmic FP64 flops of one matvec: 2 D d^2 chl chr (chl+chr) + 4 D^2 d^3 chl chr
  const double D = mpo[b].r;
  const double mv_flops = 2.0 * D * d * d * chl * chr * (chl + chr) + 4.0 * D * D * d * d * d * chl * chr;
  // The inner Lanczos loop is a cached CUDA graph per (bond, direction); its key
  // covers everything the captured matvec depends on (shapes and buffers).
  uint64_t key = 1469598103934665603ull;
  for (uint64_t v : {static_cast<uint64_t>(b), static_cast<uint64_t>(chlp), static_cast<uint64_t>(chrp),
                     reinterpret_cast<uint64_t>(L[b].p), reinterpret_cast<uint64_t>(R[b + 1].p),
                     reinterpret_cast<uint64_t>(c.ws_a.p), reinterpret_cast<uint64_t>(c.ws_b.p),
                     reinterpret_cast<uint64_t>(c.ws_split.p)})
    key = (key ^ v) * 1099511628211ull;
  c.acc.begin(EventAcc::kMatvec, c.stream);  // the whole eigensolve (matvecs + orthogonalisation)
  // graph mode: enqueued without a host wait; read back with the bond selection below
  eigs_lowest_async(
      c, lz,
      [&](const double* in, double* out) {
        c.acc.begin(EventAcc::kHeff, c.stream);  // skipped while the Lanczos graph is captured
        heff_apply(c, op, in, out);
        c.acc.end(c.stream, mv_flops);
      },
      nvec, dim, theta.p,
      cfg.eig_tol, cfg.eig_max_iter, vec.p, 2 * b + (right ? 1 : 0), key, &op);
  c.acc.end(c.stream, 0.0);  // flops added once the matvec count is known
  if (profile) c.sync();
  const auto t1 = clk::now();
  const SvdSide side = right ? SvdSide::kRows : SvdSide::kCols;
  c.acc.begin(EventAcc::kSvd, c.stream);
  const int sm_ = chlp * d, sn_ = d * chrp, smt = chl * d, snt = d * chr;
  VKeep& vk = vkeep[2 * static_cast<size_t>(b) + (right ? 1 : 0)];
  const bool warm = warm_svd && vk.valid && vk.m == sm_ && vk.n == sn_ && vk.mt == smt && vk.nt == snt;
  static const char* dump_path = std::getenv("ACHI_SVD_DUMP");  // debug: input of a failing SVD
  static const int dump_at = [] {  // study: ACHI_SVD_DUMP_AT=sweep*100000+bond*2+right dumps that visit
    const char* e = std::getenv("ACHI_SVD_DUMP_AT");
    return e ? std::atoi(e) : -1;
  }();
  const bool dump_now = dump_path && dump_at == sweep_index * 100000 + 2 * b + (right ? 1 : 0);
  std::vector<double> dump;
  if (dump_path) {
    dump.resize(static_cast<size_t>(sm_) * sn_);
    ACHI_CUDA(cudaMemcpyAsync(dump.data(), vec.p, sizeof(double) * dump.size(),
                              cudaMemcpyDeviceToHost, c.stream));
  }
  SvdResultDev sr = svd_device(c, svd, vec.p, sm_, sn_, smt, snt, side, 1, 0, nullptr, true,
                               warm ? vk.v.p : nullptr);
  c.acc.end(c.stream, 0.0);
  // the fused bond selection is queued behind the SVD; one host sync serves both
  bond_select(c, sr.sigma, sr.r_true, cfg, states.p, b, sweep_index, right ? 1 : 0,
              trace.p + slot, visits.p + slot, bout.p, bout_h.p);
  c.sync();  // the one host wait of the visit: eigensolve outcome, SVD sweeps, kept rank
  const EigsOut eig = eigs_finish(c, lz);  // throws EigenNonConvergence / InvalidMatrix
  if (c.acc.enabled) c.acc.work[EventAcc::kMatvec] += eig.matvecs * mv_flops;
  auto write_dump = [&] {
    if (FILE* f = std::fopen(dump_path, "wb")) {
      const int32_t hdr[6] = {sm_, sn_, smt, snt, right ? 1 : 0, warm ? 1 : 0};
      std::fwrite(hdr, sizeof(hdr), 1, f);
      std::fwrite(dump.data(), sizeof(double), dump.size(), f);
      std::fclose(f);
    }
  };
  int svd_sweeps = 0;
  try {
    svd_sweeps = sr.sweeps();
  } catch (const Error&) {
    if (dump_path) write_dump();
    throw;
  }
  if (dump_now) write_dump();
  // algorithmic FP64 flops of the blocked Jacobi: per sweep
  // C(ng/16, 2) block pairs x 2 * 32^2 * (2 mg + ng) (Gram + rotation of G,
  // rotation of V) ~= 4 ng^2 (2 mg + ng)
  if (c.acc.enabled)
    c.acc.work[EventAcc::kSvd] += 4.0 * svd_sweeps * static_cast<double>(sr.ng) * sr.ng *
                                  (2.0 * sr.mg + sr.ng);
  const auto t2 = clk::now();
  static const int visit_log = [] {  // 1: slow visits only, 2: every visit
    const char* e = std::getenv("ACHI_VISIT_LOG");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  if (visit_log) {
    const double svd_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    const double lz_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (visit_log >= 2 || svd_ms > 5.0 || lz_ms > 20.0)
      std::fprintf(stderr, "[visit] sweep %d bond %d %s chl %d chr %d lanczos %.2f ms svd %.2f ms "
                   "(%d Jacobi sweeps, warm %d)\n", sweep_index, b, right ? "R" : "L", chl, chr,
                   lz_ms, svd_ms, svd_sweeps, warm ? 1 : 0);
  }
  const BondOut bo = *bout_h.p;
  const auto t3 = clk::now();
  if (bo.err == ACHI_E_DEGENERATE_SPECTRUM) fail(bo.err, "dmrg: zero two-site block");
  if (bo.err) fail(bo.err, "controller_update: invalid controller state or config");
  const int kept = bo.kept;
  if (!(bo.lam_norm > 0)) fail(ACHI_E_DEGENERATE_SPECTRUM, "dmrg: empty truncation");
  svd_phase_signs(c, svd, sr, kept);  // (joins the V replay, which ran beside the bond selection)
  if (warm_svd) {  // keep this factor for the next visit of the bond in this direction
    const size_t nv = static_cast<size_t>(sr.ng) * sr.ng;
    vk.v.reserve(nv);
    ACHI_CUDA(cudaMemcpyAsync(vk.v.p, sr.V, sizeof(double) * nv, cudaMemcpyDeviceToDevice, c.stream));
    vk.m = sm_;
    vk.n = sn_;
    vk.mt = smt;
    vk.nt = snt;
    vk.valid = true;
  }
  absorb(c, sr, svd.sign.p, kept, bout.p, chl, chr, d, right, site[b].p, site[b + 1].p);
  chi[b + 1] = kept;
  const int kp = pad2i(kept);
  {
    const double De = right ? mpo[b].r : mpo[b + 1].l, ch0 = right ? chl : chr;
    c.acc.begin(EventAcc::kEnv, c.stream);
    if (right)
      env_left(c, L[b].p, site[b].p, chlp, kp, d, mpo[b].l, mpo[b].r, mleft[b], L[b + 1].p);
    else
      env_right(c, R[b + 1].p, site[b + 1].p, chrp, kp, d, mpo[b + 1].l, mpo[b + 1].r,
                mright[b + 1], R[b].p);
    c.acc.end(c.stream, 2.0 * De * d * ch0 * kept * (ch0 + kept) + 2.0 * De * De * d * d * ch0 * kept);
  }
  vh[slot] = VisitHost{eig.eigenvalue, eig.residual, eig.matvecs};
  if (profile) c.sync();
  const auto t4 = clk::now();
  auto sec = [](auto a, auto z) { return std::chrono::duration<double>(z - a).count(); };
  stats.merge_lanczos += sec(t0, t1);
  stats.svd += sec(t1, t2);
  stats.select += sec(t2, t3);
  stats.absorb_env += sec(t3, t4);
  stats.matvecs += eig.matvecs;
  stats.svd_sweeps += svd_sweeps;
  stats.visits += 1;
}

// two_site_sweep (dmrg.cpp:175-214)
void Chain::sweep(int sweep_index, achi_sweep_record* rec, int32_t* chi_profile, double* entropy,
                  achi_trace_row* trace_out, achi_visit_record* visits_out) {
  Ctx& c = *ctx;
  c.sync();
  auto t0 = std::chrono::steady_clock::now();
  int slot = 0;
  for (int b = 0; b <= n - 2; ++b) visit(b, true, sweep_index, slot++);
  for (int b = n - 2; b >= 0; --b) visit(b, false, sweep_index, slot++);
  c.sync();
  c.acc.resolve();
  auto t1 = std::chrono::steady_clock::now();
  const int nv = 2 * (n - 1);
  std::vector<achi_visit_record> vr(nv);
  ACHI_CUDA(cudaMemcpyAsync(vr.data(), visits.p, sizeof(achi_visit_record) * nv,
                            cudaMemcpyDeviceToHost, c.stream));
  if (trace_out)
    ACHI_CUDA(cudaMemcpyAsync(trace_out, trace.p, sizeof(achi_trace_row) * nv,
                              cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  achi_sweep_record r{};
  r.sweep_index = sweep_index;
  std::vector<double> ent(n - 1, 0.0);
  for (int i = 0; i < nv; ++i) {
    vr[i].energy = vh[i].energy;
    vr[i].matvecs = vh[i].matvecs;
    vr[i].lanczos_residual = vh[i].residual;
    r.max_chi_used = std::max(r.max_chi_used, vr[i].kept);
    r.max_trunc_error = std::max(r.max_trunc_error, vr[i].trunc_error);
    ent[vr[i].bond] = vr[i].entropy;
  }
  r.energy = vh[nv - 1].energy;
  r.wall_time = std::chrono::duration<double>(t1 - t0).count();
  long pc = 0;
  double avg = 0;
  for (int k = 0; k < n; ++k) pc += static_cast<long>(chi[k]) * d * chi[k + 1];
  for (int k = 1; k < n; ++k) avg += chi[k];
  r.parameter_count = pc;
  r.average_chi = avg / static_cast<double>(n - 1);
  if (rec) *rec = r;
  if (chi_profile)
    for (int k = 1; k < n; ++k) chi_profile[k - 1] = chi[k];
  if (entropy)
    for (int k = 0; k < n - 1; ++k) entropy[k] = ent[k];
  if (visits_out)
    for (int i = 0; i < nv; ++i) visits_out[i] = vr[i];
}

}  // namespace achi
