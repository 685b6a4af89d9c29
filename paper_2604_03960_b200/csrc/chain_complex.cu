// complex128 chain (achi_dmrg_config.arithmetic = ACHI_ARITH_COMPLEX, or the
// complex random_mps start): the reference's own arithmetic (tensor.hpp:14-21,
// DenseMatrix = MatrixXcd) for states that are not real in any gauge.
//
// Storage: every site, environment and two-site tensor is planar -- two planes
// [Re; Im] of the real padded layout -- so the contractions are the real DMMA
// GEMMs of contract.cu with doubled M and K (contract.cuh, "complex128").  The
// eigensolve is the real restarted Lanczos on the realified vector [Re; Im]:
// for a Hermitian H_eff the complex Lanczos recurrence has real alpha/beta, so
// its Krylov vectors are those of the real iteration on [Re; Im] (the same
// eigenvalue, eigenvector and matvec count up to rounding; linalg.cpp:107-178).
// The truncated SVD is the complex svd_full of svd_complex.cu (fix_phases
// included); bond selection and the controller read only sigma and are shared
// with the real path.
#include <algorithm>
#include <chrono>
#include <random>

#include "chain.cuh"

namespace achi {

std::vector<int> capped_bond_dims(int n, int d, int chi);  // chain.cu

namespace {

// C (M x N) = A (M x K) . B (K x N), interleaved complex, row-major
__global__ void cmatmul_kernel(const double2* __restrict__ A, const double2* __restrict__ B,
                               double2* __restrict__ C, int M, int N, int K) {
  __shared__ double2 as[16][17], bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double2 acc = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < K; k0 += 16) {
    as[ty][tx] = (row < M && k0 + tx < K) ? A[static_cast<long>(row) * K + k0 + tx] : make_double2(0.0, 0.0);
    bs[ty][tx] = (k0 + ty < K && col < N) ? B[static_cast<long>(k0 + ty) * N + col] : make_double2(0.0, 0.0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 a = as[ty][k], b = bs[k][tx];
      acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
      acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
    }
    __syncthreads();
  }
  if (row < M && col < N) C[static_cast<long>(row) * N + col] = acc;
}

// U (rows x k interleaved): column q *= sigma[q]
__global__ void scale_cols_c_kernel(double2* U, long rows, int k, const double* __restrict__ sigma) {
  const long tot = rows * k;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const double s = sigma[t % k];
    U[t].x *= s;
    U[t].y *= s;
  }
}

// interleaved (l, m, r) -> planar padded (lp, m, rp), zero pads
__global__ void c2planar3_kernel(const double2* __restrict__ src, int l, int m, int r, int lp, int rp,
                                 double* __restrict__ dst) {
  const long plane = static_cast<long>(lp) * m * rp;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < plane;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const long row = t / rp;
    const int j = static_cast<int>(t - row * rp);
    const long i = row / m;
    double re = 0.0, im = 0.0;
    if (i < l && j < r) {
      const double2 v = src[row * r + j];
      re = v.x;
      im = v.y;
    }
    dst[t] = re;
    dst[plane + t] = im;
  }
}

// planar padded (lp, m, rp) -> interleaved (l, m, r)
__global__ void planar2c3_kernel(const double* __restrict__ src, int l, int m, int r, int lp, int rp,
                                 double2* __restrict__ dst) {
  const long plane = static_cast<long>(lp) * m * rp;
  const long tot = static_cast<long>(l) * m * r;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const long row = t / r;
    const int j = static_cast<int>(t - row * r);
    const long o = row * rp + j;
    dst[t] = make_double2(src[o], src[plane + o]);
  }
}

// truncate / normalise / absorb (dmrg.cpp:144-158) from the complex SVD
// factors U (m x rk) and V^dagger (rk x n), m = chl d, n = d chr: site b
// (chlp, d, keptp) and site b+1 (keptp, d, chrp) as planes; lambda / ||lambda||
// goes into site b+1 when moving right, into site b otherwise.
struct AbsorbC {
  const double2* U;
  const double2* Vd;
  const double* sigma;
  const BondOut* bo;
  int rk, n, kept, keptp, chl, chlp, chr, chrp, d, right;
  double* site_b;
  double* site_b1;
};

__global__ void absorb_c_kernel(AbsorbC a) {
  const long n_b = static_cast<long>(a.chlp) * a.d * a.keptp;
  const long n_b1 = static_cast<long>(a.keptp) * a.d * a.chrp;
  const double inv_lam = 1.0 / a.bo->lam_norm;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n_b + n_b1;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (t < n_b) {
      const long row = t / a.keptp;
      const int k = static_cast<int>(t - row * a.keptp);
      if (k < a.kept && row < static_cast<long>(a.chl) * a.d) {
        v = a.U[row * a.rk + k];
        if (!a.right) {
          const double s = a.sigma[k] * inv_lam;
          v.x *= s;
          v.y *= s;
        }
      }
      a.site_b[t] = v.x;
      a.site_b[n_b + t] = v.y;
    } else {
      const long u = t - n_b;
      const int k = static_cast<int>(u / (static_cast<long>(a.d) * a.chrp));
      const long c = u - static_cast<long>(k) * a.d * a.chrp;
      const int s2 = static_cast<int>(c / a.chrp), jr = static_cast<int>(c % a.chrp);
      if (k < a.kept && jr < a.chr) {
        v = a.Vd[static_cast<long>(k) * a.n + s2 * a.chr + jr];
        if (a.right) {
          const double s = a.sigma[k] * inv_lam;
          v.x *= s;
          v.y *= s;
        }
      }
      a.site_b1[u] = v.x;
      a.site_b1[n_b1 + u] = v.y;
    }
  }
}

__global__ void scale_all_c_kernel(double* x, long n, const double* nrm2, int* bad) {
  const double s = *nrm2;
  if (!(s > 0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *bad = 1;
    return;
  }
  const double inv = 1.0 / sqrt(s);
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long>(gridDim.x) * blockDim.x)
    x[t] *= inv;
}

int grid_for(const Ctx& c, long tot) {
  return static_cast<int>(std::max<long>(1, std::min<long>(cdiv(tot, 256), 8L * c.num_sms)));
}

void to_planar3(Ctx& c, const double* src, int l, int m, int r, double* dst) {
  const int lp = pad2i(l), rp = pad2i(r);
  c2planar3_kernel<<<grid_for(c, static_cast<long>(lp) * m * rp), 256, 0, c.stream>>>(
      reinterpret_cast<const double2*>(src), l, m, r, lp, rp, dst);
  ACHI_LAUNCHED(c);
}

void from_planar3(Ctx& c, const double* src, int l, int m, int r, double* dst) {
  planar2c3_kernel<<<grid_for(c, static_cast<long>(l) * m * r), 256, 0, c.stream>>>(
      src, l, m, r, pad2i(l), pad2i(r), reinterpret_cast<double2*>(dst));
  ACHI_LAUNCHED(c);
}

// push_left on sites n-1..1 (mps.cpp:186-210) with the complex SVD in place
// of Householder QR: site i as M (l x d r) = (U S) V^dagger; site i <- V^dagger,
// site i-1 <- site i-1 (U S).  Same bond dimensions min(l, d r), same state,
// another gauge of each bond (a unitary), which the sweep is covariant under.
void device_canonicalize_left_c(Ctx& c, std::vector<DevBuf>& s, std::vector<int>& dims, int d) {
  const int n = static_cast<int>(s.size());
  SvdWs ws;
  for (int i = n - 1; i >= 1; --i) {
    const int l = dims[i], r = dims[i + 1], cols = d * r, k = std::min(l, cols), ll = dims[i - 1];
    DevBuf U, VD, sig, nb;
    U.reserve(2 * static_cast<size_t>(l) * k);
    VD.reserve(2 * static_cast<size_t>(k) * cols);
    sig.reserve(k);
    svd_complex_device(c, ws, s[i].p, l, cols, sig.p, U.p, VD.p, 1);  // V^dagger orthonormal
    scale_cols_c_kernel<<<grid_for(c, static_cast<long>(l) * k), 256, 0, c.stream>>>(
        reinterpret_cast<double2*>(U.p), l, k, sig.p);
    ACHI_LAUNCHED(c);
    nb.reserve(2 * static_cast<size_t>(ll) * d * k);
    cmatmul_kernel<<<dim3(cdiv(k, 16), cdiv(static_cast<long>(ll) * d, 16)), dim3(16, 16), 0, c.stream>>>(
        reinterpret_cast<const double2*>(s[i - 1].p), reinterpret_cast<const double2*>(U.p),
        reinterpret_cast<double2*>(nb.p), ll * d, k, l);
    ACHI_LAUNCHED(c);
    c.sync();
    s[i] = std::move(VD);
    s[i - 1] = std::move(nb);
    dims[i] = k;
  }
}

}  // namespace

std::vector<std::vector<double>> random_complex_sites(int n, int d, int chi, uint64_t seed,
                                                      std::vector<int>& dims_out) {
  if (chi < 1) fail(ACHI_E_INVALID_RANK, "random_mps: chi must be >= 1");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  const auto cd = capped_bond_dims(n, d, chi);
  std::vector<int> dims(n + 1, 1);
  for (int k = 1; k < n; ++k) dims[k] = cd[k - 1];
  std::vector<std::vector<double>> s(n);
  for (int i = 0; i < n; ++i) {
    s[i].resize(2 * static_cast<size_t>(dims[i]) * d * dims[i + 1]);
    for (size_t t = 0; t < s[i].size(); t += 2) {
      // Cplx(gauss(rng), gauss(rng)) (mps.cpp:86): the constructor arguments are
      // evaluated right to left by g++ (the reference's toolchain), so the
      // imaginary part is the first draw of each pair
      const double im = gauss(rng);
      const double re = gauss(rng);
      s[i][t] = re;
      s[i][t + 1] = im;
    }
  }
  dims_out = dims;
  return s;
}

std::vector<DevBuf> canonical_on_device_c(Ctx& c, const std::vector<std::vector<double>>& hs,
                                          std::vector<int>& dims, int d, int times) {
  std::vector<DevBuf> ds(hs.size());
  for (size_t k = 0; k < hs.size(); ++k) {
    ds[k].reserve(hs[k].size());
    ACHI_CUDA(cudaMemcpyAsync(ds[k].p, hs[k].data(), sizeof(double) * hs[k].size(),
                              cudaMemcpyHostToDevice, c.stream));
  }
  for (int t = 0; t < times; ++t) {
    device_canonicalize_left_c(c, ds, dims, d);
    if (t + 1 < times) {  // normalise the centre site (random_mps, mps.cpp:90-94)
      const long n0 = 2L * dims[0] * d * dims[1];
      DevBuf nrm;
      DevArr<int> bad;
      nrm.reserve(1);
      int* pb = bad.reserve(1);
      ACHI_CUDA(cudaMemsetAsync(pb, 0, sizeof(int), c.stream));
      device_norm2(c, ds[0].p, n0, nrm.p);
      scale_all_c_kernel<<<grid_for(c, n0), 256, 0, c.stream>>>(ds[0].p, n0, nrm.p, pb);
      ACHI_LAUNCHED(c);
      int hb = 0;
      ACHI_CUDA(cudaMemcpyAsync(&hb, pb, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (hb) fail(ACHI_E_NUMERICAL_FAILURE, "random_mps: zero-norm state");
    }
  }
  return ds;
}

void Chain::upload_sites_c(const std::vector<std::vector<double>>& hs) {
  for (int k = 0; k < n; ++k) {
    const int l = chi[k], r = chi[k + 1];
    if (static_cast<long>(hs[k].size()) != 2L * l * d * r) fail(ACHI_E_INTERNAL, "upload_sites: size mismatch");
    DevBuf t;
    t.reserve(hs[k].size());
    ACHI_CUDA(cudaMemcpyAsync(t.p, hs[k].data(), sizeof(double) * hs[k].size(), cudaMemcpyHostToDevice,
                              ctx->stream));
    to_planar3(*ctx, t.p, l, d, r, site[k].p);
    ctx->sync();
  }
}

void Chain::copy_sites_device_c(const std::vector<DevBuf>& ds) {
  for (int k = 0; k < n; ++k) to_planar3(*ctx, ds[k].p, chi[k], d, chi[k + 1], site[k].p);
  ctx->sync();
}

void Chain::download_site_c(int k, double* out) {
  const int l = chi[k], r = chi[k + 1];
  DevBuf t;
  t.reserve(2 * static_cast<size_t>(l) * d * r);
  from_planar3(*ctx, site[k].p, l, d, r, t.p);
  ACHI_CUDA(cudaMemcpyAsync(out, t.p, sizeof(double) * 2 * l * d * r, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
}

// visit_bond (dmrg.cpp:84-171) in complex128
void Chain::visit_complex(int b, bool right, int sweep_index, int slot) {
  Ctx& c = *ctx;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int chl = chi[b], chm = chi[b + 1], chr = chi[b + 2];
  const int chlp = pad2i(chl), chmp = pad2i(chm), chrp = pad2i(chr);
  const long nvec = static_cast<long>(chlp) * d * d * chrp;  // one plane
  const long dim = static_cast<long>(chl) * d * d * chr;     // complex dimension
  theta_merge_c(c, site[b].p, site[b + 1].p, chlp, chmp, chrp, d, scr.p, theta.p);
  heff_prepare_c(c, L[b].p, chlp, mpo[b].l, R[b + 1].p, chrp, mpo[b + 1].r, lhat.p, rhat.p);
  HeffOpsC op{lhat.p, rhat.p, chlp, chrp, d, mpo[b].l, mpo[b + 1].r, mheff[b]};
  const double D = mpo[b].r;
  const double mv_flops =
      4.0 * (2.0 * D * d * d * chl * chr * (chl + chr)) + 2.0 * (2.0 * D * D * d * d * d * chl * chr);
  uint64_t key = 0x9e3779b97f4a7c15ull;
  for (uint64_t v : {static_cast<uint64_t>(b), static_cast<uint64_t>(chlp), static_cast<uint64_t>(chrp),
                     reinterpret_cast<uint64_t>(lhat.p), reinterpret_cast<uint64_t>(rhat.p),
                     reinterpret_cast<uint64_t>(c.ws_a.p), reinterpret_cast<uint64_t>(c.ws_b.p),
                     reinterpret_cast<uint64_t>(c.ws_split.p)})
    key = (key ^ v) * 1099511628211ull;
  c.acc.begin(EventAcc::kMatvec, c.stream);
  eigs_lowest_async(
      c, lz,
      [&](const double* in, double* out) {
        c.acc.begin(EventAcc::kHeff, c.stream);
        heff_apply_c(c, op, in, out);
        c.acc.end(c.stream, mv_flops);
      },
      2 * nvec, dim, theta.p, cfg.eig_tol, cfg.eig_max_iter, vec.p, 2 * b + (right ? 1 : 0), key, nullptr);
  c.acc.end(c.stream, 0.0);
  const auto t1 = clk::now();
  // svd_full of theta as (chl d) x (d chr) (dmrg.cpp:117)
  const int m = chl * d, nn = d * chr, rk = std::min(m, nn);
  c.acc.begin(EventAcc::kSvd, c.stream);
  from_planar3(c, vec.p, chl, d * d, chr, cth.p);
  // the factor that stays canonical is the orthonormal one (U moving right, V^dagger left);
  // warm start from the previous decomposition of this bond and direction (as the real path)
  const SvdSide side = right ? SvdSide::kRows : SvdSide::kCols;
  const int ngw = svd_working_cols(2 * m, 2 * nn, side);
  VKeep& vk = vkeep[2 * static_cast<size_t>(b) + (right ? 1 : 0)];
  const bool warm = warm_svd && vk.valid && vk.m == 2 * m && vk.n == 2 * nn;
  cv_keep.reserve(static_cast<size_t>(ngw) * ngw);
  const int svd_sweeps = svd_complex_stage1(c, svd, cplan, cth.p, m, nn, csig.p, right ? 0 : 1,
                                            warm ? vk.v.p : nullptr, warm_svd ? cv_keep.p : nullptr);
  if (warm_svd) {  // the buffers rotate: this bond keeps the new factor
    std::swap(vk.v, cv_keep);
    vk.m = 2 * m;
    vk.n = 2 * nn;
    vk.valid = true;
  }
  c.acc.end(c.stream, 0.0);
  bond_select(c, csig.p, rk, cfg, states.p, b, sweep_index, right ? 1 : 0, trace.p + slot,
              visits.p + slot, bout.p, bout_h.p);
  c.sync();
  const EigsOut eig = eigs_finish(c, lz);
  if (c.acc.enabled) c.acc.work[EventAcc::kMatvec] += eig.matvecs * mv_flops;
  const auto t2 = clk::now();
  const BondOut bo = *bout_h.p;
  if (bo.err == ACHI_E_DEGENERATE_SPECTRUM) fail(bo.err, "dmrg: zero two-site block");
  if (bo.err) fail(bo.err, "controller_update: invalid controller state or config");
  const int kept = bo.kept;
  if (!(bo.lam_norm > 0)) fail(ACHI_E_DEGENERATE_SPECTRUM, "dmrg: empty truncation");
  const int kp = pad2i(kept);
  svd_complex_stage2(c, cplan, kept, cu.p, cv.p);  // the kept vectors only
  {
    AbsorbC a{reinterpret_cast<const double2*>(cu.p), reinterpret_cast<const double2*>(cv.p), csig.p,
              bout.p, rk, nn, kept, kp, chl, chlp, chr, chrp, d, right ? 1 : 0, site[b].p, site[b + 1].p};
    const long tot = static_cast<long>(chlp) * d * kp + static_cast<long>(kp) * d * chrp;
    absorb_c_kernel<<<grid_for(c, tot), 256, 0, c.stream>>>(a);
    ACHI_LAUNCHED(c);
  }
  chi[b + 1] = kept;
  {
    const double De = right ? mpo[b].r : mpo[b + 1].l, ch0 = right ? chl : chr;
    c.acc.begin(EventAcc::kEnv, c.stream);
    if (right)
      env_left_c(c, L[b].p, site[b].p, chlp, kp, d, mpo[b].l, mpo[b].r, mleft[b], scr.p, L[b + 1].p);
    else
      env_right_c(c, R[b + 1].p, site[b + 1].p, chrp, kp, d, mpo[b + 1].l, mpo[b + 1].r, mright[b + 1],
                  scr.p, R[b].p);
    c.acc.end(c.stream, 4.0 * (2.0 * De * d * ch0 * kept * (ch0 + kept)) + 4.0 * De * De * d * d * ch0 * kept);
  }
  vh[slot] = VisitHost{eig.eigenvalue, eig.residual, eig.matvecs};
  if (profile) c.sync();
  const auto t3 = clk::now();
  auto sec = [](auto a, auto z) { return std::chrono::duration<double>(z - a).count(); };
  stats.merge_lanczos += sec(t0, t1);
  stats.svd += sec(t1, t2);
  stats.absorb_env += sec(t2, t3);
  stats.matvecs += eig.matvecs;
  stats.svd_sweeps += svd_sweeps;
  stats.visits += 1;
}

}  // namespace achi
