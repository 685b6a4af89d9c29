// Reference-style tests of the C++ host mirror (paper_2604_03960_b200/host/
// adaptchi_b200.hpp) on the GPU.  Cases restate the reference's own tests
// (tests/test_linalg.cpp, test_mps.cpp, test_controller.cpp, test_dmrg.cpp in
// /root/reference/proj) against the same API names; the exact-diagonalisation
// energies come from argv (computed by the oracle in tests/test_host_mirror.py).
//
// Build: g++ -std=c++17 -O2 test_host_mirror.cpp -L<_build> -ladaptchi_b200
// Usage: test_host_mirror E_heis8_pauli E_tfim8_h1
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <random>

#include "../../paper_2604_03960_b200/host/adaptchi_b200.hpp"

using namespace adaptchi;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                             \
  do {                                                                       \
    ++g_checks;                                                              \
    bool ok = false;                                                         \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const T&) {                                                     \
      ok = true;                                                             \
    } catch (...) {                                                          \
    }                                                                        \
    if (!ok) {                                                               \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                        \
  } while (0)

static bool approx(double a, double b, double eps) {
  return std::abs(a - b) <= eps * std::max(1.0, std::max(std::abs(a), std::abs(b)));
}
static mps::SingularSpectrum spec_of(std::initializer_list<double> v) {
  return {RVector(v), 0};
}
static DenseMatrix random_real(long r, long c, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  DenseMatrix m(r, c);
  for (auto& x : m.d) x = g(rng);
  return m;
}
static DenseMatrix random_complex(long r, long c, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  DenseMatrix m(r, c);
  for (auto& x : m.d) {
    const double re = g(rng);
    x = Cplx(re, g(rng));
  }
  return m;
}
static double recon_error(const DenseMatrix& m, const linalg::SvdResult& r) {
  double e = 0;
  for (long i = 0; i < m.rows(); ++i)
    for (long j = 0; j < m.cols(); ++j) {
      Cplx s = 0;
      for (long k = 0; k < static_cast<long>(r.sigma.size()); ++k) s += r.u(i, k) * r.sigma[k] * r.v_dagger(k, j);
      e = std::max(e, std::abs(s - m(i, j)));
    }
  return e;
}
// max |U^H U - I| over the first k columns
static double unitarity_error(const DenseMatrix& u, long k) {
  double e = 0;
  for (long a = 0; a < k; ++a)
    for (long b = 0; b < k; ++b) {
      Cplx s = 0;
      for (long i = 0; i < u.rows(); ++i) s += std::conj(u(i, a)) * u(i, b);
      e = std::max(e, std::abs(s - (a == b ? 1.0 : 0.0)));
    }
  return e;
}

static models::ModelSpec heisenberg(int n, models::SpinConvention conv) {
  models::ModelSpec s;
  s.n = n;
  s.convention = conv;
  return s;
}
static models::ModelSpec tfim(int n, double h) {
  models::ModelSpec s;
  s.family = models::ModelFamily::transverse_ising;
  s.n = n;
  s.jz = 1.0;
  s.h = h;
  return s;
}
static dmrg::DmrgConfig fixed_config(int chi) {
  dmrg::DmrgConfig cfg;
  cfg.controller.mode = ctrl::ControlMode::fixed;
  cfg.controller.chi_max = chi;
  cfg.controller.chi_min = std::min(2, chi);
  return cfg;
}
static dmrg::DmrgConfig adaptive_config(int chi_max, double eps = 1e-10) {
  dmrg::DmrgConfig cfg;
  cfg.controller.mode = ctrl::ControlMode::pid;
  cfg.controller.chi_max = chi_max;
  cfg.controller.eps_trunc = eps;
  return cfg;
}

static void test_linalg() {
  {  // svd_full identity 2x2 (test_linalg.cpp:38)
    auto r = linalg::svd_full(DenseMatrix::Identity(2, 2));
    CHECK(approx(r.sigma[0], 1.0, 1e-12) && approx(r.sigma[1], 1.0, 1e-12));
    CHECK(std::abs(r.u(0, 0) - 1.0) <= 1e-12 && std::abs(r.u(1, 1) - 1.0) <= 1e-12);
    CHECK(std::abs(r.v_dagger(0, 0) - 1.0) <= 1e-12 && std::abs(r.v_dagger(0, 1)) <= 1e-12);
  }
  {  // diag(3,2)
    DenseMatrix m(2, 2);
    m(0, 0) = 3;
    m(1, 1) = 2;
    auto r = linalg::svd_full(m);
    CHECK(approx(r.sigma[0], 3.0, 1e-13) && approx(r.sigma[1], 2.0, 1e-13));
  }
  for (auto [rows, cols] : {std::pair<long, long>{8, 8}, {5, 9}, {9, 5}, {1, 7}, {7, 1}}) {
    DenseMatrix m = random_real(rows, cols, 42);
    auto r = linalg::svd_full(m);
    CHECK(r.rank == std::min(rows, cols));
    CHECK(recon_error(m, r) <= 1e-12);
    double fro = 0, s2 = 0;
    for (Cplx x : m.d) fro += std::norm(x);
    for (double s : r.sigma) s2 += s * s;
    CHECK(approx(fro, s2, 1e-12));
    for (size_t k = 1; k < r.sigma.size(); ++k) CHECK(r.sigma[k] <= r.sigma[k - 1]);
    auto r2 = linalg::svd_full(m);  // determinism
    CHECK(r2.sigma == r.sigma);
  }
  CHECK_THROWS_AS(linalg::svd_full(DenseMatrix(0, 3)), InvalidMatrix);
  {  // svd_truncated diagonal / range / degenerate cut (test_linalg.cpp:98-144)
    DenseMatrix m(3, 3);
    m(0, 0) = 3;
    m(1, 1) = 2;
    m(2, 2) = 1;
    auto r = linalg::svd_truncated(m, 2);
    CHECK(r.rank == 2 && approx(r.sigma[0], 3, 1e-13) && approx(r.sigma[1], 2, 1e-13));
    CHECK_THROWS_AS(linalg::svd_truncated(m, 0), InvalidRank);
    CHECK_THROWS_AS(linalg::svd_truncated(m, 4), InvalidRank);
    DenseMatrix d(3, 3);
    d(0, 0) = 2;
    d(1, 1) = 1;
    d(2, 2) = 1;
    CHECK(linalg::svd_truncated(d, 2).degenerate_cut);
    CHECK(!linalg::svd_truncated(d, 1).degenerate_cut);
  }
  {  // eigs_lowest on diag(-1,0,1) and the two-spin singlet (test_linalg.cpp:170-193)
    DenseMatrix h(3, 3);
    h(0, 0) = -1;
    h(2, 2) = 1;
    auto r = linalg::eigs_lowest(h, CVector(3, 1.0), 1e-12, 100);
    CHECK(approx(r.eigenvalue, -1.0, 1e-10));
    CHECK(approx(std::abs(r.eigenvector[0]), 1.0, 1e-8));
    DenseMatrix s(4, 4);
    s(0, 0) = s(3, 3) = 0.25;
    s(1, 1) = s(2, 2) = -0.25;
    s(1, 2) = s(2, 1) = 0.5;
    auto q = linalg::eigs_lowest(s, CVector{0.3, -0.7, 0.2, 0.9}, 1e-12, 100);
    CHECK(approx(q.eigenvalue, -0.75, 1e-10));
    CHECK_THROWS_AS(linalg::eigs_lowest(s, CVector(4, 0.0), 1e-10, 10), InvalidMatrix);
    DenseMatrix a = random_real(32, 32, 12), hs(32, 32);
    for (long i = 0; i < 32; ++i)
      for (long j = 0; j < 32; ++j) hs(i, j) = 0.5 * (a(i, j) + a(j, i));
    bool threw = false;
    try {
      linalg::eigs_lowest(hs, CVector(32, 1.0), 1e-14, 3);
    } catch (const EigenNonConvergence& e) {
      threw = std::isfinite(e.best_residual) && e.best_residual > 0;
    }
    CHECK(threw);
  }
  {  // complex svd_full (test_linalg.cpp:25-82 on MatrixXcd::Random): reconstruction,
     // isometric factors, non-increasing sigma, fix_phases, sum sigma^2 = ||A||_F^2
    for (auto [rows, cols] : {std::pair<long, long>{8, 8}, {5, 9}, {9, 5}, {1, 7}, {40, 30}}) {
      DenseMatrix m = random_complex(rows, cols, 7);
      auto r = linalg::svd_full(m);
      const long k = std::min(rows, cols);
      CHECK(r.rank == k && recon_error(m, r) <= 1e-12);
      CHECK(unitarity_error(r.u, k) <= 1e-10);
      double fro = 0, s2 = 0;
      for (Cplx x : m.d) fro += std::norm(x);
      for (double x : r.sigma) s2 += x * x;
      CHECK(approx(fro, s2, 1e-12));
      for (long q = 0; q < k; ++q) {  // first largest |u| entry real and positive
        long imax = 0;
        double best = 0;
        for (long i = 0; i < rows; ++i)
          if (std::abs(r.u(i, q)) > best) best = std::abs(r.u(i, q)), imax = i;
        CHECK(r.u(imax, q).real() > 0 && std::abs(r.u(imax, q).imag()) <= 1e-15 * best);
      }
    }
    DenseMatrix bad(2, 2);
    bad(0, 1) = Cplx(0, std::nan(""));
    CHECK_THROWS_AS(linalg::svd_full(bad), InvalidMatrix);
  }
  {  // eigs_lowest(LinearMap, ...) (linalg.hpp:71-78): real and complex Hermitian operators
    DenseMatrix h(3, 3);
    h(0, 0) = -1;
    h(2, 2) = 1;
    linalg::LinearMap op = [&](const CVector& x, CVector& y) {
      for (long i = 0; i < 3; ++i) {
        y[i] = 0;
        for (long j = 0; j < 3; ++j) y[i] += h(i, j) * x[j];
      }
    };
    auto r = linalg::eigs_lowest(op, 3, CVector(3, 1.0), 1e-12, 100);
    CHECK(approx(r.eigenvalue, -1.0, 1e-10));
    // a random complex Hermitian 6 x 6: LinearMap path (realified) vs the dense path
    DenseMatrix c = random_complex(6, 6, 99), hc(6, 6);
    for (long i = 0; i < 6; ++i)
      for (long j = 0; j < 6; ++j) hc(i, j) = 0.5 * (c(i, j) + std::conj(c(j, i)));
    linalg::LinearMap opc = [&](const CVector& x, CVector& y) {
      for (long i = 0; i < 6; ++i) {
        y[i] = 0;
        for (long j = 0; j < 6; ++j) y[i] += hc(i, j) * x[j];
      }
    };
    auto rc = linalg::eigs_lowest(opc, 6, CVector(6, 1.0), 1e-11, 200);
    auto rd = linalg::eigs_lowest(hc, CVector(6, 1.0), 1e-11, 200);
    CHECK(approx(rc.eigenvalue, rd.eigenvalue, 1e-9));
    double res = 0;  // |H v - E v|
    for (long i = 0; i < 6; ++i) {
      Cplx y = 0;
      for (long j = 0; j < 6; ++j) y += hc(i, j) * rc.eigenvector[j];
      res += std::norm(y - rc.eigenvalue * rc.eigenvector[i]);
    }
    CHECK(std::sqrt(res) <= 1e-9);
  }
  {  // split_two_site / merge_two_site (mps.cpp:124-166, 317-324; test_mps.cpp)
    const int d = 2, cl = 3, cr = 4;
    DenseMatrix theta = random_complex(d * cl, d * cr, 17);
    auto sp = mps::split_two_site(theta, d, cl, cr, 6);
    CHECK(sp.outcome.kept_chi == 6 && sp.left.dim(2) == 6 && sp.right.dim(0) == 6);
    mps::MatrixProductState psi({sp.left, sp.right});
    DenseMatrix back = mps::merge_two_site(psi, 0);
    double e = 0;
    for (long i = 0; i < theta.rows(); ++i)
      for (long j = 0; j < theta.cols(); ++j) e = std::max(e, std::abs(back(i, j) - theta(i, j)));
    CHECK(e <= 1e-12);
    auto sp2 = mps::split_two_site(theta, d, cl, cr, 2, 1e-14, mps::AbsorbSide::left);
    CHECK(sp2.outcome.kept_chi == 2 && sp2.lambda.values.size() == 2);
    CHECK(approx(sp2.outcome.truncation_error, mps::truncation_error(sp2.outcome.spectrum, 2), 1e-14));
    CHECK_THROWS_AS(mps::split_two_site(theta, d, cl, cr + 1, 2), InvalidMatrix);
    CHECK_THROWS_AS(mps::split_two_site(theta, d, cl, cr, 0), InvalidRank);
    CHECK_THROWS_AS(mps::split_two_site(DenseMatrix(d * cl, d * cr), d, cl, cr, 2), DegenerateSpectrum);
  }
  {  // select_backend threshold dispatch (test_linalg.cpp:228)
    linalg::BackendRegistry registry;
    linalg::BackendPolicy policy;
    CHECK(linalg::select_backend(policy, 32, registry) == linalg::BackendId::reference);
    CHECK(linalg::select_backend(policy, 2048, registry) == linalg::BackendId::reference);
    registry.register_external(std::make_unique<linalg::B200SvdBackend>());
    CHECK(linalg::select_backend(policy, 32, registry) == linalg::BackendId::reference);
    CHECK(linalg::select_backend(policy, 64, registry) == linalg::BackendId::external);
    DenseMatrix m = random_real(6, 4, 3);
    auto r = linalg::svd_dispatch(m, policy, 128, registry);
    CHECK(recon_error(m, r) <= 1e-12);
  }
}

static void test_spectrum() {
  // test_mps.cpp:76-122
  CHECK(std::abs(mps::entropy_from_spectrum(spec_of({1.0}))) <= 1e-15);
  CHECK(approx(mps::entropy_from_spectrum(spec_of({M_SQRT1_2, M_SQRT1_2})), std::log(2.0), 1e-12));
  CHECK(approx(mps::entropy_from_spectrum(spec_of({std::sqrt(0.9), std::sqrt(0.1)})),
               0.3250829733914482, 1e-12));
  CHECK(mps::entropy_from_spectrum(spec_of({1.0, 1e-15})) == 0.0);
  CHECK_THROWS_AS(mps::entropy_from_spectrum(spec_of({0.0, 0.0})), DegenerateSpectrum);
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int trial = 0; trial < 20; ++trial) {
    long len = 1 + static_cast<long>(uni(rng) * 20);
    RVector v(len);
    for (auto& x : v) x = uni(rng);
    std::sort(v.begin(), v.end(), std::greater<double>());
    CHECK(mps::entropy_from_spectrum({v, 0}) <= std::log(static_cast<double>(len)) + 1e-12);
  }
  auto sp = spec_of({std::sqrt(0.8), std::sqrt(0.2)});
  CHECK(std::abs(mps::truncation_error(sp, 2)) <= 1e-15);
  CHECK(approx(mps::truncation_error(sp, 1), 0.4472135954999579, 1e-12));
  CHECK(std::abs(mps::truncation_error(spec_of({1.0, 0.0}), 1)) <= 1e-15);
  CHECK_THROWS_AS(mps::truncation_error(sp, 0), InvalidRank);
  CHECK_THROWS_AS(mps::truncation_error(sp, 3), InvalidRank);
  auto big = spec_of({0.9, 0.5, 0.3, 0.1, 0.01});
  for (int k = 1; k < 5; ++k)
    CHECK(mps::truncation_error(big, k + 1) <= mps::truncation_error(big, k) + 1e-15);
  // test_controller.cpp:217
  RVector v{0.9, 0.4, 0.1, 0.01};
  CHECK(ctrl::rank_for_discarded_weight(v, 1e-6) == 4);
  CHECK(ctrl::rank_for_discarded_weight(v, 1e-3) == 3);
  CHECK(ctrl::rank_for_discarded_weight(v, 0.05) == 2);
  CHECK(ctrl::rank_for_discarded_weight(v, 0.5) == 1);
}

static void test_controller() {
  // test_controller.cpp:227-295
  ctrl::ControllerConfig cfg;
  cfg.chi_min = 1;
  cfg.chi_max = 64;
  {
    cfg.mode = ctrl::ControlMode::fixed;
    ctrl::BondControllerState st;
    for (int t = 0; t < 5; ++t) CHECK(ctrl::controller_update(st, spec_of({0.9, 0.3, 0.01}), cfg).chi == 64);
  }
  {
    auto c = cfg;
    c.mode = ctrl::ControlMode::direct;
    c.gamma_margin = 1.0;
    c.alpha_ema = 0.5;
    c.predictor_order = ctrl::PredictorOrder::off;
    ctrl::BondControllerState st;
    int chi = 0;
    for (int t = 0; t < 60; ++t) chi = ctrl::controller_update(st, spec_of({M_SQRT1_2, M_SQRT1_2}), c).chi;
    CHECK(chi == 2);
  }
  {
    auto c = cfg;
    c.mode = ctrl::ControlMode::threshold;
    c.eps_trunc = 1e-6;
    ctrl::BondControllerState st;
    CHECK(ctrl::controller_update(st, spec_of({1.0, 1e-2, 1e-9}), c).chi == 2);
  }
  {
    auto c = cfg;
    c.mode = ctrl::ControlMode::pid;
    c.alpha_ema = 1.0;
    c.predictor_order = ctrl::PredictorOrder::off;
    c.s_target = std::log(2.0);
    ctrl::BondControllerState st;
    st.chi = 8;
    st.initialized = true;
    std::vector<int> last;
    for (int t = 0; t < 40; ++t) last.push_back(ctrl::controller_update(st, spec_of({M_SQRT1_2, M_SQRT1_2}), c).chi);
    for (size_t t = 30; t < last.size(); ++t) CHECK(std::abs(last[t] - last[29]) <= 1);
  }
  {  // clamp containment
    std::mt19937_64 rng(8);
    std::uniform_real_distribution<double> uni(0, 2.5);
    ctrl::ControllerConfig c;
    c.chi_min = 3;
    c.chi_max = 17;
    c.s_target = 1.0;
    ctrl::BondControllerState st;
    st.chi = 5;
    st.initialized = true;
    for (int t = 0; t < 100; ++t) {
      RVector v(6);
      for (auto& x : v) x = uni(rng) + 1e-6;
      std::sort(v.begin(), v.end(), std::greater<double>());
      auto d = ctrl::controller_update(st, {v, 0}, c);
      CHECK(d.chi >= 3 && d.chi <= 17);
    }
  }
}

static void test_dmrg(double e_heis8, double e_tfim8) {
  {  // test_dmrg.cpp:111
    auto r = dmrg::run_dmrg(heisenberg(2, models::SpinConvention::spin_half), fixed_config(4));
    CHECK(approx(r.energy, -0.75, 1e-9));
  }
  {  // test_dmrg.cpp:117
    auto cfg = fixed_config(16);
    cfg.eps_conv = 1e-10;
    auto r = dmrg::run_dmrg(heisenberg(8, models::SpinConvention::pauli), cfg);
    CHECK(r.converged);
    CHECK(r.sweeps.size() <= 5);
    CHECK(std::abs(r.energy - e_heis8) <= 1e-8);
  }
  {  // test_dmrg.cpp:128
    auto r = dmrg::run_dmrg(heisenberg(10, models::SpinConvention::pauli), fixed_config(24));
    for (size_t s = 1; s < r.sweeps.size(); ++s) CHECK(r.sweeps[s].energy <= r.sweeps[s - 1].energy + 1e-10);
    CHECK(r.max_monotonicity_violation <= 1e-10);
  }
  {  // test_dmrg.cpp:136
    auto r1 = dmrg::run_dmrg(heisenberg(8, models::SpinConvention::pauli), adaptive_config(32));
    for (const auto& s : r1.sweeps) CHECK(s.energy >= e_heis8 - 1e-9);
    // the reference's automatic start for TFIM is a random complex MPS
    // (dmrg.cpp:230-236): complex arithmetic runs it unchanged
    auto tc = adaptive_config(32);
    tc.arithmetic = dmrg::DmrgConfig::Arithmetic::complex;
    auto r2 = dmrg::run_dmrg(tfim(8, 1.0), tc);
    for (const auto& s : r2.sweeps) CHECK(s.energy >= e_tfim8 - 1e-9);
    CHECK(std::abs(r2.energy - e_tfim8) <= 1e-8);
    // the chain's state comes back as complex tensors: the complex random
    // start (mps.cpp:75-95) has unit norm and genuinely complex entries
    dmrg::Chain ch(tfim(8, 1.0), tc);
    auto psi = ch.state();
    CHECK(psi.size() == 8);
    double nrm = 0, imag = 0;
    for (long i = 0; i < psi.site(0).size(); ++i) nrm += std::norm(psi.site(0).data()[i]);
    for (int k = 0; k < psi.size(); ++k)
      for (long i = 0; i < psi.site(k).size(); ++i) imag = std::max(imag, std::abs(psi.site(k).data()[i].imag()));
    CHECK(std::abs(nrm - 1.0) <= 1e-12);
    CHECK(imag > 1e-3);
  }
  {  // test_dmrg.cpp:144, 254, 270
    ctrl::ControllerTrace trace;
    auto r = dmrg::run_dmrg(heisenberg(12, models::SpinConvention::pauli), adaptive_config(32, 1e-9), &trace);
    CHECK(r.converged);
    CHECK(r.max_monotonicity_violation <= 1e-6 * std::abs(r.energy));
    CHECK(trace.rows().size() == r.sweeps.size() * 2 * 11);
    for (const auto& s : r.sweeps) {
      CHECK(s.chi_profile.size() == 11 && s.entropy_profile.size() == 11);
      CHECK(*std::max_element(s.chi_profile.begin(), s.chi_profile.end()) <= 32);
    }
    CHECK(r.bond_dims == r.sweeps.back().chi_profile);
  }
  CHECK_THROWS_AS(dmrg::run_dmrg(heisenberg(1, models::SpinConvention::pauli), fixed_config(4)), Error);
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::printf("usage: %s E_heis8_pauli E_tfim8_h1\n", argv[0]);
    return 2;
  }
  const double e_heis8 = std::atof(argv[1]), e_tfim8 = std::atof(argv[2]);
  try {
    test_linalg();
    test_spectrum();
    test_controller();
    test_dmrg(e_heis8, e_tfim8);
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught exception: %s\n", e.what());
    return 1;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
