// ============================================================================
// TEST INFRASTRUCTURE ONLY — CPU ORACLE.
//
// A C++ restatement of the reference (arxiv/paper_2604_03960, /root/reference/
// proj) two-site DMRG hot path, used as the parity checker for the B200
// kernels.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load it.  The product library
// (paper_2604_03960_b200) never links, loads or calls anything here.
//
// Why a restatement: the reference itself cannot be built in this image
// (Eigen3, doctest, nlohmann/json and CLI11 are absent; proj/CMakeLists.txt:
// 5,13).  Eigen's arithmetic is replaced by the bundled OpenBLAS 0.3.30
// (numpy.libs/libscipy_openblas64_, ILP64):
//   - Tensor::contract GEMM (tensor.hpp:195-196)        -> dgemm / zgemm
//   - Eigen::BDCSVD thin U/V (linalg.cpp:38)            -> dgesdd / zgesdd ('S')
//   - SelfAdjointEigenSolver::computeFromTridiagonal    -> dstev ('V')
//     (linalg.cpp:144-145)
//   - HouseholderQR (mps.cpp:176,191)                   -> geqrf + orgqr/ungqr
// Departures are rounding-level only (reduction orders; D&C SVD variants).
// Parity pinning: the oracle is checked against every known answer the
// reference's own tests hold for this path (tests/test_oracle_golden.py).
//
// Templated on the scalar: complex128 with the reference MPO is the faithful
// restatement (and the CPU baseline "port"); double with the real-gauge MPO
// is the arithmetic the GPU path performs.
// ============================================================================
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace oracle {

using cd = std::complex<double>;
using lint = long long;

// ---- error taxonomy (errors.hpp:8-59) --------------------------------------
struct Error : std::runtime_error {
  int code;
  double residual = 0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum {
  E_ERROR = 1, E_INVALID_MATRIX = 2, E_NUMERICAL_FAILURE = 3, E_INVALID_RANK = 4,
  E_EIGEN_NONCONV = 5, E_INVALID_BASIS = 6, E_SIZE_GUARD = 7, E_DEGENERATE = 8,
  E_UNSUPPORTED = 9, E_INVALID_CONFIG = 10, E_INTERNAL = 11
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

// ---- BLAS/LAPACK (ILP64, scipy_ prefix, 64_ suffix) ------------------------
extern "C" {
void scipy_dgemm_64_(const char*, const char*, const lint*, const lint*, const lint*,
                     const double*, const double*, const lint*, const double*,
                     const lint*, const double*, double*, const lint*, size_t, size_t);
void scipy_zgemm_64_(const char*, const char*, const lint*, const lint*, const lint*,
                     const cd*, const cd*, const lint*, const cd*, const lint*,
                     const cd*, cd*, const lint*, size_t, size_t);
void scipy_dgesdd_64_(const char*, const lint*, const lint*, double*, const lint*,
                      double*, double*, const lint*, double*, const lint*, double*,
                      const lint*, lint*, lint*, size_t);
void scipy_zgesdd_64_(const char*, const lint*, const lint*, cd*, const lint*, double*,
                      cd*, const lint*, cd*, const lint*, cd*, const lint*, double*,
                      lint*, lint*, size_t);
void scipy_dstev_64_(const char*, const lint*, double*, double*, double*, const lint*,
                     double*, lint*, size_t);
void scipy_dgeqrf_64_(const lint*, const lint*, double*, const lint*, double*, double*,
                      const lint*, lint*);
void scipy_dorgqr_64_(const lint*, const lint*, const lint*, double*, const lint*,
                      const double*, double*, const lint*, lint*);
void scipy_zgeqrf_64_(const lint*, const lint*, cd*, const lint*, cd*, cd*, const lint*,
                      lint*);
void scipy_zungqr_64_(const lint*, const lint*, const lint*, cd*, const lint*, const cd*,
                      cd*, const lint*, lint*);
void scipy_openblas_set_num_threads64_(int);
}

inline double conj_(double x) { return x; }
inline cd conj_(cd x) { return std::conj(x); }
inline double real_(double x) { return x; }
inline double real_(cd x) { return x.real(); }
inline double abs2_(double x) { return x * x; }
inline double abs2_(cd x) { return std::norm(x); }

// C(m x n, row-major) = A(m x k, row-major) * B(k x n, row-major)
inline void gemm_rm(lint m, lint n, lint k, const double* a, const double* b, double* c) {
  const double one = 1, zero = 0;
  if (m == 0 || n == 0) return;
  if (k == 0) { std::fill(c, c + m * n, 0.0); return; }
  scipy_dgemm_64_("N", "N", &n, &m, &k, &one, b, &n, a, &k, &zero, c, &n, 1, 1);
}
inline void gemm_rm(lint m, lint n, lint k, const cd* a, const cd* b, cd* c) {
  const cd one = 1, zero = 0;
  if (m == 0 || n == 0) return;
  if (k == 0) { std::fill(c, c + m * n, cd(0)); return; }
  scipy_zgemm_64_("N", "N", &n, &m, &k, &one, b, &n, a, &k, &zero, c, &n, 1, 1);
}

// ---- Tensor (tensor.hpp:26-198) ---------------------------------------------
template <class T>
struct Tensor {
  std::vector<long> shape;
  std::vector<T> data;
  Tensor() = default;
  explicit Tensor(std::vector<long> s) : shape(std::move(s)) {
    long n = 1;
    for (long x : shape) {
      if (x < 1) fail(E_INVALID_MATRIX, "tensor dimension must be >= 1");
      n *= x;
    }
    data.assign(static_cast<size_t>(n), T(0));
  }
  long dim(int a) const { return shape[static_cast<size_t>(a)]; }
  int rank() const { return static_cast<int>(shape.size()); }
  long size() const { return static_cast<long>(data.size()); }
  T& operator()(long i, long j, long k) { return data[(i * shape[1] + j) * shape[2] + k]; }
  T operator()(long i, long j, long k) const { return data[(i * shape[1] + j) * shape[2] + k]; }
  T& operator()(long i, long j, long k, long l) {
    return data[((i * shape[1] + j) * shape[2] + k) * shape[3] + l];
  }
  T operator()(long i, long j, long k, long l) const {
    return data[((i * shape[1] + j) * shape[2] + k) * shape[3] + l];
  }
  Tensor conjugated() const {
    Tensor t = *this;
    for (auto& v : t.data) v = conj_(v);
    return t;
  }
  double norm() const {
    double s = 0;
    for (const auto& v : data) s += abs2_(v);
    return std::sqrt(s);
  }

  // tensor.hpp:122-150: element-by-element stride walk
  Tensor permuted(const std::vector<int>& axes) const {
    const int n = rank();
    std::vector<long> ns(n);
    for (int i = 0; i < n; ++i) ns[i] = shape[axes[i]];
    Tensor out(ns);
    std::vector<long> out_strides(n, 1), new_for_old(n, 0);
    for (int i = n - 2; i >= 0; --i) out_strides[i] = out_strides[i + 1] * ns[i + 1];
    for (int i = 0; i < n; ++i) new_for_old[axes[i]] = out_strides[i];
    std::vector<long> idx(n, 0);
    long dst = 0;
    const long total = size();
    for (long src = 0; src < total; ++src) {
      out.data[dst] = data[src];
      for (int ax = n - 1; ax >= 0; --ax) {
        dst += new_for_old[ax];
        if (++idx[ax] < shape[ax]) break;
        dst -= idx[ax] * new_for_old[ax];
        idx[ax] = 0;
      }
    }
    return out;
  }

  // tensor.hpp:152-198: permute to (free, contracted) x (contracted, free), one GEMM
  Tensor contract(const std::vector<int>& axes_a, const Tensor& other,
                  const std::vector<int>& axes_b) const {
    if (axes_a.size() != axes_b.size()) fail(E_INTERNAL, "contract: axis count mismatch");
    const int na = rank(), nb = other.rank();
    std::vector<int> free_a, free_b;
    std::vector<bool> ua(na, false), ub(nb, false);
    for (size_t i = 0; i < axes_a.size(); ++i) {
      if (dim(axes_a[i]) != other.dim(axes_b[i])) fail(E_INTERNAL, "contract: dimension mismatch");
      ua[axes_a[i]] = true;
      ub[axes_b[i]] = true;
    }
    for (int i = 0; i < na; ++i) if (!ua[i]) free_a.push_back(i);
    for (int i = 0; i < nb; ++i) if (!ub[i]) free_b.push_back(i);
    std::vector<int> pa = free_a;
    pa.insert(pa.end(), axes_a.begin(), axes_a.end());
    std::vector<int> pb(axes_b.begin(), axes_b.end());
    pb.insert(pb.end(), free_b.begin(), free_b.end());
    Tensor ta = permuted(pa), tb = other.permuted(pb);
    long m = 1, k = 1, n = 1;
    std::vector<long> os;
    for (int ax : free_a) { m *= dim(ax); os.push_back(dim(ax)); }
    for (int ax : axes_a) k *= dim(ax);
    for (int ax : free_b) { n *= other.dim(ax); os.push_back(other.dim(ax)); }
    if (os.empty()) os.push_back(1);
    Tensor out(os);
    gemm_rm(m, n, k, ta.data.data(), tb.data.data(), out.data.data());
    return out;
  }
};

// Column-major dense matrix (the reference's Eigen::MatrixXcd DenseMatrix).
template <class T>
struct Mat {
  long rows = 0, cols = 0;
  std::vector<T> d;
  Mat() = default;
  Mat(long r, long c) : rows(r), cols(c), d(static_cast<size_t>(r * c), T(0)) {}
  T& operator()(long i, long j) { return d[i + j * rows]; }
  T operator()(long i, long j) const { return d[i + j * rows]; }
};

// ---- SVD engine (linalg.cpp:11-89) -------------------------------------------
template <class T>
struct SvdResult {
  Mat<T> u;                  // m x r
  std::vector<double> sigma; // r
  Mat<T> vt;                 // r x n
  long rank = 0;
  bool degenerate_cut = false;
};

template <class T>
void check_input(const Mat<T>& m) {  // linalg.cpp:11-15
  if (m.rows < 1 || m.cols < 1) fail(E_INVALID_MATRIX, "svd: matrix must be at least 1x1");
  for (const auto& v : m.d)
    if (!std::isfinite(real_(v)) || !std::isfinite(std::imag(std::complex<double>(v))))
      fail(E_INVALID_MATRIX, "svd: non-finite entries");
}

// linalg.cpp:19-35: largest-|u| entry of each U column real positive (first max wins)
template <class T>
void fix_phases(Mat<T>& u, Mat<T>& vt) {
  for (long j = 0; j < u.cols; ++j) {
    long imax = 0;
    double best = 0;
    for (long i = 0; i < u.rows; ++i) {
      double a = std::abs(u(i, j));
      if (a > best) { best = a; imax = i; }
    }
    if (best <= 0) continue;
    T f = conj_(u(imax, j)) / best;
    for (long i = 0; i < u.rows; ++i) u(i, j) *= f;
    if (j < vt.rows)
      for (long c = 0; c < vt.cols; ++c) vt(j, c) *= conj_(f);
  }
}

inline void gesdd(Mat<double>& a, std::vector<double>& s, Mat<double>& u, Mat<double>& vt) {
  lint m = a.rows, n = a.cols, r = std::min(m, n), lwork = -1, info = 0;
  s.assign(r, 0); u = Mat<double>(m, r); vt = Mat<double>(r, n);
  std::vector<lint> iwork(8 * r);
  double wq;
  lint ldu = m, ldvt = r;
  scipy_dgesdd_64_("S", &m, &n, a.d.data(), &m, s.data(), u.d.data(), &ldu, vt.d.data(), &ldvt,
                   &wq, &lwork, iwork.data(), &info, 1);
  lwork = static_cast<lint>(wq) + 1;
  std::vector<double> work(lwork);
  scipy_dgesdd_64_("S", &m, &n, a.d.data(), &m, s.data(), u.d.data(), &ldu, vt.d.data(), &ldvt,
                   work.data(), &lwork, iwork.data(), &info, 1);
  if (info != 0) fail(E_NUMERICAL_FAILURE, "svd: decomposition did not converge");
}
inline void gesdd(Mat<cd>& a, std::vector<double>& s, Mat<cd>& u, Mat<cd>& vt) {
  lint m = a.rows, n = a.cols, r = std::min(m, n), lwork = -1, info = 0;
  s.assign(r, 0); u = Mat<cd>(m, r); vt = Mat<cd>(r, n);
  std::vector<lint> iwork(8 * r);
  lint mx = std::max(m, n);
  std::vector<double> rwork(std::max<lint>(5 * r * r + 5 * r, 2 * mx * r + 2 * r * r + r) + 1);
  cd wq;
  lint ldu = m, ldvt = r;
  scipy_zgesdd_64_("S", &m, &n, a.d.data(), &m, s.data(), u.d.data(), &ldu, vt.d.data(), &ldvt,
                   &wq, &lwork, rwork.data(), iwork.data(), &info, 1);
  lwork = static_cast<lint>(wq.real()) + 1;
  std::vector<cd> work(lwork);
  scipy_zgesdd_64_("S", &m, &n, a.d.data(), &m, s.data(), u.d.data(), &ldu, vt.d.data(), &ldvt,
                   work.data(), &lwork, rwork.data(), iwork.data(), &info, 1);
  if (info != 0) fail(E_NUMERICAL_FAILURE, "svd: decomposition did not converge");
}

// reference_svd + svd_full (linalg.cpp:37-48,67-70)
template <class T>
SvdResult<T> svd_full(const Mat<T>& m) {
  check_input(m);
  Mat<T> a = m;
  SvdResult<T> r;
  gesdd(a, r.sigma, r.u, r.vt);
  r.rank = static_cast<long>(r.sigma.size());
  fix_phases(r.u, r.vt);
  return r;
}

// svd_truncated (linalg.cpp:72-89)
template <class T>
SvdResult<T> svd_truncated(const Mat<T>& m, long keep) {
  check_input(m);
  const long rmax = std::min(m.rows, m.cols);
  if (keep < 1 || keep > rmax) fail(E_INVALID_RANK, "svd_truncated: keep out of range [1, min(rows,cols)]");
  SvdResult<T> full = svd_full(m);
  SvdResult<T> r;
  r.u = Mat<T>(m.rows, keep);
  for (long j = 0; j < keep; ++j)
    for (long i = 0; i < m.rows; ++i) r.u(i, j) = full.u(i, j);
  r.sigma.assign(full.sigma.begin(), full.sigma.begin() + keep);
  r.vt = Mat<T>(keep, m.cols);
  for (long j = 0; j < m.cols; ++j)
    for (long i = 0; i < keep; ++i) r.vt(i, j) = full.vt(i, j);
  r.rank = keep;
  if (keep < full.rank)
    r.degenerate_cut = std::abs(full.sigma[keep - 1] - full.sigma[keep]) <= 1e-12 * full.sigma[0];
  return r;
}

// ---- Lanczos (linalg.cpp:107-178) --------------------------------------------
template <class T>
struct EigsResult {
  double eigenvalue = 0;
  std::vector<T> eigenvector;
  int matvec_count = 0;
  double residual = 0;
};

template <class T>
T vdot(const std::vector<T>& a, const std::vector<T>& b) {  // Eigen a.dot(b) = sum conj(a) b
  T s = T(0);
  for (size_t i = 0; i < a.size(); ++i) s += conj_(a[i]) * b[i];
  return s;
}
template <class T>
double vnorm(const std::vector<T>& a) {
  double s = 0;
  for (const auto& x : a) s += abs2_(x);
  return std::sqrt(s);
}

// lowest eigenpair of the k x k symmetric tridiagonal (diag, sub) (Eigen computeFromTridiagonal)
inline void tridiag_lowest(const std::vector<double>& diag, const std::vector<double>& sub, int k,
                           double& theta, std::vector<double>& s) {
  std::vector<double> d(diag.begin(), diag.begin() + k), e(std::max(k - 1, 1), 0.0);
  for (int i = 0; i + 1 < k; ++i) e[i] = sub[i];
  std::vector<double> z(static_cast<size_t>(k) * k), work(std::max(1, 2 * k - 2));
  lint n = k, ldz = k, info = 0;
  scipy_dstev_64_("V", &n, d.data(), e.data(), z.data(), &ldz, work.data(), &info, 1);
  if (info != 0) fail(E_NUMERICAL_FAILURE, "tridiagonal eigensolver failed");
  theta = d[0];
  s.assign(z.begin(), z.begin() + k);  // column 0 (column-major)
}

template <class T, class F>
EigsResult<T> eigs_lowest(F&& apply_h, long dim, const std::vector<T>& v0, double tol, int max_iter) {
  if (static_cast<long>(v0.size()) != dim) fail(E_INVALID_MATRIX, "eigs_lowest: v0 size mismatch");
  double n0 = vnorm(v0);
  if (!(n0 > 0)) fail(E_INVALID_MATRIX, "eigs_lowest: v0 must have norm > 0");
  const int block = static_cast<int>(std::min<long>(dim, 48));
  std::vector<T> q(v0);
  for (auto& x : q) x /= n0;
  double best_residual = std::numeric_limits<double>::infinity();
  int matvecs = 0;
  std::vector<std::vector<T>> basis;
  std::vector<T> w(dim), ritz(dim);
  while (matvecs < max_iter) {
    basis.clear();
    basis.push_back(q);
    std::vector<double> alpha, beta;
    for (int j = 0; j < block && matvecs < max_iter; ++j) {
      apply_h(basis[j], w);
      ++matvecs;
      double a = real_(vdot(basis[j], w));
      alpha.push_back(a);
      for (long x = 0; x < dim; ++x) w[x] -= a * basis[j][x];
      if (j > 0)
        for (long x = 0; x < dim; ++x) w[x] -= beta[j - 1] * basis[j - 1][x];
      for (const auto& b : basis) {  // full reorthogonalisation (MGS)
        T c = vdot(b, w);
        for (long x = 0; x < dim; ++x) w[x] -= c * b[x];
      }
      double bnorm = vnorm(w);
      const int k = j + 1;
      double theta;
      std::vector<double> s;
      tridiag_lowest(alpha, beta, k, theta, s);
      double res_bound = bnorm * std::abs(s[k - 1]);
      bool breakdown = bnorm <= 1e-14 * std::max(1.0, std::abs(theta));
      if (res_bound <= tol * std::max(1.0, std::abs(theta)) || breakdown || k == block ||
          matvecs >= max_iter) {
        std::fill(ritz.begin(), ritz.end(), T(0));
        for (int i = 0; i < k; ++i)
          for (long x = 0; x < dim; ++x) ritz[x] += s[i] * basis[i][x];
        double rn = vnorm(ritz);
        for (auto& x : ritz) x /= rn;
        apply_h(ritz, w);
        ++matvecs;
        double ev = real_(vdot(ritz, w));
        std::vector<T> rv(dim);
        for (long x = 0; x < dim; ++x) rv[x] = w[x] - ev * ritz[x];
        double res = vnorm(rv);
        best_residual = std::min(best_residual, res);
        if (res <= tol * std::max(1.0, std::abs(ev))) return {ev, ritz, matvecs, res};
        if (breakdown && res > tol * std::max(1.0, std::abs(ev))) {
          double rvn = vnorm(rv);
          for (long x = 0; x < dim; ++x) q[x] = ritz[x] + 1e-8 * (rv[x] / rvn);
          double qn = vnorm(q);
          for (auto& x : q) x /= qn;
        } else {
          q = ritz;
        }
        break;
      }
      beta.push_back(bnorm);
      std::vector<T> nb(dim);
      for (long x = 0; x < dim; ++x) nb[x] = w[x] / bnorm;
      basis.push_back(std::move(nb));
    }
  }
  Error e(E_EIGEN_NONCONV, "eigs_lowest: no convergence within max_iter");
  e.residual = best_residual;
  throw e;
}

// ---- MPS core (mps.cpp) -----------------------------------------------------
// entropy_from_spectrum (mps.cpp:97-113)
inline double entropy_from_spectrum(const std::vector<double>& v) {
  if (v.empty()) fail(E_DEGENERATE, "entropy: empty spectrum");
  double lmax = v[0];
  if (!(lmax > 0)) fail(E_DEGENERATE, "entropy: all-zero spectrum");
  double cutoff = 1e-14 * lmax, total = 0;
  for (double x : v) if (x > cutoff) total += x * x;
  double s = 0;
  for (double x : v) {
    if (x <= cutoff) continue;
    double p = x * x / total;
    if (p > 0) s -= p * std::log(p);
  }
  return s;
}
// truncation_error (mps.cpp:115-122)
inline double truncation_error(const std::vector<double>& v, int kept) {
  if (kept < 1 || kept > static_cast<int>(v.size())) fail(E_INVALID_RANK, "truncation_error: kept out of range");
  double tail = 0;
  for (size_t k = kept; k < v.size(); ++k) tail += v[k] * v[k];
  return std::sqrt(std::max(0.0, tail));
}

template <class T>
struct MPS {
  std::vector<Tensor<T>> sites;
  int center = -1;
  int size() const { return static_cast<int>(sites.size()); }
  int phys_dim() const { return static_cast<int>(sites.front().dim(1)); }
  std::vector<int> bond_dims() const {  // mps.cpp:24-29
    std::vector<int> d;
    for (size_t i = 0; i + 1 < sites.size(); ++i) d.push_back(static_cast<int>(sites[i].dim(2)));
    return d;
  }
};

template <class T>
MPS<T> product_state(int n, int d, const std::vector<int>& local) {  // mps.cpp:40-57
  if (static_cast<int>(local.size()) != n) fail(E_INVALID_BASIS, "product_state: need one basis index per site");
  MPS<T> psi;
  for (int i = 0; i < n; ++i) {
    int s = local[i];
    if (s < 0 || s >= d) fail(E_INVALID_BASIS, "product_state: basis index out of range");
    Tensor<T> t({1, d, 1});
    t(0, s, 0) = T(1);
    psi.sites.push_back(std::move(t));
  }
  psi.center = 0;
  return psi;
}

// Householder QR, thin Q (m x k) and R (k x ncol), column-major
inline void qr_thin(Mat<double>& a, Mat<double>& q, Mat<double>& r) {
  lint m = a.rows, n = a.cols, k = std::min(m, n), info = 0, lwork = -1;
  std::vector<double> tau(std::max<lint>(k, 1));
  double wq;
  scipy_dgeqrf_64_(&m, &n, a.d.data(), &m, tau.data(), &wq, &lwork, &info);
  lwork = static_cast<lint>(wq) + 1;
  std::vector<double> work(lwork);
  scipy_dgeqrf_64_(&m, &n, a.d.data(), &m, tau.data(), work.data(), &lwork, &info);
  r = Mat<double>(k, n);
  for (lint j = 0; j < n; ++j)
    for (lint i = 0; i <= std::min<lint>(j, k - 1); ++i) r(i, j) = a(i, j);
  q = Mat<double>(m, k);
  for (lint j = 0; j < k; ++j)
    for (lint i = 0; i < m; ++i) q(i, j) = a(i, j);
  lwork = -1;
  scipy_dorgqr_64_(&m, &k, &k, q.d.data(), &m, tau.data(), &wq, &lwork, &info);
  lwork = static_cast<lint>(wq) + 1;
  work.assign(lwork, 0);
  scipy_dorgqr_64_(&m, &k, &k, q.d.data(), &m, tau.data(), work.data(), &lwork, &info);
}
inline void qr_thin(Mat<cd>& a, Mat<cd>& q, Mat<cd>& r) {
  lint m = a.rows, n = a.cols, k = std::min(m, n), info = 0, lwork = -1;
  std::vector<cd> tau(std::max<lint>(k, 1));
  cd wq;
  scipy_zgeqrf_64_(&m, &n, a.d.data(), &m, tau.data(), &wq, &lwork, &info);
  lwork = static_cast<lint>(wq.real()) + 1;
  std::vector<cd> work(lwork);
  scipy_zgeqrf_64_(&m, &n, a.d.data(), &m, tau.data(), work.data(), &lwork, &info);
  r = Mat<cd>(k, n);
  for (lint j = 0; j < n; ++j)
    for (lint i = 0; i <= std::min<lint>(j, k - 1); ++i) r(i, j) = a(i, j);
  q = Mat<cd>(m, k);
  for (lint j = 0; j < k; ++j)
    for (lint i = 0; i < m; ++i) q(i, j) = a(i, j);
  lwork = -1;
  scipy_zungqr_64_(&m, &k, &k, q.d.data(), &m, tau.data(), &wq, &lwork, &info);
  lwork = static_cast<lint>(wq.real()) + 1;
  work.assign(lwork, cd(0));
  scipy_zungqr_64_(&m, &k, &k, q.d.data(), &m, tau.data(), work.data(), &lwork, &info);
}

// row-major (rows x cols) view of a tensor -> column-major Mat
template <class T>
Mat<T> to_mat(const Tensor<T>& t, long rows, long cols) {
  Mat<T> m(rows, cols);
  for (long i = 0; i < rows; ++i)
    for (long j = 0; j < cols; ++j) m(i, j) = t.data[i * cols + j];
  return m;
}
template <class T>
Tensor<T> from_mat(const Mat<T>& m, std::vector<long> shape) {  // tensor.hpp:105-109
  Tensor<T> t(std::move(shape));
  for (long i = 0; i < m.rows; ++i)
    for (long j = 0; j < m.cols; ++j) t.data[i * m.cols + j] = m(i, j);
  return t;
}
template <class T>
Mat<T> matmul(const Mat<T>& a, const Mat<T>& b) {
  Mat<T> c(a.rows, b.cols);
  for (long j = 0; j < b.cols; ++j)
    for (long k = 0; k < a.cols; ++k) {
      T bk = b(k, j);
      for (long i = 0; i < a.rows; ++i) c(i, j) += a(i, k) * bk;
    }
  return c;
}
template <class T>
Mat<T> adjoint(const Mat<T>& a) {
  Mat<T> c(a.cols, a.rows);
  for (long i = 0; i < a.rows; ++i)
    for (long j = 0; j < a.cols; ++j) c(j, i) = conj_(a(i, j));
  return c;
}

// canonicalize (mps.cpp:171-210) via push_right / push_left
template <class T>
void push_right(MPS<T>& psi, int i) {
  Tensor<T>& a = psi.sites[i];
  long l = a.dim(0), d = a.dim(1), r = a.dim(2);
  Mat<T> m = to_mat(a, l * d, r), q, rr;
  qr_thin(m, q, rr);
  long k = std::min(l * d, r);
  psi.sites[i] = from_mat(q, {l, d, k});
  Tensor<T>& b = psi.sites[i + 1];
  Mat<T> bm = to_mat(b, b.dim(0), b.dim(1) * b.dim(2));
  Mat<T> bn = matmul(rr, bm);
  psi.sites[i + 1] = from_mat(bn, {k, b.dim(1), b.dim(2)});
}
template <class T>
void push_left(MPS<T>& psi, int i) {
  Tensor<T>& a = psi.sites[i];
  long l = a.dim(0), d = a.dim(1), r = a.dim(2);
  Mat<T> m = adjoint(to_mat(a, l, d * r)), q, rr;
  qr_thin(m, q, rr);
  long k = std::min(d * r, l);
  psi.sites[i] = from_mat(adjoint(q), {k, d, r});
  Tensor<T>& b = psi.sites[i - 1];
  Mat<T> bm = to_mat(b, b.dim(0) * b.dim(1), b.dim(2));
  Mat<T> bn = matmul(bm, adjoint(rr));
  psi.sites[i - 1] = from_mat(bn, {b.dim(0), b.dim(1), k});
}
template <class T>
void canonicalize(MPS<T>& psi, int center) {
  const int n = psi.size();
  if (center < 0 || center >= n) fail(E_INVALID_RANK, "canonicalize: center out of range");
  for (int i = 0; i < center; ++i) push_right(psi, i);
  for (int i = n - 1; i > center; --i) push_left(psi, i);
  psi.center = center;
}

// random_mps (mps.cpp:60-95): complex Gaussian, mt19937_64 + normal_distribution
inline std::vector<int> capped_bond_dims(int n, int d, int chi) {
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
inline MPS<cd> random_mps(int n, int d, int chi, uint64_t seed) {
  if (chi < 1) fail(E_INVALID_RANK, "random_mps: chi must be >= 1");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  auto dims = capped_bond_dims(n, d, chi);
  MPS<cd> psi;
  for (int i = 0; i < n; ++i) {
    long l = i == 0 ? 1 : dims[i - 1];
    long r = i == n - 1 ? 1 : dims[i];
    Tensor<cd> t({l, d, r});
    for (long k = 0; k < t.size(); ++k) {
      // mps.cpp:86 writes Cplx(gauss(rng), gauss(rng)); the order of the two
      // draws is unspecified in C++ and g++ (the reference's toolchain)
      // evaluates constructor arguments right to left: the imaginary part is
      // the first draw (checked with g++ here)
      double im = gauss(rng);
      double re = gauss(rng);
      t.data[k] = cd(re, im);
    }
    psi.sites.push_back(std::move(t));
  }
  canonicalize(psi, 0);
  double nrm = psi.sites[0].norm();
  if (!(nrm > 0)) fail(E_NUMERICAL_FAILURE, "random_mps: zero-norm state");
  for (auto& x : psi.sites[0].data) x *= 1.0 / nrm;
  return psi;
}

// Real-valued variant of random_mps for the real FP64 path: the same
// mt19937_64(seed) normal sequence, one draw per entry (not part of the
// reference; the product path's ACHI_INIT_RANDOM_REAL mirrors it).
template <class T>
MPS<T> random_mps_real(int n, int d, int chi, uint64_t seed) {
  if (chi < 1) fail(E_INVALID_RANK, "random_mps: chi must be >= 1");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  auto dims = capped_bond_dims(n, d, chi);
  MPS<T> psi;
  for (int i = 0; i < n; ++i) {
    long l = i == 0 ? 1 : dims[i - 1];
    long r = i == n - 1 ? 1 : dims[i];
    Tensor<T> t({l, d, r});
    for (long k = 0; k < t.size(); ++k) t.data[k] = T(gauss(rng));
    psi.sites.push_back(std::move(t));
  }
  canonicalize(psi, 0);
  double nrm = psi.sites[0].norm();
  if (!(nrm > 0)) fail(E_NUMERICAL_FAILURE, "random_mps: zero-norm state");
  for (auto& x : psi.sites[0].data) x *= 1.0 / nrm;
  return psi;
}

// ---- controller (controller.cpp:12-190) -------------------------------------
struct ControllerConfig {
  int mode = 3;  // fixed, threshold, direct, pid
  double alpha_ema = 0.3, gamma_margin = 1.2, s_target = -1.0;
  double kp = 2.0, ki = 0.1, kd = 0.5;
  double beta_predict = 0.4;
  int predictor_order = 1;  // off, linear, quadratic
  int chi_min = 2, chi_max = 64;
  int pid_scale = 0;  // additive, multiplicative
  double eps_trunc = 1e-10;
  double resolved_s_target() const {  // controller.cpp:12-15
    if (s_target >= 0) return s_target;
    return std::log(static_cast<double>(chi_max)) - 0.5;
  }
  void validate() const {  // controller.cpp:17-33
    if (chi_min < 1) fail(E_INVALID_CONFIG, "controller: chi_min must be >= 1");
    if (chi_min > chi_max) fail(E_INVALID_CONFIG, "controller: chi_min must be <= chi_max");
    if (!(alpha_ema > 0.0) || alpha_ema > 1.0) fail(E_INVALID_CONFIG, "controller: alpha_ema must lie in (0, 1]");
    if (gamma_margin < 1.0) fail(E_INVALID_CONFIG, "controller: gamma_margin must be >= 1");
    if (beta_predict < 0.0) fail(E_INVALID_CONFIG, "controller: beta_predict must be >= 0");
    if (!(eps_trunc >= 0.0)) fail(E_INVALID_CONFIG, "controller: eps_trunc must be >= 0");
    if (kp < 0 || ki < 0 || kd < 0 || !std::isfinite(kp) || !std::isfinite(ki) || !std::isfinite(kd))
      fail(E_INVALID_CONFIG, "controller: gains must be finite and >= 0");
  }
};

struct BondState {
  double ema = 0, prev_error = 0, integral = 0;
  double history[3] = {0, 0, 0};
  int chi = 1, history_len = 0;
  bool initialized = false;
  void push_history(double v) {  // controller.cpp:35-42
    if (history_len < 3) {
      history[history_len++] = v;
    } else {
      history[0] = history[1];
      history[1] = history[2];
      history[2] = v;
    }
  }
  double history_at(int back) const { return history[history_len - 1 - back]; }
};

struct Decision {
  int chi = 0;
  double s_raw = 0, s_ema = 0, s_pred = 0, error = 0, p_term = 0, i_term = 0, d_term = 0;
  long delta_chi = 0;
  bool clamped = false;
};

inline void ema_update(BondState& st, double s_raw, double alpha) {  // controller.cpp:49-60
  if (!(alpha > 0.0) || alpha > 1.0) fail(E_INVALID_CONFIG, "ema_update: alpha must lie in (0, 1]");
  if (s_raw < 0) fail(E_INVALID_CONFIG, "ema_update: entropy must be >= 0");
  if (!st.initialized) {
    st.ema = s_raw;
    st.initialized = true;
  } else {
    st.ema = alpha * s_raw + (1.0 - alpha) * st.ema;
  }
  st.push_history(st.ema);
}

inline int chi_target_direct(double s, double gamma, int chi_min, int chi_max) {  // :71-82
  if (s < 0) fail(E_INVALID_CONFIG, "chi_target_direct: entropy must be >= 0");
  if (gamma < 1.0) fail(E_INVALID_CONFIG, "chi_target_direct: gamma must be >= 1");
  double target = std::ceil(gamma * std::exp(s) - 1e-9);
  double c = std::clamp(target, static_cast<double>(chi_min), static_cast<double>(chi_max));
  return static_cast<int>(c);
}

inline Decision pid_step(BondState& st, double s_input, const ControllerConfig& cfg) {  // :84-117
  if (!st.initialized) fail(E_INVALID_CONFIG, "pid_step: state not initialized (no EMA update yet)");
  Decision d;
  d.s_ema = st.ema;
  d.s_pred = s_input;
  d.error = s_input - cfg.resolved_s_target();
  d.p_term = cfg.kp * d.error;
  st.integral += cfg.ki * d.error;
  d.i_term = st.integral;
  d.d_term = cfg.kd * (d.error - st.prev_error);
  double u = d.p_term + d.i_term + d.d_term;
  long raw;
  if (cfg.pid_scale == 0) {
    d.delta_chi = std::llround(u);
    raw = st.chi + d.delta_chi;
  } else {
    raw = std::llround(st.chi * (1.0 + u / 10.0));
    d.delta_chi = raw - st.chi;
  }
  long cl = std::clamp<long>(raw, cfg.chi_min, cfg.chi_max);
  d.clamped = cl != raw;
  if (d.clamped) {
    st.integral -= cfg.ki * d.error;
    d.i_term = st.integral;
  }
  st.prev_error = d.error;
  st.chi = static_cast<int>(cl);
  d.chi = st.chi;
  return d;
}

inline double predict_entropy(const BondState& st, double beta, int order, bool* fallback) {  // :119-132
  const int need = order == 2 ? 3 : 2;
  if (order == 0 || st.history_len < need) {
    if (fallback) *fallback = true;
    return st.ema;
  }
  double s0 = st.history_at(0), s1 = st.history_at(1);
  double v = s0 + beta * (s0 - s1);
  if (order == 2) v += beta * (s0 - 2.0 * s1 + st.history_at(2));
  if (fallback) *fallback = false;
  return std::max(0.0, v);
}

// rank_for_discarded_weight (controller.cpp:134-148); margin = relative distance to threshold
inline int rank_for_discarded_weight(const std::vector<double>& v, double eps, double* margin = nullptr) {
  const long n = static_cast<long>(v.size());
  if (n == 0) fail(E_DEGENERATE, "rank_for_discarded_weight: empty");
  double total = 0;
  for (double x : v) total += x * x;
  if (!(total > 0)) fail(E_DEGENERATE, "rank_for_discarded_weight: all-zero spectrum");
  double tail = 0, thr = eps * total;
  double m = std::numeric_limits<double>::infinity();
  for (long k = n - 1; k >= 1; --k) {
    tail += v[k] * v[k];
    if (thr > 0) m = std::min(m, std::abs(tail - thr) / thr);
    if (tail > thr) {
      if (margin) *margin = m;
      return static_cast<int>(k + 1);
    }
  }
  if (margin) *margin = m;
  return 1;
}

inline Decision controller_update(BondState& st, const std::vector<double>& spec,
                                  const ControllerConfig& cfg) {  // :150-190
  double s_raw = entropy_from_spectrum(spec);
  ema_update(st, s_raw, cfg.alpha_ema);
  double s_in = predict_entropy(st, cfg.beta_predict, cfg.predictor_order, nullptr);
  Decision d;
  switch (cfg.mode) {
    case 0:
      d.chi = cfg.chi_max;
      st.chi = d.chi;
      break;
    case 1: {
      int r = rank_for_discarded_weight(spec, cfg.eps_trunc);
      d.chi = std::clamp(r, cfg.chi_min, cfg.chi_max);
      st.chi = d.chi;
      break;
    }
    case 2:
      d.chi = chi_target_direct(s_in, cfg.gamma_margin, cfg.chi_min, cfg.chi_max);
      st.chi = d.chi;
      break;
    default:
      d = pid_step(st, s_in, cfg);
      break;
  }
  d.s_raw = s_raw;
  d.s_ema = st.ema;
  d.s_pred = s_in;
  return d;
}

// ---- models (models.cpp:19-109) ----------------------------------------------
struct ModelSpec {
  int family = 0;  // heisenberg_xxz, transverse_ising
  int n = 2;
  double jx = 1, jy = 1, jz = 1, h = 0;
  int convention = 1;  // spin_half, pauli
  void validate() const {
    if (n < 2) fail(E_INVALID_CONFIG, "model: n must be >= 2");
    if (!std::isfinite(jx) || !std::isfinite(jy) || !std::isfinite(jz) || !std::isfinite(h))
      fail(E_INVALID_CONFIG, "model: couplings must be finite");
  }
};

// real_gauge: Y -> iY = [[0,1],[-1,0]] and jy*Y -> -jy*iY: same H, real W.
template <class T>
std::vector<Tensor<T>> build_mpo(const ModelSpec& spec, bool real_gauge) {
  spec.validate();
  const double sc = spec.convention == 0 ? 0.5 : 1.0;
  using Op = std::array<T, 4>;  // (so, si) row-major
  Op id{T(1), T(0), T(0), T(1)};
  Op x{T(0), T(sc), T(sc), T(0)};
  Op z{T(sc), T(0), T(0), T(-sc)};
  Op y_in{}, y_out{};
  if (real_gauge) {
    y_in = Op{T(0), T(sc), T(-sc), T(0)};
    for (int i = 0; i < 4; ++i) y_out[i] = -spec.jy * y_in[i];
  } else {
    if constexpr (std::is_same_v<T, double>) {
      if (spec.family == 0 && spec.jy != 0)
        fail(E_UNSUPPORTED, "build_mpo: complex sigma^y channel needs complex arithmetic");
    } else {
      y_in = Op{T(0), T(cd(0, -sc)), T(cd(0, sc)), T(0)};
      for (int i = 0; i < 4; ++i) y_out[i] = spec.jy * y_in[i];
    }
  }
  long w;
  Tensor<T> bulk;
  auto put = [&](long row, long col, const Op& op) {
    for (long so = 0; so < 2; ++so)
      for (long si = 0; si < 2; ++si) bulk(row, so, si, col) = op[so * 2 + si];
  };
  auto scaled = [](const Op& op, double f) {
    Op o;
    for (int i = 0; i < 4; ++i) o[i] = f * op[i];
    return o;
  };
  if (spec.family == 0) {
    w = 5;
    bulk = Tensor<T>({w, 2, 2, w});
    put(0, 0, id);
    put(1, 0, x);
    put(2, 0, y_in);
    put(3, 0, z);
    put(4, 0, scaled(z, -spec.h));
    put(4, 1, scaled(x, spec.jx));
    put(4, 2, y_out);
    put(4, 3, scaled(z, spec.jz));
    put(4, 4, id);
  } else if (spec.family == 1) {
    w = 3;
    bulk = Tensor<T>({w, 2, 2, w});
    put(0, 0, id);
    put(1, 0, z);
    put(2, 0, scaled(x, -spec.h));
    put(2, 1, scaled(z, -spec.jz));
    put(2, 2, id);
  } else {
    fail(E_UNSUPPORTED, "build_mpo: unknown model family");
  }
  Tensor<T> first({1, 2, 2, w}), last({w, 2, 2, 1});
  for (long so = 0; so < 2; ++so)
    for (long si = 0; si < 2; ++si) {
      for (long c = 0; c < w; ++c) first(0, so, si, c) = bulk(w - 1, so, si, c);
      for (long r = 0; r < w; ++r) last(r, so, si, 0) = bulk(r, so, si, 0);
    }
  std::vector<Tensor<T>> sites;
  sites.push_back(first);
  for (int i = 1; i < spec.n - 1; ++i) sites.push_back(bulk);
  sites.push_back(last);
  return sites;
}

template <class T>
std::vector<Tensor<T>> identity_mpo(int n, int d) {  // models.cpp:99-109
  std::vector<Tensor<T>> s;
  for (int i = 0; i < n; ++i) {
    Tensor<T> t({1, d, d, 1});
    for (long k = 0; k < d; ++k) t(0, k, k, 0) = T(1);
    s.push_back(t);
  }
  return s;
}

// matrix-free XXZ exact ground energy (models.cpp:177-223): Lanczos tol 1e-12, 800 matvecs
inline double exact_ground_energy_xxz(const ModelSpec& spec, int cap) {
  spec.validate();
  if (spec.n > cap) fail(E_SIZE_GUARD, "exact_ground_energy: n exceeds the Lanczos tier cap");
  const double s2 = spec.convention == 1 ? 1.0 : 0.25, sf = spec.convention == 1 ? 1.0 : 0.5;
  const long dim = 1L << spec.n;
  const double flip = (spec.jx + spec.jy) * s2, raise = (spec.jx - spec.jy) * s2;
  auto apply = [&](const std::vector<cd>& in, std::vector<cd>& out) {
    std::fill(out.begin(), out.end(), cd(0));
    for (long idx = 0; idx < dim; ++idx) {
      double diag = 0;
      for (int i = 0; i + 1 < spec.n; ++i) {
        bool si = (idx >> i) & 1, sj = (idx >> (i + 1)) & 1;
        diag += spec.jz * s2 * (si == sj ? 1.0 : -1.0);
        long f = idx ^ (3L << i);
        if (si != sj) {
          if (flip != 0) out[f] += flip * in[idx];
        } else if (raise != 0) {
          out[f] += raise * in[idx];
        }
      }
      for (int i = 0; i < spec.n; ++i) diag -= spec.h * sf * (((idx >> i) & 1) ? -1.0 : 1.0);
      out[idx] += diag * in[idx];
    }
  };
  std::mt19937_64 rng(12345);
  std::normal_distribution<double> g(0.0, 1.0);
  std::vector<cd> v0(dim);
  for (long i = 0; i < dim; ++i) v0[i] = cd(g(rng), 0.0);
  return eigs_lowest<cd>(apply, dim, v0, 1e-12, 800).eigenvalue;
}

// ---- DMRG (dmrg.cpp) ---------------------------------------------------------
struct DmrgConfig {
  int max_sweeps = 24;
  double eps_conv = 1e-8, eig_tol = 1e-10;
  int eig_max_iter = 200;
  ControllerConfig controller{};
  int initial_state = 0;  // automatic, neel, random
  uint64_t seed = 1234;
  double noise_floor = 1e-14;
  void validate() const {  // dmrg.cpp:8-16
    if (max_sweeps < 1) fail(E_INVALID_CONFIG, "dmrg: max_sweeps must be >= 1");
    if (!(eps_conv > 0)) fail(E_INVALID_CONFIG, "dmrg: eps_conv must be > 0");
    if (!(eig_tol > 0)) fail(E_INVALID_CONFIG, "dmrg: eig_tol must be > 0");
    if (eig_max_iter < 1) fail(E_INVALID_CONFIG, "dmrg: eig_max_iter must be >= 1");
    controller.validate();
  }
};

template <class T>
struct Environment {  // dmrg.cpp:18-56
  std::vector<Tensor<T>> left, right;
  explicit Environment(int n) : left(n), right(n) {
    Tensor<T> triv({1, 1, 1});
    triv.data[0] = T(1);
    left[0] = triv;
    right[n - 1] = triv;
  }
  void update_left(int k, const MPS<T>& psi, const std::vector<Tensor<T>>& mpo) {
    const Tensor<T>& l = left[k - 1];
    const Tensor<T>& a = psi.sites[k - 1];
    const Tensor<T>& w = mpo[k - 1];
    Tensor<T> t = l.contract({2}, a, {0});
    t = t.contract({1, 2}, w, {0, 2});
    t = a.conjugated().contract({0, 1}, t, {0, 2});
    left[k] = t.permuted({0, 2, 1});
  }
  void update_right(int k, const MPS<T>& psi, const std::vector<Tensor<T>>& mpo) {
    const Tensor<T>& r = right[k + 1];
    const Tensor<T>& a = psi.sites[k + 1];
    const Tensor<T>& w = mpo[k + 1];
    Tensor<T> t = a.contract({2}, r, {2});
    t = t.contract({1, 3}, w, {2, 3});
    t = a.conjugated().contract({1, 2}, t, {3, 1});
    right[k] = t.permuted({0, 2, 1});
  }
  void rebuild(const MPS<T>& psi, const std::vector<Tensor<T>>& mpo, int center) {
    for (int k = 1; k <= center; ++k) update_left(k, psi, mpo);
    for (int k = psi.size() - 2; k >= center; --k) update_right(k, psi, mpo);
  }
};

template <class T>
Tensor<T> apply_effective_hamiltonian(const Tensor<T>& l, const Tensor<T>& w1, const Tensor<T>& w2,
                                      const Tensor<T>& r, const Tensor<T>& theta) {  // dmrg.cpp:58-71
  Tensor<T> t = l.contract({2}, theta, {0});
  t = t.contract({1, 2}, w1, {0, 2});
  t = t.contract({4, 1}, w2, {0, 2});
  t = t.contract({4, 1}, r, {1, 2});
  return t;
}

struct VisitLog {
  int sweep, bond, moving_right, kept, floor_rank, significant, n_sigma, matvecs, degenerate_cut;
  double energy, entropy, trunc_error, floor_margin, sigma_kept, sigma_next, residual;
};
struct TraceRow {
  int sweep, bond;
  Decision d;
};
struct SweepRecord {
  int sweep_index = 0;
  double energy = 0, delta_e_rel = 0;
  std::vector<int> chi_profile;
  std::vector<double> entropy_profile;
  double max_trunc_error = 0, wall_time = 0;
  long parameter_count = 0;
  double average_chi = 0;
  int max_chi_used = 0;
};

template <class T>
struct DmrgRun {
  std::vector<SweepRecord> sweeps;
  std::vector<TraceRow> trace;
  std::vector<VisitLog> visits;
  bool converged = false;
  double energy = 0, max_monotonicity_violation = 0;
  int max_chi_used = 0;
  MPS<T> psi;
};

// visit_bond (dmrg.cpp:84-171)
template <class T>
VisitLog visit_bond(MPS<T>& psi, const std::vector<Tensor<T>>& mpo, Environment<T>& env,
                    const DmrgConfig& cfg, std::vector<BondState>& states, int bond,
                    bool moving_right, int sweep, std::vector<TraceRow>* trace) {
  const long d = psi.phys_dim();
  const long chl = psi.sites[bond].dim(0), chr = psi.sites[bond + 1].dim(2);
  Tensor<T> theta0 = psi.sites[bond].contract({2}, psi.sites[bond + 1], {0});
  Tensor<T> tin({chl, d, d, chr});
  auto apply = [&](const std::vector<T>& in, std::vector<T>& out) {
    tin.data = in;
    Tensor<T> tout = apply_effective_hamiltonian(env.left[bond], mpo[bond], mpo[bond + 1],
                                                 env.right[bond + 1], tin);
    out = tout.data;
  };
  EigsResult<T> eig = eigs_lowest<T>(apply, theta0.size(), theta0.data, cfg.eig_tol, cfg.eig_max_iter);
  Mat<T> theta(chl * d, d * chr);
  for (long i = 0; i < chl * d; ++i)
    for (long j = 0; j < d * chr; ++j) theta(i, j) = eig.eigenvector[i * d * chr + j];
  BondState& st = states[bond];
  const ControllerConfig& cc = cfg.controller;
  int request = st.chi;
  SvdResult<T> svd = svd_full(theta);
  double s1 = svd.sigma.empty() ? 0.0 : svd.sigma[0];
  if (!(s1 > 0)) fail(E_DEGENERATE, "dmrg: zero two-site block");
  VisitLog log{};
  int floor_rank = rank_for_discarded_weight(svd.sigma, cc.eps_trunc, &log.floor_margin);
  int kept = cc.mode == 0 ? cc.chi_max : std::clamp(std::max(request, floor_rank), cc.chi_min, cc.chi_max);
  int significant = 0;
  for (double s : svd.sigma) if (s > cfg.noise_floor * s1) ++significant;
  if (cc.mode != 0) kept = std::min(kept, std::max(significant, 1));
  kept = std::min<long>(kept, static_cast<long>(svd.sigma.size()));
  kept = std::max(kept, 1);
  Decision dec = controller_update(st, svd.sigma, cc);
  if (trace) trace->push_back({sweep, bond, dec});
  long r = svd.rank;
  Mat<T> u(chl * d, kept), vt(kept, d * chr);
  std::vector<double> lam(svd.sigma.begin(), svd.sigma.begin() + kept);
  double ln = 0;
  for (double x : lam) ln += x * x;
  ln = std::sqrt(ln);
  if (!(ln > 0)) fail(E_DEGENERATE, "dmrg: empty truncation");
  for (auto& x : lam) x /= ln;
  for (long j = 0; j < kept; ++j)
    for (long i = 0; i < chl * d; ++i) u(i, j) = svd.u(i, j) * (moving_right ? 1.0 : lam[j]);
  for (long c = 0; c < d * chr; ++c)
    for (long i = 0; i < kept; ++i) vt(i, c) = svd.vt(i, c) * (moving_right ? lam[i] : 1.0);
  psi.sites[bond] = from_mat(u, {chl, d, kept});
  psi.sites[bond + 1] = from_mat(vt, {kept, d, chr});
  psi.center = moving_right ? bond + 1 : bond;
  if (moving_right)
    env.update_left(bond + 1, psi, mpo);
  else
    env.update_right(bond, psi, mpo);
  log.sweep = sweep;
  log.bond = bond;
  log.moving_right = moving_right;
  log.kept = kept;
  log.floor_rank = floor_rank;
  log.significant = significant;
  log.n_sigma = static_cast<int>(r);
  log.matvecs = eig.matvec_count;
  log.degenerate_cut = kept < r && std::abs(svd.sigma[kept - 1] - svd.sigma[kept]) <= 1e-12 * s1;
  log.energy = eig.eigenvalue;
  log.entropy = entropy_from_spectrum(svd.sigma);
  log.trunc_error = truncation_error(svd.sigma, kept);
  log.sigma_kept = svd.sigma[kept - 1] / s1;
  log.sigma_next = kept < r ? svd.sigma[kept] / s1 : 0.0;
  log.residual = eig.residual;
  return log;
}

// two_site_sweep (dmrg.cpp:175-214)
template <class T>
SweepRecord two_site_sweep(MPS<T>& psi, const std::vector<Tensor<T>>& mpo, Environment<T>& env,
                           const DmrgConfig& cfg, std::vector<BondState>& states, int sweep,
                           std::vector<TraceRow>* trace, std::vector<VisitLog>* visits) {
  const int n = psi.size();
  SweepRecord rec;
  rec.sweep_index = sweep;
  rec.entropy_profile.assign(n - 1, 0.0);
  double energy = 0;
  auto t0 = std::chrono::steady_clock::now();
  auto one = [&](int bond, bool right) {
    VisitLog v = visit_bond(psi, mpo, env, cfg, states, bond, right, sweep, trace);
    energy = v.energy;
    rec.max_chi_used = std::max(rec.max_chi_used, v.kept);
    rec.max_trunc_error = std::max(rec.max_trunc_error, v.trunc_error);
    rec.entropy_profile[bond] = v.entropy;
    if (visits) visits->push_back(v);
  };
  for (int b = 0; b <= n - 2; ++b) one(b, true);
  for (int b = n - 2; b >= 0; --b) one(b, false);
  auto t1 = std::chrono::steady_clock::now();
  rec.wall_time = std::chrono::duration<double>(t1 - t0).count();
  rec.energy = energy;
  rec.chi_profile = psi.bond_dims();
  long pc = 0;
  for (const auto& s : psi.sites) pc += s.dim(0) * s.dim(1) * s.dim(2);
  rec.parameter_count = pc;
  double avg = 0;
  for (int x : rec.chi_profile) avg += x;
  rec.average_chi = avg / static_cast<double>(rec.chi_profile.size());
  return rec;
}

template <class T>
void init_run(const ModelSpec& spec, const DmrgConfig& cfg, MPS<T>& psi) {
  int init = cfg.initial_state;
  // automatic (dmrg.cpp:222-225): TFIM -> random; on the real path random_real
  if (init == 0) init = spec.family == 0 ? 1 : (std::is_same_v<T, cd> ? 2 : 3);
  if (init == 3) {
    psi = random_mps_real<T>(spec.n, 2, cfg.controller.chi_min, cfg.seed);
  } else if (init == 1) {
    std::vector<int> basis(spec.n);
    for (int i = 0; i < spec.n; ++i) basis[i] = i % 2;
    psi = product_state<T>(spec.n, 2, basis);
  } else {
    if constexpr (std::is_same_v<T, cd>) {
      psi = random_mps(spec.n, 2, cfg.controller.chi_min, cfg.seed);
    } else {
      fail(E_UNSUPPORTED, "random complex initial state needs complex arithmetic");
    }
  }
  canonicalize(psi, 0);
}

// run_dmrg (dmrg.cpp:216-282); max_sweeps_override < 0 -> cfg.max_sweeps
template <class T>
DmrgRun<T> run_dmrg(const ModelSpec& spec, const DmrgConfig& cfg, bool real_gauge) {
  spec.validate();
  cfg.validate();
  auto mpo = build_mpo<T>(spec, real_gauge);
  DmrgRun<T> out;
  MPS<T> psi;
  init_run(spec, cfg, psi);
  Environment<T> env(spec.n);
  env.rebuild(psi, mpo, 0);
  std::vector<BondState> states(spec.n - 1);
  for (auto& st : states) {
    st.chi = cfg.controller.chi_min;
    st.ema = 0.0;
    st.initialized = true;
    st.push_history(0.0);
  }
  double prev = 0;
  bool have_prev = false;
  for (int sweep = 0; sweep < cfg.max_sweeps; ++sweep) {
    SweepRecord rec = two_site_sweep(psi, mpo, env, cfg, states, sweep, &out.trace, &out.visits);
    out.max_chi_used = std::max(out.max_chi_used, rec.max_chi_used);
    if (have_prev) {
      double delta = rec.energy - prev;
      rec.delta_e_rel = std::abs(delta) / std::max(std::abs(rec.energy), 1e-300);
      if (delta > 0) out.max_monotonicity_violation = std::max(out.max_monotonicity_violation, delta);
    } else {
      rec.delta_e_rel = std::numeric_limits<double>::infinity();
    }
    out.sweeps.push_back(rec);
    if (have_prev && rec.delta_e_rel < cfg.eps_conv) {
      out.converged = true;
      prev = rec.energy;
      break;
    }
    prev = rec.energy;
    have_prev = true;
  }
  out.energy = prev;
  out.psi = std::move(psi);
  return out;
}

}  // namespace oracle
