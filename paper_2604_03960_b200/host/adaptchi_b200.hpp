// adaptchi_b200.hpp — C++ host mirror of the reference interface over the C-ABI.
//
// Header-only, C++17.  Names, argument meaning, defaults and exception types
// follow /root/reference/proj/include/adaptchi/{errors,models,controller,mps,
// linalg,dmrg,tensor}.hpp so that reference-style code and tests compile
// against the B200 backend with a changed include.  Eigen types are replaced
// by small value types with the reference's scalar type: DenseMatrix is a
// complex column-major matrix (Eigen::MatrixXcd), CVector a complex vector;
// real-valued blocks take the real FP64 device path, complex ones the complex
// device SVD / the realified Lanczos.  Every computation runs
// on the GPU through include/adaptchi_b200.h; there is no host fallback.
#pragma once

#include <cmath>
#include <complex>
#include <functional>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../../include/adaptchi_b200.h"

namespace adaptchi {

// ---- errors.hpp:8-59 --------------------------------------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidMatrix : Error { using Error::Error; };
struct NumericalFailure : Error { using Error::Error; };
struct InvalidRank : Error { using Error::Error; };
struct EigenNonConvergence : Error {
  double best_residual;
  EigenNonConvergence(const std::string& m, double r) : Error(m), best_residual(r) {}
};
struct InvalidBasisState : Error { using Error::Error; };
struct SizeGuard : Error { using Error::Error; };
struct DegenerateSpectrum : Error { using Error::Error; };
struct UnsupportedModel : Error { using Error::Error; };
struct InvalidConfig : Error { using Error::Error; };
struct InternalConsistency : Error { using Error::Error; };

namespace b200 {

// One process-wide context on device 0 (a DMRG run is sequential).
class Device {
 public:
  static Device& get() {
    static Device d;
    return d;
  }
  achi_ctx* ctx() const { return ctx_; }
  ~Device() {
    if (ctx_) achi_ctx_destroy(ctx_);
  }

 private:
  Device() {
    if (achi_ctx_create(0, &ctx_) != ACHI_OK) throw Error("adaptchi_b200: no sm_100 device");
  }
  achi_ctx* ctx_ = nullptr;
};

[[noreturn]] inline void rethrow(int rc) {
  achi_ctx* ctx = Device::get().ctx();
  char msg[1024];
  achi_last_error(ctx, msg, sizeof msg);
  switch (rc) {
    case ACHI_E_INVALID_MATRIX: throw InvalidMatrix(msg);
    case ACHI_E_NUMERICAL_FAILURE: throw NumericalFailure(msg);
    case ACHI_E_INVALID_RANK: throw InvalidRank(msg);
    case ACHI_E_EIGEN_NONCONVERGENCE: throw EigenNonConvergence(msg, achi_last_residual(ctx));
    case ACHI_E_INVALID_BASIS_STATE: throw InvalidBasisState(msg);
    case ACHI_E_SIZE_GUARD: throw SizeGuard(msg);
    case ACHI_E_DEGENERATE_SPECTRUM: throw DegenerateSpectrum(msg);
    case ACHI_E_UNSUPPORTED_MODEL: throw UnsupportedModel(msg);
    case ACHI_E_INVALID_CONFIG: throw InvalidConfig(msg);
    case ACHI_E_INTERNAL: throw InternalConsistency(msg);
    default: throw Error(msg);
  }
}
inline void check(int rc) {
  if (rc != ACHI_OK) rethrow(rc);
}

}  // namespace b200

// tensor.hpp:14-17
using Cplx = std::complex<double>;
using CVector = std::vector<Cplx>;
using RVector = std::vector<double>;

// Complex column-major dense matrix (stands in for Eigen::MatrixXcd, tensor.hpp:15).
struct DenseMatrix {
  long r = 0, c = 0;
  std::vector<Cplx> d;
  DenseMatrix() = default;
  DenseMatrix(long rows, long cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols), Cplx(0, 0)) {}
  static DenseMatrix Identity(long n, long m) {
    DenseMatrix x(n, m);
    for (long i = 0; i < std::min(n, m); ++i) x(i, i) = 1.0;
    return x;
  }
  long rows() const { return r; }
  long cols() const { return c; }
  Cplx& operator()(long i, long j) { return d[static_cast<size_t>(i + j * r)]; }
  Cplx operator()(long i, long j) const { return d[static_cast<size_t>(i + j * r)]; }
  bool is_real() const {
    for (const Cplx& x : d)
      if (x.imag() != 0.0) return false;
    return true;
  }
  std::vector<double> real_row_major() const {
    std::vector<double> o(d.size());
    for (long i = 0; i < r; ++i)
      for (long j = 0; j < c; ++j) o[static_cast<size_t>(i * c + j)] = (*this)(i, j).real();
    return o;
  }
  std::vector<double> interleaved_row_major() const {
    std::vector<double> o(2 * d.size());
    for (long i = 0; i < r; ++i)
      for (long j = 0; j < c; ++j) {
        o[static_cast<size_t>(2 * (i * c + j))] = (*this)(i, j).real();
        o[static_cast<size_t>(2 * (i * c + j) + 1)] = (*this)(i, j).imag();
      }
    return o;
  }
  static DenseMatrix from_real_row_major(long rows, long cols, const double* p) {
    DenseMatrix x(rows, cols);
    for (long i = 0; i < rows; ++i)
      for (long j = 0; j < cols; ++j) x(i, j) = p[i * cols + j];
    return x;
  }
  static DenseMatrix from_interleaved_row_major(long rows, long cols, const double* p) {
    DenseMatrix x(rows, cols);
    for (long i = 0; i < rows; ++i)
      for (long j = 0; j < cols; ++j) x(i, j) = Cplx(p[2 * (i * cols + j)], p[2 * (i * cols + j) + 1]);
    return x;
  }
};

// Row-major complex tensor of small rank (tensor.hpp:26-120; contractions run
// on the device through the mirror's operations, not here).
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<long> shape) : shape_(std::move(shape)), data_(size_of(shape_), Cplx(0, 0)) {}
  static size_t size_of(const std::vector<long>& shape) {
    long n = 1;
    for (long s : shape) {
      if (s < 1) throw InvalidMatrix("tensor dimension must be >= 1");
      n *= s;
    }
    return static_cast<size_t>(n);
  }
  const std::vector<long>& shape() const { return shape_; }
  long dim(int axis) const { return shape_[static_cast<size_t>(axis)]; }
  int rank() const { return static_cast<int>(shape_.size()); }
  long size() const { return static_cast<long>(data_.size()); }
  Cplx* data() { return data_.data(); }
  const Cplx* data() const { return data_.data(); }
  Cplx& operator()(long i, long j, long k) { return data_[static_cast<size_t>((i * shape_[1] + j) * shape_[2] + k)]; }
  Cplx operator()(long i, long j, long k) const {
    return data_[static_cast<size_t>((i * shape_[1] + j) * shape_[2] + k)];
  }
  // row-major copy of a matrix into the given shape (tensor.hpp:105-109)
  static Tensor from_matrix(const DenseMatrix& m, std::vector<long> shape) {
    Tensor t(std::move(shape));
    if (static_cast<long>(t.data_.size()) != m.rows() * m.cols()) throw InternalConsistency("reshape size mismatch");
    for (long i = 0; i < m.rows(); ++i)
      for (long j = 0; j < m.cols(); ++j) t.data_[static_cast<size_t>(i * m.cols() + j)] = m(i, j);
    return t;
  }

 private:
  std::vector<long> shape_;
  std::vector<Cplx> data_;
};

// ---- models.hpp:7-56 ------------------------------------------------------
namespace models {
enum class ModelFamily { heisenberg_xxz, transverse_ising };
enum class SpinConvention { spin_half, pauli };
struct ModelSpec {
  ModelFamily family = ModelFamily::heisenberg_xxz;
  int n = 2;
  double jx = 1.0, jy = 1.0, jz = 1.0, h = 0.0;
  SpinConvention convention = SpinConvention::pauli;
  achi_model_spec c() const {
    return {family == ModelFamily::heisenberg_xxz ? ACHI_HEISENBERG_XXZ : ACHI_TRANSVERSE_ISING,
            n, jx, jy, jz, h, convention == SpinConvention::pauli ? ACHI_PAULI : ACHI_SPIN_HALF, 0};
  }
};
inline double bethe_reference() { return 0.25 - std::log(2.0); }  // models.cpp:261
inline double bethe_reference_pauli() { return 4.0 * bethe_reference(); }
}  // namespace models

// ---- controller.hpp:11-134 ------------------------------------------------
namespace ctrl {
enum class ControlMode { fixed, threshold, direct, pid };
enum class PredictorOrder { off, linear, quadratic };
enum class PidScale { additive, multiplicative };
struct PidGains {
  double kp = 2.0, ki = 0.1, kd = 0.5;
};
struct ControllerConfig {
  ControlMode mode = ControlMode::pid;
  double alpha_ema = 0.3;
  double gamma_margin = 1.2;
  double s_target = -1.0;
  PidGains gains{};
  double beta_predict = 0.4;
  PredictorOrder predictor_order = PredictorOrder::linear;
  int chi_min = 2;
  int chi_max = 64;
  PidScale pid_scale = PidScale::additive;
  double eps_trunc = 1e-10;
  double resolved_s_target() const {
    return s_target >= 0 ? s_target : std::log(static_cast<double>(chi_max)) - 0.5;
  }
  achi_controller_config c() const {
    return {static_cast<int32_t>(mode), static_cast<int32_t>(predictor_order), alpha_ema,
            gamma_margin, s_target, gains.kp, gains.ki, gains.kd, beta_predict, chi_min, chi_max,
            static_cast<int32_t>(pid_scale), 0, eps_trunc};
  }
};
struct BondControllerState {
  double ema = 0.0, prev_error = 0.0, integral = 0.0;
  int chi = 1;
  double history[3] = {0, 0, 0};
  int history_len = 0;
  bool initialized = false;
  achi_bond_state c() const {
    achi_bond_state s{};
    s.ema = ema;
    s.prev_error = prev_error;
    s.integral = integral;
    for (int i = 0; i < 3; ++i) s.history[i] = history[i];
    s.chi = chi;
    s.history_len = history_len;
    s.initialized = initialized ? 1 : 0;
    return s;
  }
  void from(const achi_bond_state& s) {
    ema = s.ema;
    prev_error = s.prev_error;
    integral = s.integral;
    for (int i = 0; i < 3; ++i) history[i] = s.history[i];
    chi = s.chi;
    history_len = s.history_len;
    initialized = s.initialized != 0;
  }
};
struct ControllerDecision {
  int chi = 0;
  double s_raw = 0, s_ema = 0, s_pred = 0, error = 0, p_term = 0, i_term = 0, d_term = 0;
  long delta_chi = 0;
  bool clamped = false;
};
struct TraceRow {
  int sweep = 0, bond = 0;
  ControllerDecision d{};
};
class ControllerTrace {  // controller.hpp:122-132
 public:
  void add(int sweep, int bond, const ControllerDecision& d) { rows_.push_back({sweep, bond, d}); }
  const std::vector<TraceRow>& rows() const { return rows_; }
  void write_csv(std::ostream& os) const {
    os << "sweep,bond,s_raw,s_ema,s_pred,e,P,I,D,delta_chi,chi,clamped\n";
    for (const auto& r : rows_)
      os << r.sweep << ',' << r.bond << ',' << r.d.s_raw << ',' << r.d.s_ema << ',' << r.d.s_pred
         << ',' << r.d.error << ',' << r.d.p_term << ',' << r.d.i_term << ',' << r.d.d_term << ','
         << r.d.delta_chi << ',' << r.d.chi << ',' << (r.d.clamped ? 1 : 0) << '\n';
  }

 private:
  std::vector<TraceRow> rows_;
};
inline ControllerDecision from_c(const achi_trace_row& t) {
  ControllerDecision d;
  d.chi = t.chi;
  d.s_raw = t.s_raw;
  d.s_ema = t.s_ema;
  d.s_pred = t.s_pred;
  d.error = t.error;
  d.p_term = t.p_term;
  d.i_term = t.i_term;
  d.d_term = t.d_term;
  d.delta_chi = static_cast<long>(t.delta_chi);
  d.clamped = t.clamped != 0;
  return d;
}
}  // namespace ctrl

// ---- mps.hpp spectrum helpers (mps.cpp:97-122) ------------------------------
namespace mps {
struct SingularSpectrum {
  RVector values;
  int bond_index = -1;
};
inline double entropy_from_spectrum(const SingularSpectrum& s) {
  double out[4];
  b200::check(achi_spectrum_stats(b200::Device::get().ctx(), static_cast<int>(s.values.size()),
                                  s.values.data(), 1, 0.0, out));
  return out[0];
}
inline double truncation_error(const SingularSpectrum& s, int kept) {
  double out[4];
  b200::check(achi_spectrum_stats(b200::Device::get().ctx(), static_cast<int>(s.values.size()),
                                  s.values.data(), kept, 0.0, out));
  return out[1];
}
}  // namespace mps

namespace ctrl {
// rank_for_discarded_weight (controller.cpp:134-148) on the device
inline int rank_for_discarded_weight(const RVector& values, double eps) {
  double out[4];
  b200::check(achi_spectrum_stats(b200::Device::get().ctx(), static_cast<int>(values.size()),
                                  values.data(), 1, eps, out));
  return static_cast<int>(out[2]);
}
// controller_update (controller.cpp:150-190) through the fused K7 kernel
inline ControllerDecision controller_update(BondControllerState& state,
                                            const mps::SingularSpectrum& spectrum,
                                            const ControllerConfig& cfg) {
  achi_dmrg_config dc{};
  dc.noise_floor = 1e-14;
  dc.controller = cfg.c();
  achi_bond_state st = state.c();
  achi_trace_row row{};
  b200::check(achi_bond_select(b200::Device::get().ctx(), &dc,
                               static_cast<int>(spectrum.values.size()), spectrum.values.data(),
                               &st, 0, spectrum.bond_index, &row, nullptr));
  state.from(st);
  return from_c(row);
}
}  // namespace ctrl

// ---- linalg.hpp:9-80 --------------------------------------------------------
namespace linalg {
struct SvdResult {
  DenseMatrix u;      // m x r
  RVector sigma;      // r, non-increasing
  DenseMatrix v_dagger;  // r x n
  long rank = 0;
  bool degenerate_cut = false;
};
enum class BackendId { reference, external };
struct BackendPolicy {
  long accelerator_threshold = 64;
  BackendId preferred = BackendId::external;
};
class SvdBackend {
 public:
  virtual ~SvdBackend() = default;
  virtual SvdResult svd(const DenseMatrix& m) const = 0;
  virtual std::string_view name() const = 0;
};

// svd_full (linalg.cpp:67-70) on the GPU Jacobi kernel, fix_phases convention
// (linalg.cpp:19-35).  A block with an all-zero imaginary part takes the real
// FP64 path (achi_svd: real factors, the same convention); any other complex
// block the complex path (achi_svd_complex).  Non-finite entries ->
// InvalidMatrix (check_input, linalg.cpp:11-15).
inline SvdResult svd_full(const DenseMatrix& m) {
  if (m.rows() < 1 || m.cols() < 1) throw InvalidMatrix("svd: matrix must be at least 1x1");
  const long r = std::min(m.rows(), m.cols());
  SvdResult out;
  out.sigma.assign(static_cast<size_t>(r), 0.0);
  out.rank = r;
  int sweeps = 0;
  if (m.is_real()) {
    std::vector<double> a = m.real_row_major(), u(static_cast<size_t>(m.rows() * r)),
                        vt(static_cast<size_t>(r * m.cols()));
    b200::check(achi_svd(b200::Device::get().ctx(), static_cast<int>(m.rows()),
                         static_cast<int>(m.cols()), a.data(), out.sigma.data(), u.data(), vt.data(),
                         &sweeps));
    out.u = DenseMatrix::from_real_row_major(m.rows(), r, u.data());
    out.v_dagger = DenseMatrix::from_real_row_major(r, m.cols(), vt.data());
  } else {
    std::vector<double> a = m.interleaved_row_major(), u(static_cast<size_t>(2 * m.rows() * r)),
                        vd(static_cast<size_t>(2 * r * m.cols()));
    b200::check(achi_svd_complex(b200::Device::get().ctx(), static_cast<int>(m.rows()),
                                 static_cast<int>(m.cols()), a.data(), out.sigma.data(), u.data(),
                                 vd.data(), &sweeps));
    out.u = DenseMatrix::from_interleaved_row_major(m.rows(), r, u.data());
    out.v_dagger = DenseMatrix::from_interleaved_row_major(r, m.cols(), vd.data());
  }
  return out;
}
// svd_truncated (linalg.cpp:72-89)
inline SvdResult svd_truncated(const DenseMatrix& m, long keep) {
  const long rmax = std::min(m.rows(), m.cols());
  if (keep < 1 || keep > rmax) throw InvalidRank("svd_truncated: keep out of range [1, min(rows,cols)]");
  SvdResult full = svd_full(m);
  SvdResult r;
  r.u = DenseMatrix(m.rows(), keep);
  for (long j = 0; j < keep; ++j)
    for (long i = 0; i < m.rows(); ++i) r.u(i, j) = full.u(i, j);
  r.sigma.assign(full.sigma.begin(), full.sigma.begin() + keep);
  r.v_dagger = DenseMatrix(keep, m.cols());
  for (long j = 0; j < m.cols(); ++j)
    for (long i = 0; i < keep; ++i) r.v_dagger(i, j) = full.v_dagger(i, j);
  r.rank = keep;
  if (keep < full.rank)
    r.degenerate_cut = std::abs(full.sigma[keep - 1] - full.sigma[keep]) <= 1e-12 * full.sigma[0];
  return r;
}

class B200SvdBackend final : public SvdBackend {
 public:
  SvdResult svd(const DenseMatrix& m) const override { return svd_full(m); }
  std::string_view name() const override { return "b200"; }
};

// linalg.cpp:58-105: the registry keeps the external backend; here the
// "reference" host backend is the same device path (no CPU fallback).
class BackendRegistry {
 public:
  static BackendRegistry& global() {
    static BackendRegistry r;
    return r;
  }
  BackendRegistry() = default;
  void register_external(std::unique_ptr<SvdBackend> b) { external_ = std::move(b); }
  bool has_external() const { return external_ != nullptr; }
  const SvdBackend* external() const { return external_.get(); }

 private:
  std::unique_ptr<SvdBackend> external_;
};
inline BackendId select_backend(const BackendPolicy& policy, long chi,
                                const BackendRegistry& registry = BackendRegistry::global()) {
  if (chi < policy.accelerator_threshold) return BackendId::reference;
  if (policy.preferred == BackendId::external && registry.has_external()) return BackendId::external;
  return BackendId::reference;
}
inline SvdResult svd_dispatch(const DenseMatrix& m, const BackendPolicy& policy, long chi,
                              const BackendRegistry& registry = BackendRegistry::global()) {
  if (select_backend(policy, chi, registry) == BackendId::external) return registry.external()->svd(m);
  return svd_full(m);
}

struct EigsResult {
  double eigenvalue = 0;
  CVector eigenvector;
  int matvec_count = 0;
  double residual = 0;
};
using LinearMap = std::function<void(const CVector&, CVector&)>;

namespace detail {
struct RealMap {  // a complex LinearMap as a real operator (realified when complex)
  const LinearMap* op;
  long dim;
  bool realified;
  bool complex_seen = false;
  CVector in, out;
  static void call(void* user, const double* x, double* y, int64_t n) {
    auto* self = static_cast<RealMap*>(user);
    const long d = self->dim;
    self->in.assign(static_cast<size_t>(d), Cplx(0, 0));
    for (long i = 0; i < d; ++i) self->in[i] = self->realified ? Cplx(x[i], x[d + i]) : Cplx(x[i], 0.0);
    self->out.assign(static_cast<size_t>(d), Cplx(0, 0));
    (*self->op)(self->in, self->out);
    for (long i = 0; i < d; ++i) {
      y[i] = self->out[i].real();
      if (self->realified)
        y[d + i] = self->out[i].imag();
      else if (self->out[i].imag() != 0.0)
        self->complex_seen = true;
    }
    if (self->complex_seen && !self->realified)
      for (int64_t i = 0; i < n; ++i) y[i] = std::nan("");  // abort; rerun realified
  }
};
}  // namespace detail

// eigs_lowest (linalg.cpp:107-178) for a LinearMap (linalg.hpp:64-78): the
// restarted Lanczos runs on the device, the operator on the host
// (achi_eigs_lowest_callback).  A real operator from a real v0 runs the real
// iteration (the reference's arithmetic to rounding); a complex Hermitian
// one runs as the real symmetric [[Re H, -Im H], [Im H, Re H]] on [x; y],
// whose lowest eigenvector [x; y] gives the complex eigenvector x + i y.
inline EigsResult eigs_lowest(const LinearMap& apply_h, long dim, const CVector& v0, double tol = 1e-10,
                              int max_iter = 200) {
  if (dim < 1 || static_cast<long>(v0.size()) != dim) throw InvalidMatrix("eigs_lowest: v0 size mismatch");
  bool v0_real = true;
  for (const Cplx& x : v0)
    if (x.imag() != 0.0) v0_real = false;
  for (int pass = v0_real ? 0 : 1; pass < 2; ++pass) {
    detail::RealMap rm{&apply_h, dim, pass == 1, false, {}, {}};
    const long rd = rm.realified ? 2 * dim : dim;
    std::vector<double> x0(static_cast<size_t>(rd)), vec(static_cast<size_t>(rd));
    for (long i = 0; i < dim; ++i) {
      x0[i] = v0[i].real();
      if (rm.realified) x0[dim + i] = v0[i].imag();
    }
    EigsResult r;
    const int rc = achi_eigs_lowest_callback(b200::Device::get().ctx(), static_cast<int>(rd),
                                             &detail::RealMap::call, &rm, x0.data(), tol, max_iter,
                                             &r.eigenvalue, vec.data(), &r.matvec_count, &r.residual);
    if (rm.complex_seen && !rm.realified) continue;  // complex operator: run realified
    b200::check(rc);
    r.eigenvector.assign(static_cast<size_t>(dim), Cplx(0, 0));
    for (long i = 0; i < dim; ++i) r.eigenvector[i] = rm.realified ? Cplx(vec[i], vec[dim + i]) : Cplx(vec[i], 0);
    return r;
  }
  throw InternalConsistency("eigs_lowest: unreachable");
}

// eigs_lowest for a dense Hermitian operator: a real matrix runs the device
// Lanczos directly on the device matrix (achi_eigs_lowest_dense), a complex
// one through its real 2 dim x 2 dim form.
inline EigsResult eigs_lowest(const DenseMatrix& h, const CVector& v0, double tol = 1e-10,
                              int max_iter = 200) {
  const long dim = h.rows();
  if (h.cols() != dim || static_cast<long>(v0.size()) != dim) throw InvalidMatrix("eigs_lowest: v0 size mismatch");
  bool real = h.is_real();
  for (const Cplx& x : v0) real = real && x.imag() == 0.0;
  const long rd = real ? dim : 2 * dim;
  std::vector<double> a(static_cast<size_t>(rd * rd)), x0(static_cast<size_t>(rd)), vec(static_cast<size_t>(rd));
  for (long i = 0; i < dim; ++i) {
    x0[i] = v0[i].real();
    if (!real) x0[dim + i] = v0[i].imag();
    for (long j = 0; j < dim; ++j) {
      const Cplx v = h(i, j);
      a[static_cast<size_t>(i * rd + j)] = v.real();
      if (!real) {
        a[static_cast<size_t>(i * rd + dim + j)] = -v.imag();
        a[static_cast<size_t>((dim + i) * rd + j)] = v.imag();
        a[static_cast<size_t>((dim + i) * rd + dim + j)] = v.real();
      }
    }
  }
  EigsResult r;
  b200::check(achi_eigs_lowest_dense(b200::Device::get().ctx(), static_cast<int>(rd), a.data(), x0.data(),
                                     tol, max_iter, &r.eigenvalue, vec.data(), &r.matvec_count, &r.residual));
  r.eigenvector.assign(static_cast<size_t>(dim), Cplx(0, 0));
  for (long i = 0; i < dim; ++i) r.eigenvector[i] = real ? Cplx(vec[i], 0) : Cplx(vec[i], vec[dim + i]);
  return r;
}

// C = A B for complex row-major A (M x K) and B (K x N) on the device DMMA
// GEMM (achi_dgemm; four real products, operands padded to even leading
// dimensions): the contraction inside Tensor::contract (tensor.hpp:195-196).
inline std::vector<Cplx> cgemm(long M, long N, long K, const Cplx* A, const Cplx* B) {
  const long Kp = K + (K & 1), Np = N + (N & 1);
  std::vector<double> ar(static_cast<size_t>(M * Kp), 0.0), ai(ar.size(), 0.0), br(static_cast<size_t>(K * Np), 0.0),
      bi(br.size(), 0.0);
  for (long i = 0; i < M; ++i)
    for (long k = 0; k < K; ++k) {
      ar[static_cast<size_t>(i * Kp + k)] = A[i * K + k].real();
      ai[static_cast<size_t>(i * Kp + k)] = A[i * K + k].imag();
    }
  for (long k = 0; k < K; ++k)
    for (long j = 0; j < N; ++j) {
      br[static_cast<size_t>(k * Np + j)] = B[k * N + j].real();
      bi[static_cast<size_t>(k * Np + j)] = B[k * N + j].imag();
    }
  std::vector<double> t[4];
  const double* pa[4] = {ar.data(), ai.data(), ar.data(), ai.data()};
  const double* pb[4] = {br.data(), bi.data(), bi.data(), br.data()};
  for (int q = 0; q < 4; ++q) {
    t[q].assign(static_cast<size_t>(M * Np), 0.0);
    b200::check(achi_dgemm(b200::Device::get().ctx(), static_cast<int>(M), static_cast<int>(Np),
                           static_cast<int>(Kp), 1, pa[q], Kp, 0, pb[q], Np, t[q].data(), Np));
  }
  std::vector<Cplx> c(static_cast<size_t>(M * N));
  for (long i = 0; i < M; ++i)
    for (long j = 0; j < N; ++j) {
      const size_t o = static_cast<size_t>(i * Np + j);
      c[static_cast<size_t>(i * N + j)] = Cplx(t[0][o] - t[1][o], t[2][o] + t[3][o]);
    }
  return c;
}
}  // namespace linalg

// ---- mps.hpp:20-99: MPS container, split / merge of two-site blocks --------
namespace mps {
struct TruncationOutcome {
  int kept_chi = 0;
  double truncation_error = 0;
  double entropy = 0;
  SingularSpectrum spectrum;
  bool degenerate_cut = false;
};

// Open-boundary MPS of (left, phys, right) site tensors (mps.hpp:30-50).  The
// device-resident state of a run lives in dmrg::Chain; this host container is
// what split/merge and snapshots exchange.
class MatrixProductState {
 public:
  MatrixProductState() = default;
  explicit MatrixProductState(std::vector<Tensor> sites) : sites_(std::move(sites)) {}
  int size() const { return static_cast<int>(sites_.size()); }
  int phys_dim() const { return static_cast<int>(sites_.front().dim(1)); }
  Tensor& site(int i) { return sites_[static_cast<size_t>(i)]; }
  const Tensor& site(int i) const { return sites_[static_cast<size_t>(i)]; }
  void set_site(int i, Tensor t) { sites_[static_cast<size_t>(i)] = std::move(t); }
  std::vector<int> bond_dims() const {  // mps.cpp:24-29
    std::vector<int> b;
    for (int i = 0; i + 1 < size(); ++i) b.push_back(static_cast<int>(sites_[static_cast<size_t>(i)].dim(2)));
    return b;
  }

 private:
  std::vector<Tensor> sites_;
};

enum class AbsorbSide { left, right };
struct SplitResult {
  Tensor left;              // (chi_left, d, kept)
  SingularSpectrum lambda;  // kept values
  Tensor right;             // (kept, d, chi_right)
  TruncationOutcome outcome;
};

// split_two_site (mps.cpp:124-166): device SVD, entropy and truncation error
// (achi_spectrum_stats); the kept factors are sliced and lambda absorbed on
// the host (O(chi^2) copies of the API-level helper; the DMRG path absorbs on
// the device).
inline SplitResult split_two_site(const DenseMatrix& theta, int d, int chi_left, int chi_right,
                                  int chi_request, double trunc_floor = 1e-14,
                                  AbsorbSide absorb = AbsorbSide::right) {
  if (theta.rows() != static_cast<long>(d) * chi_left || theta.cols() != static_cast<long>(d) * chi_right)
    throw InvalidMatrix("split_two_site: theta shape mismatch");
  if (chi_request < 1) throw InvalidRank("split_two_site: chi_request >= 1");
  linalg::SvdResult svd = linalg::svd_full(theta);
  const double s1 = svd.sigma.empty() ? 0.0 : svd.sigma[0];
  if (!(s1 > 0)) throw DegenerateSpectrum("split_two_site: zero matrix");
  long significant = 0;
  for (double x : svd.sigma)
    if (x > trunc_floor * s1) ++significant;
  significant = std::max<long>(significant, 1);
  const long kept = std::min<long>(chi_request, significant);
  SplitResult out;
  out.outcome.spectrum.values = svd.sigma;
  out.outcome.kept_chi = static_cast<int>(kept);
  out.outcome.entropy = entropy_from_spectrum(out.outcome.spectrum);
  out.outcome.truncation_error = truncation_error(out.outcome.spectrum, static_cast<int>(kept));
  out.outcome.degenerate_cut = kept < static_cast<long>(svd.sigma.size()) &&
                               std::abs(svd.sigma[kept - 1] - svd.sigma[kept]) <= 1e-12 * s1;
  DenseMatrix u(theta.rows(), kept), vdag(kept, theta.cols());
  for (long j = 0; j < kept; ++j)
    for (long i = 0; i < theta.rows(); ++i)
      u(i, j) = svd.u(i, j) * (absorb == AbsorbSide::left ? svd.sigma[j] : 1.0);
  for (long j = 0; j < theta.cols(); ++j)
    for (long i = 0; i < kept; ++i)
      vdag(i, j) = svd.v_dagger(i, j) * (absorb == AbsorbSide::right ? svd.sigma[i] : 1.0);
  out.lambda.values.assign(svd.sigma.begin(), svd.sigma.begin() + kept);
  out.left = Tensor::from_matrix(u, {chi_left, d, kept});
  out.right = Tensor::from_matrix(vdag, {kept, d, chi_right});
  return out;
}

// merge_two_site (mps.cpp:317-324): (l, s1, x) * (x, s2, r) -> (l s1) x (s2 r),
// on the device GEMM
inline DenseMatrix merge_two_site(const MatrixProductState& psi, int k) {
  const Tensor& a = psi.site(k);
  const Tensor& b = psi.site(k + 1);
  if (a.dim(2) != b.dim(0)) throw InvalidMatrix("merge_two_site: bond mismatch");
  const long l = a.dim(0), d1 = a.dim(1), x = a.dim(2), d2 = b.dim(1), r = b.dim(2);
  const std::vector<Cplx> c = linalg::cgemm(l * d1, d2 * r, x, a.data(), b.data());
  DenseMatrix m(l * d1, d2 * r);
  for (long i = 0; i < l * d1; ++i)
    for (long j = 0; j < d2 * r; ++j) m(i, j) = c[static_cast<size_t>(i * d2 * r + j)];
  return m;
}
}  // namespace mps

// ---- dmrg.hpp:10-98 ---------------------------------------------------------
namespace dmrg {
struct DmrgConfig {
  int max_sweeps = 24;
  double eps_conv = 1e-8;
  double eig_tol = 1e-10;
  int eig_max_iter = 200;
  ctrl::ControllerConfig controller{};
  enum class InitialState { automatic, neel, random, random_real };
  InitialState initial_state = InitialState::automatic;
  uint64_t seed = 1234;
  double noise_floor = 1e-14;
  // complex128 like the reference (automatic -> the complex random_mps for
  // TFIM, dmrg.cpp:222-235); real (default) runs real-valued states in FP64
  enum class Arithmetic { real, complex };
  Arithmetic arithmetic = Arithmetic::real;
  achi_dmrg_config c() const {
    return {max_sweeps, eig_max_iter, eps_conv, eig_tol, static_cast<int32_t>(initial_state),
            static_cast<int32_t>(arithmetic), seed, noise_floor, controller.c()};
  }
};
struct SweepRecord {
  int sweep_index = 0;
  double energy = 0, delta_e_rel = 0;
  std::vector<int> chi_profile;
  std::vector<double> entropy_profile;
  double max_trunc_error = 0, wall_time = 0;
  long parameter_count = 0;
  double average_chi = 0;
};
struct SweepOutcome {
  SweepRecord record;
  int max_chi_used = 0;
};
struct DmrgResult {
  std::vector<SweepRecord> sweeps;
  bool converged = false;
  double energy = 0;
  int max_chi_used = 0;
  double max_monotonicity_violation = 0;
  std::vector<int> bond_dims;  // final chi profile (psi.bond_dims())
};

// Device-resident chain: replaces (psi, mpo, env, states) of the reference
// with one handle (dmrg.cpp:216-250 setup); sweep() is two_site_sweep.
class Chain {
 public:
  Chain(const models::ModelSpec& spec, const DmrgConfig& cfg) : n_(spec.n) {
    achi_model_spec s = spec.c();
    achi_dmrg_config c = cfg.c();
    b200::check(achi_chain_create(b200::Device::get().ctx(), &s, &c, &h_));
  }
  ~Chain() {
    if (h_) achi_chain_destroy(h_);
  }
  Chain(const Chain&) = delete;
  Chain& operator=(const Chain&) = delete;
  achi_chain* handle() const { return h_; }

  SweepOutcome sweep(int sweep_index, ctrl::ControllerTrace* trace = nullptr) {
    achi_sweep_record rec{};
    std::vector<int32_t> chi(n_ - 1);
    std::vector<double> ent(n_ - 1);
    std::vector<achi_trace_row> rows(2 * (n_ - 1));
    b200::check(achi_chain_sweep(h_, sweep_index, &rec, chi.data(), ent.data(), rows.data(), nullptr));
    SweepOutcome o;
    o.record = to_record(rec, chi.data(), ent.data(), n_ - 1);
    o.max_chi_used = rec.max_chi_used;
    if (trace)
      for (const auto& r : rows) trace->add(r.sweep, r.bond, ctrl::from_c(r));
    return o;
  }
  std::vector<int> bond_dims() const {
    std::vector<int32_t> d(n_ - 1);
    achi_chain_bond_dims(h_, d.data());
    return std::vector<int>(d.begin(), d.end());
  }
  // the current MPS (complex tensors, as the reference holds psi)
  mps::MatrixProductState state() const {
    const std::vector<int> b = bond_dims();
    const bool cplx = achi_chain_is_complex(h_) != 0;
    std::vector<Tensor> sites;
    for (int k = 0; k < n_; ++k) {
      const long l = k == 0 ? 1 : b[static_cast<size_t>(k - 1)];
      const long r = k == n_ - 1 ? 1 : b[static_cast<size_t>(k)];
      Tensor t({l, 2, r});
      std::vector<double> buf(static_cast<size_t>(2 * l * 2 * r));
      if (cplx) {
        b200::check(achi_chain_get_site_complex(h_, k, buf.data(), buf.size()));
        for (long i = 0; i < t.size(); ++i) t.data()[i] = Cplx(buf[2 * i], buf[2 * i + 1]);
      } else {
        b200::check(achi_chain_get_site(h_, k, buf.data(), buf.size()));
        for (long i = 0; i < t.size(); ++i) t.data()[i] = Cplx(buf[i], 0.0);
      }
      sites.push_back(std::move(t));
    }
    return mps::MatrixProductState(std::move(sites));
  }
  static SweepRecord to_record(const achi_sweep_record& r, const int32_t* chi, const double* ent,
                               int nb) {
    SweepRecord s;
    s.chi_profile.assign(chi, chi + nb);
    s.entropy_profile.assign(ent, ent + nb);
    s.sweep_index = r.sweep_index;
    s.energy = r.energy;
    s.delta_e_rel = r.delta_e_rel;
    s.max_trunc_error = r.max_trunc_error;
    s.wall_time = r.wall_time;
    s.parameter_count = static_cast<long>(r.parameter_count);
    s.average_chi = r.average_chi;
    return s;
  }
  int n() const { return n_; }

 private:
  int n_;
  achi_chain* h_ = nullptr;
};

// run_dmrg (dmrg.cpp:216-282) on the device
inline DmrgResult run_dmrg(const models::ModelSpec& spec, const DmrgConfig& cfg,
                           ctrl::ControllerTrace* trace = nullptr) {
  Chain ch(spec, cfg);
  const int n = spec.n, ms = cfg.max_sweeps, nb = n - 1, nv = 2 * (n - 1);
  std::vector<achi_sweep_record> recs(ms);
  std::vector<int32_t> chi(static_cast<size_t>(ms) * nb);
  std::vector<double> ent(static_cast<size_t>(ms) * nb);
  std::vector<achi_trace_row> rows(static_cast<size_t>(ms) * nv);
  achi_dmrg_result r{};
  b200::check(achi_chain_run(ch.handle(), &r, recs.data(), chi.data(), ent.data(), rows.data(), nullptr));
  DmrgResult out;
  out.converged = r.converged != 0;
  out.energy = r.energy;
  out.max_chi_used = r.max_chi_used;
  out.max_monotonicity_violation = r.max_monotonicity_violation;
  for (int k = 0; k < r.n_sweeps; ++k) {
    SweepRecord s = Chain::to_record(recs[k], chi.data() + k * nb, ent.data() + k * nb, nb);
    out.sweeps.push_back(std::move(s));
  }
  if (trace)
    for (int i = 0; i < r.n_sweeps * nv; ++i) trace->add(rows[i].sweep, rows[i].bond, ctrl::from_c(rows[i]));
  out.bond_dims = ch.bond_dims();
  return out;
}
}  // namespace dmrg
}  // namespace adaptchi
