// adaptchi_b200.hpp — C++ host mirror of the reference interface over the C-ABI.
//
// Header-only, C++17.  Names, argument meaning, defaults and exception types
// follow /root/reference/proj/include/adaptchi/{errors,models,controller,mps,
// linalg,dmrg}.hpp so that reference-style code and tests compile against the
// B200 backend with a changed include.  Eigen types are replaced by small
// value types (DenseMatrix is a real column-major matrix: the device path is
// real FP64).  Every computation runs on the GPU through
// include/adaptchi_b200.h; there is no host fallback.
#pragma once

#include <cmath>
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

// Real column-major dense matrix (stands in for Eigen::MatrixXcd, tensor.hpp:15).
struct DenseMatrix {
  long r = 0, c = 0;
  std::vector<double> d;
  DenseMatrix() = default;
  DenseMatrix(long rows, long cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols), 0.0) {}
  static DenseMatrix Identity(long n, long m) {
    DenseMatrix x(n, m);
    for (long i = 0; i < std::min(n, m); ++i) x(i, i) = 1.0;
    return x;
  }
  long rows() const { return r; }
  long cols() const { return c; }
  double& operator()(long i, long j) { return d[static_cast<size_t>(i + j * r)]; }
  double operator()(long i, long j) const { return d[static_cast<size_t>(i + j * r)]; }
  std::vector<double> row_major() const {
    std::vector<double> o(d.size());
    for (long i = 0; i < r; ++i)
      for (long j = 0; j < c; ++j) o[static_cast<size_t>(i * c + j)] = (*this)(i, j);
    return o;
  }
  static DenseMatrix from_row_major(long rows, long cols, const double* p) {
    DenseMatrix x(rows, cols);
    for (long i = 0; i < rows; ++i)
      for (long j = 0; j < cols; ++j) x(i, j) = p[i * cols + j];
    return x;
  }
};
using RVector = std::vector<double>;

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
inline SvdResult svd_full(const DenseMatrix& m) {
  if (m.rows() < 1 || m.cols() < 1) throw InvalidMatrix("svd: matrix must be at least 1x1");
  const long r = std::min(m.rows(), m.cols());
  std::vector<double> a = m.row_major(), s(r), u(m.rows() * r), vt(r * m.cols());
  int sweeps = 0;
  b200::check(achi_svd(b200::Device::get().ctx(), static_cast<int>(m.rows()),
                       static_cast<int>(m.cols()), a.data(), s.data(), u.data(), vt.data(), &sweeps));
  SvdResult out;
  out.u = DenseMatrix::from_row_major(m.rows(), r, u.data());
  out.sigma = s;
  out.v_dagger = DenseMatrix::from_row_major(r, m.cols(), vt.data());
  out.rank = r;
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
  RVector eigenvector;
  int matvec_count = 0;
  double residual = 0;
};
// eigs_lowest (linalg.cpp:107-178) for a dense symmetric operator (the
// reference's host std::function operator cannot run on the device; on the DMRG
// path the Lanczos runs inside dmrg::two_site_sweep on H_eff).
inline EigsResult eigs_lowest(const DenseMatrix& h, const RVector& v0, double tol = 1e-10,
                              int max_iter = 200) {
  const int dim = static_cast<int>(h.rows());
  if (static_cast<int>(v0.size()) != dim) throw InvalidMatrix("eigs_lowest: v0 size mismatch");
  std::vector<double> a = h.row_major();
  EigsResult r;
  r.eigenvector.assign(dim, 0.0);
  b200::check(achi_eigs_lowest_dense(b200::Device::get().ctx(), dim, a.data(), v0.data(), tol,
                                     max_iter, &r.eigenvalue, r.eigenvector.data(),
                                     &r.matvec_count, &r.residual));
  return r;
}
}  // namespace linalg

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
  achi_dmrg_config c() const {
    return {max_sweeps, eig_max_iter, eps_conv, eig_tol, static_cast<int32_t>(initial_state), 0,
            seed, noise_floor, controller.c()};
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
