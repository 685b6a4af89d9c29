// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle for ctypes
// (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).  See
// adaptchi_oracle.hpp for what is restated and from where.
#include <cstdio>

#include "../include/adaptchi_b200.h"
#include "adaptchi_oracle.hpp"

using namespace oracle;

namespace {

int set_err(char* err, size_t len, const std::exception& e) {
  if (err && len) std::snprintf(err, len, "%s", e.what());
  if (auto* oe = dynamic_cast<const Error*>(&e)) return oe->code;
  return E_ERROR;
}

ModelSpec to_spec(const achi_model_spec* s) {
  ModelSpec m;
  m.family = s->family;
  m.n = s->n;
  m.jx = s->jx;
  m.jy = s->jy;
  m.jz = s->jz;
  m.h = s->h;
  m.convention = s->convention;
  return m;
}

ControllerConfig to_cc(const achi_controller_config* c) {
  ControllerConfig cc;
  cc.mode = c->mode;
  cc.predictor_order = c->predictor_order;
  cc.alpha_ema = c->alpha_ema;
  cc.gamma_margin = c->gamma_margin;
  cc.s_target = c->s_target;
  cc.kp = c->kp;
  cc.ki = c->ki;
  cc.kd = c->kd;
  cc.beta_predict = c->beta_predict;
  cc.chi_min = c->chi_min;
  cc.chi_max = c->chi_max;
  cc.pid_scale = c->pid_scale;
  cc.eps_trunc = c->eps_trunc;
  return cc;
}

DmrgConfig to_cfg(const achi_dmrg_config* c) {
  DmrgConfig d;
  d.max_sweeps = c->max_sweeps;
  d.eps_conv = c->eps_conv;
  d.eig_tol = c->eig_tol;
  d.eig_max_iter = c->eig_max_iter;
  d.initial_state = c->initial_state;
  d.seed = c->seed;
  d.noise_floor = c->noise_floor;
  d.controller = to_cc(&c->controller);
  return d;
}

BondState to_state(const achi_bond_state* s) {
  BondState b;
  b.ema = s->ema;
  b.prev_error = s->prev_error;
  b.integral = s->integral;
  for (int i = 0; i < 3; ++i) b.history[i] = s->history[i];
  b.chi = s->chi;
  b.history_len = s->history_len;
  b.initialized = s->initialized != 0;
  return b;
}
void from_state(const BondState& b, achi_bond_state* s) {
  s->ema = b.ema;
  s->prev_error = b.prev_error;
  s->integral = b.integral;
  for (int i = 0; i < 3; ++i) s->history[i] = b.history[i];
  s->chi = b.chi;
  s->history_len = b.history_len;
  s->initialized = b.initialized ? 1 : 0;
}
void to_row(int sweep, int bond, const Decision& d, achi_trace_row* r) {
  r->sweep = sweep;
  r->bond = bond;
  r->chi = d.chi;
  r->clamped = d.clamped;
  r->delta_chi = d.delta_chi;
  r->s_raw = d.s_raw;
  r->s_ema = d.s_ema;
  r->s_pred = d.s_pred;
  r->error = d.error;
  r->p_term = d.p_term;
  r->i_term = d.i_term;
  r->d_term = d.d_term;
}
void to_visit(const VisitLog& v, achi_visit_record* o) {
  o->sweep = v.sweep;
  o->bond = v.bond;
  o->moving_right = v.moving_right;
  o->kept = v.kept;
  o->floor_rank = v.floor_rank;
  o->significant = v.significant;
  o->n_sigma = v.n_sigma;
  o->matvecs = v.matvecs;
  o->degenerate_cut = v.degenerate_cut;
  o->energy = v.energy;
  o->entropy = v.entropy;
  o->trunc_error = v.trunc_error;
  o->floor_margin = v.floor_margin;
  o->sigma_kept = v.sigma_kept;
  o->sigma_next = v.sigma_next;
  o->lanczos_residual = v.residual;
}

Tensor<double> tens(std::vector<long> shape, const double* p) {
  Tensor<double> t(std::move(shape));
  std::copy(p, p + t.size(), t.data.begin());
  return t;
}

template <class T>
int run_impl(const achi_model_spec* spec, const achi_dmrg_config* cfg, bool real_gauge,
             achi_dmrg_result* res, achi_sweep_record* recs, int32_t* chi, double* ent,
             achi_trace_row* trace, achi_visit_record* visits, int32_t* dims_out,
             double* sites_out, size_t sites_cap) {
  auto run = run_dmrg<T>(to_spec(spec), to_cfg(cfg), real_gauge);
  const int n = spec->n;
  if (res) {
    res->n_sweeps = static_cast<int>(run.sweeps.size());
    res->converged = run.converged;
    res->max_chi_used = run.max_chi_used;
    res->energy = run.energy;
    res->max_monotonicity_violation = run.max_monotonicity_violation;
  }
  for (size_t s = 0; s < run.sweeps.size(); ++s) {
    const SweepRecord& r = run.sweeps[s];
    if (recs) {
      recs[s].sweep_index = r.sweep_index;
      recs[s].max_chi_used = r.max_chi_used;
      recs[s].energy = r.energy;
      recs[s].delta_e_rel = r.delta_e_rel;
      recs[s].max_trunc_error = r.max_trunc_error;
      recs[s].wall_time = r.wall_time;
      recs[s].parameter_count = r.parameter_count;
      recs[s].average_chi = r.average_chi;
    }
    for (int b = 0; b < n - 1; ++b) {
      if (chi) chi[s * (n - 1) + b] = r.chi_profile[b];
      if (ent) ent[s * (n - 1) + b] = r.entropy_profile[b];
    }
  }
  if (trace)
    for (size_t i = 0; i < run.trace.size(); ++i)
      to_row(run.trace[i].sweep, run.trace[i].bond, run.trace[i].d, &trace[i]);
  if (visits)
    for (size_t i = 0; i < run.visits.size(); ++i) to_visit(run.visits[i], &visits[i]);
  if (dims_out) {
    auto d = run.psi.bond_dims();
    for (int b = 0; b < n - 1; ++b) dims_out[b] = d[b];
  }
  if (sites_out) {
    size_t off = 0;
    for (const auto& s : run.psi.sites) {
      if (off + s.size() > sites_cap) fail(E_SIZE_GUARD, "sites_out capacity");
      for (long k = 0; k < s.size(); ++k) sites_out[off + k] = real_(s.data[k]);
      off += s.size();
    }
  }
  return 0;
}

}  // namespace

// ---- step-wise chain (run_dmrg setup + two_site_sweep), for timed baselines ----
struct OracleChainBase {
  virtual ~OracleChainBase() = default;
  virtual SweepRecord sweep(int s) = 0;
};
template <class T>
struct OracleChain : OracleChainBase {
  ModelSpec ms;
  DmrgConfig dc;
  std::vector<Tensor<T>> mpo;
  MPS<T> psi;
  Environment<T> env;
  std::vector<BondState> states;
  OracleChain(const ModelSpec& s, const DmrgConfig& c)
      : ms(s), dc(c), mpo(build_mpo<T>(s, !std::is_same_v<T, cd>)), env(s.n) {
    ms.validate();
    dc.validate();
    init_run(ms, dc, psi);
    env.rebuild(psi, mpo, 0);
    states.assign(ms.n - 1, BondState{});
    for (auto& st : states) {  // dmrg.cpp:243-250
      st.chi = dc.controller.chi_min;
      st.ema = 0.0;
      st.initialized = true;
      st.push_history(0.0);
    }
  }
  SweepRecord sweep(int s) override {
    return two_site_sweep(psi, mpo, env, dc, states, s, nullptr, nullptr);
  }
};


extern "C" {

void oracle_set_threads(int n) { scipy_openblas_set_num_threads64_(n); }

// run_dmrg (dmrg.cpp:216-282).  complex_mode=1: complex128 with the reference
// MPO (faithful); 0: real FP64 with the real-gauge MPO (the GPU's arithmetic).
int oracle_run_dmrg(const achi_model_spec* spec, const achi_dmrg_config* cfg, int complex_mode,
                    achi_dmrg_result* res, achi_sweep_record* recs, int32_t* chi, double* ent,
                    achi_trace_row* trace, achi_visit_record* visits, int32_t* dims_out,
                    double* sites_out, size_t sites_cap, char* err, size_t errlen) {
  try {
    if (complex_mode)
      return run_impl<cd>(spec, cfg, false, res, recs, chi, ent, trace, visits, dims_out,
                          sites_out, sites_cap);
    return run_impl<double>(spec, cfg, true, res, recs, chi, ent, trace, visits, dims_out,
                            sites_out, sites_cap);
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// Time `visits` consecutive bond visits of one sweep starting at bond `first`
// (sampled CPU baseline for configs too large to run in full).  The chain is
// first driven through `warm_sweeps` complete sweeps.
int oracle_sample_visits(const achi_model_spec* spec, const achi_dmrg_config* cfg,
                         int complex_mode, int warm_sweeps, int first, int count,
                         double* seconds, int32_t* dims_out, char* err, size_t errlen) {
  try {
    auto body = [&](auto tag) -> int {
      using T = decltype(tag);
      ModelSpec ms = to_spec(spec);
      DmrgConfig dc = to_cfg(cfg);
      auto mpo = build_mpo<T>(ms, !std::is_same_v<T, cd>);
      MPS<T> psi;
      init_run(ms, dc, psi);
      Environment<T> env(ms.n);
      env.rebuild(psi, mpo, 0);
      std::vector<BondState> states(ms.n - 1);
      for (auto& st : states) {
        st.chi = dc.controller.chi_min;
        st.initialized = true;
        st.push_history(0.0);
      }
      for (int s = 0; s < warm_sweeps; ++s)
        two_site_sweep(psi, mpo, env, dc, states, s, nullptr, nullptr);
      auto t0 = std::chrono::steady_clock::now();
      for (int v = 0; v < count && first + v <= ms.n - 2; ++v)
        visit_bond(psi, mpo, env, dc, states, first + v, true, warm_sweeps, nullptr);
      auto t1 = std::chrono::steady_clock::now();
      *seconds = std::chrono::duration<double>(t1 - t0).count();
      if (dims_out) {
        auto d = psi.bond_dims();
        for (int b = 0; b < ms.n - 1; ++b) dims_out[b] = d[b];
      }
      return 0;
    };
    return complex_mode ? body(cd{}) : body(double{});
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// Time `count` right-moving bond visits starting at `first` from a given
// right-canonical real MPS (centre 0) and controller states: the sampled CPU
// baseline for sweeps too long to run in full on the host.
int oracle_time_visits_from_state(const achi_model_spec* spec, const achi_dmrg_config* cfg,
                                  int complex_mode, const int32_t* dims, const double* const* sites,
                                  const achi_bond_state* states, int first, int count,
                                  double* seconds, int32_t* matvecs, char* err, size_t errlen) {
  try {
    auto body = [&](auto tag) -> int {
      using T = decltype(tag);
      ModelSpec ms = to_spec(spec);
      DmrgConfig dc = to_cfg(cfg);
      auto mpo = build_mpo<T>(ms, !std::is_same_v<T, cd>);
      MPS<T> psi;
      for (int k = 0; k < ms.n; ++k) {
        long l = k == 0 ? 1 : dims[k - 1], r = k == ms.n - 1 ? 1 : dims[k];
        Tensor<T> t({l, 2, r});
        for (long i = 0; i < t.size(); ++i) t.data[i] = T(sites[k][i]);
        psi.sites.push_back(std::move(t));
      }
      // move the canonical centre to `first` (QR sweeps, state unchanged) and
      // build the environments there (Environment::rebuild, dmrg.cpp:51-56)
      canonicalize(psi, first);
      Environment<T> env(ms.n);
      env.rebuild(psi, mpo, first);
      std::vector<BondState> st(ms.n - 1);
      for (int b = 0; b < ms.n - 1; ++b) st[b] = to_state(&states[b]);
      for (int v = 0; v < count && first + v <= ms.n - 2; ++v) {
        auto t0 = std::chrono::steady_clock::now();
        VisitLog lg = visit_bond(psi, mpo, env, dc, st, first + v, true, 0, nullptr);
        auto t1 = std::chrono::steady_clock::now();
        seconds[v] = std::chrono::duration<double>(t1 - t0).count();
        if (matvecs) matvecs[v] = lg.matvecs;
      }
      return 0;
    };
    return complex_mode ? body(cd{}) : body(double{});
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

void* oracle_chain_create(const achi_model_spec* spec, const achi_dmrg_config* cfg, int complex_mode,
                          char* err, size_t errlen) {
  try {
    if (complex_mode) return new OracleChain<cd>(to_spec(spec), to_cfg(cfg));
    return new OracleChain<double>(to_spec(spec), to_cfg(cfg));
  } catch (const std::exception& e) {
    set_err(err, errlen, e);
    return nullptr;
  }
}
int oracle_chain_sweep(void* h, int sweep, achi_sweep_record* rec, int32_t* chi, char* err,
                       size_t errlen) {
  try {
    SweepRecord r = static_cast<OracleChainBase*>(h)->sweep(sweep);
    rec->sweep_index = r.sweep_index;
    rec->max_chi_used = r.max_chi_used;
    rec->energy = r.energy;
    rec->max_trunc_error = r.max_trunc_error;
    rec->wall_time = r.wall_time;
    rec->parameter_count = r.parameter_count;
    rec->average_chi = r.average_chi;
    for (size_t b = 0; b < r.chi_profile.size(); ++b) chi[b] = r.chi_profile[b];
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
void oracle_chain_destroy(void* h) { delete static_cast<OracleChainBase*>(h); }

// apply_effective_hamiltonian (dmrg.cpp:58-71), real
int oracle_heff_apply(int chl, int chr, int d, int D1, int D2, int D3, const double* L,
                      const double* W1, const double* W2, const double* R, const double* theta,
                      double* out, char* err, size_t errlen) {
  try {
    auto t = apply_effective_hamiltonian(tens({chl, D1, chl}, L), tens({D1, d, d, D2}, W1),
                                         tens({D2, d, d, D3}, W2), tens({chr, D3, chr}, R),
                                         tens({chl, d, d, chr}, theta));
    std::copy(t.data.begin(), t.data.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// Environment::update_left / update_right (dmrg.cpp:26-49), real
int oracle_env_update_left(int chl, int chn, int d, int Dl, int Dr, const double* L,
                           const double* A, const double* W, double* out, char* err,
                           size_t errlen) {
  try {
    auto l = tens({chl, Dl, chl}, L), a = tens({chl, d, chn}, A), w = tens({Dl, d, d, Dr}, W);
    Tensor<double> t = l.contract({2}, a, {0});
    t = t.contract({1, 2}, w, {0, 2});
    t = a.conjugated().contract({0, 1}, t, {0, 2});
    t = t.permuted({0, 2, 1});
    std::copy(t.data.begin(), t.data.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_env_update_right(int chr, int chn, int d, int Dl, int Dr, const double* R,
                            const double* B, const double* W, double* out, char* err,
                            size_t errlen) {
  try {
    auto r = tens({chr, Dr, chr}, R), a = tens({chn, d, chr}, B), w = tens({Dl, d, d, Dr}, W);
    Tensor<double> t = a.contract({2}, r, {2});
    t = t.contract({1, 3}, w, {2, 3});
    t = a.conjugated().contract({1, 2}, t, {3, 1});
    t = t.permuted({0, 2, 1});
    std::copy(t.data.begin(), t.data.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// svd_full (linalg.cpp:67-70): a is m x n row-major; outputs row-major
int oracle_svd(int m, int n, const double* a, double* sigma, double* u, double* vt, char* err,
               size_t errlen) {
  try {
    Mat<double> mat(m, n);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) mat(i, j) = a[static_cast<long>(i) * n + j];
    auto r = svd_full(mat);
    const long k = r.rank;
    for (long i = 0; i < k; ++i) sigma[i] = r.sigma[i];
    if (u)
      for (long i = 0; i < m; ++i)
        for (long j = 0; j < k; ++j) u[i * k + j] = r.u(i, j);
    if (vt)
      for (long i = 0; i < k; ++i)
        for (long j = 0; j < n; ++j) vt[i * n + j] = r.vt(i, j);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
// complex svd_full on interleaved (re, im) row-major input; sigma only (timing / C2 complex)
int oracle_svd_complex(int m, int n, const double* a_interleaved, double* sigma, char* err,
                       size_t errlen) {
  try {
    Mat<cd> mat(m, n);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        long o = 2 * (static_cast<long>(i) * n + j);
        mat(i, j) = cd(a_interleaved[o], a_interleaved[o + 1]);
      }
    auto r = svd_full(mat);
    for (long i = 0; i < r.rank; ++i) sigma[i] = r.sigma[i];
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
// svd_truncated (linalg.cpp:72-89): sigma[keep], degenerate flag
int oracle_svd_truncated(int m, int n, const double* a, int keep, double* sigma, int* degenerate,
                         char* err, size_t errlen) {
  try {
    Mat<double> mat(m, n);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) mat(i, j) = a[static_cast<long>(i) * n + j];
    auto r = svd_truncated(mat, keep);
    for (long i = 0; i < keep; ++i) sigma[i] = r.sigma[i];
    *degenerate = r.degenerate_cut;
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// eigs_lowest (linalg.cpp:107-178) on a dense symmetric real operator (row-major)
int oracle_eigs_lowest_dense(int dim, const double* h, const double* v0, double tol, int max_iter,
                             double* ev, double* vec, int* matvecs, double* residual, char* err,
                             size_t errlen) {
  try {
    std::vector<double> v(v0, v0 + dim);
    auto apply = [&](const std::vector<double>& in, std::vector<double>& out) {
      for (int i = 0; i < dim; ++i) {
        double s = 0;
        for (int j = 0; j < dim; ++j) s += h[static_cast<long>(i) * dim + j] * in[j];
        out[i] = s;
      }
    };
    auto r = eigs_lowest<double>(apply, dim, v, tol, max_iter);
    *ev = r.eigenvalue;
    std::copy(r.eigenvector.begin(), r.eigenvector.end(), vec);
    *matvecs = r.matvec_count;
    *residual = r.residual;
    return 0;
  } catch (const Error& e) {
    if (residual) *residual = e.residual;
    return set_err(err, errlen, e);
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// ---- controller / spectrum helpers -----------------------------------------
int oracle_entropy(int n, const double* v, double* out, char* err, size_t errlen) {
  try {
    *out = entropy_from_spectrum(std::vector<double>(v, v + n));
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_truncation_error(int n, const double* v, int kept, double* out, char* err,
                            size_t errlen) {
  try {
    *out = truncation_error(std::vector<double>(v, v + n), kept);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_rank_for_discarded_weight(int n, const double* v, double eps, int* out,
                                     double* margin, char* err, size_t errlen) {
  try {
    *out = rank_for_discarded_weight(std::vector<double>(v, v + n), eps, margin);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_chi_target_direct(double s, double gamma, int chi_min, int chi_max, int* out,
                             char* err, size_t errlen) {
  try {
    *out = chi_target_direct(s, gamma, chi_min, chi_max);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_ema_update(achi_bond_state* st, double s_raw, double alpha, char* err, size_t errlen) {
  try {
    BondState b = to_state(st);
    ema_update(b, s_raw, alpha);
    from_state(b, st);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_pid_step(achi_bond_state* st, double s_input, const achi_controller_config* cfg,
                    achi_trace_row* row, char* err, size_t errlen) {
  try {
    BondState b = to_state(st);
    Decision d = pid_step(b, s_input, to_cc(cfg));
    from_state(b, st);
    if (row) to_row(0, 0, d, row);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}
int oracle_predict_entropy(const achi_bond_state* st, double beta, int order, double* value,
                           int* fallback) {
  bool fb = false;
  *value = predict_entropy(to_state(st), beta, order, &fb);
  *fallback = fb;
  return 0;
}
int oracle_controller_update(achi_bond_state* st, int n, const double* spectrum,
                             const achi_controller_config* cfg, achi_trace_row* row, char* err,
                             size_t errlen) {
  try {
    BondState b = to_state(st);
    Decision d = controller_update(b, std::vector<double>(spectrum, spectrum + n), to_cc(cfg));
    from_state(b, st);
    if (row) to_row(0, 0, d, row);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// build_mpo site tensor k (models.cpp:49-97): real gauge (1) -> real out; reference
// gauge (0) -> interleaved complex out.  Returns the 4 dims.
int oracle_build_mpo_site(const achi_model_spec* spec, int real_gauge, int k, int64_t* dims,
                          double* out, char* err, size_t errlen) {
  try {
    if (real_gauge) {
      auto s = build_mpo<double>(to_spec(spec), true);
      for (int i = 0; i < 4; ++i) dims[i] = s[k].shape[i];
      if (out) std::copy(s[k].data.begin(), s[k].data.end(), out);
    } else {
      auto s = build_mpo<cd>(to_spec(spec), false);
      for (int i = 0; i < 4; ++i) dims[i] = s[k].shape[i];
      if (out)
        for (long i = 0; i < s[k].size(); ++i) {
          out[2 * i] = s[k].data[i].real();
          out[2 * i + 1] = s[k].data[i].imag();
        }
    }
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

// exact_ground_energy, XXZ family (models.cpp:177-223)
int oracle_exact_ground_energy(const achi_model_spec* spec, int cap, double* out, char* err,
                               size_t errlen) {
  try {
    *out = exact_ground_energy_xxz(to_spec(spec), cap);
    return 0;
  } catch (const std::exception& e) {
    return set_err(err, errlen, e);
  }
}

}  // extern "C"
