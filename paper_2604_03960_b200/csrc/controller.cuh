// Scalar adaptive-chi controller (controller.cpp:12-190), compiled for the
// device: the fused bond-select kernel runs it in one thread after the
// spectrum reductions, so the per-bond state never leaves the GPU.
#pragma once

#include <cmath>

#include "../../include/adaptchi_b200.h"

namespace achi {

struct Decision {
  int chi = 0;
  double s_raw = 0, s_ema = 0, s_pred = 0, error = 0, p_term = 0, i_term = 0, d_term = 0;
  long long delta_chi = 0;
  bool clamped = false;
};

// returns 0 or an ACHI_E_* code (InvalidConfig paths of the reference)
__host__ __device__ inline double resolved_s_target(const achi_controller_config& c) {
  if (c.s_target >= 0) return c.s_target;  // controller.cpp:12-15
  return log(static_cast<double>(c.chi_max)) - 0.5;
}

__host__ __device__ inline void push_history(achi_bond_state& s, double v) {  // :35-42
  if (s.history_len < 3) {
    s.history[s.history_len++] = v;
  } else {
    s.history[0] = s.history[1];
    s.history[1] = s.history[2];
    s.history[2] = v;
  }
}
__host__ __device__ inline double history_at(const achi_bond_state& s, int back) {
  return s.history[s.history_len - 1 - back];
}

__host__ __device__ inline int ema_update(achi_bond_state& s, double s_raw, double alpha) {  // :49-60
  if (!(alpha > 0.0) || alpha > 1.0) return ACHI_E_INVALID_CONFIG;
  if (s_raw < 0) return ACHI_E_INVALID_CONFIG;
  if (!s.initialized) {
    s.ema = s_raw;
    s.initialized = 1;
  } else {
    s.ema = alpha * s_raw + (1.0 - alpha) * s.ema;
  }
  push_history(s, s.ema);
  return 0;
}

__host__ __device__ inline int chi_target_direct(double s, double gamma, int chi_min, int chi_max,
                                                 int* out) {  // :71-82
  if (s < 0 || gamma < 1.0) return ACHI_E_INVALID_CONFIG;
  double target = ceil(gamma * exp(s) - 1e-9);
  double lo = chi_min, hi = chi_max;
  double c = target < lo ? lo : (target > hi ? hi : target);
  *out = static_cast<int>(c);
  return 0;
}

__host__ __device__ inline int pid_step(achi_bond_state& s, double s_in,
                                        const achi_controller_config& c, Decision& d) {  // :84-117
  if (!s.initialized) return ACHI_E_INVALID_CONFIG;
  d.s_ema = s.ema;
  d.s_pred = s_in;
  d.error = s_in - resolved_s_target(c);
  d.p_term = c.kp * d.error;
  s.integral += c.ki * d.error;
  d.i_term = s.integral;
  d.d_term = c.kd * (d.error - s.prev_error);
  const double u = d.p_term + d.i_term + d.d_term;
  long long raw;
  if (c.pid_scale == ACHI_PID_ADDITIVE) {
    d.delta_chi = llround(u);
    raw = s.chi + d.delta_chi;
  } else {
    raw = llround(s.chi * (1.0 + u / 10.0));
    d.delta_chi = raw - s.chi;
  }
  long long cl = raw < c.chi_min ? c.chi_min : (raw > c.chi_max ? c.chi_max : raw);
  d.clamped = cl != raw;
  if (d.clamped) {
    s.integral -= c.ki * d.error;  // anti-windup
    d.i_term = s.integral;
  }
  s.prev_error = d.error;
  s.chi = static_cast<int>(cl);
  d.chi = s.chi;
  return 0;
}

__host__ __device__ inline double predict_entropy(const achi_bond_state& s, double beta, int order,
                                                  bool* fallback) {  // :119-132
  const int need = order == ACHI_PREDICT_QUADRATIC ? 3 : 2;
  if (order == ACHI_PREDICT_OFF || s.history_len < need) {
    if (fallback) *fallback = true;
    return s.ema;
  }
  const double s0 = history_at(s, 0), s1 = history_at(s, 1);
  double v = s0 + beta * (s0 - s1);
  if (order == ACHI_PREDICT_QUADRATIC) v += beta * (s0 - 2.0 * s1 + history_at(s, 2));
  if (fallback) *fallback = false;
  return v > 0.0 ? v : 0.0;
}

// controller_update (:150-190) with the entropy and the threshold-mode rank
// already reduced from the spectrum by the caller.
__host__ __device__ inline int controller_update(achi_bond_state& s, double s_raw,
                                                 int threshold_rank,
                                                 const achi_controller_config& c, Decision& d) {
  int rc = ema_update(s, s_raw, c.alpha_ema);
  if (rc) return rc;
  const double s_in = predict_entropy(s, c.beta_predict, c.predictor_order, nullptr);
  switch (c.mode) {
    case ACHI_MODE_FIXED:
      d.chi = c.chi_max;
      s.chi = d.chi;
      break;
    case ACHI_MODE_THRESHOLD: {
      int r = threshold_rank;
      d.chi = r < c.chi_min ? c.chi_min : (r > c.chi_max ? c.chi_max : r);
      s.chi = d.chi;
      break;
    }
    case ACHI_MODE_DIRECT:
      rc = chi_target_direct(s_in, c.gamma_margin, c.chi_min, c.chi_max, &d.chi);
      if (rc) return rc;
      s.chi = d.chi;
      break;
    default:
      rc = pid_step(s, s_in, c, d);
      if (rc) return rc;
      break;
  }
  d.s_raw = s_raw;
  d.s_ema = s.ema;
  d.s_pred = s_in;
  return 0;
}

}  // namespace achi
