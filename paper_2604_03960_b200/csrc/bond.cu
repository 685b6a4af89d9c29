// Fused bond-select and absorb kernels (see bond.cuh).
#include <cmath>

#include "bond.cuh"
#include "controller.cuh"

namespace achi {

namespace {

constexpr int BS_THREADS = 1024;

__device__ double bs_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (w == 0) {
    r = l < (blockDim.x >> 5) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (l == 0) sh[32] = r;
  }
  __syncthreads();
  return sh[32];
}

__device__ int bs_max_int(int v, int* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    int r = l < (blockDim.x >> 5) ? sh[l] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = max(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (l == 0) sh[32] = r;
  }
  __syncthreads();
  return sh[32];
}

// dynamic smem: suf[r + 1] (suffix sums of sigma^2), seg[BS_THREADS]
__device__ __forceinline__ void bond_select_body(
    const double* __restrict__ sigma, int r, const achi_dmrg_config& cfg, achi_bond_state* states, int bond,
    int sweep, int moving_right, achi_trace_row* trace, achi_visit_record* visit, BondOut* out) {
  extern __shared__ double dyn[];
  double* suf = dyn;                 // r + 1
  double* seg = dyn + r + 1;         // BS_THREADS
  __shared__ double shd[33];
  __shared__ int shi[33];
  const achi_controller_config& cc = cfg.controller;
  const double s1 = r > 0 ? sigma[0] : 0.0;
  if (!(s1 > 0)) {
    if (threadIdx.x == 0) out->err = ACHI_E_DEGENERATE_SPECTRUM;
    return;
  }
  // ---- suffix sums of sigma^2 (deterministic segmented scan) ----
  const int per = (r + BS_THREADS - 1) / BS_THREADS;
  const int lo = threadIdx.x * per, hi = min(r, lo + per);
  double acc = 0.0;
  for (int k = hi - 1; k >= lo; --k) {
    acc += sigma[k] * sigma[k];
    suf[k] = acc;  // local suffix within the segment
  }
  seg[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    // exclusive suffix over later segments, fixed order; only the first nseg threads
    // hold values (the others added exact zeros: skipping them changes no bit)
    const int nseg = (r + per - 1) / per;
    double run = 0.0;
    for (int t = nseg - 1; t >= 0; --t) {
      const double v = seg[t];
      seg[t] = run;
      run += v;
    }
    suf[r] = 0.0;
  }
  __syncthreads();
  for (int k = lo; k < hi; ++k) suf[k] += seg[threadIdx.x];
  __syncthreads();
  const double total = suf[0];

  // ---- rank_for_discarded_weight (controller.cpp:134-148) ----
  const double thr = cc.eps_trunc * total;
  int kstar = 0;  // largest k in [1, r-1] with suf[k] > thr
  for (int k = max(lo, 1); k < hi; ++k)
    if (suf[k] > thr) kstar = max(kstar, k);
  kstar = bs_max_int(kstar, shi);
  const int floor_rank = kstar >= 1 ? kstar + 1 : 1;

  // ---- significant count (dmrg.cpp:130-132) and entropy (mps.cpp:97-113) ----
  const double noise = cfg.noise_floor * s1, cutoff = 1e-14 * s1;
  double cnt = 0.0, tot_e = 0.0;
  for (int k = threadIdx.x; k < r; k += BS_THREADS) {
    const double v = sigma[k];
    cnt += v > noise ? 1.0 : 0.0;
    if (v > cutoff) tot_e += v * v;
  }
  const int significant = static_cast<int>(bs_sum(cnt, shd) + 0.5);
  tot_e = bs_sum(tot_e, shd);
  double ent = 0.0;
  for (int k = threadIdx.x; k < r; k += BS_THREADS) {
    const double v = sigma[k];
    if (v > cutoff) {
      const double p = v * v / tot_e;
      if (p > 0) ent -= p * log(p);
    }
  }
  ent = bs_sum(ent, shd);

  if (threadIdx.x == 0) {
    // kept-rank rule (dmrg.cpp:113-136)
    achi_bond_state st = states[bond];
    const int request = st.chi;
    int kept;
    if (cc.mode == ACHI_MODE_FIXED) {
      kept = cc.chi_max;
    } else {
      kept = max(request, floor_rank);
      kept = kept < cc.chi_min ? cc.chi_min : (kept > cc.chi_max ? cc.chi_max : kept);
    }
    if (cc.mode != ACHI_MODE_FIXED) kept = min(kept, max(significant, 1));
    kept = min(kept, r);
    kept = max(kept, 1);
    // controller update from the full spectrum (dmrg.cpp:138-142)
    Decision d;
    const int rc = controller_update(st, ent, floor_rank, cc, d);
    if (rc) {
      out->err = rc;
      return;
    }
    states[bond] = st;
    const double tail = kept < r ? suf[kept] : 0.0;
    const double lam2 = total - tail;
    double margin = INFINITY;
    if (thr > 0) {
      if (kstar >= 1) {
        margin = fabs(suf[kstar] - thr) / thr;
        if (kstar + 1 <= r - 1) margin = fmin(margin, fabs(suf[kstar + 1] - thr) / thr);
      } else if (r >= 2) {
        margin = fabs(suf[1] - thr) / thr;
      }
    }
    out->kept = kept;
    out->err = 0;
    out->floor_rank = floor_rank;
    out->significant = significant;
    out->lam_norm = sqrt(lam2 > 0 ? lam2 : 0.0);
    out->total = total;
    out->entropy = ent;
    out->trunc_error = sqrt(tail > 0 ? tail : 0.0);
    if (trace) {
      trace->sweep = sweep;
      trace->bond = bond;
      trace->chi = d.chi;
      trace->clamped = d.clamped ? 1 : 0;
      trace->delta_chi = d.delta_chi;
      trace->s_raw = d.s_raw;
      trace->s_ema = d.s_ema;
      trace->s_pred = d.s_pred;
      trace->error = d.error;
      trace->p_term = d.p_term;
      trace->i_term = d.i_term;
      trace->d_term = d.d_term;
    }
    if (visit) {
      visit->sweep = sweep;
      visit->bond = bond;
      visit->moving_right = moving_right;
      visit->kept = kept;
      visit->floor_rank = floor_rank;
      visit->significant = significant;
      visit->n_sigma = r;
      visit->degenerate_cut = kept < r && fabs(sigma[kept - 1] - sigma[kept]) <= 1e-12 * s1;
      visit->entropy = ent;
      visit->trunc_error = out->trunc_error;
      visit->floor_margin = margin;
      visit->sigma_kept = sigma[kept - 1] / s1;
      visit->sigma_next = kept < r ? sigma[kept] / s1 : 0.0;
    }
  }
}

// out_host (optional, pinned): the record for the host, written by the kernel
// itself (no separate device-to-host copy on the stream)
__global__ void __launch_bounds__(BS_THREADS) bond_select_kernel(
    const double* __restrict__ sigma, int r, achi_dmrg_config cfg, achi_bond_state* states, int bond,
    int sweep, int moving_right, achi_trace_row* trace, achi_visit_record* visit, BondOut* out,
    BondOut* out_host) {
  pdl_wait();  // launched with launch_pdl (common.cuh)
  bond_select_body(sigma, r, cfg, states, bond, sweep, moving_right, trace, visit, out);
  if (out_host && threadIdx.x == 0) *out_host = *out;  // thread 0 wrote every field of *out
}

// Standalone spectrum reductions (entropy, truncation error at `kept`,
// discarded-weight floor rank, significant count) with the same deterministic
// orders as bond_select_kernel.  out[4]; *err = ACHI_E_* or 0.
__global__ void __launch_bounds__(BS_THREADS) spectrum_stats_kernel(const double* __restrict__ sigma,
                                                                    int r, int kept, double eps,
                                                                    double* out, int* err) {
  extern __shared__ double dyn[];
  double* suf = dyn;
  double* seg = dyn + r + 1;
  __shared__ double shd[33];
  __shared__ int shi[33];
  const double s1 = sigma[0];
  if (!(s1 > 0)) {
    if (threadIdx.x == 0) *err = ACHI_E_DEGENERATE_SPECTRUM;
    return;
  }
  const int per = (r + BS_THREADS - 1) / BS_THREADS;
  const int lo = threadIdx.x * per, hi = min(r, lo + per);
  double acc = 0.0;
  for (int k = hi - 1; k >= lo; --k) {
    acc += sigma[k] * sigma[k];
    suf[k] = acc;
  }
  seg[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    for (int t = (r + per - 1) / per - 1; t >= 0; --t) {  // (segments past r hold zeros)
      const double v = seg[t];
      seg[t] = run;
      run += v;
    }
    suf[r] = 0.0;
  }
  __syncthreads();
  for (int k = lo; k < hi; ++k) suf[k] += seg[threadIdx.x];
  __syncthreads();
  const double thr = eps * suf[0];
  int kstar = 0;
  for (int k = max(lo, 1); k < hi; ++k)
    if (suf[k] > thr) kstar = max(kstar, k);
  kstar = bs_max_int(kstar, shi);
  const double cutoff = 1e-14 * s1;
  double cnt = 0.0, tot_e = 0.0;
  for (int k = threadIdx.x; k < r; k += BS_THREADS) {
    const double v = sigma[k];
    cnt += v > cutoff ? 1.0 : 0.0;
    if (v > cutoff) tot_e += v * v;
  }
  const double significant = bs_sum(cnt, shd);
  tot_e = bs_sum(tot_e, shd);
  double ent = 0.0;
  for (int k = threadIdx.x; k < r; k += BS_THREADS) {
    const double v = sigma[k];
    if (v > cutoff) {
      const double p = v * v / tot_e;
      if (p > 0) ent -= p * log(p);
    }
  }
  ent = bs_sum(ent, shd);
  if (threadIdx.x == 0) {
    out[0] = ent;
    const double tail = (kept >= 1 && kept < r) ? suf[kept] : 0.0;
    out[1] = sqrt(tail > 0 ? tail : 0.0);
    out[2] = kstar >= 1 ? kstar + 1 : 1;
    out[3] = significant;
    *err = 0;
  }
}

struct AbsorbArgs {
  const double* G;
  const double* V;
  long mg, ng;
  const int* perm;
  const double* sorted;
  const double* sign;
  const BondOut* bo;
  int kept, keptp, chl, chlp, chr, chrp, d, right;
  double* site_b;
  double* site_b1;
};

__global__ void absorb_kernel(AbsorbArgs a) {
  pdl_wait();  // launched with launch_pdl (common.cuh)
  const long n_b = static_cast<long>(a.chlp) * a.d * a.keptp;
  const long n_b1 = static_cast<long>(a.keptp) * a.d * a.chrp;
  const double inv_lam = 1.0 / a.bo->lam_norm;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < n_b + n_b1;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    if (t < n_b) {
      const long row = t / a.keptp;
      const int k = static_cast<int>(t - row * a.keptp);
      double v = 0.0;
      if (k < a.kept && row < static_cast<long>(a.chl) * a.d) {
        const long col = a.perm[k];
        if (a.right) {
          v = a.V[col * a.ng + row] * a.sign[k];  // U
        } else {
          v = a.sorted[k] > 0 ? a.G[col * a.mg + row] * a.sign[k] * inv_lam : 0.0;  // U lambda
        }
      }
      a.site_b[t] = v;
    } else {
      const long u = t - n_b;
      const int k = static_cast<int>(u / (static_cast<long>(a.d) * a.chrp));
      const long c = u - static_cast<long>(k) * a.d * a.chrp;
      const int jr = static_cast<int>(c % a.chrp);
      double v = 0.0;
      if (k < a.kept && jr < a.chr) {
        const long col = a.perm[k];
        if (a.right) {
          v = a.sorted[k] > 0 ? a.G[col * a.mg + c] * a.sign[k] * inv_lam : 0.0;  // lambda V^T
        } else {
          v = a.V[col * a.ng + c] * a.sign[k];  // V^T
        }
      }
      a.site_b1[u] = v;
    }
  }
}

}  // namespace

void bond_select(Ctx& ctx, const double* sigma, int r, const achi_dmrg_config& cfg,
                 achi_bond_state* states, int bond, int sweep, int moving_right,
                 achi_trace_row* trace_slot, achi_visit_record* visit_slot, BondOut* out,
                 BondOut* out_host) {
  const size_t smem = sizeof(double) * (static_cast<size_t>(r) + 1 + BS_THREADS);
  per_device_once("bond_select_kernel", ctx.device, [] {
    ACHI_CUDA(cudaFuncSetAttribute(bond_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    return 1;
  });
  if (smem > 200 * 1024) fail(ACHI_E_SIZE_GUARD, "bond_select: spectrum too long");
  ACHI_CUDA(launch_pdl(bond_select_kernel, 1, BS_THREADS, smem, ctx.stream, sigma, r, cfg, states, bond, sweep,
                       moving_right, trace_slot, visit_slot, out, out_host));
  ACHI_LAUNCHED(ctx);
}

void spectrum_stats(Ctx& ctx, const double* sigma, int r, int kept, double eps, double* out,
                    int* err) {
  const size_t smem = sizeof(double) * (static_cast<size_t>(r) + 1 + BS_THREADS);
  per_device_once("spectrum_stats_kernel", ctx.device, [] {
    ACHI_CUDA(cudaFuncSetAttribute(spectrum_stats_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return 1;
  });
  if (smem > 200 * 1024) fail(ACHI_E_SIZE_GUARD, "spectrum_stats: spectrum too long");
  spectrum_stats_kernel<<<1, BS_THREADS, smem, ctx.stream>>>(sigma, r, kept, eps, out, err);
  ACHI_LAUNCHED(ctx);
}

void absorb(Ctx& ctx, const SvdResultDev& r, const double* sign, int kept, const BondOut* bo,
            int chl, int chr, int d, bool moving_right, double* site_b, double* site_b1) {
  AbsorbArgs a;
  a.G = r.G;
  a.V = r.V;
  a.mg = r.mg;
  a.ng = r.ng;
  a.perm = r.perm;
  a.sorted = r.sigma;
  a.sign = sign;
  a.bo = bo;
  a.kept = kept;
  a.keptp = pad2i(kept);
  a.chl = chl;
  a.chlp = pad2i(chl);
  a.chr = chr;
  a.chrp = pad2i(chr);
  a.d = d;
  a.right = moving_right ? 1 : 0;
  a.site_b = site_b;
  a.site_b1 = site_b1;
  const long tot = static_cast<long>(a.chlp) * d * a.keptp + static_cast<long>(a.keptp) * d * a.chrp;
  const int blocks = static_cast<int>(std::min<long>(cdiv(tot, 256), 8L * ctx.num_sms));
  ACHI_CUDA(launch_pdl(absorb_kernel, blocks, 256, 0, ctx.stream, a));
  ACHI_LAUNCHED(ctx);
}

}  // namespace achi
