// Fused bond selection (K7) and truncate/absorb (K8) of one bond visit
// (dmrg.cpp:113-158): entropy monitor, discarded-weight floor, noise guard,
// kept-rank rule, EMA/predictor/PID controller update, truncation error and
// the normalised absorption of lambda into the new site tensors.
#pragma once

#include "common.cuh"
#include "svd_jacobi.cuh"

namespace achi {

struct BondOut {
  int32_t kept, err, floor_rank, significant;
  double lam_norm, total, entropy, trunc_error;
};

// One CTA; sigma (device, r values, non-increasing).  Updates states[bond],
// writes trace[slot]/visit[slot] (either may be null) and *out.
// out_host (optional, pinned host memory): *out is also written there by the kernel.
void bond_select(Ctx& ctx, const double* sigma, int r, const achi_dmrg_config& cfg,
                 achi_bond_state* states, int bond, int sweep, int moving_right,
                 achi_trace_row* trace_slot, achi_visit_record* visit_slot, BondOut* out,
                 BondOut* out_host = nullptr);

// entropy / truncation error / floor rank / significant count of one spectrum
void spectrum_stats(Ctx& ctx, const double* sigma, int r, int kept, double eps, double* out,
                    int* err);

// Write site b (chl~, d, kept~) and site b+1 (kept~, d, chr~) from the SVD
// factors (dmrg.cpp:144-158); moving_right absorbs lambda/||lambda|| into
// site b+1, otherwise into site b.  Pads are written as zeros.
void absorb(Ctx& ctx, const SvdResultDev& r, const double* sign, int kept, const BondOut* bo,
            int chl, int chr, int d, bool moving_right, double* site_b, double* site_b1);

}  // namespace achi
