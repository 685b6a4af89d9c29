// Tensor-network contractions of the two-site local update, each written as
// DMMA GEMM -> sparse MPO mixing -> DMMA GEMM with no permutation copies.
//
// Device layouts are the reference's row-major layouts with every bond
// dimension stored padded to even (chi~ = chi + chi%2, pad entries exactly
// zero) so that all TMA row strides are 16-byte multiples.  Zero pads are
// preserved by every kernel (GEMMs of zero rows/cols give zero; the mixing
// is linear).
#pragma once

#include "gemm_dmma.cuh"

namespace achi {

// Sparse mixing matrix (CSR by output row) for one MPO contraction step.
struct MixMatrix {
  int nout = 0, nin = 0;
  std::vector<int> rowptr, col;
  std::vector<double> val;
};

// Device copy of a MixMatrix: int rowptr[nout+1], int col[nnz], double val[nnz].
struct DevMix {
  int nout = 0, nin = 0, nnz = 0;
  const int* rowptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
};

// MPO tensor W(l, so, si, r) (models.hpp:25-26), row-major, host copy.
struct HostMpo {
  int l, d, r;
  std::vector<double> w;
  double at(int a, int so, int si, int b) const {
    return w[((static_cast<size_t>(a) * d + so) * d + si) * r + b];
  }
};

// H_eff mixing W12[(s1',s2',e),(a,s1,s2)] = sum_c W1(a,s1',s1,c) W2(c,s2',s2,e)
MixMatrix mix_heff(const HostMpo& w1, const HostMpo& w2);
// env-left mixing WL[(s',a'),(a,s)] = W(a,s',s,a')
MixMatrix mix_env_left(const HostMpo& w);
// env-right mixing WR[(s',a),(e,s)] = W(a,s',s,e)
MixMatrix mix_env_right(const HostMpo& w);

// Upload a set of mixing matrices into one device block; returns descriptors.
struct MixStore {
  DevArr<unsigned char> blob;
  std::vector<DevMix> upload(Ctx& ctx, const std::vector<MixMatrix>& ms);
};

// Operands of the local update at one bond (device pointers, padded dims).
struct HeffOps {
  const double* L;  // (chl~, D1, chl~)
  const double* R;  // (chr~, D3, chr~)
  int chl, chr;     // padded
  int d, D1, D3;
  DevMix mix;       // mix_heff(W_b, W_{b+1})
};

// out = H_eff theta (dmrg.cpp:58-71); theta/out (chl~, d, d, chr~).  Bonds with
// chl~, chr~ <= 128 take the fused one-launch path (heff_small.cu), larger ones
// the TMA GEMM -> mixing -> GEMM path.
void heff_apply(Ctx& ctx, const HeffOps& op, const double* theta, double* out);
bool heff_small_applicable(const HeffOps& op);
void heff_apply_small(Ctx& ctx, const HeffOps& op, const double* theta, double* out);

// Lnew (chn~, Dr, chn~) from L (chl~, Dl, chl~) and A (chl~, d, chn~) (dmrg.cpp:26-37)
void env_left(Ctx& ctx, const double* L, const double* A, int chl, int chn, int d, int Dl, int Dr,
              const DevMix& mix, double* Lnew);
// Rnew (chn~, Dl, chn~) from R (chr~, Dr, chr~) and B (chn~, d, chr~) (dmrg.cpp:39-49)
void env_right(Ctx& ctx, const double* R, const double* B, int chr, int chn, int d, int Dl, int Dr,
               const DevMix& mix, double* Rnew);
// theta (chl~, d, d, chr~) = A (chl~, d, chm~) . B (chm~, d, chr~)  (dmrg.cpp:94)
void theta_merge(Ctx& ctx, const double* A, const double* B, int chl, int chm, int chr, int d,
                 double* theta);

// Copy a host (l, d, r) tensor into a padded device tensor (l~, d, r~) with zero pads.
void upload_padded3(Ctx& ctx, const double* host, int l, int d, int r, double* dev);
// Copy a padded device tensor (l~, m, r~) to host (l, m, r).
void download_padded3(Ctx& ctx, const double* dev, int l, int m, int r, double* host);

}  // namespace achi
