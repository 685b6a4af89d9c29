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

// ---------------------------------------------------------------------------
// complex128 (planar).  A complex tensor is stored as two planes [Re; Im], each
// in the real padded layout above (plane stride = one plane's element count).
// Every complex contraction is one real DMMA GEMM of doubled M and K:
//   C_planar = realify(A) . B_planar,  realify(A) = [[Ar, -Ai], [Ai, Ar]]
// with the left operand realified (rows (q, m), cols (p, k)) and the right
// operand planar with the contracted index leading (rows (p, k)); the output
// is planar with its M index leading.  Where the H_eff's second GEMM has the
// intermediate on the left, the intermediate is written with the plane inside
// its rows (Y[m, (p, k)]) and each output plane is one GEMM against one half of
// the realified environment.  4 real multiplies per complex one (4M), all on
// the FP64 tensor cores; the MPO mixing stays real (real-gauge W).
// ---------------------------------------------------------------------------

// dst (2M x 2K row-major) = realify of the matrix view z(m, k) = src[m sm + k sk]
// (+ plane offset for the imaginary part), conjugated when `conj`.
void realify(Ctx& ctx, const double* src, long plane, long M, long K, long sm, long sk, bool conj,
             double* dst);
// planar dst[p][k][n] = src[p][n][k] (two planes of rows x cols -> cols x rows)
void planar_transpose(Ctx& ctx, const double* src, long rows, long cols, double* dst);

struct HeffOpsC {
  const double* Lhat;  // realify(L as [(bl, a), jl]): (2 chl~ D1) x (2 chl~)
  const double* Rhat;  // realify(R as [br, (e, jr)]): (2 chr~) x (2 D3 chr~)
  int chl, chr;        // padded
  int d, D1, D3;
  DevMix mix;
};
// out = H_eff theta on planar (chl~, d, d, chr~) complex tensors (dmrg.cpp:58-71)
void heff_apply_c(Ctx& ctx, const HeffOpsC& op, const double* theta, double* out);
// Lhat / Rhat of HeffOpsC from planar environments
void heff_prepare_c(Ctx& ctx, const double* L, int chl, int D1, const double* R, int chr, int D3,
                    double* Lhat, double* Rhat);
// planar environment updates (update_left / update_right, dmrg.cpp:26-49); scr
// holds >= max(4 chl~^2 Dl, 4 chn~ chl~ d) (left) / max(4 chr~^2 Dr, 4 chn~ d chr~)
// + 2 chn~ d chr~ (right) doubles
void env_left_c(Ctx& ctx, const double* L, const double* A, int chl, int chn, int d, int Dl, int Dr,
                const DevMix& mix, double* scr, double* Lnew);
void env_right_c(Ctx& ctx, const double* R, const double* B, int chr, int chn, int d, int Dl,
                 int Dr, const DevMix& mix, double* scr, double* Rnew);
// planar theta (chl~, d, d, chr~) = A . B; scr >= 4 chl~ d chm~ doubles
void theta_merge_c(Ctx& ctx, const double* A, const double* B, int chl, int chm, int chr, int d,
                   double* scr, double* theta);

// Copy a host (l, d, r) tensor into a padded device tensor (l~, d, r~) with zero pads.
void upload_padded3(Ctx& ctx, const double* host, int l, int d, int r, double* dev);
// Copy a padded device tensor (l~, m, r~) to host (l, m, r).
void download_padded3(Ctx& ctx, const double* dev, int l, int m, int r, double* host);

}  // namespace achi
