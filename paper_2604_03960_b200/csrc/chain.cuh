// Device-resident DMRG chain: MPS sites, left/right environment blocks and
// per-bond controller states live in HBM; the host drives the sweep
// (two_site_sweep, dmrg.cpp:175-214) and reads back only the kept rank per
// visit plus Lanczos convergence scalars.
#pragma once

#include <vector>

#include "bond.cuh"
#include "contract.cuh"
#include "lanczos.cuh"
#include "svd_jacobi.cuh"

struct achi_ctx {
  achi::Ctx c;
};

namespace achi {

// models.cpp:49-97 with the sigma^y channel in the real gauge (iY, -jy*iY)
std::vector<HostMpo> build_mpo_real(const achi_model_spec& spec);
void validate_spec(const achi_model_spec& spec);
void validate_config(const achi_dmrg_config& cfg);

struct VisitHost {
  double energy, residual;
  int matvecs;
};

// canonicalize(psi, 0) (mps.cpp:172-210) on the device: host site tensors
// (l, d, r row-major) in, unpadded device site tensors out (`times` passes,
// the centre site normalised between passes as random_mps does).
std::vector<DevBuf> canonical_on_device(Ctx& c, const std::vector<std::vector<double>>& sites,
                                        std::vector<int>& dims, int d, int times = 1);

// complex128 counterparts (chain_complex.cu): canonicalize(psi, 0) of host
// sites given as interleaved (re, im) (l, d, r) tensors, on the device by
// complex SVD push_left; returns unpadded interleaved device sites.
std::vector<DevBuf> canonical_on_device_c(Ctx& c, const std::vector<std::vector<double>>& sites,
                                          std::vector<int>& dims, int d, int times = 1);
// random_mps (mps.cpp:75-95): the reference's mt19937_64 complex draws
std::vector<std::vector<double>> random_complex_sites(int n, int d, int chi, uint64_t seed,
                                                      std::vector<int>& dims_out);

struct Chain {
  Ctx* ctx = nullptr;
  achi_ctx* owner = nullptr;
  achi_model_spec spec{};
  achi_dmrg_config cfg{};
  int n = 0, d = 2;
  std::vector<HostMpo> mpo;
  MixStore mixes;
  std::vector<DevMix> mheff, mleft, mright;
  std::vector<int> chi, cap;  // chi[k]: bond between sites k-1 and k (chi[0] = chi[n] = 1)
  std::vector<DevBuf> site, L, R;
  DevArr<achi_bond_state> states;
  DevArr<achi_trace_row> trace;
  DevArr<achi_visit_record> visits;
  DevArr<BondOut> bout;
  PinnedArr<BondOut> bout_h;
  DevBuf theta, vec;
  LanczosWs lz;
  SvdWs svd;
  // SVD warm start (svd_device v_init): the last orthogonal factor of each bond
  // per sweep direction with the padded/true theta shape it belongs to.  Once
  // the state has converged, the same bond's block changes little between
  // sweeps, so the previous factor nearly diagonalises it.
  struct VKeep {
    DevBuf v;
    int m = 0, n = 0, mt = 0, nt = 0;
    bool valid = false;
  };
  std::vector<VKeep> vkeep;  // [2 b + moving_right]
  bool warm_svd = true;
  std::vector<VisitHost> vh;
  // phase wall-clock accounting (host steady_clock at the existing sync points)
  struct Stats {
    double merge_lanczos = 0, svd = 0, select = 0, absorb_env = 0;
    long matvecs = 0, svd_sweeps = 0, visits = 0;
  } stats;
  bool profile = false;  // sync after each visit so phase times are exact
  // complex128 chain: every site / environment / theta buffer holds two planes
  // [Re; Im] of the real padded layout (contract.cuh); lhat / rhat are the
  // realified environments of the current visit, scr the realified operands of
  // the merge and the environment updates, cth / cu / cv / csig the
  // interleaved theta and SVD factors of the complex SVD.
  bool cplx = false;
  DevBuf lhat, rhat, scr, cth, cu, cv, csig, cv_keep;
  CsvdPlan cplan;
  // run-level bookkeeping (dmrg.cpp:255-281)
  double prev_energy = 0;
  bool have_prev = false;

  void create(Ctx& c, const achi_model_spec& s, const achi_dmrg_config& g);
  void rebuild_envs();
  double expectation_energy();
  void upload_sites(const std::vector<std::vector<double>>& host_sites);
  void copy_sites_device(const std::vector<DevBuf>& device_sites);
  void visit(int bond, bool moving_right, int sweep, int slot);
  void visit_complex(int bond, bool moving_right, int sweep, int slot);
  // interleaved complex sites: host (l, d, r) -> padded planar storage, and back
  void upload_sites_c(const std::vector<std::vector<double>>& host_sites);
  void copy_sites_device_c(const std::vector<DevBuf>& device_sites);
  void download_site_c(int k, double* out);
  void sweep(int sweep_index, achi_sweep_record* rec, int32_t* chi_profile, double* entropy,
             achi_trace_row* trace_out, achi_visit_record* visits_out);
  long site_size(int k) const { return static_cast<long>(pad2i(chi[k])) * d * pad2i(chi[k + 1]); }
};

}  // namespace achi

struct achi_chain {
  achi::Chain ch;
};
