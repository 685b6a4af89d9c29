// extern "C" boundary (include/adaptchi_b200.h): typed errors -> int codes.
#include <cmath>
#include <cstring>
#include <memory>

#include "chain.cuh"
#include "ozaki.cuh"

using namespace achi;

namespace {

int guard(achi_ctx* ctx, const std::function<void()>& f) {
  AllocStream as(ctx ? ctx->c.stream : nullptr);
  try {
    // a thread may drive contexts on several GPUs, or one created elsewhere
    if (ctx) ACHI_CUDA(cudaSetDevice(ctx->c.device));
    f();
    if (ctx) ctx->c.last_error.clear();
    return ACHI_OK;
  } catch (const Error& e) {
    if (ctx) {
      ctx->c.last_error = e.what();
      ctx->c.last_residual = e.residual;
    }
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.last_error = e.what();
    return ACHI_E_ERROR;
  }
}

__global__ void dense_gemv_kernel(const double* __restrict__ h, int dim, const double* __restrict__ x,
                                  double* __restrict__ y) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= dim) return;
  double s = 0.0;
  for (int j = lane; j < dim; j += 32) s += h[static_cast<long>(row) * dim + j] * x[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// deterministic pseudo-random fill in [-1, 1) (splitmix64), for timing hooks
__global__ void fill_random_kernel(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull + seed * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = static_cast<double>(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

void fill_random(Ctx& c, double* p, size_t n, unsigned long long seed) {
  fill_random_kernel<<<4 * c.num_sms, 256, 0, c.stream>>>(p, n, seed);
  ACHI_LAUNCHED(c);
}

HostMpo host_mpo(const double* w, int l, int d, int r) {
  HostMpo m{l, d, r, std::vector<double>(w, w + static_cast<size_t>(l) * d * d * r)};
  return m;
}

void h2d(Ctx& c, double* dst, const double* src, size_t n) {
  ACHI_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
}
void d2h(Ctx& c, double* dst, const double* src, size_t n) {
  ACHI_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
}

}  // namespace

extern "C" {

int achi_ctx_create(int device, achi_ctx** out) {
  return guard(nullptr, [&] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device)
      fail(ACHI_E_NO_DEVICE, "no CUDA device");
    cudaDeviceProp prop;
    ACHI_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(ACHI_E_NO_DEVICE, "device is not sm_100 (B200)");
    ACHI_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<achi_ctx>();
    ctx->c.device = device;
    ctx->c.num_sms = prop.multiProcessorCount;
    ACHI_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    ACHI_CUDA(cudaStreamCreateWithFlags(&ctx->c.aux, cudaStreamNonBlocking));
    ACHI_CUDA(cudaEventCreateWithFlags(&ctx->c.ev_fork, cudaEventDisableTiming));
    ACHI_CUDA(cudaEventCreateWithFlags(&ctx->c.ev_join, cudaEventDisableTiming));
    ACHI_CUDA(cudaStreamCreateWithFlags(&ctx->c.vstream, cudaStreamNonBlocking));
    ACHI_CUDA(cudaEventCreateWithFlags(&ctx->c.ev_v0, cudaEventDisableTiming));
    ACHI_CUDA(cudaEventCreateWithFlags(&ctx->c.ev_v1, cudaEventDisableTiming));
    // keep freed pool memory cached (stream-ordered allocations, common.cuh)
    cudaMemPool_t pool;
    ACHI_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    ACHI_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    {
      // the split-K workspace is used inside captured graphs: size it up front
      AllocStream as(ctx->c.stream);
      ctx->c.ws_split.reserve(4096UL * 592);
    }
    *out = ctx.release();
  });
}

int achi_ctx_set_grid_cap(achi_ctx* ctx, int max_ctas) {
  return guard(ctx, [&] {
    if (max_ctas < 0) fail(ACHI_E_INVALID_CONFIG, "grid cap must be >= 0");
    ctx->c.grid_cap = max_ctas;
  });
}

int achi_ctx_destroy(achi_ctx* ctx) {
  if (!ctx) return ACHI_OK;
  cudaSetDevice(ctx->c.device);
  cudaStream_t s = ctx->c.stream, aux = ctx->c.aux, vs = ctx->c.vstream;
  cudaEvent_t e1 = ctx->c.ev_fork, e2 = ctx->c.ev_join, e3 = ctx->c.ev_v0, e4 = ctx->c.ev_v1;
  cudaStreamSynchronize(vs);  // no V replay may outlive the buffers it writes
  {
    AllocStream as(s);
    delete ctx;
  }
  cudaStreamSynchronize(s);
  cudaStreamSynchronize(aux);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  cudaEventDestroy(e3);
  cudaEventDestroy(e4);
  cudaStreamDestroy(vs);
  cudaStreamDestroy(aux);
  cudaStreamDestroy(s);
  return ACHI_OK;
}

int achi_last_error(const achi_ctx* ctx, char* buf, size_t len) {
  if (!ctx || !buf || !len) return ACHI_OK;
  std::snprintf(buf, len, "%s", ctx->c.last_error.c_str());
  return ACHI_OK;
}

double achi_last_residual(const achi_ctx* ctx) { return ctx ? ctx->c.last_residual : 0.0; }
int64_t achi_launch_count(const achi_ctx* ctx) { return ctx ? ctx->c.launches : 0; }
int achi_synchronize(achi_ctx* ctx) {
  return guard(ctx, [&] { ctx->c.sync(); });
}

int achi_timer_start(achi_ctx* ctx) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (!c.ev0) {
      ACHI_CUDA(cudaEventCreate(&c.ev0));
      ACHI_CUDA(cudaEventCreate(&c.ev1));
    }
    c.sync();
    ACHI_CUDA(cudaEventRecord(c.ev0, c.stream));
  });
}

int achi_timer_stop(achi_ctx* ctx, double* ms) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    ACHI_CUDA(cudaEventRecord(c.ev1, c.stream));
    ACHI_CUDA(cudaEventSynchronize(c.ev1));
    float f = 0;
    ACHI_CUDA(cudaEventElapsedTime(&f, c.ev0, c.ev1));
    *ms = f;
  });
}

int achi_flush_l2(achi_ctx* ctx, size_t bytes) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const size_t n = bytes / sizeof(double);
    c.flush.reserve(n);
    ACHI_CUDA(cudaMemsetAsync(c.flush.p, 0, n * sizeof(double), c.stream));
  });
}

int achi_ctx_set_ozaki(achi_ctx* ctx, int slices, double min_flops) {
  return guard(ctx, [&] {
    if (slices != 0 && (slices < 2 || slices > OZ_MAX_SLICES)) fail(ACHI_E_INVALID_CONFIG, "ozaki: slices 0 or 2..9");
    ctx->c.ozaki_slices = slices;
    ctx->c.ozaki_min_flops = min_flops;
  });
}

int achi_ctx_set_lanczos_graph(achi_ctx* ctx, int mode) {
  return guard(ctx, [&] { ctx->c.lanczos_graph = mode < 0 ? -1 : (mode ? 1 : 0); });
}

int achi_device_times(achi_ctx* ctx, int enable, int reset, double* out9) {
  return achi_device_times_ex(ctx, enable, reset, out9, 3);
}

int achi_device_times_ex(achi_ctx* ctx, int enable, int reset, double* out, int n_phases) {
  return guard(ctx, [&] {
    if (n_phases < 0 || n_phases > EventAcc::kNumTags) fail(ACHI_E_INVALID_CONFIG, "device_times: n_phases");
    EventAcc& a = ctx->c.acc;
    ctx->c.sync();
    a.resolve();
    if (out)
      for (int t = 0; t < n_phases; ++t) {
        out[t] = a.ms[t];
        out[n_phases + t] = a.work[t];
        out[2 * n_phases + t] = static_cast<double>(a.count[t]);
      }
    if (reset)
      for (int t = 0; t < EventAcc::kNumTags; ++t) a.ms[t] = a.work[t] = 0, a.count[t] = 0;
    if (enable >= 0) {
      a.enabled = enable != 0;
      a.sample = std::max(1, enable);  // enable = n > 1: time one chain visit in n
      a.visit_seq = 0;
    }
  });
}

// ---- chain ----
int achi_chain_create(achi_ctx* ctx, const achi_model_spec* spec, const achi_dmrg_config* cfg,
                      achi_chain** out) {
  return guard(ctx, [&] {
    auto ch = std::make_unique<achi_chain>();
    ch->ch.owner = ctx;
    ch->ch.create(ctx->c, *spec, *cfg);
    *out = ch.release();
  });
}

int achi_chain_destroy(achi_chain* chain) {
  if (chain) {
    AllocStream as(chain->ch.ctx->stream);
    try {
      svd_wait_v(*chain->ch.ctx, chain->ch.svd);  // its buffers are freed on the main stream
    } catch (...) {
    }
    delete chain;
  }
  return ACHI_OK;
}

int achi_chain_sweep(achi_chain* chain, int sweep_index, achi_sweep_record* rec,
                     int32_t* chi_profile, double* entropy_profile, achi_trace_row* trace,
                     achi_visit_record* visits) {
  achi_ctx* ctx = chain->ch.owner;
  return guard(ctx, [&] {
    chain->ch.sweep(sweep_index, rec, chi_profile, entropy_profile, trace, visits);
  });
}

// run_dmrg sweep loop + convergence (dmrg.cpp:255-281)
int achi_chain_run(achi_chain* chain, achi_dmrg_result* result, achi_sweep_record* records,
                   int32_t* chi_profiles, double* entropy_profiles, achi_trace_row* trace,
                   achi_visit_record* visits) {
  Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    const int nb = ch.n - 1, nv = 2 * (ch.n - 1);
    achi_dmrg_result res{};
    double prev = 0;
    bool have_prev = false;
    for (int s = 0; s < ch.cfg.max_sweeps; ++s) {
      achi_sweep_record rec{};
      ch.sweep(s, &rec, chi_profiles ? chi_profiles + static_cast<long>(s) * nb : nullptr,
               entropy_profiles ? entropy_profiles + static_cast<long>(s) * nb : nullptr,
               trace ? trace + static_cast<long>(s) * nv : nullptr,
               visits ? visits + static_cast<long>(s) * nv : nullptr);
      res.max_chi_used = std::max(res.max_chi_used, rec.max_chi_used);
      if (have_prev) {
        const double delta = rec.energy - prev;
        rec.delta_e_rel = std::fabs(delta) / std::max(std::fabs(rec.energy), 1e-300);
        if (delta > 0) res.max_monotonicity_violation = std::max(res.max_monotonicity_violation, delta);
      } else {
        rec.delta_e_rel = std::numeric_limits<double>::infinity();
      }
      if (records) records[s] = rec;
      res.n_sweeps = s + 1;
      if (have_prev && rec.delta_e_rel < ch.cfg.eps_conv) {
        res.converged = 1;
        prev = rec.energy;
        break;
      }
      prev = rec.energy;
      have_prev = true;
    }
    res.energy = prev;
    if (result) *result = res;
  });
}

int achi_chain_stats(achi_chain* chain, int profile, double* out8) {
  Chain& ch = chain->ch;
  ch.profile = profile != 0;
  if (out8) {
    out8[0] = ch.stats.merge_lanczos;
    out8[1] = ch.stats.svd;
    out8[2] = ch.stats.select;
    out8[3] = ch.stats.absorb_env;
    out8[4] = static_cast<double>(ch.stats.matvecs);
    out8[5] = static_cast<double>(ch.stats.svd_sweeps);
    out8[6] = static_cast<double>(ch.stats.visits);
    out8[7] = 0;
  }
  return ACHI_OK;
}

int achi_chain_bond_dims(const achi_chain* chain, int32_t* dims) {
  for (int k = 1; k < chain->ch.n; ++k) dims[k - 1] = chain->ch.chi[k];
  return ACHI_OK;
}

int achi_chain_get_site(const achi_chain* chain, int k, double* out, size_t capacity) {
  const Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    if (k < 0 || k >= ch.n) fail(ACHI_E_INVALID_RANK, "site index out of range");
    if (ch.cplx) fail(ACHI_E_UNSUPPORTED_MODEL, "complex chain: use achi_chain_get_site_complex");
    const int l = ch.chi[k], r = ch.chi[k + 1];
    if (capacity < static_cast<size_t>(l) * ch.d * r) fail(ACHI_E_SIZE_GUARD, "capacity");
    download_padded3(*ch.ctx, ch.site[k].p, l, ch.d, r, out);
  });
}

int achi_chain_is_complex(const achi_chain* chain) { return chain && chain->ch.cplx ? 1 : 0; }

int achi_chain_get_site_complex(const achi_chain* chain, int k, double* out, size_t capacity) {
  achi_chain* ch_ = const_cast<achi_chain*>(chain);
  Chain& ch = ch_->ch;
  return guard(ch.owner, [&] {
    if (k < 0 || k >= ch.n) fail(ACHI_E_INVALID_RANK, "site index out of range");
    if (!ch.cplx) fail(ACHI_E_UNSUPPORTED_MODEL, "real chain: use achi_chain_get_site");
    const int l = ch.chi[k], r = ch.chi[k + 1];
    if (capacity < 2 * static_cast<size_t>(l) * ch.d * r) fail(ACHI_E_SIZE_GUARD, "capacity");
    ch.download_site_c(k, out);
  });
}

int achi_chain_load_mps_complex(achi_chain* chain, const int32_t* bond_dims, const double* const* sites,
                                int canonicalize) {
  Chain& ch = chain->ch;
  return guard(ch.owner, [&] {
    if (!ch.cplx) fail(ACHI_E_UNSUPPORTED_MODEL, "real chain: use achi_chain_load_mps");
    std::vector<int> dims(ch.n + 1, 1);
    for (int k = 1; k < ch.n; ++k) {
      if (bond_dims[k - 1] < 1) fail(ACHI_E_INVALID_RANK, "load_mps: bond dimension must be >= 1");
      dims[k] = bond_dims[k - 1];
    }
    std::vector<std::vector<double>> hs(ch.n);
    for (int k = 0; k < ch.n; ++k) {
      const size_t sz = 2 * static_cast<size_t>(dims[k]) * ch.d * dims[k + 1];
      hs[k].assign(sites[k], sites[k] + sz);
      for (double x : hs[k])
        if (!std::isfinite(x)) fail(ACHI_E_INVALID_MATRIX, "load_mps: non-finite site entry");
    }
    std::vector<DevBuf> ds;
    if (canonicalize) ds = canonical_on_device_c(*ch.ctx, hs, dims, ch.d);
    for (int k = 1; k < ch.n; ++k)
      if (dims[k] > ch.cap[k]) fail(ACHI_E_INVALID_RANK, "load_mps: bond dimension exceeds capacity");
    for (int k = 1; k < ch.n; ++k) ch.chi[k] = dims[k];
    if (canonicalize)
      ch.copy_sites_device_c(ds);
    else
      ch.upload_sites_c(hs);
    ch.rebuild_envs();
    ch.ctx->sync();
  });
}

int achi_chain_get_env(const achi_chain* chain, int which, int k, int64_t* shape3, double* out,
                       size_t capacity) {
  const Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    if (k < 0 || k >= ch.n) fail(ACHI_E_INVALID_RANK, "env index out of range");
    if (ch.cplx) fail(ACHI_E_UNSUPPORTED_MODEL, "complex chain: environments are planar complex");
    const int chi = which == 0 ? ch.chi[k] : ch.chi[k + 1];
    const int D = which == 0 ? ch.mpo[k].l : ch.mpo[k].r;
    shape3[0] = chi;
    shape3[1] = D;
    shape3[2] = chi;
    if (out) {
      if (capacity < static_cast<size_t>(chi) * D * chi) fail(ACHI_E_SIZE_GUARD, "capacity");
      download_padded3(*ch.ctx, which == 0 ? ch.L[k].p : ch.R[k].p, chi, D, chi, out);
    }
  });
}

int achi_chain_get_states(const achi_chain* chain, achi_bond_state* out) {
  const Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    ACHI_CUDA(cudaMemcpyAsync(out, ch.states.p, sizeof(achi_bond_state) * (ch.n - 1),
                              cudaMemcpyDeviceToHost, ch.ctx->stream));
    ch.ctx->sync();
  });
}

int achi_chain_set_states(achi_chain* chain, const achi_bond_state* in) {
  Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    ACHI_CUDA(cudaMemcpyAsync(ch.states.p, in, sizeof(achi_bond_state) * (ch.n - 1),
                              cudaMemcpyHostToDevice, ch.ctx->stream));
    ch.ctx->sync();
  });
}

int achi_chain_load_mps(achi_chain* chain, const int32_t* bond_dims, const double* const* sites,
                        int canonicalize) {
  Chain& ch = chain->ch;
  achi_ctx* ctx = ch.owner;
  return guard(ctx, [&] {
    if (ch.cplx) fail(ACHI_E_UNSUPPORTED_MODEL, "complex chain: use achi_chain_load_mps_complex");
    std::vector<int> dims(ch.n + 1, 1);
    for (int k = 1; k < ch.n; ++k) {
      if (bond_dims[k - 1] < 1) fail(ACHI_E_INVALID_RANK, "load_mps: bond dimension must be >= 1");
      dims[k] = bond_dims[k - 1];
    }
    std::vector<std::vector<double>> hs(ch.n);
    for (int k = 0; k < ch.n; ++k) {
      const size_t sz = static_cast<size_t>(dims[k]) * ch.d * dims[k + 1];
      hs[k].assign(sites[k], sites[k] + sz);
      for (double x : hs[k])
        if (!std::isfinite(x)) fail(ACHI_E_INVALID_MATRIX, "load_mps: non-finite site entry");
    }
    std::vector<DevBuf> ds;
    if (canonicalize) ds = canonical_on_device(*ch.ctx, hs, dims, ch.d);  // canonicalize(psi, 0), mps.cpp:204-210
    for (int k = 1; k < ch.n; ++k)
      if (dims[k] > ch.cap[k]) fail(ACHI_E_INVALID_RANK, "load_mps: bond dimension exceeds capacity");
    for (int k = 1; k < ch.n; ++k) ch.chi[k] = dims[k];
    if (canonicalize)
      ch.copy_sites_device(ds);
    else
      ch.upload_sites(hs);
    ch.rebuild_envs();
    ch.ctx->sync();
  });
}

int achi_chain_load_state(achi_chain* chain, const int32_t* bond_dims, const double* const* sites) {
  return achi_chain_load_mps(chain, bond_dims, sites, 0);
}

int achi_chain_energy(achi_chain* chain, double* energy) {
  Chain& ch = chain->ch;
  return guard(ch.owner, [&] {
    if (!energy) fail(ACHI_E_INVALID_CONFIG, "chain_energy: null output");
    *energy = ch.expectation_energy();
  });
}

// ---- local kernels on host buffers ----
int achi_heff_apply(achi_ctx* ctx, int chl, int chr, int d, int D1, int D2, int D3,
                    const double* L, const double* W1, const double* W2, const double* R,
                    const double* theta, double* out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const int lp = pad2i(chl), rp = pad2i(chr);
    DevBuf dL, dR, dT, dO;
    dL.reserve(static_cast<size_t>(lp) * D1 * lp);
    dR.reserve(static_cast<size_t>(rp) * D3 * rp);
    dT.reserve(static_cast<size_t>(lp) * d * d * rp);
    dO.reserve(static_cast<size_t>(lp) * d * d * rp);
    upload_padded3(c, L, chl, D1, chl, dL.p);
    upload_padded3(c, R, chr, D3, chr, dR.p);
    upload_padded3(c, theta, chl, d * d, chr, dT.p);
    MixStore ms;
    auto mix = ms.upload(c, {mix_heff(host_mpo(W1, D1, d, D2), host_mpo(W2, D2, d, D3))});
    HeffOps op{dL.p, dR.p, lp, rp, d, D1, D3, mix[0]};
    heff_apply(c, op, dT.p, dO.p);
    download_padded3(c, dO.p, chl, d * d, chr, out);
  });
}

int achi_env_update_left(achi_ctx* ctx, int chl, int chn, int d, int Dl, int Dr, const double* L,
                         const double* A, const double* W, double* Lnew) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const int lp = pad2i(chl), np = pad2i(chn);
    DevBuf dL, dA, dO;
    dL.reserve(static_cast<size_t>(lp) * Dl * lp);
    dA.reserve(static_cast<size_t>(lp) * d * np);
    dO.reserve(static_cast<size_t>(np) * Dr * np);
    upload_padded3(c, L, chl, Dl, chl, dL.p);
    upload_padded3(c, A, chl, d, chn, dA.p);
    MixStore ms;
    auto mix = ms.upload(c, {mix_env_left(host_mpo(W, Dl, d, Dr))});
    env_left(c, dL.p, dA.p, lp, np, d, Dl, Dr, mix[0], dO.p);
    download_padded3(c, dO.p, chn, Dr, chn, Lnew);
  });
}

int achi_env_update_right(achi_ctx* ctx, int chr, int chn, int d, int Dl, int Dr, const double* R,
                          const double* B, const double* W, double* Rnew) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const int rp = pad2i(chr), np = pad2i(chn);
    DevBuf dR, dB, dO;
    dR.reserve(static_cast<size_t>(rp) * Dr * rp);
    dB.reserve(static_cast<size_t>(np) * d * rp);
    dO.reserve(static_cast<size_t>(np) * Dl * np);
    upload_padded3(c, R, chr, Dr, chr, dR.p);
    upload_padded3(c, B, chn, d, chr, dB.p);
    MixStore ms;
    auto mix = ms.upload(c, {mix_env_right(host_mpo(W, Dl, d, Dr))});
    env_right(c, dR.p, dB.p, rp, np, d, Dl, Dr, mix[0], dO.p);
    download_padded3(c, dO.p, chn, Dl, chn, Rnew);
  });
}

int achi_svd(achi_ctx* ctx, int m, int n, const double* a, double* sigma, double* u, double* vt,
             int* sweeps_out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (m < 1 || n < 1) fail(ACHI_E_INVALID_MATRIX, "svd: matrix must be at least 1x1");
    for (long i = 0; i < static_cast<long>(m) * n; ++i)
      if (!std::isfinite(a[i])) fail(ACHI_E_INVALID_MATRIX, "svd: non-finite entries");
    DevBuf dA, dS, dU, dV;
    dA.reserve(static_cast<size_t>(m) * n);
    h2d(c, dA.p, a, static_cast<size_t>(m) * n);
    SvdWs ws;
    ws.vrecover = true;
    const SvdSide side = m <= n ? SvdSide::kRows : SvdSide::kCols;
    SvdResultDev r = svd_device(c, ws, dA.p, m, n, m, n, side);
    const int k = r.r_true;
    svd_phase_signs(c, ws, r, k);
    dU.reserve(static_cast<size_t>(m) * k);
    dV.reserve(static_cast<size_t>(k) * n);
    svd_gather(c, ws, r, k, dU.p, dV.p);
    if (sigma) d2h(c, sigma, r.sigma, k);
    if (u) d2h(c, u, dU.p, static_cast<size_t>(m) * k);
    if (vt) d2h(c, vt, dV.p, static_cast<size_t>(k) * n);
    c.sync();
    if (sweeps_out) *sweeps_out = r.sweeps();
  });
}

int achi_svd_batched(achi_ctx* ctx, int batch, int m, int n, const double* a, double* sigma) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const long mn = static_cast<long>(m) * n;
    DevBuf dA, dS;
    dA.reserve(static_cast<size_t>(mn) * batch);
    const int k = std::min(m, n);
    dS.reserve(static_cast<size_t>(k) * batch);
    h2d(c, dA.p, a, static_cast<size_t>(mn) * batch);
    SvdWs ws;
    svd_device(c, ws, dA.p, m, n, m, n, m <= n ? SvdSide::kRows : SvdSide::kCols, batch, mn, dS.p,
               false);
    d2h(c, sigma, dS.p, static_cast<size_t>(k) * batch);
    c.sync();
  });
}

int achi_svd_batched_device(achi_ctx* ctx, int batch, int m, int n, const double* d_a,
                            double* d_sigma, int* sweeps_out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    static thread_local SvdWs ws;  // reused across benchmark calls (no realloc per call)
    SvdResultDev r = svd_device(c, ws, d_a, m, n, m, n, m <= n ? SvdSide::kRows : SvdSide::kCols,
                                batch, static_cast<long>(m) * n, d_sigma, false);
    c.sync();
    if (sweeps_out) *sweeps_out = r.sweeps();
  });
}

int achi_svd_device(achi_ctx* ctx, int m, int n, const double* d_a, double* d_sigma, double* d_u,
                    double* d_vt, int* sweeps_out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (m < 1 || n < 1) fail(ACHI_E_INVALID_MATRIX, "svd: matrix must be at least 1x1");
    static thread_local SvdWs ws;
    ws.vrecover = true;
    static const int side_env = [] {  // study knob: force the orthogonalised side (rows|cols)
      const char* e = std::getenv("ACHI_SVD_SIDE");
      return e ? (e[0] == 'r' ? 0 : 1) : -1;
    }();
    const SvdSide side = side_env < 0 ? (m <= n ? SvdSide::kRows : SvdSide::kCols)
                                      : (side_env == 0 ? SvdSide::kRows : SvdSide::kCols);
    SvdResultDev r = svd_device(c, ws, d_a, m, n, m, n, side);
    const int k = r.r_true;
    svd_phase_signs(c, ws, r, k);
    svd_gather(c, ws, r, k, d_u, d_vt);
    if (d_sigma)
      ACHI_CUDA(cudaMemcpyAsync(d_sigma, r.sigma, sizeof(double) * k, cudaMemcpyDeviceToDevice, c.stream));
    c.sync();
    if (sweeps_out) *sweeps_out = r.sweeps();
  });
}

int achi_svd_complex_device(achi_ctx* ctx, int m, int n, const double* d_a, double* d_sigma,
                            double* d_u, double* d_vdag, int* sweeps_out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (m < 1 || n < 1) fail(ACHI_E_INVALID_MATRIX, "svd: matrix must be at least 1x1");
    SvdWs ws;
    ws.vrecover = true;
    const int sw = svd_complex_device(c, ws, d_a, m, n, d_sigma, d_u, d_vdag);
    if (sweeps_out) *sweeps_out = sw;
  });
}

int achi_svd_complex(achi_ctx* ctx, int m, int n, const double* a, double* sigma, double* u,
                     double* vdag, int* sweeps_out) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (m < 1 || n < 1) fail(ACHI_E_INVALID_MATRIX, "svd: matrix must be at least 1x1");
    const size_t mn2 = 2 * static_cast<size_t>(m) * n;
    for (size_t i = 0; i < mn2; ++i)
      if (!std::isfinite(a[i])) fail(ACHI_E_INVALID_MATRIX, "svd: non-finite entries");
    const int r = std::min(m, n);
    DevBuf dA, dS, dU, dV;
    dA.reserve(mn2);
    dS.reserve(r);
    dU.reserve(2 * static_cast<size_t>(m) * r);
    dV.reserve(2 * static_cast<size_t>(r) * n);
    h2d(c, dA.p, a, mn2);
    SvdWs ws;
    ws.vrecover = true;
    const int sw = svd_complex_device(c, ws, dA.p, m, n, dS.p, dU.p, dV.p);
    if (sigma) d2h(c, sigma, dS.p, r);
    if (u) d2h(c, u, dU.p, 2 * static_cast<size_t>(m) * r);
    if (vdag) d2h(c, vdag, dV.p, 2 * static_cast<size_t>(r) * n);
    c.sync();
    if (sweeps_out) *sweeps_out = sw;
  });
}

int achi_bond_select(achi_ctx* ctx, const achi_dmrg_config* cfg, int n_sigma, const double* sigma,
                     achi_bond_state* state, int sweep, int bond, achi_trace_row* row,
                     achi_visit_record* visit) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n_sigma < 1) fail(ACHI_E_DEGENERATE_SPECTRUM, "entropy: empty spectrum");
    DevBuf dS;
    DevArr<achi_bond_state> dst;
    DevArr<achi_trace_row> dtr;
    DevArr<achi_visit_record> dvr;
    DevArr<BondOut> dbo;
    dS.reserve(n_sigma);
    dst.reserve(1);
    dtr.reserve(1);
    dvr.reserve(1);
    dbo.reserve(1);
    h2d(c, dS.p, sigma, n_sigma);
    ACHI_CUDA(cudaMemcpyAsync(dst.p, state, sizeof(achi_bond_state), cudaMemcpyHostToDevice, c.stream));
    ACHI_CUDA(cudaMemsetAsync(dbo.p, 0, sizeof(BondOut), c.stream));
    bond_select(c, dS.p, n_sigma, *cfg, dst.p, 0, sweep, 0, dtr.p, dvr.p, dbo.p);
    BondOut bo;
    ACHI_CUDA(cudaMemcpyAsync(&bo, dbo.p, sizeof(BondOut), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (bo.err == ACHI_E_DEGENERATE_SPECTRUM) fail(bo.err, "entropy: all-zero spectrum");
    if (bo.err) fail(bo.err, "controller_update: invalid state or config");
    ACHI_CUDA(cudaMemcpyAsync(state, dst.p, sizeof(achi_bond_state), cudaMemcpyDeviceToHost, c.stream));
    if (row) ACHI_CUDA(cudaMemcpyAsync(row, dtr.p, sizeof(achi_trace_row), cudaMemcpyDeviceToHost, c.stream));
    if (visit)
      ACHI_CUDA(cudaMemcpyAsync(visit, dvr.p, sizeof(achi_visit_record), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (row) row->bond = bond;
    if (visit) visit->bond = bond;
  });
}

int achi_dgemm(achi_ctx* ctx, int M, int N, int K, int a_kmajor, const double* a, long lda,
               int b_kmajor, const double* b, long ldb, double* c, long ldc) {
  return guard(ctx, [&] {
    Ctx& cx = ctx->c;
    const size_t na = static_cast<size_t>(a_kmajor ? M : K) * lda;
    const size_t nb = static_cast<size_t>(b_kmajor ? N : K) * ldb;
    const size_t nc = static_cast<size_t>(M) * ldc;
    DevBuf dA, dB, dC;
    dA.reserve(na);
    dB.reserve(nb);
    dC.reserve(nc);
    h2d(cx, dA.p, a, na);
    h2d(cx, dB.p, b, nb);
    ACHI_CUDA(cudaMemsetAsync(dC.p, 0, nc * sizeof(double), cx.stream));
    gemm(cx, M, N, K, Operand{dA.p, lda, a_kmajor ? Major::kK : Major::kMN},
         Operand{dB.p, ldb, b_kmajor ? Major::kK : Major::kMN}, dC.p, ldc);
    d2h(cx, c, dC.p, nc);
    cx.sync();
  });
}

int achi_dgemm_device(achi_ctx* ctx, int M, int N, int K, int a_kmajor, const double* d_a, long lda,
                      int b_kmajor, const double* d_b, long ldb, double* d_c, long ldc) {
  return guard(ctx, [&] {
    Ctx& cx = ctx->c;
    gemm(cx, M, N, K, Operand{d_a, lda, a_kmajor ? Major::kK : Major::kMN},
         Operand{d_b, ldb, b_kmajor ? Major::kK : Major::kMN}, d_c, ldc);
  });
}

int achi_spectrum_stats(achi_ctx* ctx, int n_sigma, const double* sigma, int kept, double eps,
                        double* out4) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (n_sigma < 1) fail(ACHI_E_DEGENERATE_SPECTRUM, "entropy: empty spectrum");
    if (kept < 1 || kept > n_sigma) fail(ACHI_E_INVALID_RANK, "truncation_error: kept out of range");
    DevBuf dS, dO;
    DevArr<int> dE;
    dS.reserve(n_sigma);
    dO.reserve(4);
    dE.reserve(1);
    h2d(c, dS.p, sigma, n_sigma);
    spectrum_stats(c, dS.p, n_sigma, kept, eps, dO.p, dE.p);
    int err = 0;
    d2h(c, out4, dO.p, 4);
    ACHI_CUDA(cudaMemcpyAsync(&err, dE.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (err) fail(err, "entropy: all-zero spectrum");
  });
}

int achi_heff_bench(achi_ctx* ctx, int chi, int reps, double* ms_per_matvec, double* tflops) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    const int cp = pad2i(chi), d = 2, D = 5;
    achi_model_spec spec{ACHI_HEISENBERG_XXZ, 4, 1.0, 1.0, 1.0, 0.0, ACHI_SPIN_HALF, 0};
    auto mpo = build_mpo_real(spec);
    MixStore ms;
    auto mix = ms.upload(c, {mix_heff(mpo[1], mpo[2])});
    DevBuf dL, dR, dT, dO;
    const size_t nenv = static_cast<size_t>(cp) * D * cp, nvec = static_cast<size_t>(cp) * d * d * cp;
    fill_random(c, dL.reserve(nenv), nenv, 1);
    fill_random(c, dR.reserve(nenv), nenv, 2);
    fill_random(c, dT.reserve(nvec), nvec, 3);
    dO.reserve(nvec);
    HeffOps op{dL.p, dR.p, cp, cp, d, D, D, mix[0]};
    heff_apply(c, op, dT.p, dO.p);  // warm-up (tensor maps, attributes)
    cudaEvent_t e0, e1;
    ACHI_CUDA(cudaEventCreate(&e0));
    ACHI_CUDA(cudaEventCreate(&e1));
    ACHI_CUDA(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < reps; ++r) heff_apply(c, op, dT.p, dO.p);
    ACHI_CUDA(cudaEventRecord(e1, c.stream));
    ACHI_CUDA(cudaEventSynchronize(e1));
    float f = 0;
    ACHI_CUDA(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double x = chi, flops = 2.0 * D * d * d * x * x * (2 * x) + 4.0 * D * D * d * d * d * x * x;
    *ms_per_matvec = f / reps;
    *tflops = flops / (*ms_per_matvec * 1e-3) / 1e12;
  });
}

int achi_eigs_lowest_dense(achi_ctx* ctx, int dim, const double* h, const double* v0, double tol,
                           int max_iter, double* eigenvalue, double* eigenvector, int* matvecs,
                           double* residual) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    DevBuf dH, dV, dO;
    dH.reserve(static_cast<size_t>(dim) * dim);
    dV.reserve(dim);
    dO.reserve(dim);
    h2d(c, dH.p, h, static_cast<size_t>(dim) * dim);
    h2d(c, dV.p, v0, dim);
    LanczosWs ws;
    EigsOut e = eigs_lowest(
        c, ws,
        [&](const double* in, double* out) {
          dense_gemv_kernel<<<cdiv(dim, 8), 256, 0, c.stream>>>(dH.p, dim, in, out);
          ACHI_LAUNCHED(c);
        },
        dim, dim, dV.p, tol, max_iter, dO.p);
    d2h(c, eigenvector, dO.p, dim);
    c.sync();
    *eigenvalue = e.eigenvalue;
    *matvecs = e.matvecs;
    *residual = e.residual;
  });
}

int achi_dgemm_ozaki_device(achi_ctx* ctx, int M, int N, int K, const double* d_a, long lda, int a_trans,
                            const double* d_b, long ldb, int b_kmajor, double* d_c, long ldc, int slices) {
  return guard(ctx, [&] {
    if (M < 1 || N < 1 || K < 1) fail(ACHI_E_INVALID_MATRIX, "ozaki: empty operand");
    dgemm_ozaki(ctx->c, M, N, K, d_a, lda, a_trans != 0, d_b, ldb, b_kmajor != 0, d_c, ldc, slices);
  });
}

int achi_eigs_lowest_callback(achi_ctx* ctx, int dim, achi_matvec_fn fn, void* user, const double* v0,
                              double tol, int max_iter, double* eigenvalue, double* eigenvector,
                              int* matvecs, double* residual) {
  return guard(ctx, [&] {
    Ctx& c = ctx->c;
    if (dim < 1 || !fn) fail(ACHI_E_INVALID_MATRIX, "eigs_lowest: dim >= 1 and an operator are required");
    DevBuf dV, dO;
    dV.reserve(dim);
    dO.reserve(dim);
    h2d(c, dV.p, v0, dim);
    std::vector<double> hin(dim), hout(dim);
    LanczosWs ws;
    // the host operator cannot run inside a graph: this call steps the Lanczos from the host
    struct GraphMode {
      Ctx& c;
      int prev;
      ~GraphMode() { c.lanczos_graph = prev; }
    } gm{c, c.lanczos_graph};
    c.lanczos_graph = 0;
    EigsOut e = eigs_lowest(
        c, ws,
        [&](const double* in, double* out) {
          d2h(c, hin.data(), in, dim);
          c.sync();
          fn(user, hin.data(), hout.data(), dim);
          for (int i = 0; i < dim; ++i)
            if (!std::isfinite(hout[i])) fail(ACHI_E_INVALID_MATRIX, "eigs_lowest: operator returned non-finite values");
          h2d(c, out, hout.data(), dim);
          c.sync();
        },
        dim, dim, dV.p, tol, max_iter, dO.p);
    d2h(c, eigenvector, dO.p, dim);
    c.sync();
    *eigenvalue = e.eigenvalue;
    *matvecs = e.matvecs;
    *residual = e.residual;
  });
}

}  // extern "C"
