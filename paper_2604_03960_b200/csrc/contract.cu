// H_eff matvec, environment updates, theta merge (see contract.cuh).
#include <cstring>

#include "contract.cuh"

namespace achi {

// ---------------------------------------------------------------------------
// Mixing matrices (host, built once per chain from the MPO)
// ---------------------------------------------------------------------------
namespace {

MixMatrix from_dense(int nout, int nin, const std::vector<double>& dense) {
  MixMatrix m;
  m.nout = nout;
  m.nin = nin;
  m.rowptr.push_back(0);
  for (int o = 0; o < nout; ++o) {
    for (int i = 0; i < nin; ++i) {
      double v = dense[static_cast<size_t>(o) * nin + i];
      if (v != 0.0) {
        m.col.push_back(i);
        m.val.push_back(v);
      }
    }
    m.rowptr.push_back(static_cast<int>(m.col.size()));
  }
  return m;
}

}  // namespace

MixMatrix mix_heff(const HostMpo& w1, const HostMpo& w2) {
  const int d = w1.d, D1 = w1.l, D2 = w1.r, D3 = w2.r;
  if (w2.l != D2 || w2.d != d) fail(ACHI_E_INTERNAL, "mix_heff: MPO bond mismatch");
  const int nin = D1 * d * d, nout = d * d * D3;
  std::vector<double> dense(static_cast<size_t>(nin) * nout, 0.0);
  for (int a = 0; a < D1; ++a)
    for (int s1 = 0; s1 < d; ++s1)
      for (int s2 = 0; s2 < d; ++s2)
        for (int p1 = 0; p1 < d; ++p1)
          for (int p2 = 0; p2 < d; ++p2)
            for (int e = 0; e < D3; ++e) {
              double acc = 0;
              for (int c = 0; c < D2; ++c) acc += w1.at(a, p1, s1, c) * w2.at(c, p2, s2, e);
              const int in = (a * d + s1) * d + s2;
              const int out = (p1 * d + p2) * D3 + e;
              dense[static_cast<size_t>(out) * nin + in] = acc;
            }
  return from_dense(nout, nin, dense);
}

MixMatrix mix_env_left(const HostMpo& w) {
  const int d = w.d, Dl = w.l, Dr = w.r;
  const int nin = Dl * d, nout = d * Dr;
  std::vector<double> dense(static_cast<size_t>(nin) * nout, 0.0);
  for (int a = 0; a < Dl; ++a)
    for (int s = 0; s < d; ++s)
      for (int p = 0; p < d; ++p)
        for (int b = 0; b < Dr; ++b)
          dense[static_cast<size_t>(p * Dr + b) * nin + (a * d + s)] = w.at(a, p, s, b);
  return from_dense(nout, nin, dense);
}

MixMatrix mix_env_right(const HostMpo& w) {
  const int d = w.d, Dl = w.l, Dr = w.r;
  const int nin = Dr * d, nout = d * Dl;
  std::vector<double> dense(static_cast<size_t>(nin) * nout, 0.0);
  for (int a = 0; a < Dl; ++a)
    for (int p = 0; p < d; ++p)
      for (int s = 0; s < d; ++s)
        for (int e = 0; e < Dr; ++e)
          dense[static_cast<size_t>(p * Dl + a) * nin + (e * d + s)] = w.at(a, p, s, e);
  return from_dense(nout, nin, dense);
}

std::vector<DevMix> MixStore::upload(Ctx& ctx, const std::vector<MixMatrix>& ms) {
  // layout per matrix: [val (double) nnz][rowptr int nout+1][col int nnz], 16-byte aligned
  std::vector<size_t> offs;
  size_t total = 0;
  auto align = [](size_t x) { return (x + 15) & ~size_t(15); };
  for (const auto& m : ms) {
    offs.push_back(total);
    total = align(total + m.val.size() * sizeof(double));
    total = align(total + m.rowptr.size() * sizeof(int));
    total = align(total + m.col.size() * sizeof(int));
  }
  std::vector<unsigned char> host(total + 16, 0);
  std::vector<DevMix> out;
  unsigned char* dev = blob.reserve(total + 16);
  for (size_t k = 0; k < ms.size(); ++k) {
    const auto& m = ms[k];
    size_t o = offs[k];
    DevMix dm;
    dm.nout = m.nout;
    dm.nin = m.nin;
    dm.nnz = static_cast<int>(m.val.size());
    std::memcpy(host.data() + o, m.val.data(), m.val.size() * sizeof(double));
    dm.val = reinterpret_cast<const double*>(dev + o);
    o = align(o + m.val.size() * sizeof(double));
    std::memcpy(host.data() + o, m.rowptr.data(), m.rowptr.size() * sizeof(int));
    dm.rowptr = reinterpret_cast<const int*>(dev + o);
    o = align(o + m.rowptr.size() * sizeof(int));
    std::memcpy(host.data() + o, m.col.data(), m.col.size() * sizeof(int));
    dm.col = reinterpret_cast<const int*>(dev + o);
    out.push_back(dm);
  }
  ACHI_CUDA(cudaMemcpyAsync(dev, host.data(), total, cudaMemcpyHostToDevice, ctx.stream));
  ctx.sync();
  return out;
}

// ---------------------------------------------------------------------------
// MPO mixing kernel: for every (outer o, inner t), y_vec = W x_vec with
//   x(i1,i2) at o*sxo + t*sxt + i1*sx1 + i2*sx2  (i = i1*nin2 + i2)
//   y(j1,j2) at o*syo + t*syt + j1*sy1 + j2*sy2  (j = j1*nout2 + j2)
// Memory-bound; W is sparse (<= ~50 nonzeros of 400 for XXZ) and staged in smem.
// ---------------------------------------------------------------------------
struct MixGeom {
  int nin2, nout2;
  long sxo, sxt, sx1, sx2;
  long syo, syt, sy1, sy2;
  long outer, inner;
};

constexpr int MIX_THREADS = 128;
constexpr int MIX_MAXIN = 32;

__global__ void __launch_bounds__(MIX_THREADS) mpo_mix_kernel(const double* __restrict__ x,
                                                              double* __restrict__ y, DevMix W,
                                                              MixGeom g) {
  pdl_wait();  // launched with launch_pdl / the PDL attribute (common.cuh)
  __shared__ double xs[MIX_MAXIN][MIX_THREADS];
  __shared__ double sval[512];
  __shared__ int scol[512];
  __shared__ int srow[MIX_MAXIN + 1];
  for (int i = threadIdx.x; i < W.nnz; i += blockDim.x) {
    sval[i] = W.val[i];
    scol[i] = W.col[i];
  }
  for (int i = threadIdx.x; i <= W.nout; i += blockDim.x) srow[i] = W.rowptr[i];
  __syncthreads();
  const long total = g.outer * g.inner;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const long o = idx / g.inner, t = idx - o * g.inner;
    const double* xb = x + o * g.sxo + t * g.sxt;
    for (int i = 0; i < W.nin; ++i) {
      const int i1 = i / g.nin2, i2 = i - i1 * g.nin2;
      xs[i][threadIdx.x] = __ldg(xb + i1 * g.sx1 + i2 * g.sx2);
    }
    double* yb = y + o * g.syo + t * g.syt;
    for (int j = 0; j < W.nout; ++j) {
      double acc = 0.0;
      for (int e = srow[j]; e < srow[j + 1]; ++e) acc += sval[e] * xs[scol[e]][threadIdx.x];
      const int j1 = j / g.nout2, j2 = j - j1 * g.nout2;
      yb[j1 * g.sy1 + j2 * g.sy2] = acc;
    }
  }
}

namespace {

void mix(Ctx& ctx, const double* x, double* y, const DevMix& W, const MixGeom& g) {
  if (W.nin > MIX_MAXIN || W.nout > MIX_MAXIN || W.nnz > 512)
    fail(ACHI_E_UNSUPPORTED_MODEL, "MPO mixing larger than the kernel's staging (D*d^2 > 32)");
  const long total = g.outer * g.inner;
  if (total <= 0) return;
  const int blocks = static_cast<int>(std::min<long>(cdiv(total, MIX_THREADS), 16L * ctx.num_sms));
  ACHI_CUDA(launch_pdl(mpo_mix_kernel, blocks, MIX_THREADS, 0, ctx.stream, x, y, W, g));
  ACHI_LAUNCHED(ctx);
}

}  // namespace

// ---------------------------------------------------------------------------
// Contractions
// ---------------------------------------------------------------------------
void heff_apply(Ctx& ctx, const HeffOps& op, const double* theta, double* out) {
  static const bool small_on = [] {
    const char* e = std::getenv("ACHI_HEFF_SMALL");
    return !(e && e[0] == '0');
  }();
  // largest chi on the fused path: the wide instantiation (chi 129..256) measured
  // slower than the TMA GEMM path (53/70/127 vs 43/49/102 us at chi 160/192/256,
  // profiles/heff_study_r01.txt), so the crossover stays at 128 unless overridden
  static const int small_max = [] {
    const char* e = std::getenv("ACHI_HEFF_SMALL_MAX");
    return e ? std::atoi(e) : 128;
  }();
  if (small_on && std::max(op.chl, op.chr) <= small_max && heff_small_applicable(op)) {
    heff_apply_small(ctx, op, theta, out);
    return;
  }
  const long chl = op.chl, chr = op.chr, d = op.d, D1 = op.D1, D3 = op.D3;
  double* X = ctx.ws_a.reserve(static_cast<size_t>(chl * D1 * d * d * chr));
  double* Y = ctx.ws_b.reserve(static_cast<size_t>(chl * d * d * D3 * chr));
  // X[(bl,a),(s1,s2,jr)] = L[(bl,a), jl] theta[jl, (s1,s2,jr)]
  gemm(ctx, static_cast<int>(chl * D1), static_cast<int>(d * d * chr), static_cast<int>(chl),
       Operand{op.L, chl, Major::kK}, Operand{theta, d * d * chr, Major::kMN}, X, d * d * chr);
  // Y[(bl,s1',s2'),(e,jr)] = sum W12 X
  MixGeom g{static_cast<int>(d * d), static_cast<int>(D3),
            D1 * d * d * chr, 1, d * d * chr, chr,
            d * d * D3 * chr, 1, D3 * chr, chr,
            chl, chr};
  mix(ctx, X, Y, op.mix, g);
  // out[(bl,s1',s2'), br] = Y[(bl s1' s2'), (e jr)] R[br, (e jr)]
  gemm(ctx, static_cast<int>(chl * d * d), static_cast<int>(chr), static_cast<int>(D3 * chr),
       Operand{Y, D3 * chr, Major::kK}, Operand{op.R, D3 * chr, Major::kK}, out, chr);
}

void env_left(Ctx& ctx, const double* L, const double* A, int chl_, int chn_, int d_, int Dl_,
              int Dr_, const DevMix& W, double* Lnew) {
  const long chl = chl_, chn = chn_, d = d_, Dl = Dl_, Dr = Dr_;
  double* T1 = ctx.ws_a.reserve(static_cast<size_t>(chl * Dl * d * chn));
  double* T2 = ctx.ws_b.reserve(static_cast<size_t>(chl * d * Dr * chn));
  // T1[(b,a),(s,j')] = L[(b,a), j] A[j, (s,j')]
  gemm(ctx, static_cast<int>(chl * Dl), static_cast<int>(d * chn), static_cast<int>(chl),
       Operand{L, chl, Major::kK}, Operand{A, d * chn, Major::kMN}, T1, d * chn);
  // T2[(b,s'),(a',j')] = sum_{a,s} W(a,s',s,a') T1[(b,a),(s,j')]
  MixGeom g{static_cast<int>(d), static_cast<int>(Dr),
            Dl * d * chn, 1, d * chn, chn,
            d * Dr * chn, 1, Dr * chn, chn,
            chl, chn};
  mix(ctx, T1, T2, W, g);
  // Lnew[b', (a',j')] = sum_{(b,s')} A[(b,s'), b'] T2[(b,s'), (a',j')]
  gemm(ctx, static_cast<int>(chn), static_cast<int>(Dr * chn), static_cast<int>(chl * d),
       Operand{A, chn, Major::kMN}, Operand{T2, Dr * chn, Major::kMN}, Lnew, Dr * chn);
}

void env_right(Ctx& ctx, const double* R, const double* B, int chr_, int chn_, int d_, int Dl_,
               int Dr_, const DevMix& W, double* Rnew) {
  const long chr = chr_, chn = chn_, d = d_, Dl = Dl_, Dr = Dr_;
  double* T1 = ctx.ws_a.reserve(static_cast<size_t>(chr * Dr * chn * d));
  double* T2 = ctx.ws_b.reserve(static_cast<size_t>(d * chr * Dl * chn));
  // T1[(b,e),(j,s)] = sum_j'' R[(b,e), j''] B[(j,s), j'']
  gemm(ctx, static_cast<int>(chr * Dr), static_cast<int>(chn * d), static_cast<int>(chr),
       Operand{R, chr, Major::kK}, Operand{B, chr, Major::kK}, T1, chn * d);
  // T2[(s',b),(a,j)] = sum_{e,s} W(a,s',s,e) T1[(b,e),(j,s)]
  MixGeom g{static_cast<int>(d), static_cast<int>(Dl),
            Dr * chn * d, d, chn * d, 1,
            Dl * chn, 1, chr * Dl * chn, chn,
            chr, chn};
  mix(ctx, T1, T2, W, g);
  // Rnew[b', (a,j)] = sum_{(s',b)} B[b', (s',b)] T2[(s',b), (a,j)]
  gemm(ctx, static_cast<int>(chn), static_cast<int>(Dl * chn), static_cast<int>(d * chr),
       Operand{B, d * chr, Major::kK}, Operand{T2, Dl * chn, Major::kMN}, Rnew, Dl * chn);
}

void theta_merge(Ctx& ctx, const double* A, const double* B, int chl, int chm, int chr, int d,
                 double* theta) {
  gemm(ctx, chl * d, d * chr, chm, Operand{A, chm, Major::kK},
       Operand{B, static_cast<long>(d) * chr, Major::kMN}, theta, static_cast<long>(d) * chr);
}

// ---------------------------------------------------------------------------
// complex128, planar (contract.cuh)
// ---------------------------------------------------------------------------
namespace {

__global__ void realify_kernel(const double* __restrict__ src, long plane, long M, long K, long sm,
                               long sk, int conj, double* __restrict__ dst) {
  const long tot = M * K, ld = 2 * K;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < tot;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const long m = t / K, k = t - m * K;
    const long o = m * sm + k * sk;
    const double re = src[o], im = conj ? -src[o + plane] : src[o + plane];
    dst[m * ld + k] = re;
    dst[m * ld + K + k] = -im;
    dst[(m + M) * ld + k] = im;
    dst[(m + M) * ld + K + k] = re;
  }
}

__global__ void ptranspose_kernel(const double* __restrict__ src, long rows, long cols,
                                  double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const long plane = rows * cols;
  const long r0 = static_cast<long>(blockIdx.y) * 32, c0 = static_cast<long>(blockIdx.x) * 32;
  for (int p = 0; p < 2; ++p) {
    const double* s = src + p * plane;
    double* dd = dst + p * plane;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const long r = r0 + i, c = c0 + threadIdx.x;
      tile[i][threadIdx.x] = (r < rows && c < cols) ? s[r * cols + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const long c = c0 + i, r = r0 + threadIdx.x;
      if (r < rows && c < cols) dd[c * rows + r] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

}  // namespace

void realify(Ctx& ctx, const double* src, long plane, long M, long K, long sm, long sk, bool conj,
             double* dst) {
  const long tot = M * K;
  if (tot <= 0) return;
  const int blocks = static_cast<int>(std::min<long>(cdiv(tot, 256), 8L * ctx.num_sms));
  realify_kernel<<<blocks, 256, 0, ctx.stream>>>(src, plane, M, K, sm, sk, conj ? 1 : 0, dst);
  ACHI_LAUNCHED(ctx);
}

void planar_transpose(Ctx& ctx, const double* src, long rows, long cols, double* dst) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid(static_cast<unsigned>(cdiv(cols, 32)), static_cast<unsigned>(cdiv(rows, 32)));
  ptranspose_kernel<<<grid, dim3(32, 8), 0, ctx.stream>>>(src, rows, cols, dst);
  ACHI_LAUNCHED(ctx);
}

void heff_prepare_c(Ctx& ctx, const double* L, int chl_, int D1_, const double* R, int chr_,
                    int D3_, double* Lhat, double* Rhat) {
  const long chl = chl_, D1 = D1_, chr = chr_, D3 = D3_;
  // L as [(bl, a), jl]; R as [br, (e, jr)]
  realify(ctx, L, chl * D1 * chl, chl * D1, chl, chl, 1, false, Lhat);
  realify(ctx, R, chr * D3 * chr, chr, D3 * chr, D3 * chr, 1, false, Rhat);
}

void heff_apply_c(Ctx& ctx, const HeffOpsC& op, const double* theta, double* out) {
  const long chl = op.chl, chr = op.chr, d = op.d, D1 = op.D1, D3 = op.D3;
  double* X = ctx.ws_a.reserve(static_cast<size_t>(2 * chl * D1 * d * d * chr));
  double* Y = ctx.ws_b.reserve(static_cast<size_t>(2 * chl * d * d * D3 * chr));
  // X[(q,bl,a),(s1,s2,jr)] = Lhat[(q,bl,a),(p,jl)] theta[(p,jl),(s1,s2,jr)]
  gemm(ctx, static_cast<int>(2 * chl * D1), static_cast<int>(d * d * chr), static_cast<int>(2 * chl),
       Operand{op.Lhat, 2 * chl, Major::kK}, Operand{theta, d * d * chr, Major::kMN}, X, d * d * chr);
  // Y[(bl,s1',s2'),(q,e,jr)]: the plane inside each row
  for (long q = 0; q < 2; ++q) {
    MixGeom g{static_cast<int>(d * d), static_cast<int>(D3),
              D1 * d * d * chr, 1, d * d * chr, chr,
              d * d * 2 * D3 * chr, 1, 2 * D3 * chr, chr,
              chl, chr};
    mix(ctx, X + q * chl * D1 * d * d * chr, Y + q * D3 * chr, op.mix, g);
  }
  // out_q[(bl,s1',s2'), br] = Y[(bl,s1',s2'), (p,e,jr)] Rhat[(q,br), (p,e,jr)]
  for (long q = 0; q < 2; ++q)
    gemm(ctx, static_cast<int>(chl * d * d), static_cast<int>(chr), static_cast<int>(2 * D3 * chr),
         Operand{Y, 2 * D3 * chr, Major::kK}, Operand{op.Rhat + q * chr * 2 * D3 * chr, 2 * D3 * chr, Major::kK},
         out + q * chl * d * d * chr, chr);
}

void env_left_c(Ctx& ctx, const double* L, const double* A, int chl_, int chn_, int d_, int Dl_,
                int Dr_, const DevMix& W, double* scr, double* Lnew) {
  const long chl = chl_, chn = chn_, d = d_, Dl = Dl_, Dr = Dr_;
  double* T1 = ctx.ws_a.reserve(static_cast<size_t>(2 * chl * Dl * d * chn));
  double* T2 = ctx.ws_b.reserve(static_cast<size_t>(2 * chl * d * Dr * chn));
  // T1 planar [(q,b,a),(s,j')] = realify(L as [(b,a), j]) . A planar [(p,j),(s,j')]
  realify(ctx, L, chl * Dl * chl, chl * Dl, chl, chl, 1, false, scr);
  gemm(ctx, static_cast<int>(2 * chl * Dl), static_cast<int>(d * chn), static_cast<int>(2 * chl),
       Operand{scr, 2 * chl, Major::kK}, Operand{A, d * chn, Major::kMN}, T1, d * chn);
  // T2 planar [(q,b,s'),(a',j')]: the planes are one more outer index of uniform stride
  MixGeom g{static_cast<int>(d), static_cast<int>(Dr),
            Dl * d * chn, 1, d * chn, chn,
            d * Dr * chn, 1, Dr * chn, chn,
            2 * chl, chn};
  mix(ctx, T1, T2, W, g);
  // Lnew planar [(q,b'),(a',j')] = realify(A^dagger as [b', (b,s')]) . T2 planar
  realify(ctx, A, chl * d * chn, chn, chl * d, 1, chn, true, scr);
  gemm(ctx, static_cast<int>(2 * chn), static_cast<int>(Dr * chn), static_cast<int>(2 * chl * d),
       Operand{scr, 2 * chl * d, Major::kK}, Operand{T2, Dr * chn, Major::kMN}, Lnew, Dr * chn);
}

void env_right_c(Ctx& ctx, const double* R, const double* B, int chr_, int chn_, int d_, int Dl_,
                 int Dr_, const DevMix& W, double* scr, double* Rnew) {
  const long chr = chr_, chn = chn_, d = d_, Dl = Dl_, Dr = Dr_;
  double* T1 = ctx.ws_a.reserve(static_cast<size_t>(2 * chr * Dr * chn * d));
  double* T2 = ctx.ws_b.reserve(static_cast<size_t>(2 * d * chr * Dl * chn));
  double* Bt = scr + std::max(4 * chr * chr * Dr, 4 * chn * d * chr);
  // T1 planar [(q,b,e),(j,s)] = realify(R as [(b,e), j'']) . B^T planar [(p,j''),(j,s)]
  planar_transpose(ctx, B, chn * d, chr, Bt);
  realify(ctx, R, chr * Dr * chr, chr * Dr, chr, chr, 1, false, scr);
  gemm(ctx, static_cast<int>(2 * chr * Dr), static_cast<int>(chn * d), static_cast<int>(2 * chr),
       Operand{scr, 2 * chr, Major::kK}, Operand{Bt, chn * d, Major::kMN}, T1, chn * d);
  // T2 planar [(q,s',b),(a,j)], one mixing launch per plane
  for (long q = 0; q < 2; ++q) {
    MixGeom g{static_cast<int>(d), static_cast<int>(Dl),
              Dr * chn * d, d, chn * d, 1,
              Dl * chn, 1, chr * Dl * chn, chn,
              chr, chn};
    mix(ctx, T1 + q * chr * Dr * chn * d, T2 + q * d * chr * Dl * chn, W, g);
  }
  // Rnew planar [(q,b'),(a,j)] = realify(conj(B) as [b', (s',b)]) . T2 planar
  realify(ctx, B, chn * d * chr, chn, d * chr, d * chr, 1, true, scr);
  gemm(ctx, static_cast<int>(2 * chn), static_cast<int>(Dl * chn), static_cast<int>(2 * d * chr),
       Operand{scr, 2 * d * chr, Major::kK}, Operand{T2, Dl * chn, Major::kMN}, Rnew, Dl * chn);
}

void theta_merge_c(Ctx& ctx, const double* A, const double* B, int chl_, int chm_, int chr_, int d_,
                   double* scr, double* theta) {
  const long chl = chl_, chm = chm_, chr = chr_, d = d_;
  realify(ctx, A, chl * d * chm, chl * d, chm, chm, 1, false, scr);
  gemm(ctx, static_cast<int>(2 * chl * d), static_cast<int>(d * chr), static_cast<int>(2 * chm),
       Operand{scr, 2 * chm, Major::kK}, Operand{B, d * chr, Major::kMN}, theta, d * chr);
}

void upload_padded3(Ctx& ctx, const double* host, int l, int d, int r, double* dev) {
  const int lp = pad2i(l), rp = pad2i(r);
  ACHI_CUDA(cudaMemsetAsync(dev, 0, sizeof(double) * lp * d * rp, ctx.stream));
  ACHI_CUDA(cudaMemcpy2DAsync(dev, sizeof(double) * rp, host, sizeof(double) * r,
                              sizeof(double) * r, static_cast<size_t>(l) * d,
                              cudaMemcpyHostToDevice, ctx.stream));
}

void download_padded3(Ctx& ctx, const double* dev, int l, int m, int r, double* host) {
  const int rp = pad2i(r);
  ACHI_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * r, dev, sizeof(double) * rp,
                              sizeof(double) * r, static_cast<size_t>(l) * m,
                              cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
}

}  // namespace achi
