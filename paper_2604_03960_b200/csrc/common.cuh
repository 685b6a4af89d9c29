// Common infrastructure for the B200-native DMRG hot path: error handling,
// device buffers, the context (device + stream + launch counter).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/adaptchi_b200.h"

namespace achi {

// Typed error carrying an ACHI_E_* code (one per reference exception type,
// errors.hpp:8-59).
struct Error : std::runtime_error {
  int code;
  double residual = 0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    fail(ACHI_E_CUDA, buf);
  }
}
#define ACHI_CUDA(x) ::achi::cuda_check((x), #x, __FILE__, __LINE__)
#define ACHI_LAUNCHED(ctx)                                            \
  do {                                                                \
    ::achi::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    ++(ctx).launches;                                                 \
  } while (0)

// Programmatic dependent launch: a kernel launched with launch_pdl may have its CTAs
// scheduled while the previous kernel of the stream drains (the kernel-boundary gap of
// the small per-visit kernels overlaps), so such a kernel calls pdl_wait() before it
// touches memory: griddepcontrol.wait returns once the previous grid has completed and
// its writes are visible (a no-op in a kernel launched without the attribute).
// ACHI_PDL=0: plain stream serialization.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ACHI_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// not while the stream is being captured (the Lanczos graphs keep plain kernel edges)
inline bool pdl_allowed(cudaStream_t s) {
  if (!pdl_enabled()) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_allowed(s) ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kern, args...);
}

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync /
// cudaFreeAsync on the stream of the context being driven, see AllocStream),
// whose release threshold is raised at context creation: buffers that grow
// while chi grows reuse cached pool memory instead of a synchronising
// cudaFree + cudaMalloc (which stalled sweeps for up to ~0.5 s).
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
// RAII: route allocations of this thread to `s` for the scope of a C-ABI call
struct AllocStream {
  cudaStream_t prev;
  explicit AllocStream(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~AllocStream() { alloc_stream() = prev; }
};
inline void* dev_alloc(size_t bytes) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (alloc_stream()) cudaStreamIsCapturing(alloc_stream(), &cs);
  if (cs != cudaStreamCaptureStatusNone)  // buffers must be sized before graph capture
    fail(ACHI_E_INTERNAL, "device allocation inside a stream capture");
  void* p = nullptr;
  ACHI_CUDA(cudaMallocAsync(&p, bytes, alloc_stream()));
  return p;
}
inline void dev_free(void* p) {
  if (p) cudaFreeAsync(p, alloc_stream());
}

// Owning device allocation (capacity-based, grows but never shrinks).
struct DevBuf {
  double* p = nullptr;
  size_t cap = 0;  // elements
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; cap = o.cap; o.p = nullptr; o.cap = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    dev_free(p);
    p = nullptr;
    cap = 0;
  }
  // ensure capacity (contents not preserved on growth)
  double* reserve(size_t n) {
    if (n > cap) {
      release();
      p = static_cast<double*>(dev_alloc((n == 0 ? 1 : n) * sizeof(double)));
      cap = n;
    }
    return p;
  }
};

template <class T>
struct DevArr {
  T* p = nullptr;
  size_t cap = 0;
  DevArr() = default;
  DevArr(const DevArr&) = delete;
  DevArr& operator=(const DevArr&) = delete;
  ~DevArr() { dev_free(p); }
  T* reserve(size_t n) {
    if (n > cap) {
      dev_free(p);
      p = static_cast<T*>(dev_alloc((n == 0 ? 1 : n) * sizeof(T)));
      cap = n;
    }
    return p;
  }
};

// Pinned host scratch for small device->host status reads.
template <class T>
struct PinnedArr {
  T* p = nullptr;
  size_t cap = 0;
  ~PinnedArr() { if (p) cudaFreeHost(p); }
  T* reserve(size_t n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      ACHI_CUDA(cudaMallocHost(&p, (n == 0 ? 1 : n) * sizeof(T)));
      cap = n;
    }
    return p;
  }
};

// Lanczos step status written by the device (read by the host driver loop).
struct LanczosStatus {
  double theta;      // lowest Ritz value of the current tridiagonal
  double res_bound;  // beta_j * |s_{k-1}|
  double bnorm;      // ||w|| after reorthogonalisation
  double alpha;      // q_j . H q_j
  double ev;         // Rayleigh quotient of the Ritz vector (after explicit check)
  double res;        // ||H r - ev r||
  double aux;
  int32_t flags, pad;
};

// Device-time accounting: event pairs recorded on the context stream around a
// phase, resolved into per-tag totals after a sync the caller already pays (the
// chain resolves once per sweep: the per-visit host cost is the records alone).
// Phases nest (kHeff, the H_eff applications, sits inside kMatvec, the whole
// eigensolve); nothing is recorded while the stream is being captured.
struct EventAcc {
  enum Tag { kMatvec = 0, kSvd = 1, kEnv = 2, kHeff = 3, kNumTags = 4 };
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, int>> stack;  // open phases: (tag, index of start event)
  struct Closed { int tag, start, stop; };
  std::vector<Closed> closed;
  size_t used = 0;
  double ms[kNumTags] = {0, 0, 0, 0};
  double work[kNumTags] = {0, 0, 0, 0};  // algorithmic flops or bytes
  long count[kNumTags] = {0, 0, 0, 0};
  bool enabled = false;
  bool in_capture = false;  // set by the Lanczos graph builder while ctx.stream is captured
  // timing events cost device time (~4 us per bond visit at C3): a chain times one
  // visit in `sample` (rotating over the bonds when sample is coprime with 2(N-1))
  int sample = 1;
  long visit_seq = 0;
  bool visit_timed() { return enabled && (visit_seq++ % sample) == 0; }
  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(int tag, cudaStream_t s) {
    if (!enabled) return;
    if (in_capture) {
      stack.emplace_back(tag, -1);
      return;
    }
    const int i = static_cast<int>(used);
    cudaEventRecord(next(), s);
    stack.emplace_back(tag, i);
  }
  void end(cudaStream_t s, double w) {
    if (!enabled || stack.empty()) return;
    const auto [tag, i] = stack.back();
    stack.pop_back();
    if (i < 0) return;
    const int j = static_cast<int>(used);
    cudaEventRecord(next(), s);
    closed.push_back(Closed{tag, i, j});
    work[tag] += w;
    count[tag] += 1;
  }
  // call after a stream sync: fold all closed pairs into the totals
  void resolve() {
    for (const Closed& c : closed) {
      float f = 0;
      if (cudaEventElapsedTime(&f, pool[c.start], pool[c.stop]) == cudaSuccess) ms[c.tag] += f;
    }
    closed.clear();
    if (stack.empty()) used = 0;
  }
  ~EventAcc() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// suspends the accounting for one untimed visit
struct EventAccPause {
  EventAcc& a;
  bool prev;
  EventAccPause(EventAcc& acc, bool pause) : a(acc), prev(acc.enabled) {
    if (pause) a.enabled = false;
  }
  ~EventAccPause() { a.enabled = prev; }
};

struct Ctx {
  EventAcc acc;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int num_sms = 148;
  // cap on the CTAs of this context's cooperative kernels (0: none); several
  // contexts sharing a GPU (ensemble chains in flight) each get a share
  int grid_cap = 0;
  // Lanczos inner loop as a conditional CUDA graph (1), stepped from the host
  // (0: every kernel visible to ncu and to the per-matvec event accounting),
  // or the process default (-1: ACHI_LANCZOS_GRAPH, on unless "0")
  int lanczos_graph = -1;
  // emulated-FP64 contractions on the int8 tensor cores (ozaki.cu): digits per
  // operand entry (0: off, the DMMA engine) for GEMMs of at least ozaki_min_flops
  int ozaki_slices = 0;
  double ozaki_min_flops = 1e9;
  DevBuf oz_digits;
  DevArr<int> oz_ex;
  int cap_grid(long want) const {
    return static_cast<int>(grid_cap > 0 ? std::min<long>(want, grid_cap) : want);
  }
  std::string last_error;
  double last_residual = 0;
  // scratch
  DevBuf ws_a, ws_b, ws_c, ws_split;  // GEMM / contraction intermediates
  DevBuf red;                          // reduction partials
  DevBuf small;                        // small device scalars (h coefficients, s vector, ...)
  PinnedArr<double> host_small;
  PinnedArr<LanczosStatus> status;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // second stream for fork/join inside captured graphs (Lanczos: the
  // tridiagonal step runs beside the next matvec)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // side stream of the cluster SVD's V replay (svd_jacobi.cu, SvdWs::defer_v)
  cudaStream_t vstream = nullptr;
  cudaEvent_t ev_v0 = nullptr, ev_v1 = nullptr;
  DevBuf flush;
  void sync() { ACHI_CUDA(cudaStreamSynchronize(stream)); }
};

// One-time per-device setup (kernel attributes, occupancy-derived grid sizes),
// thread-safe and keyed by (site, device): a second GPU gets its own
// attributes, and concurrent contexts on worker threads do not race.
template <class F>
int per_device_once(const std::string& site, int device, F&& f) {
  static std::mutex mu;
  static std::map<std::pair<std::string, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(site, device);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int v = f();
  cache.emplace(key, v);
  return v;
}

inline size_t pad2(size_t x) { return x + (x & 1); }
inline int pad2i(int x) { return x + (x & 1); }
inline int cdiv(long a, long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace achi
