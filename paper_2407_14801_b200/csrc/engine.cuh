// engine.cuh -- the host level scheduler of libsquaresort.so (included by the
// per-key-type translation units inst_*.cu and by the C ABI in api.cu).
//
// The scheduler runs SquareSort (Alg 1) level by level: a level is
// one batched grid per step for ALL segments that are too large to sort on
// chip, so the recursion -- shallow (O(log log n)) but very wide --
// costs a handful of launches per level rather than one per recursive call.
// Segments that fit on chip are sorted by the batched block sort (the GPU's
// simple_sort), grouped in power-of-two size classes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>
#include <chrono>
#include <set>
#include <tuple>

#include "../../include/squaresort.h"
#include "skew.cuh"
#include "binclust.cuh"

namespace sq {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline thread_local std::string g_errmsg;
inline thread_local sq_stats g_stats;

#define SQ_CUDA(call)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      if (e_ == cudaErrorMemoryAllocation) throw Error(SQ_ERR_OUT_OF_MEMORY, cudaGetErrorString(e_)); \
      throw Error(SQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    }                                                                                        \
  } while (0)

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(SQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_stats.kernel_launches++;
}

// ------------------------------------------------------------------ per-kernel timing
// When enabled (sq_profile), every launch is bracketed by CUDA events on its
// stream; elapsed times accumulate per kernel role after the call's final sync.
inline int cur_device() {
  int dev = 0;
  SQ_CUDA(cudaGetDevice(&dev));
  return dev;
}

// ------------------------------------------------------------------ per-device state
// Everything that is bound to a device (kernel attributes, the SM count, the
// library's memory pool, events, side streams) is kept per device ordinal, so a
// process may sort on several GPUs (one thread or many).
constexpr int kMaxDevices = 64;
struct DeviceState {
  std::mutex mu;
  int checked = 0;  // 1 ok (sm_100), 2 unsupported
  int sms = 0;
  cudaMemPool_t pool = nullptr;  // library-owned stream-ordered pool: scratch is cached between calls
  std::set<std::pair<const void*, size_t>> smem_set;
  std::map<std::tuple<const void*, int, size_t>, int> grids;
};
inline DeviceState& dev_state(int dev) {
  static DeviceState st[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) throw Error(SQ_ERR_UNSUPPORTED_DEVICE, "device ordinal out of range");
  return st[dev];
}

// Thread-local, per-device resources (events, side streams, pinned staging) are
// released when the thread exits.
struct EventPool {
  std::map<int, std::vector<cudaEvent_t>> free;
  ~EventPool() {
    for (auto& kv : free)
      for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
  }
};
inline thread_local EventPool g_events;

inline cudaEvent_t pool_event(int dev) {
  auto& v = g_events.free[dev];
  if (!v.empty()) {
    cudaEvent_t e = v.back();
    v.pop_back();
    return e;
  }
  cudaEvent_t e;
  SQ_CUDA(cudaEventCreate(&e));
  return e;
}
inline void pool_return(int dev, cudaEvent_t e) { g_events.free[dev].push_back(e); }

// ------------------------------------------------------------------ per-kernel timing
// When enabled (sq_profile), every launch is bracketed by CUDA events on its
// stream; elapsed times accumulate per kernel role after the call's final sync.
struct ProfEntry {
  const char* name;
  int dev;
  cudaEvent_t a, b;
};
inline std::atomic<bool> g_prof{false};
inline thread_local std::vector<ProfEntry> g_prof_pending;
inline std::mutex g_prof_mu;
inline std::map<std::string, std::pair<uint64_t, double>> g_prof_acc;

struct ProfScope {
  cudaStream_t st;
  const char* name;
  int dev = 0;
  cudaEvent_t a = nullptr;
  ProfScope(const char* n, cudaStream_t s) : st(s), name(n) {
    if (g_prof.load()) {
      dev = cur_device();
      a = pool_event(dev);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = nullptr;
      try {
        b = pool_event(dev);
      } catch (...) {
        pool_return(dev, a);
        return;
      }
      cudaEventRecord(b, st);
      g_prof_pending.push_back({name, dev, a, b});
    }
  }
};

inline void prof_collect() {  // after a stream sync
  if (g_prof_pending.empty()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_prof_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) {
      auto& v = g_prof_acc[e.name];
      v.first++;
      v.second += ms;
    }
    pool_return(e.dev, e.a);
    pool_return(e.dev, e.b);
  }
  g_prof_pending.clear();
}

// ------------------------------------------------------------------ host trace
// SQ_HOST_TRACE=1 prints host timestamps of the level phases to stderr (diagnostics).
inline bool g_trace = getenv("SQ_HOST_TRACE") != nullptr;
inline void htrace(const char* what, size_t a = 0, size_t b = 0) {
  if (!g_trace) return;
  static const auto t0 = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  fprintf(stderr, "[sq %10.1f us] %s %zu %zu\n", us, what, a, b);
}

// ------------------------------------------------------------------ options
inline uint32_t g_max_tile = 0;  // 0 = default
// buckets larger than one CTA's tile: 0 = another SquareSort level,
// 1 = multi-CTA merge sort (default), 2 = thread-block cluster sort
inline int g_big_mode = getenv("SQ_BIG_MODE") ? atoi(getenv("SQ_BIG_MODE")) : 1;
// bucket-sort size classes run concurrently on side streams (SQ_CONCURRENT_CLASSES=0
// serialises them on the caller's stream; measured 6.47 vs 6.61 ms at cfg5)
inline int g_concurrent_classes = getenv("SQ_CONCURRENT_CLASSES") ? atoi(getenv("SQ_CONCURRENT_CLASSES")) : 1;

// on-chip base case for 32- and 64-bit sort keys (keys, u32-key pairs): 1 = counting
// sort + network fix-up (binsort.cuh, default, where its shared memory fits),
// 0 = merge sort (blocksort.cuh)
// small levels (graph replay, two bucket-sort classes): n at most this; see GraphCache below
inline size_t g_graph_max_n = getenv("SQ_GRAPH_MAX_N") ? (size_t)atoll(getenv("SQ_GRAPH_MAX_N")) : (size_t(1) << 22);
// samples of at least this many pivots are gathered by k_sample_gather (a huge value turns it off)
inline uint32_t g_sample_split = getenv("SQ_SAMPLE_SPLIT") ? (uint32_t)atoi(getenv("SQ_SAMPLE_SPLIT")) : 4096u;
inline int g_small_classes = getenv("SQ_SMALL_CLASSES") ? atoi(getenv("SQ_SMALL_CLASSES")) : 1;
inline int g_base_case = getenv("SQ_BASE_CASE") ? atoi(getenv("SQ_BASE_CASE")) : 1;
constexpr size_t kMaxSmem = 232448;  // dynamic shared memory per CTA on sm_100 (227 KB)
template <bool B, typename F>
void with_bin(F&& f) {
  f(std::integral_constant<bool, B>{});
}

// ------------------------------------------------------------------ device check
// The device must be an sm_100 part.  Scratch comes from a pool the library owns
// (the device's default pool and other users' allocations are left alone); freed
// scratch stays reserved in it between calls so that a repeated sort does not
// re-map gigabytes of memory, and sq_trim_memory() returns it to the system.
inline void check_device() {
  const int dev = cur_device();
  DeviceState& ds = dev_state(dev);
  std::lock_guard<std::mutex> lk(ds.mu);
  if (ds.checked == 0) {
    cudaDeviceProp p;
    SQ_CUDA(cudaGetDeviceProperties(&p, dev));
    ds.checked = (p.major == 10 && p.minor == 0) ? 1 : 2;
    ds.sms = p.multiProcessorCount;
    if (ds.checked == 2)
      throw Error(SQ_ERR_UNSUPPORTED_DEVICE,
                  "device is sm_" + std::to_string(p.major) + std::to_string(p.minor) + ", need sm_100 (B200)");
  }
  if (ds.checked == 2) throw Error(SQ_ERR_UNSUPPORTED_DEVICE, "device is not sm_100 (B200)");
  if (!ds.pool) {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    SQ_CUDA(cudaMemPoolCreate(&ds.pool, &pp));
    uint64_t thr = UINT64_MAX;
    SQ_CUDA(cudaMemPoolSetAttribute(ds.pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
}

inline cudaMemPool_t lib_pool() {
  DeviceState& ds = dev_state(cur_device());
  std::lock_guard<std::mutex> lk(ds.mu);
  if (!ds.pool) throw Error(SQ_ERR_CUDA, "library memory pool missing (check_device not called)");
  return ds.pool;
}

// ------------------------------------------------------------------ small transfers
// Descriptor uploads and size read-backs between pinned (UVA-mapped) host
// staging and device memory are done by SM loads/stores, not by the copy
// engines: a 1 GB copy of another batch item queued on a copy engine would
// otherwise hold the sort's few-KB transfers back (sq_sort_*_host_batch).
static __global__ void k_xfer(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t bytes) {
  const size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x, T = size_t(gridDim.x) * blockDim.x;
  if (((uintptr_t(src) | uintptr_t(dst)) & 15) == 0) {
    const size_t n16 = bytes >> 4;
    for (size_t i = t; i < n16; i += T) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = (n16 << 4) + t; i < bytes; i += T) dst[i] = src[i];
  } else {
    for (size_t i = t; i < bytes; i += T) dst[i] = src[i];
  }
}

inline void xfer(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  const uint32_t g = (uint32_t)std::min<size_t>((bytes + 4095) / 4096, 148);
  k_xfer<<<g, 256, 0, st>>>((const uint8_t*)src, (uint8_t*)dst, bytes);
  check_launch("k_xfer");
}

// ------------------------------------------------------------------ per-call memory
// Pinned host staging for descriptor uploads and size read-backs: one bump
// pool per host thread, reused across calls (page-locking is expensive).
struct PinnedPool {
  std::vector<std::pair<char*, size_t>> blocks;
  size_t cur = 0, used = 0;
  void* get(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    while (cur < blocks.size() && used + bytes > blocks[cur].second) {
      cur++;
      used = 0;
    }
    if (cur == blocks.size()) {
      size_t sz = std::max<size_t>(bytes, size_t(8) << 20);
      char* p = nullptr;
      SQ_CUDA(cudaMallocHost((void**)&p, sz));
      blocks.push_back({p, sz});
      used = 0;
    }
    void* r = blocks[cur].first + used;
    used += bytes;
    return r;
  }
  void reset() { cur = 0; used = 0; }
  ~PinnedPool() {
    for (auto& b : blocks) cudaFreeHost(b.first);
  }
};
inline thread_local PinnedPool g_pinned;

// Per-call memory: stream-ordered scratch from the library pool and pinned staging
// from the thread's bump pool.  A bump Arena (graph capture of a level, see
// GraphCache) instead hands out consecutive pieces of two caller-owned regions and
// never frees; every Arena counts the bytes it hands out, so that a level's needs
// are known after one ordinary run.
struct Arena {
  cudaStream_t st;
  std::vector<void*> dev;
  bool used_host = false;
  cudaMemPool_t pool;
  size_t dev_bytes = 0, pin_bytes = 0;  // handed out so far (rounded up to 256 bytes)
  char* bump_dev = nullptr;             // bump mode: regions and capacities
  char* bump_pin = nullptr;
  size_t bump_dev_cap = 0, bump_pin_cap = 0;
  static size_t rnd(size_t b) { return ((b ? b : 16) + 255) & ~size_t(255); }
  explicit Arena(cudaStream_t s) : st(s), pool(lib_pool()) {}
  Arena(cudaStream_t s, char* d, size_t dcap, char* h, size_t hcap)
      : st(s), pool(nullptr), bump_dev(d), bump_pin(h), bump_dev_cap(dcap), bump_pin_cap(hcap) {}
  void* alloc(size_t bytes) {
    if (bump_dev) {
      if (dev_bytes + rnd(bytes) > bump_dev_cap) throw Error(SQ_ERR_CUDA, "graph scratch region exhausted");
      void* p = bump_dev + dev_bytes;
      dev_bytes += rnd(bytes);
      return p;
    }
    void* p = nullptr;
    SQ_CUDA(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, st));
    dev.push_back(p);
    dev_bytes += rnd(bytes);
    return p;
  }
  void release(void* p) {
    auto it = std::find(dev.begin(), dev.end(), p);
    if (it != dev.end()) {
      cudaFreeAsync(p, st);
      dev.erase(it);
    }
  }
  void* pinned(size_t bytes) {
    if (bump_pin) {
      if (pin_bytes + rnd(bytes) > bump_pin_cap) throw Error(SQ_ERR_CUDA, "graph staging region exhausted");
      void* p = bump_pin + pin_bytes;
      pin_bytes += rnd(bytes);
      return p;
    }
    used_host = true;
    pin_bytes += rnd(bytes);
    return g_pinned.get(bytes);
  }
  // Several host arrays in one staging block and one transfer (one k_xfer launch
  // instead of one per array); returns their device addresses in order.
  std::vector<void*> upload_all(const std::vector<std::pair<const void*, size_t>>& parts) {
    size_t tot = 0;
    for (auto& p : parts) tot += (p.second + 15) & ~size_t(15);
    std::vector<void*> out;
    char* d = (char*)alloc(tot);
    char* h = tot ? (char*)pinned(tot) : nullptr;
    size_t o = 0;
    for (auto& p : parts) {
      if (p.second) memcpy(h + o, p.first, p.second);
      out.push_back(d + o);
      o += (p.second + 15) & ~size_t(15);
    }
    xfer(d, h, tot, st);
    return out;
  }
  template <typename T>
  static std::pair<const void*, size_t> part(const std::vector<T>& v) {
    return {v.data(), v.size() * sizeof(T)};
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* d = (T*)alloc(v.size() * sizeof(T));
    if (!v.empty()) {
      T* h = (T*)pinned(v.size() * sizeof(T));
      memcpy(h, v.data(), v.size() * sizeof(T));
      xfer(d, h, v.size() * sizeof(T), st);
    }
    return d;
  }
  ~Arena() {
    for (void* p : dev) cudaFreeAsync(p, st);
    if (used_host) {
      cudaStreamSynchronize(st);  // staging may be reused by the next call
      g_pinned.reset();
    }
  }
};

constexpr int kBinClusterTag = 100;  // cls_cl entries above it: counting-sort clusters of (entry - tag) CTAs

// ------------------------------------------------------------------ size classes
// On-chip tiles (threads x keys per thread) for 32-bit sort keys and for
// 64-bit sort keys (u64 keys, pair composites).
inline constexpr uint32_t kTiles[] = {64, 128, 256, 512, 1024, 2048, 3072, 4096, 6144, 8192, 12288, 16384, 24576, 32768};

template <typename SK> constexpr uint32_t key_max_tile() {
  return sizeof(SK) == 4 ? 32768u : (sizeof(SK) == 8 ? 16384u : 8192u);
}

inline uint32_t tile_for(uint32_t len) {
  for (uint32_t t : kTiles)
    if (len <= t) return t;
  return 0;
}

// Launch as a programmatic dependent of the previous kernel in the stream (it may
// start before that one finishes; it must execute griddepcontrol.wait before it
// touches that kernel's outputs).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*f)(KArgs...), uint32_t grid, uint32_t block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SQ_CUDA(cudaLaunchKernelEx(&cfg, f, std::forward<Args>(args)...));
}

// Dynamic shared memory above 48 KB must be opted into per kernel and per
// device; done once per (kernel, size) on each device.
template <typename F>
void set_smem(F f, size_t bytes) {
  DeviceState& ds = dev_state(cur_device());
  std::lock_guard<std::mutex> lk(ds.mu);
  const auto key = std::make_pair((const void*)f, bytes);
  if (ds.smem_set.count(key)) return;
  SQ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  ds.smem_set.insert(key);
}

template <int N> using IC = std::integral_constant<int, N>;

// f(IC<NT>, IC<V>) for the block shape of `tile` with sort key type SK.
template <typename SK, typename F>
void with_tile(uint32_t tile, F&& f) {
  if constexpr (sizeof(SK) == 4) {
    switch (tile) {
      case 64: return f(IC<32>{}, IC<2>{});
      case 128: return f(IC<32>{}, IC<4>{});
      case 256: return f(IC<32>{}, IC<8>{});
      case 512: return f(IC<32>{}, IC<16>{});
      case 1024: return f(IC<32>{}, IC<32>{});
      case 2048: return f(IC<64>{}, IC<32>{});
      case 3072: return f(IC<96>{}, IC<32>{});
      case 4096: return f(IC<128>{}, IC<32>{});
      case 6144: return f(IC<192>{}, IC<32>{});
      case 8192: return f(IC<256>{}, IC<32>{});
      case 12288: return f(IC<384>{}, IC<32>{});
      case 16384: return f(IC<512>{}, IC<32>{});
      case 24576: return f(IC<768>{}, IC<32>{});
      case 32768: return f(IC<1024>{}, IC<32>{});
    }
  } else if constexpr (sizeof(SK) == 16) {  // u64-key pair composites: 8 keys (32 registers) per thread
    switch (tile) {
      case 64: return f(IC<32>{}, IC<2>{});
      case 128: return f(IC<32>{}, IC<4>{});
      case 256: return f(IC<32>{}, IC<8>{});
      case 512: return f(IC<64>{}, IC<8>{});
      case 1024: return f(IC<128>{}, IC<8>{});
      case 2048: return f(IC<256>{}, IC<8>{});
      case 3072: return f(IC<384>{}, IC<8>{});
      case 4096: return f(IC<512>{}, IC<8>{});
      case 6144: return f(IC<768>{}, IC<8>{});
      case 8192: return f(IC<1024>{}, IC<8>{});
    }
  } else {
    switch (tile) {
      case 64: return f(IC<32>{}, IC<2>{});
      case 128: return f(IC<32>{}, IC<4>{});
      case 256: return f(IC<32>{}, IC<8>{});
      case 512: return f(IC<64>{}, IC<8>{});
      case 1024: return f(IC<128>{}, IC<8>{});
      case 2048: return f(IC<256>{}, IC<8>{});
      case 3072: return f(IC<192>{}, IC<16>{});
      case 4096: return f(IC<256>{}, IC<16>{});
      case 6144: return f(IC<384>{}, IC<16>{});
      case 8192: return f(IC<512>{}, IC<16>{});
      case 12288: return f(IC<768>{}, IC<16>{});
      case 16384: return f(IC<1024>{}, IC<16>{});
    }
  }
  throw Error(SQ_ERR_CUDA, "no block shape for tile " + std::to_string(tile));
}

// Latency shapes for the tiles of small levels (32-bit sort keys): a 512-2048 key
// tile sorted by 2-8 warps of 8 keys per thread (merge sort) instead of one or two
// warps of 32 -- a small level runs few CTAs, so a CTA's own latency is the level's.
template <typename SK, typename F>
void with_tile_lat(bool lat, uint32_t tile, F&& f) {
  if constexpr (sizeof(SK) == 4) {
    if (lat) switch (tile) {
      case 512: return f(IC<64>{}, IC<8>{});
      case 1024: return f(IC<128>{}, IC<8>{});
      case 2048: return f(IC<256>{}, IC<8>{});
    }
  }
  return with_tile<SK>(tile, std::forward<F>(f));
}

inline int num_sms() {
  DeviceState& ds = dev_state(cur_device());
  std::lock_guard<std::mutex> lk(ds.mu);
  if (!ds.sms) {
    int dev = cur_device();
    SQ_CUDA(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return ds.sms;
}

// One full wave of resident CTAs for a persistent kernel (sets the kernel's
// shared-memory attribute first), cached per device.
template <typename F>
int wave_grid(F f, int nt, size_t smem) {
  set_smem(f, smem);
  const int sms = num_sms();
  DeviceState& ds = dev_state(cur_device());
  std::lock_guard<std::mutex> lk(ds.mu);
  const auto key = std::make_tuple((const void*)f, nt, smem);
  auto it = ds.grids.find(key);
  if (it != ds.grids.end()) return it->second;
  int occ = 0;
  SQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, nt, smem));
  const int g = std::max(1, occ) * sms;
  ds.grids[key] = g;
  return g;
}

// count kernel configuration per key type (standalone SkewTranspose)
template <typename K> struct CountCfg;
template <> struct CountCfg<uint32_t> { static constexpr int NT = 512, STAGE = 16384, KSMEM = 16384; };
template <> struct CountCfg<uint64_t> { static constexpr int NT = 512, STAGE = 8192, KSMEM = 16384; };

// transpose configuration per (key type, pairs)
template <typename K, bool PAIRS> struct TrCfg;
template <> struct TrCfg<uint32_t, false> { static constexpr int NT = 256, S = 4096, G = 256; };
template <> struct TrCfg<uint32_t, true> { static constexpr int NT = 256, S = 4096, G = 256; };
template <> struct TrCfg<uint64_t, false> { static constexpr int NT = 256, S = 4096, G = 256; };
// piece-major transpose (sort path): threads, piece size, fragments per piece
constexpr int kPlanFW = 128;  // piece-plan window (columns); <= the transpose's F = 128
template <typename K, bool PAIRS> struct PmTr;
template <> struct PmTr<uint32_t, false> { static constexpr int NT = 256, S = 4096, F = 128, XNT = 256; };
template <> struct PmTr<uint32_t, true> { static constexpr int NT = 256, S = 4096, F = 128, XNT = 256; };
template <> struct PmTr<uint64_t, false> { static constexpr int NT = 256, S = 4096, F = 128, XNT = 256; };
template <> struct PmTr<uint64_t, true> { static constexpr int NT = 256, S = 4096, F = 128, XNT = 256; };

// cluster bucket sort: per-CTA tile (threads x keys) for 32-bit / 64-bit sort keys
// (small per-CTA tiles keep 3 CTAs per SM resident; the big one serves the
// rare buckets beyond 16 small tiles)
template <typename SK> struct ClusterCfg;
template <> struct ClusterCfg<uint32_t> { static constexpr int NT = 256, V = 32, TILE = 8192; };
template <> struct ClusterCfg<uint64_t> { static constexpr int NT = 256, V = 16, TILE = 4096; };
template <typename SK> struct ClusterBig;
template <> struct ClusterBig<uint32_t> { static constexpr int NT = 512, V = 32, TILE = 16384; };
template <> struct ClusterBig<uint64_t> { static constexpr int NT = 512, V = 16, TILE = 8192; };
// largest bucket one CTA sorts when clusters are on (2 CTAs per SM stay resident)
// (the counting-sort base case sorts up to 32K 32-bit keys per CTA at full rate;
// SQ_ONE_CAP overrides it for experiments)
// largest unit of packed small buckets (SQ_UNIT_MAX; 0 = the largest one-CTA class)
// (measured: 16K units 4.41 ms vs 32K 4.47 ms at cfg5 -- the 16K class runs two CTAs per SM)
inline uint32_t g_unit_max = getenv("SQ_UNIT_MAX") ? (uint32_t)atoi(getenv("SQ_UNIT_MAX")) : 16384u;
inline uint32_t g_one_cap = getenv("SQ_ONE_CAP") ? (uint32_t)atoi(getenv("SQ_ONE_CAP")) : 32768u;
// largest bucket one CTA sorts for 64-bit sort keys (u64 keys, u32-key pairs): the 12K
// counting-sort tile (cfg5p 7.27 -> 6.47 ms against 8K; a 16K pair tile does not fit
// the counting sort and runs the merge sort: 7.81 ms)
inline uint32_t g_one_cap8 = getenv("SQ_ONE_CAP8") ? (uint32_t)atoi(getenv("SQ_ONE_CAP8")) : 12288u;
// a bucket-sort class to leave out (its buckets go to the next larger class): the 24K
// class runs 24 warps per SM (80 registers), the 32K class 32 -- measured 4.392 vs
// 4.413-4.424 ms at cfg5 without it (SQ_SKIP_TILE=0 restores it)
inline uint32_t g_skip_tile = getenv("SQ_SKIP_TILE") ? (uint32_t)atoi(getenv("SQ_SKIP_TILE")) : 24576u;
// value-split sorts of big buckets (mode 4): the CTA tile and how full its ranges
// are planned (SQ_SPLIT_TILE: 0 = per key type default; SQ_SPLIT_FILL percent;
// SQ_SPLIT_QMAX: most ranges per bucket, larger buckets take the merge path)
inline uint32_t g_split_tile = getenv("SQ_SPLIT_TILE") ? (uint32_t)atoi(getenv("SQ_SPLIT_TILE")) : 0u;
inline uint32_t g_split_fill = getenv("SQ_SPLIT_FILL") ? (uint32_t)atoi(getenv("SQ_SPLIT_FILL")) : 85u;
inline uint32_t g_split_qmax = getenv("SQ_SPLIT_QMAX") ? (uint32_t)atoi(getenv("SQ_SPLIT_QMAX")) : 16u;
// the split kernel's tiles (a few shapes, to bound the instantiations)
inline constexpr uint32_t kSplitTiles[] = {256, 1024, 4096, 8192, 12288, 16384, 32768};
template <typename SK> uint32_t split_tile(uint32_t one) {
  uint32_t want = g_split_tile ? g_split_tile : (sizeof(SK) == 4 ? 16384u : 8192u);
  want = std::min(want, std::max(256u, one));
  uint32_t t = 256;
  for (uint32_t c : kSplitTiles)
    if (c <= want && c <= key_max_tile<SK>()) t = c;
  return t;
}
template <typename SK, typename F>
void with_split_tile(uint32_t tile, F&& f) {
  switch (tile) {
    case 256: return with_tile<SK>(256, f);
    case 1024: return with_tile<SK>(1024, f);
    case 4096: return with_tile<SK>(4096, f);
    case 8192: return with_tile<SK>(8192, f);
    case 12288: return with_tile<SK>(12288, f);
    case 16384: if constexpr (sizeof(SK) <= 8) return with_tile<SK>(16384, f); break;
    case 32768: if constexpr (sizeof(SK) == 4) return with_tile<SK>(32768, f); break;
  }
  throw Error(SQ_ERR_CUDA, "no split tile " + std::to_string(tile));
}

template <typename SK> uint32_t single_cap() {
  return sizeof(SK) == 4 ? (g_base_case ? g_one_cap : 16384u) : (sizeof(SK) == 8 ? g_one_cap8 : 4096u);
}

// merge passes: threads x outputs per thread (tile = NT * VM keys)
template <typename K, bool PAIRS> struct MergeCfg {
  static constexpr int NT = 128, VM = PAIRS ? 16 : 32;
};

// Side streams for running the bucket-class kernels concurrently, per host
// thread and device (destroyed when the thread exits).
struct SideStreams {
  static constexpr int N = 4;
  cudaStream_t s[N] = {};
};
struct SideStreamSet {
  std::map<int, SideStreams> per_dev;
  ~SideStreamSet() {
    for (auto& kv : per_dev)
      for (cudaStream_t x : kv.second.s)
        if (x) cudaStreamDestroy(x);
  }
};
inline thread_local SideStreamSet g_side;
inline SideStreams& side_streams() {
  const int dev = cur_device();
  auto it = g_side.per_dev.find(dev);
  if (it != g_side.per_dev.end()) return it->second;
  // streams 0-1 carry the critical path (chunk sorts, then the merge passes):
  // highest priority, so their CTAs are scheduled before the other classes'
  SideStreams ss;
  int lo = 0, hi = 0;
  SQ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int i = 0; i < SideStreams::N; i++)
    SQ_CUDA(cudaStreamCreateWithPriority(&ss.s[i], cudaStreamNonBlocking, i < 2 ? hi : lo));
  return g_side.per_dev[dev] = ss;
}

// `waiter` waits for everything enqueued on `on` so far.
inline void stream_wait(cudaStream_t waiter, cudaStream_t on) {
  const int dev = cur_device();
  cudaEvent_t e = pool_event(dev);
  cudaError_t r = cudaEventRecord(e, on);
  if (r == cudaSuccess) r = cudaStreamWaitEvent(waiter, e, 0);
  pool_return(dev, e);
  if (r != cudaSuccess) throw Error(SQ_ERR_CUDA, std::string("stream_wait: ") + cudaGetErrorString(r));
}

// Fork the side streams off `st`; join them back into `st` on join() or, if an
// exception unwinds past the fork, in the destructor, so that every stream-ordered
// free on `st` (Arena) comes after all side-stream work that may use the memory.
struct ForkJoin {
  cudaStream_t st;
  SideStreams& ss;
  bool active = false;
  ForkJoin(cudaStream_t s, SideStreams& side) : st(s), ss(side) {
    for (int i = 0; i < SideStreams::N; i++) stream_wait(ss.s[i], st);
    active = true;
  }
  void join() {
    if (!active) return;
    active = false;
    for (int i = 0; i < SideStreams::N; i++) stream_wait(st, ss.s[i]);
  }
  ~ForkJoin() {
    if (!active) return;
    active = false;
    for (int i = 0; i < SideStreams::N; i++) {
      try {
        stream_wait(st, ss.s[i]);
      } catch (...) {
        cudaStreamSynchronize(ss.s[i]);  // last resort: the frees must not overtake it
      }
    }
  }
};

// ------------------------------------------------------------------ the engine
struct Seg {
  uint32_t off, len;
  uint64_t node;
};

struct DebugOut {  // sq_debug_level_u32 / _u64
  void* dst;       // n keys (K)
  void* pivots;    // m-1 keys (K)
  uint32_t* bucend;
  uint32_t* info;
};

// BIN: the counting-sort base case (keys-only u32); each (K, PAIRS, BIN) is
// compiled in its own translation unit (inst_*.cu).
template <typename K, bool PAIRS, bool BIN = false>
struct Engine {
  using SK = sortkey_t<K, PAIRS>;  // on-chip sort key
  cudaStream_t st;
  Arena& ar;
  K* kb[3];        // [0] caller's buffer, [1] scratch, [2] merge-sort scratch
  uint32_t* vb[3];
  size_t n;
  uint32_t cap;
  int big_mode = g_big_mode;  // this engine's mode for buckets beyond one CTA

  Engine(cudaStream_t s, Arena& a, K* keys, uint32_t* vals, size_t n_) : st(s), ar(a), n(n_) {
    kb[0] = keys;
    kb[1] = kb[2] = nullptr;
    vb[0] = vals;
    vb[1] = vb[2] = nullptr;
    cap = key_max_tile<SK>();
    if (g_max_tile && g_max_tile < cap) cap = g_max_tile;
  }

  void ensure_scratch() {
    if (!kb[1]) kb[1] = (K*)ar.alloc(n * sizeof(K));
    if (PAIRS && !vb[1]) vb[1] = (uint32_t*)ar.alloc(n * sizeof(uint32_t));
  }
  void ensure_third() {
    if (!kb[2]) kb[2] = (K*)ar.alloc(n * sizeof(K));
    if (PAIRS && !vb[2]) vb[2] = (uint32_t*)ar.alloc(n * sizeof(uint32_t));
  }

  void copy_ranges(const std::vector<SegDesc>& r, int src, int dst) {
    if (r.empty() || src == dst) return;
    const SegDesc* d = ar.upload(r);
    ProfScope ps("copy", st);
    k_copy_ranges<K><<<(uint32_t)r.size(), 256, 0, st>>>(d, kb[src], kb[dst], PAIRS ? vb[src] : nullptr,
                                                         PAIRS ? vb[dst] : nullptr);
    check_launch("k_copy_ranges");
  }

  // Contiguous segments of at most `cap` keys: one CTA each, by size class.
  void blocksort(uint32_t tile, const std::vector<SegDesc>& d, int src, int dst, const char* role) {
    const SegDesc* dd = ar.upload(d);
    const uint32_t nseg = (uint32_t)d.size();
    with_tile<SK>(tile, [&](auto nt, auto v) {
      constexpr int NT = decltype(nt)::value, V = decltype(v)::value;
      using BS = BlockSort<SK, NT, V>;
      ProfScope ps(role, st);
      if constexpr (PAIRS) {
        const size_t smem = BS::SMEM_BYTES + size_t(BS::TILE) * 4;
        set_smem(k_blocksort_pairs<K, NT, V>, smem);
        k_blocksort_pairs<K, NT, V><<<nseg, NT, smem, st>>>(dd, kb[src], vb[src], kb[dst], vb[dst]);
      } else {
        set_smem(k_blocksort<K, NT, V>, BS::SMEM_BYTES);
        k_blocksort<K, NT, V><<<nseg, NT, BS::SMEM_BYTES, st>>>(dd, kb[src], kb[dst]);
      }
      check_launch("k_blocksort");
    });
  }

  void sort_batch(const std::vector<Seg>& segs, int src, int dst, int depth, const char* role) {
    if (depth > 48) throw Error(SQ_ERR_CUDA, "recursion too deep");
    std::map<uint32_t, std::vector<SegDesc>> cls;
    std::vector<Seg> big;
    std::vector<SegDesc> bigr;
    for (const Seg& s : segs) {
      if (s.len == 0) continue;
      if (s.len > cap) {
        big.push_back(s);
        bigr.push_back({s.off, s.len});
      } else {
        cls[std::max<uint32_t>(64, tile_for(s.len))].push_back({s.off, s.len});
      }
    }
    for (auto& kv : cls) blocksort(kv.first, kv.second, src, dst, role);
    if (!big.empty()) {
      copy_ranges(bigr, src, dst);  // a level sorts a segment where it will end up
      run_level(big, dst, depth, nullptr);
    }
  }

  template <int CL, typename CC>
  void launch_cluster_t(cudaStream_t cs, const uint32_t* lst, const uint32_t* cnt, const BucketRec* recs,
                        const TileInfo* tiles, int T, int X, const uint32_t* pout, const uint16_t* ppre,
                        uint32_t nbuck) {
    using BS = BlockSort<SK, CC::NT, CC::V>;
    const size_t smem = 2 * BS::SMEM_BYTES + (PAIRS ? size_t(BS::TILE) * 4 : 0) + (3 * CC::NT + 64) * 4;
    auto f = k_clustersort<K, CC::NT, CC::V, CL, PAIRS>;
    int max_clusters = -1;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(CC::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = cs;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (max_clusters < 0) {
      set_smem(f, smem);
      if (CL > 8) SQ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));  // cheap; per device
      cfg.gridDim = dim3(CL * num_sms());
      int mc = 0;
      SQ_CUDA(cudaOccupancyMaxActiveClusters(&mc, f, &cfg));
      max_clusters = mc;
    }
    if (max_clusters <= 0) throw Error(SQ_ERR_CUDA, "cluster of " + std::to_string(CL) + " CTAs cannot be scheduled");
    cfg.gridDim = dim3(CL * std::min<uint32_t>(max_clusters, nbuck));
    ProfScope ps("clustersort", cs);
    SQ_CUDA(cudaLaunchKernelEx(&cfg, f, recs, tiles, lst, cnt, (const K*)kb[T], kb[X],
                               (const uint32_t*)(PAIRS ? vb[T] : nullptr), PAIRS ? vb[X] : nullptr, pout, ppre));
    check_launch("k_clustersort");
  }

  // Clusters of CL counting-sort tiles (mode 3, 32-bit keys): one cluster per bucket,
  // persistent over the class list; skewed buckets go to the oversize list.
  template <int CL>
  void launch_bincluster_t(cudaStream_t cs, const uint32_t* lst, const uint32_t* cnt, const BucketRec* recs,
                           const TileInfo* tiles, int T, int X, const uint32_t* pout, const uint16_t* ppre,
                           uint32_t* ovl, uint32_t* ovc, uint32_t nbuck) {
    if constexpr (std::is_same<K, uint32_t>::value && !PAIRS) {
      auto f = k_binsort_cluster<CL>;
      constexpr size_t smem = BinClusterCfg::SMEM;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(BinClusterCfg::NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = cs;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      set_smem(f, smem);
      static int max_clusters[64] = {0};  // per device ordinal
      const int dev = cur_device();
      int& mc = max_clusters[dev & 63];
      if (mc <= 0) {
        cfg.gridDim = dim3(CL * num_sms());
        SQ_CUDA(cudaOccupancyMaxActiveClusters(&mc, f, &cfg));
        if (mc <= 0) throw Error(SQ_ERR_CUDA, "cluster of " + std::to_string(CL) + " counting-sort tiles cannot be scheduled");
      }
      cfg.gridDim = dim3(CL * std::min<uint32_t>(mc, nbuck));
      std::optional<ProfScope> ps;
      if (!g_concurrent_classes) ps.emplace("bucketsort", cs);
      SQ_CUDA(cudaLaunchKernelEx(&cfg, f, recs, tiles, lst, cnt, (const uint32_t*)kb[T], (uint32_t*)kb[X], pout, ppre,
                                 ovl, ovc));
      check_launch("k_binsort_cluster");
    } else {
      throw Error(SQ_ERR_CUDA, "counting-sort clusters serve 32-bit keys only");
    }
  }
  void launch_bincluster(int cl, cudaStream_t cs, const uint32_t* lst, const uint32_t* cnt, const BucketRec* recs,
                         const TileInfo* tiles, int T, int X, const uint32_t* pout, const uint16_t* ppre,
                         uint32_t* ovl, uint32_t* ovc, uint32_t nbuck) {
    if (cl == 2) launch_bincluster_t<2>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, ovl, ovc, nbuck);
    else if (cl == 4) launch_bincluster_t<4>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, ovl, ovc, nbuck);
    else launch_bincluster_t<8>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, ovl, ovc, nbuck);
  }

  // cl > 0: clusters of `cl` small tiles; cl < 0: clusters of -cl big tiles
  void launch_cluster(int cl, cudaStream_t cs, const uint32_t* lst, const uint32_t* cnt, const BucketRec* recs,
                      const TileInfo* tiles, int T, int X, const uint32_t* pout, const uint16_t* ppre,
                      uint32_t nbuck) {
    if constexpr (sizeof(SK) == 16) {
      throw Error(SQ_ERR_CUDA, "cluster bucket sort is not built for u64 pairs");
    } else {
    using CS = ClusterCfg<SK>;
    using CB = ClusterBig<SK>;
    if (cl == 4) launch_cluster_t<4, CS>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, nbuck);
    else if (cl == 8) launch_cluster_t<8, CS>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, nbuck);
    else if (cl == 16) launch_cluster_t<16, CS>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, nbuck);
    else launch_cluster_t<16, CB>(cs, lst, cnt, recs, tiles, T, X, pout, ppre, nbuck);
    }
  }

  // One SquareSort level (Alg 1) for a batch of segments that live in buffer X,
  // their final place.  The SkewTranspose writes into the other buffer T; the
  // bucket sorts gather from T and write the sorted buckets back into X.
  void run_level(const std::vector<Seg>& segs, int X, int depth, DebugOut* dbg) {
    LevelTail lt;
    if (!launch_level(segs, X, depth, dbg, lt)) return;  // (debug: state copied out)
    finish_level(lt, X);
  }

  // What the host needs after a level's launches: the pinned read-back of the class
  // counts and the round, and where the oversize list lives.
  struct LevelTail {
    uint32_t* hcnt = nullptr;
    uint32_t* hinfo = nullptr;
    uint32_t ncls = 0, cap_per_list = 0, top_m = 0;
    const uint32_t* list = nullptr;
    const BucketRec* recs = nullptr;
    uint64_t buck_tot = 0;
    int depth = 0;
    std::vector<void*> rel;  // scratch released after the read-back
  };

  // 7. one host read per level: the oversize list (and the round, for stats);
  // oversize buckets become the next level's batch.
  void finish_level(LevelTail& lt, int X) {
    SQ_CUDA(cudaStreamSynchronize(st));
    g_stats.host_syncs++;
    if (lt.depth == 0) {
      g_stats.top_round = lt.hinfo[0] & 0x7fffffffu;
      g_stats.top_degenerate = lt.hinfo[0] >> 31;
      g_stats.top_m = lt.top_m;
    }
    const uint32_t nos = lt.hcnt[lt.ncls + 1];
    std::vector<Seg> over;
    if (nos) {
      uint32_t* hl = (uint32_t*)ar.pinned(nos * 4);
      xfer(hl, lt.list + uint64_t(lt.ncls + 1) * lt.cap_per_list, nos * 4, st);
      BucketRec* hr = (BucketRec*)ar.pinned(lt.buck_tot * sizeof(BucketRec));
      xfer(hr, lt.recs, lt.buck_tot * sizeof(BucketRec), st);
      SQ_CUDA(cudaStreamSynchronize(st));
      g_stats.host_syncs++;
      for (uint32_t q = 0; q < nos; q++) {
        const uint32_t e = hl[q];
        const uint32_t i = item_bucket(e);
        over.push_back({hr[i].out, hr[i].size, hr[i].node});
        g_stats.oversize_keys += hr[i].size;
      }
    }
    for (void* p : lt.rel) ar.release(p);
    htrace("level: done, oversize segments", over.size(), lt.depth);
    if (!over.empty()) sort_batch(over, X, X, lt.depth + 1, "bucketsort");
  }

  // Launch every kernel of one level (steps 1-6 and the read-back transfers of step
  // 7); nothing here waits for the device, so the sequence can be captured in a
  // CUDA graph.  Returns false when dbg is given (the level state was copied out).
  bool launch_level(const std::vector<Seg>& segs, int X, int depth, DebugOut* dbg, LevelTail& lt) {
    using TC = PmTr<K, PAIRS>;
    ensure_scratch();
    g_stats.levels++;
    const int T = 1 - X;
    const uint32_t ns = (uint32_t)segs.size();
    std::vector<LevelSeg> L(ns);
    std::vector<uint32_t> tile_base(ns), piece_seg_base(ns);
    std::vector<TileInfo> tiles;
    std::map<uint32_t, std::vector<ColDesc>> colcls;
    std::vector<Seg> allcols;
    std::vector<TaskDesc> mtasks;
    bool generic = false;
    uint64_t piv_tot = 0, buck_tot = 0, segmat_tot = 0, cand_tot = 0, piece_tot = 0;
    uint32_t maxnp = 0;
    for (uint32_t s = 0; s < ns; s++) {
      const Seg& g = segs[s];
      const uint32_t m = (uint32_t)ceil_sqrt(g.len);
      LevelSeg& l = L[s];
      l.off = g.off;
      l.len = g.len;
      l.rows = l.ncols = l.k = m;
      l.nbt = (m + kTB - 1) / kTB;
      l.piv_base = (uint32_t)piv_tot;
      l.buck_base = (uint32_t)buck_tot;
      l.segmat_base = segmat_tot;
      l.cand_base = cand_tot;
      l.node = g.node;
      const uint32_t np = m - 1;
      maxnp = std::max(maxnp, np);
      piv_tot += np;
      buck_tot += m;
      segmat_tot += uint64_t(m) * (l.nbt + 1);
      cand_tot += uint64_t(kCap) * np;
      tile_base[s] = (uint32_t)tiles.size();
      for (uint32_t bt = 0; bt < l.nbt; bt++) tiles.push_back({s, bt, 0, 0, 0, 0, 0});
      // windows per tile (plan_fw): at most ceil(m / kPlanFW) + size * 32 / (31 S) + 2
      const uint32_t gpt = (m + kPlanFW - 1) / kPlanFW + 2;
      piece_seg_base[s] = (uint32_t)piece_tot;
      piece_tot += 3 * (g.len / TC::S) + uint64_t(l.nbt) * (1 + gpt) + 1;
      // columns: fc full ones of m keys, then at most one ragged one
      const uint32_t fc = (uint32_t)std::min<uint64_t>(m, g.len / m);
      const uint32_t rem = fc < m ? (uint32_t)(g.len - uint64_t(fc) * m) : 0u;
      if (m > cap) {
        generic = true;
        for (uint32_t c = 0; c < fc + (rem ? 1u : 0u); c++)
          allcols.push_back({uint32_t(g.off + uint64_t(c) * m), c < fc ? m : rem, child_key(g.node, 0, c)});
      } else {
        std::vector<ColDesc>& full = colcls[std::max<uint32_t>(64, tile_for(m))];
        for (uint32_t c = 0; c < fc; c++) full.push_back({uint32_t(g.off + uint64_t(c) * m), m, s, c});
        // the ragged last column rides in the full columns' class (padded tile): a class
        // of its own is one more launch, a lone CTA after the column sort's last wave
        if (rem)
          (fc ? full : colcls[std::max<uint32_t>(64, tile_for(rem))])
              .push_back({uint32_t(g.off + uint64_t(fc) * m), rem, s, fc});
      }
      for (uint32_t c0 = 0; c0 < m; c0 += 64) mtasks.push_back({s, c0, std::min(m, c0 + 64)});
    }
    if (maxnp > key_max_tile<K>()) throw Error(SQ_ERR_INVALID_ARGUMENT, "pivot sample too large for one CTA");
    const uint32_t ntiles = (uint32_t)tiles.size();

    // every descriptor of the level in one transfer; the column descriptors too:
    // nothing but kernels may sit between the sampler, the round selection and the
    // column sort (programmatic dependent launch)
    std::vector<std::pair<const void*, size_t>> parts = {Arena::part(L), Arena::part(tiles),
                                                        Arena::part(tile_base), Arena::part(piece_seg_base),
                                                        Arena::part(mtasks)};
    if (!generic)
      for (auto& kv : colcls) parts.push_back(Arena::part(kv.second));
    htrace("level: descriptors built", ns, depth);
    const std::vector<void*> up = ar.upload_all(parts);
    htrace("level: uploaded");
    LevelSeg* dL = (LevelSeg*)up[0];
    TileInfo* dTiles = (TileInfo*)up[1];
    uint32_t* dTileBase = (uint32_t*)up[2];
    uint32_t* dPieceBase = (uint32_t*)up[3];
    TaskDesc* dM = (TaskDesc*)up[4];
    K* cand = (K*)ar.alloc(std::max<uint64_t>(cand_tot, 1) * sizeof(K));
    uint8_t* flags = (uint8_t*)ar.alloc(uint64_t(ns) * kCap);
    K* p0s = (K*)ar.alloc(uint64_t(ns) * kCap * sizeof(K));
    K* piv = (K*)ar.alloc(std::max<uint64_t>(piv_tot, 1) * sizeof(K));
    uint32_t* info = (uint32_t*)ar.alloc(ns * 4);
    uint32_t* fix = (uint32_t*)ar.alloc((ns + 1) * 4);
    K* segmin = (K*)ar.alloc(ns * sizeof(K));
    uint32_t* segmat = (uint32_t*)ar.alloc(segmat_tot * 4);
    uint32_t* pout = (uint32_t*)ar.alloc(piece_tot * 4);
    uint16_t* ppre = (uint16_t*)ar.alloc(piece_tot * kPP * 2);
    BucketRec* recs = (BucketRec*)ar.alloc(buck_tot * sizeof(BucketRec));
    SQ_CUDA(cudaMemsetAsync(fix, 0, (ns + 1) * 4, st));
    SQ_CUDA(cudaMemsetAsync(segmin, 0xff, ns * sizeof(K), st));
    SQ_CUDA(cudaMemsetAsync(segmat, 0, segmat_tot * 4, st));

    std::vector<std::pair<uint32_t, const ColDesc*>> coldesc;
    if (!generic) {
      size_t q = 5;
      for (auto& kv : colcls) coldesc.push_back({kv.first, (const ColDesc*)up[q++]});
    }
    // 1. pivots: all rounds in parallel from the level input (L9)
    uint64_t level_total = 0;
    for (const Seg& g : segs) level_total += g.len;
    const bool lat = level_total <= g_graph_max_n && g_small_classes;  // small level: latency shapes
    // (every round is one CTA alone on its SM: its latency is the sampler's, so the
    // 8K/16K-candidate sorts of 32-bit keys run twice the warps with 16 keys per thread)
    auto with_sample_tile = [&](uint32_t tile, auto&& f) {
#ifndef SQ_SAMPLE_V32
      if constexpr (sizeof(K) == 4) {
        if (tile == 16384) return f(IC<1024>{}, IC<16>{});
        if (tile == 8192) return f(IC<512>{}, IC<16>{});
      }
#endif
      return with_tile_lat<K>(lat, tile, f);
    };
    with_sample_tile(std::max<uint32_t>(64, tile_for(std::max<uint32_t>(maxnp, 1))), [&](auto nt, auto v) {
      constexpr int NT = decltype(nt)::value, V = decltype(v)::value;
      using BS = BlockSort<K, NT, V>;
      constexpr bool SB = BIN && BS::SMEM_BYTES + bin_smem<K, NT, V, false, BIN>() <= kMaxSmem;
      constexpr size_t smem = BS::SMEM_BYTES + bin_smem<K, NT, V, false, SB>();
      set_smem(k_sample_all<K, NT, V, SB>, smem);
      ProfScope ps("sample", st);
      // large samples: the random reads spread over many CTAs first (k_sample_gather)
      const bool split = maxnp >= g_sample_split;
      if (split) {
        const uint32_t nchunk = (maxnp + kSampleChunk - 1) / kSampleChunk;
        k_sample_gather<K><<<ns * kCap * nchunk, 256, 0, st>>>(dL, kb[X], cand, nchunk);
        check_launch("k_sample_gather");
        launch_pdl(k_sample_all<K, NT, V, SB>, ns * kCap, NT, smem, st, (const LevelSeg*)dL, (const K*)kb[X], cand,
                   flags, p0s, true);
      } else {
        k_sample_all<K, NT, V, SB><<<ns * kCap, NT, smem, st>>>(dL, kb[X], cand, flags, p0s, false);
      }
      check_launch("k_sample_all");
    });
    {
      ProfScope ps("select", st);
      launch_pdl(k_select_round<K>, ns, 1024, 0, st, dL, ns, (const K*)cand, (const uint8_t*)flags, (const K*)p0s,
                 (const K*)segmin, piv, info, fix, 0);
    }
    htrace("level: sampler launched");
    // 2. sort every column in place + tile boundaries + min(D).  The first
    // class launches as a programmatic dependent: its CTAs load and sort while the
    // sampler and the round selection still run, and wait for them (griddepcontrol)
    // before writing keys back (the sampler reads the unsorted level input) and
    // before reading the pivots.
    if (!generic) {
      bool first = true;
      for (auto& cd : coldesc) {
        const uint32_t ncol = (uint32_t)colcls[cd.first].size();
        with_tile_lat<SK>(lat, cd.first, [&](auto nt, auto v) {
          constexpr int NT = decltype(nt)::value, V = decltype(v)::value;
          using BS = BlockSort<SK, NT, V>;
          constexpr size_t base = BS::SMEM_BYTES + (PAIRS ? size_t(BS::TILE) * 4 : 0);
          with_bin<BIN && base + bin_smem<K, NT, V, PAIRS, BIN>() <= kMaxSmem>([&](auto bin) {
          constexpr bool UB = decltype(bin)::value;
          const size_t smem = base + bin_smem<K, NT, V, PAIRS, UB>();
          set_smem(k_colsort<K, NT, V, PAIRS, UB>, smem);
          ProfScope ps("colsort", st);
          auto f = k_colsort<K, NT, V, PAIRS, UB>;
          if (first && !g_prof.load())
            launch_pdl(f, ncol, NT, smem, st, cd.second, (const LevelSeg*)dL, kb[X], PAIRS ? vb[X] : nullptr,
                       (const K*)piv, segmat, segmin);
          else
            f<<<ncol, NT, smem, st>>>(cd.second, dL, kb[X], PAIRS ? vb[X] : nullptr, piv, segmat, segmin);
          check_launch("k_colsort");
          first = false;
          });
        });
      }
    } else {  // columns longer than a CTA holds: a recursive level sorts them
      sort_batch(allcols, X, X, depth + 1, "colsort");
      {
        ProfScope ps("colmin", st);
        k_colmin<K><<<ns, 256, 0, st>>>(dL, kb[X], segmin);
        check_launch("k_colmin");
      }
      {
        ProfScope ps("segmat", st);
        k_segmat<K><<<(uint32_t)mtasks.size(), 256, 0, st>>>(dL, dM, kb[X], piv, segmat, fix, 0);
        check_launch("k_segmat");
      }
    }
    htrace("level: columns launched");
    // 3. min-exclusion: final round; repair the boundaries if it changed
    {
      ProfScope ps("select", st);
      k_select_round<K><<<ns, 1024, 0, st>>>(dL, ns, cand, flags, p0s, segmin, piv, info, fix, 1);
      check_launch("k_select_round");
    }
    {
      ProfScope ps("segmat", st);
      k_segmat<K><<<(uint32_t)mtasks.size(), 256, 0, st>>>(dL, dM, kb[X], piv, segmat, fix, 1);
      check_launch("k_segmat");
    }
    ar.release(cand);
    // 4. tile sizes and offsets, then the SkewTranspose X -> T; the
    // transpose also accumulates the bucket sizes
    uint32_t* bsize = (uint32_t*)ar.alloc(buck_tot * 4);
    SQ_CUDA(cudaMemsetAsync(bsize, 0, buck_tot * 4, st));
    uint32_t* pcount = (uint32_t*)ar.alloc(16);  // [0] pieces
    {
      ProfScope ps("tiles", st);
      k_tile_sizes<TC::S, kPlanFW><<<ntiles, 1024, 0, st>>>(dL, dTiles, segmat);
      check_launch("k_tile_sizes");
      // (one segment: the scan also builds the dense piece list)
      k_tile_scan<<<ns, 256, 0, st>>>(dL, dTileBase, dTiles, TC::S, kPlanFW, dPieceBase, ns == 1 ? pcount : nullptr);
      check_launch("k_tile_scan");
    }
    {
      PieceDesc* pieces = (PieceDesc*)ar.alloc(piece_tot * sizeof(PieceDesc));
      {
        ProfScope ps("tiles", st);
        if (ns != 1) {
          k_piece_dense<<<1, 1024, 0, st>>>(dTiles, ntiles, pcount);
          check_launch("k_piece_dense");
        }
        k_piece_plan2<1024, TC::S, kPlanFW><<<ntiles, 1024, 0, st>>>(dL, dTiles, segmat, pieces, pout);
        check_launch("k_piece_plan2");
      }
      using XC = WsCfg<K, PAIRS, TC::S, TC::F>;
      auto f = k_transpose_ws<K, PAIRS, TC::S, TC::F>;
      const int grid = wave_grid(f, XC::NT, XC::SMEM);
      ProfScope ps("transpose", st);
      f<<<(uint32_t)std::min<uint64_t>(grid, piece_tot), XC::NT, XC::SMEM, st>>>(
          pieces, pcount, kb[X], kb[T], PAIRS ? vb[X] : nullptr, PAIRS ? vb[T] : nullptr, piv, segmat, ppre, bsize);
      check_launch("k_transpose_ws");
      ar.release(pcount);
      ar.release(pieces);
    }
    htrace("level: transpose launched");
    // 5. bucket plan: sizes, final offsets, work lists
    // mode 3 (clusters of counting-sort tiles) serves 32-bit keys with the counting
    // sort; other engines and forced tiles run mode 1 instead
    const bool bincl = big_mode == 3 && std::is_same<SK, uint32_t>::value && BIN && !g_max_tile;
    const int mode = big_mode == 3 && !bincl ? 1 : big_mode;
    PlanOut po{};
    po.ncls = 0;
    int cls_cl[20] = {0};  // 0 = one CTA; > 0 clusters of small tiles; < 0 clusters of big tiles
    uint64_t level_keys = 0, longest_seg = 0;
    for (const Seg& g : segs) {
      level_keys += g.len;
      longest_seg = std::max<uint64_t>(longest_seg, g.len);
    }
    const bool small_level = level_keys <= g_graph_max_n && (mode == 0 || mode == 1) && !g_max_tile;
    // small levels: units small enough that most SMs get one (but CTAs of >= 128
    // threads: 4K keys, or 1K keys in the latency shape of with_tile_lat)
    uint32_t small_unit = small_level && g_small_classes ? 1024 : 4096;
    while (small_unit < (1u << 15) && uint64_t(small_unit) * 2 * num_sms() < level_keys) small_unit *= 2;
    {
      const uint32_t one = bincl ? std::min<uint32_t>(cap, BinClusterCfg::TILE)
                           : (mode != 0 && !g_max_tile ? std::min(cap, single_cap<SK>()) : cap);
      // smallest bucket-sort class 1K keys: smaller chunks share it (their padding is
      // skipped), instead of a latency-bound launch per tiny class
      const uint32_t lower = std::min<uint32_t>(1024u, one);
      for (uint32_t t : kTiles)
        if (t >= lower && t <= one && t <= key_max_tile<SK>() && !(g_skip_tile && t == g_skip_tile))
          po.cls_tile[po.ncls++] = t;
      // small levels are bound by the number of dependent launches, not by the sorting:
      // three classes only -- the units' tile, four times it (the tail of the bucket
      // sizes, so that a bucket just above a unit is not sorted in a 32K tile) and
      // the one-CTA cap
      if (small_level && g_small_classes && po.ncls > 3) {
        uint32_t ut = po.cls_tile[0];
        for (uint32_t c = 0; c < po.ncls; c++)
          if (po.cls_tile[c] <= small_unit) ut = po.cls_tile[c];
        po.ncls = 0;
        for (uint32_t t : {ut, 4 * ut, one})
          if (t <= one && (!po.ncls || t > po.cls_tile[po.ncls - 1])) po.cls_tile[po.ncls++] = t;
      }
      po.max_tile = one;
      if (bincl)  // beyond one CTA: clusters of 2, 4, 8 counting-sort tiles (binclust.cuh)
        for (int cl : {2, 4, 8}) {
          cls_cl[po.ncls] = kBinClusterTag + cl;
          po.cls_tile[po.ncls++] = BinClusterCfg::cap(cl);
          po.max_tile = BinClusterCfg::cap(cl);
        }
      if constexpr (sizeof(SK) <= 8) if (mode == 2) {  // beyond one CTA: clusters of 4, 8, 16 CTAs
        const uint32_t ct = std::min<uint32_t>(ClusterCfg<SK>::TILE, cap);
        for (int cl : {4, 8, 16}) {
          if (cl * ct <= po.max_tile) continue;
          cls_cl[po.ncls] = cl;
          po.cls_tile[po.ncls++] = cl * ct;
          po.max_tile = cl * ct;
        }
        if (!g_max_tile && 16u * ClusterBig<SK>::TILE > po.max_tile) {
          cls_cl[po.ncls] = -16;
          po.cls_tile[po.ncls++] = 16u * ClusterBig<SK>::TILE;
          po.max_tile = 16u * ClusterBig<SK>::TILE;
        }
      }
    }
    po.msort_max = po.max_tile;
    po.mtile = MergeCfg<K, PAIRS>::NT * MergeCfg<K, PAIRS>::VM;
    po.mcap = 1;
    po.units = (Unit*)ar.alloc(buck_tot * sizeof(Unit));
    po.unit_max = 0;
    for (uint32_t c = 0; c < po.ncls; c++)
      if (!cls_cl[c]) po.unit_max = std::max(po.unit_max, po.cls_tile[c]);
    if (g_unit_max) po.unit_max = std::min(po.unit_max, g_unit_max);
    po.unit_max = std::min(po.unit_max, small_unit);
    po.nunits = (uint32_t*)ar.alloc(16);
    SQ_CUDA(cudaMemsetAsync(po.nunits, 0, 4, st));
    // (u64 pairs have no cluster kernel: mode 2 runs the merge base case for them)
    const bool merge = mode == 1 || mode == 4 || (mode == 2 && sizeof(SK) == 16);
    if (merge) {  // multi-CTA merge sort for buckets of up to 16 chunks
      po.msort_max = 16u * po.max_tile;
      po.mcap = (uint32_t)(level_keys / po.mtile + 9 * buck_tot + 16);
      ensure_third();
    }
    po.mlist = (MTile*)ar.alloc(uint64_t(kMaxPasses) * po.mcap * sizeof(MTile));
    po.mcount = (uint32_t*)ar.alloc(kMaxPasses * 4);
    SQ_CUDA(cudaMemsetAsync(po.mcount, 0, kMaxPasses * 4, st));
    // value split (mode 4, keys only): inner buckets of up to split_qmax ranges
    const uint32_t stile = split_tile<SK>(po.max_tile);
    if (mode == 4 && !PAIRS) {
      po.split_part = std::max<uint32_t>(1, uint32_t(uint64_t(stile) * std::min<uint32_t>(g_split_fill, 100) / 100));
      po.split_max = std::min<uint32_t>(std::max<uint32_t>(1, std::min<uint32_t>(g_split_qmax, 16)) * po.split_part,
                                        po.msort_max);
    }
    po.cap_per_list = (uint32_t)(buck_tot + level_keys / std::max<uint32_t>(std::min(po.max_tile, po.split_max ? po.split_part : ~0u), 1) + 16);
    // lists: [0, ncls) classes, ncls copy, ncls+1 oversize, ncls+2 pair, then the
    // chunks of merge-sorted buckets per class at ncls+3+c (sorted first, so that
    // the merge passes can overlap the other classes), then the value-split items
    const uint32_t nlists = 2 * po.ncls + 4;
    po.split_list = 2 * po.ncls + 3;
    po.list = (uint32_t*)ar.alloc(uint64_t(nlists) * po.cap_per_list * 4);
    po.count = (uint32_t*)ar.alloc(nlists * 4);
    SQ_CUDA(cudaMemsetAsync(po.count, 0, nlists * 4, st));
    {
      ProfScope ps("plan", st);
      k_tile_bucket_plan<K><<<(ntiles * 32 + 127) / 128, 128, 0, st>>>(dL, dTiles, ntiles, bsize, piv, recs, po);
      check_launch("k_tile_bucket_plan");
    }
    if (dbg) {
      k_bucket_gather<K, 256><<<1024, 256, 0, st>>>(recs, dTiles, nullptr, nullptr, (uint32_t)buck_tot, kb[T],
                                                    (K*)dbg->dst, nullptr, nullptr, pout, ppre);
      check_launch("k_bucket_gather");
      std::vector<BucketRec> hr(buck_tot);
      std::vector<uint32_t> hinfo(ns);
      SQ_CUDA(cudaMemcpyAsync(hr.data(), recs, buck_tot * sizeof(BucketRec), cudaMemcpyDeviceToHost, st));
      SQ_CUDA(cudaMemcpyAsync(hinfo.data(), info, ns * 4, cudaMemcpyDeviceToHost, st));
      SQ_CUDA(cudaMemcpyAsync(dbg->pivots, piv, piv_tot * sizeof(K), cudaMemcpyDeviceToDevice, st));
      SQ_CUDA(cudaStreamSynchronize(st));
      std::vector<uint32_t> be(buck_tot), inf = {hinfo[0] & 0x7fffffffu, hinfo[0] >> 31};
      for (uint64_t i = 0; i < buck_tot; i++) be[i] = hr[i].out + hr[i].size;
      uint32_t* dbe = ar.upload(be);
      uint32_t* dinf = ar.upload(inf);
      SQ_CUDA(cudaMemcpyAsync(dbg->bucend, dbe, buck_tot * 4, cudaMemcpyDeviceToDevice, st));
      SQ_CUDA(cudaMemcpyAsync(dbg->info, dinf, 8, cudaMemcpyDeviceToDevice, st));
      return false;
    }
    // 6. bucket sorts: gather from T, sort on chip, write to X.  The
    // size classes are independent: their kernels run concurrently on side streams.
    SideStreams& ss = side_streams();
    // profiling: concurrent classes overlap, so the role is timed as one span on
    // the caller's stream (fork to join); serial classes are timed per launch
    std::optional<ProfScope> span;
    if (g_concurrent_classes) span.emplace("bucketsort", st);
    // allocated on st before the fork, released on st after the join
    uint32_t* splits = merge ? (uint32_t*)ar.alloc(uint64_t(po.mcap) * 4) : nullptr;
    ForkJoin fj(st, ss);
    auto launch_class = [&](int c, uint32_t li, cudaStream_t cs) {
      const uint32_t* lst = po.list + uint64_t(li) * po.cap_per_list;
      if (cls_cl[c] > kBinClusterTag) {
        launch_bincluster(cls_cl[c] - kBinClusterTag, cs, lst, po.count + li, recs, dTiles, T, X, pout, ppre,
                          po.list + uint64_t(po.ncls + 1) * po.cap_per_list, po.count + po.ncls + 1,
                          (uint32_t)buck_tot);
        return;
      }
      if (cls_cl[c]) {
        launch_cluster(cls_cl[c], cs, lst, po.count + li, recs, dTiles, T, X, pout, ppre, (uint32_t)buck_tot);
        return;
      }
      with_tile_lat<SK>(small_level && g_small_classes, po.cls_tile[c], [&](auto nt, auto v) {
        constexpr int NT = decltype(nt)::value, V = decltype(v)::value;
        using BS = BlockSort<SK, NT, V>;
        constexpr size_t base = BS::SMEM_BYTES + (PAIRS ? size_t(BS::TILE) * 4 : 0) + (3 * NT + 64) * 4;
        with_bin<BIN && base + bin_smem<K, NT, V, PAIRS, BIN>() <= kMaxSmem>([&](auto bin) {
        constexpr bool UB = decltype(bin)::value;
        const size_t smem = base + bin_smem<K, NT, V, PAIRS, UB>();
        auto f = k_bucketsort<K, NT, V, PAIRS, UB>;
        const int grid = wave_grid(f, NT, smem);
        std::optional<ProfScope> ps;
        if (!g_concurrent_classes) ps.emplace("bucketsort", cs);
        f<<<(uint32_t)std::min<uint64_t>(grid, po.cap_per_list), NT, smem, cs>>>(
            recs, dTiles, lst, po.count + li, kb[T], kb[X], PAIRS ? vb[T] : nullptr, PAIRS ? vb[X] : nullptr, pout,
            ppre, kb[2], PAIRS ? vb[2] : nullptr, po.units);
        check_launch("k_bucketsort");
        });
      });
    };
    auto launch_split = [&](cudaStream_t cs) {  // value-split items (k_bucketsplit)
      if constexpr (!PAIRS) {
        if (!po.split_max) return;
        with_split_tile<SK>(stile, [&](auto nt, auto v) {
          constexpr int NT = decltype(nt)::value, V = decltype(v)::value;
          using BS = BlockSort<SK, NT, V>;
          constexpr size_t base = BS::SMEM_BYTES + (3 * NT + 64) * 4;
          with_bin<BIN && base + bin_smem<K, NT, V, false, BIN>() <= kMaxSmem>([&](auto bin) {
            constexpr bool UB = decltype(bin)::value;
            const size_t smem = base + bin_smem<K, NT, V, false, UB>();
            auto f = k_bucketsplit<K, NT, V, UB>;
            const int grid = wave_grid(f, NT, smem);
            std::optional<ProfScope> ps;
            if (!g_concurrent_classes) ps.emplace("bucketsort", cs);
            f<<<(uint32_t)std::min<uint64_t>(grid, po.cap_per_list), NT, smem, cs>>>(
                dL, piv, recs, dTiles, po.list + uint64_t(po.split_list) * po.cap_per_list, po.count + po.split_list,
                kb[T], kb[X], pout, ppre);
            check_launch("k_bucketsplit");
          });
        });
      }
    };
    // a bucket is no longer than its segment: passes that no bucket of this level can
    // need are not launched (small levels: each launch is latency on the critical path)
    uint32_t npasses = 0;
    while (npasses < (uint32_t)kMaxPasses && (uint64_t(po.max_tile) << npasses) < longest_seg) npasses++;
    auto launch_merges = [&](cudaStream_t ms) {  // merge passes of the multi-CTA base case (X <-> U)
      using MC = MergeCfg<K, PAIRS>;
      using BS = BlockSort<K, MC::NT, MC::VM>;
      const size_t smem = BS::SMEM_BYTES + (PAIRS ? size_t(BS::TILE) * 4 : 0);
      auto f = k_merge_pass<K, PAIRS, MC::NT, MC::VM>;
      const int grid = wave_grid(f, MC::NT, smem);
      for (uint32_t p = 0; p < npasses; p++) {
        ProfScope ps("merge", ms);
        const MTile* items = po.mlist + uint64_t(p) * po.mcap;
        k_merge_split<K><<<2 * num_sms(), 256, 0, ms>>>(recs, items, po.mcount + p, p, po.mtile, kb[X], kb[2], splits);
        check_launch("k_merge_split");
        f<<<grid, MC::NT, smem, ms>>>(recs, items, po.mcount + p, p, kb[X], kb[2], PAIRS ? vb[X] : nullptr,
                                      PAIRS ? vb[2] : nullptr, splits);
        check_launch("k_merge_pass");
      }
    };

    // (the chunk lists are filled only for merge-sorted buckets)
    if (!g_concurrent_classes) {
      if (merge)
        for (int c = (int)po.ncls - 1; c >= 0; c--) launch_class(c, po.ncls + 3 + c, st);
      launch_split(st);
      for (int c = (int)po.ncls - 1; c >= 0; c--) launch_class(c, c, st);
      if (merge) launch_merges(st);
    } else {
      // streams 0-1: the chunks of merge-sorted buckets, then (stream 0) the merge
      // passes; streams 2-3: whole buckets and units, which the merges overlap
      int rc = 0, rw = 0;
      launch_split(ss.s[1]);
      if (merge)
        for (int c = (int)po.ncls - 1; c >= 0; c--) launch_class(c, po.ncls + 3 + c, ss.s[rc++ % 2]);
      // (without chunk lists -- recursion mode, the captured small levels -- the whole
      // classes take all four streams)
      for (int c = (int)po.ncls - 1; c >= 0; c--) launch_class(c, c, merge ? ss.s[2 + rw++ % 2] : ss.s[rw++ % 4]);
      if (merge) {
        stream_wait(ss.s[0], ss.s[1]);
        launch_merges(ss.s[0]);
      }
    }
    fj.join();
    span.reset();
    if (splits) ar.release(splits);
    lt.hcnt = (uint32_t*)ar.pinned((po.ncls + 3) * 4);
    lt.hinfo = lt.hcnt + po.ncls + 2;
    {  // single-value buckets (copied) and oversize buckets (made contiguous),
       // in units of kGatherKeys keys so that huge buckets are copied by many CTAs
      ProfScope ps("gather", st);
      const uint64_t ucap = buck_tot + level_keys / kGatherKeys + 16;
      uint2* units = (uint2*)ar.alloc(ucap * sizeof(uint2));
      uint32_t* nun = (uint32_t*)ar.alloc(16);
      // both lists (ncls: single-value, ncls + 1: oversize) in one pass
      const uint32_t* lst = po.list + uint64_t(po.ncls) * po.cap_per_list;
      // (with the level's read-back: class counts (the oversize list's length) and the round)
      k_gather_units<<<1, 1024, 0, st>>>(recs, lst, po.count + po.ncls, 2, po.cap_per_list, units, nun, po.count,
                                         po.ncls + 2, info, lt.hcnt);
      check_launch("k_gather_units");
      k_bucket_gather_units<K, 256><<<4 * num_sms(), 256, 0, st>>>(
          recs, dTiles, lst, po.cap_per_list, units, nun, kb[T], kb[X], PAIRS ? vb[T] : nullptr,
          PAIRS ? vb[X] : nullptr, pout, ppre);
      check_launch("k_bucket_gather_units");
      ar.release(nun);
      ar.release(units);
    }
    htrace("level: bucket sorts launched");
    // 7. the read-back (finish_level) was written by k_gather_units
    lt.ncls = po.ncls;
    lt.cap_per_list = po.cap_per_list;
    lt.list = po.list;
    lt.recs = recs;
    lt.buck_tot = buck_tot;
    lt.top_m = L[0].k;
    lt.depth = depth;
    lt.rel = {(void*)po.units, (void*)po.nunits, (void*)segmat, (void*)pout, (void*)ppre, (void*)recs,
              (void*)po.list, (void*)po.mlist, (void*)piv, (void*)flags, (void*)p0s, (void*)info,
              (void*)fix, (void*)segmin};
    return true;
  }
};

// ------------------------------------------------------------------ ABI helpers
inline int fail(const Error& e) {
  g_errmsg = e.what();
  return e.code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  g_stats = sq_stats{};
  try {
    fn();
    prof_collect();
    return SQ_OK;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_errmsg = e.what();
    return SQ_ERR_CUDA;
  }
}

inline void need(bool cond, const char* msg) {
  if (!cond) throw Error(SQ_ERR_INVALID_ARGUMENT, msg);
}

inline bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// ------------------------------------------------------------------ graph replay of small levels
// A one-level sort of a small array is bound by the host: the level's ~40 launches,
// events and stream waits cost ~250 us of API time while its kernels run for a few
// tens of microseconds.  A call that repeats an earlier one's (device, pointers, n,
// seed, knobs) replays the level as one CUDA graph: the first call runs normally
// and records the level's scratch and staging needs, the second captures the
// level's launches (on a library stream, over entry-owned scratch: a bump Arena)
// and instantiates the graph, and every later call launches it and does the
// level's read-back (and any oversize recursion, with ordinary scratch) as usual.
// Captured levels put buckets beyond one CTA into the next level (mode 0; rare at
// these sizes) instead of the merge passes.  SQ_GRAPH_MAX_N (default 2^22; 0 = off)
// bounds n; at most kGraphEntries levels are cached per engine instantiation.
// (g_graph_max_n is defined with the other knobs above)
constexpr int kGraphEntries = 4;
// every instantiation's clear(), for sq_trim_memory
inline std::mutex g_graph_reg_mu;
inline std::vector<void (*)()> g_graph_clearers;
inline void graph_register(void (*f)()) {
  std::lock_guard<std::mutex> g(g_graph_reg_mu);
  if (std::find(g_graph_clearers.begin(), g_graph_clearers.end(), f) == g_graph_clearers.end())
    g_graph_clearers.push_back(f);
}
inline void graph_clear_all() {
  std::vector<void (*)()> fs;
  {
    std::lock_guard<std::mutex> g(g_graph_reg_mu);
    fs = g_graph_clearers;
  }
  for (auto f : fs) f();
}

template <typename K, bool PAIRS, bool BIN>
struct GraphCache {
  using E = Engine<K, PAIRS, BIN>;
  struct Entry {
    int dev = -1;
    const void* keys = nullptr;
    const void* vals = nullptr;
    size_t n = 0;
    uint64_t seed = 0, knobs = 0, last = 0;
    size_t dev_need = 0, pin_need = 0;
    char* dmem = nullptr;
    char* hmem = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool busy = false;
    uint32_t launches = 0;
    typename E::LevelTail tail;
    ~Entry() {
      if (exec) cudaGraphExecDestroy(exec);
      if (dmem) cudaFree(dmem);
      if (hmem) cudaFreeHost(hmem);
    }
  };
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::unique_ptr<Entry>>& entries() {
    static std::vector<std::unique_ptr<Entry>> v;
    return v;
  }
  static uint64_t knobs() {
    return uint64_t(g_max_tile) ^ (uint64_t(g_unit_max) << 20) ^ (uint64_t(g_concurrent_classes) << 52) ^
           (uint64_t(g_big_mode) << 56) ^ (uint64_t(g_one_cap) << 1);
  }
  static std::vector<Seg> top(size_t n, uint64_t seed) { return {{0, (uint32_t)n, root_key(seed)}}; }

  // true: sorted here; false: the caller runs the ordinary path
  static bool run(K* keys, uint32_t* vals, size_t n, uint64_t seed, cudaStream_t st) {
    static const bool reg = (graph_register(&clear), true);
    (void)reg;
    const int dev = cur_device();
    const uint64_t kn = knobs();
    static uint64_t clock = 0;
    std::unique_lock<std::mutex> lk(mu());
    auto& v = entries();
    Entry* e = nullptr;
    for (auto& p : v)
      if (p->dev == dev && p->keys == keys && p->vals == vals && p->n == n && p->seed == seed && p->knobs == kn)
        e = p.get();
    if (!e) {  // first call: an ordinary run that records the level's needs
      lk.unlock();
      Arena ar(st);
      E eng(st, ar, keys, vals, n);
      eng.big_mode = 0;
      typename E::LevelTail lt;
      eng.launch_level(top(n, seed), 0, 0, nullptr, lt);
      const size_t dn = ar.dev_bytes, pn = ar.pin_bytes;
      eng.finish_level(lt, 0);
      lk.lock();
      if (v.size() >= (size_t)kGraphEntries) {  // evict the least recently used idle entry
        auto it = std::min_element(v.begin(), v.end(), [](auto& a, auto& b) {
          return (a->busy ? UINT64_MAX : a->last) < (b->busy ? UINT64_MAX : b->last);
        });
        if ((*it)->busy) return true;
        { int cd = cur_device(); cudaSetDevice((*it)->dev); it->reset(); cudaSetDevice(cd); }
        v.erase(it);
      }
      auto ne = std::make_unique<Entry>();
      ne->dev = dev;
      ne->keys = keys;
      ne->vals = vals;
      ne->n = n;
      ne->seed = seed;
      ne->knobs = kn;
      ne->dev_need = dn;
      ne->pin_need = pn;
      ne->last = ++clock;
      v.push_back(std::move(ne));
      return true;
    }
    if (e->busy) return false;  // another thread replays it: take the ordinary path
    e->busy = true;
    e->last = ++clock;
    lk.unlock();
    struct Release {
      Entry* e;
      ~Release() {
        std::lock_guard<std::mutex> g(mu());
        e->busy = false;
      }
    } rel{e};
    if (!e->exec) capture(e, keys, vals, n, seed);
    SQ_CUDA(cudaGraphLaunch(e->exec, st));
    g_stats.levels++;
    g_stats.kernel_launches += e->launches;
    Arena ar(st);
    E eng(st, ar, keys, vals, n);
    typename E::LevelTail lt = e->tail;
    eng.finish_level(lt, 0);
    return true;
  }

  static void capture(Entry* e, K* keys, uint32_t* vals, size_t n, uint64_t seed) {
    SQ_CUDA(cudaMalloc((void**)&e->dmem, e->dev_need));
    SQ_CUDA(cudaMallocHost((void**)&e->hmem, e->pin_need));
    // captured on a library stream of its own (the caller's may be the legacy stream),
    // one per host thread and device, destroyed when the thread exits
    struct CapStreams {
      std::map<int, cudaStream_t> s;
      ~CapStreams() {
        for (auto& kv : s) {
          cudaSetDevice(kv.first);
          cudaStreamDestroy(kv.second);
        }
      }
    };
    static thread_local CapStreams cap_stream;
    cudaStream_t& cs = cap_stream.s[e->dev];
    if (!cs) SQ_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SQ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    typename E::LevelTail lt;
    const uint64_t l0 = g_stats.kernel_launches, lv0 = g_stats.levels;
    cudaGraph_t g = nullptr;
    try {
      Arena ar(cs, e->dmem, e->dev_need, e->hmem, e->pin_need);
      E eng(cs, ar, keys, vals, n);
      eng.big_mode = 0;
      eng.launch_level(top(n, seed), 0, 0, nullptr, lt);
    } catch (...) {
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    SQ_CUDA(cudaStreamEndCapture(cs, &g));
    const cudaError_t r = cudaGraphInstantiate(&e->exec, g, 0);
    cudaGraphDestroy(g);
    SQ_CUDA(r);
    e->launches = uint32_t(g_stats.kernel_launches - l0);
    g_stats.kernel_launches = l0;  // counted again when the graph is launched
    g_stats.levels = lv0;
    lt.rel.clear();  // bump scratch: nothing to release
    e->tail = lt;
  }

  static void clear() {
    std::lock_guard<std::mutex> g(mu());
    auto& v = entries();
    const int cd = cur_device();
    for (auto it = v.begin(); it != v.end();) {
      if ((*it)->busy) { ++it; continue; }
      cudaSetDevice((*it)->dev);
      it = v.erase(it);
    }
    cudaSetDevice(cd);
  }
};

template <typename K, bool PAIRS, bool BIN>
void sort_engine(K* keys, uint32_t* vals, size_t n, uint64_t seed, cudaStream_t st) {
  // (levels with the default knobs only: a forced tile or big-bucket mode runs as asked)
  if (n <= g_graph_max_n && !g_prof.load() && n > key_max_tile<sortkey_t<K, PAIRS>>() && !g_max_tile &&
      g_big_mode == 1 && GraphCache<K, PAIRS, BIN>::run(keys, vals, n, seed, st))
    return;
  Arena ar(st);
  Engine<K, PAIRS, BIN> eng(st, ar, keys, vals, n);
  std::vector<Seg> top = {{0, (uint32_t)n, root_key(seed)}};
  eng.sort_batch(top, 0, 0, 0, "smallsort");
  SQ_CUDA(cudaGetLastError());
}

template <typename K, bool BIN>
void debug_level_engine(const K* src, K* dst, size_t n, uint64_t seed, K* pivots_out, uint32_t* bucend_out,
                        uint32_t* info_out, cudaStream_t st) {
  Arena ar(st);
  K* work = (K*)ar.alloc(n * sizeof(K));
  SQ_CUDA(cudaMemcpyAsync(work, src, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
  Engine<K, false, BIN> eng(st, ar, work, nullptr, n);
  DebugOut dbg{dst, pivots_out, bucend_out, info_out};
  std::vector<Seg> top = {{0, (uint32_t)n, root_key(seed)}};
  eng.run_level(top, 0, 0, &dbg);
  SQ_CUDA(cudaStreamSynchronize(st));
}

// The engine is compiled once per (key type, pairs, base case) in its own
// translation unit (inst_*.cu, built in parallel); every other unit sees only
// these declarations.
#define SQ_ENGINE_INSTANCES(X)                                                                        \
  X template void sort_engine<uint32_t, false, true>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint32_t, false, false>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint64_t, false, false>(uint64_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint64_t, false, true>(uint64_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint32_t, true, false>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint32_t, true, true>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void sort_engine<uint64_t, true, false>(uint64_t*, uint32_t*, size_t, uint64_t, cudaStream_t); \
  X template void debug_level_engine<uint32_t, true>(const uint32_t*, uint32_t*, size_t, uint64_t, uint32_t*,   \
                                                     uint32_t*, uint32_t*, cudaStream_t);                     \
  X template void debug_level_engine<uint32_t, false>(const uint32_t*, uint32_t*, size_t, uint64_t, uint32_t*,  \
                                                      uint32_t*, uint32_t*, cudaStream_t);                    \
  X template void debug_level_engine<uint64_t, false>(const uint64_t*, uint64_t*, size_t, uint64_t, uint64_t*,  \
                                                      uint32_t*, uint32_t*, cudaStream_t);
SQ_ENGINE_INSTANCES(extern)

// Sort on the device with the selected base case (sq_set_base_case).
template <typename K, bool PAIRS>
void sort_device(K* keys, uint32_t* vals, size_t n, uint64_t seed, cudaStream_t st) {
  if constexpr (sizeof(sortkey_t<K, PAIRS>) <= 8) {
    if (g_base_case) return sort_engine<K, PAIRS, true>(keys, vals, n, seed, st);
  }
  sort_engine<K, PAIRS, false>(keys, vals, n, seed, st);
}

inline void debug_level_u32(const uint32_t* src, uint32_t* dst, size_t n, uint64_t seed, uint32_t* pivots_out,
                            uint32_t* bucend_out, uint32_t* info_out, cudaStream_t st) {
  if (g_base_case) debug_level_engine<uint32_t, true>(src, dst, n, seed, pivots_out, bucend_out, info_out, st);
  else debug_level_engine<uint32_t, false>(src, dst, n, seed, pivots_out, bucend_out, info_out, st);
}

template <typename K, bool PAIRS>
int sort_entry(K* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream, bool host) {
  return guarded([&] {
    if (n <= 1) return;
    need(keys != nullptr, "keys is NULL");
    if (PAIRS) {
      need(vals != nullptr, "vals is NULL");
      need(!overlap(keys, n * sizeof(K), vals, n * 4), "keys and vals overlap");
    }
    need(n <= (sizeof(K) == 4 ? (size_t(1) << 30) : (size_t(1) << 28)), "n exceeds the supported maximum");
    check_device();
    cudaStream_t st = (cudaStream_t)stream;
    if (!host) {
      sort_device<K, PAIRS>(keys, vals, n, seed, st);
      SQ_CUDA(cudaStreamSynchronize(st));
      return;
    }
    Arena ar(st);
    K* dk = (K*)ar.alloc(n * sizeof(K));
    uint32_t* dv = PAIRS ? (uint32_t*)ar.alloc(n * 4) : nullptr;
    SQ_CUDA(cudaMemcpyAsync(dk, keys, n * sizeof(K), cudaMemcpyHostToDevice, st));
    if (PAIRS) SQ_CUDA(cudaMemcpyAsync(dv, vals, n * 4, cudaMemcpyHostToDevice, st));
    sort_device<K, PAIRS>(dk, dv, n, seed, st);
    SQ_CUDA(cudaMemcpyAsync(keys, dk, n * sizeof(K), cudaMemcpyDeviceToHost, st));
    if (PAIRS) SQ_CUDA(cudaMemcpyAsync(vals, dv, n * 4, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaStreamSynchronize(st));
  });
}

// Signed and floating-point keys: an order-preserving bijection
// onto unsigned keys of the same width, applied in place before the unsigned sort
// and inverted after it (reading L25).  Signed: flip the sign bit.
// IEEE-754 binary32/64: flip every bit of a negative value, only the sign bit of a
// non-negative one -- the totalOrder of IEEE 754-2008 5.10 (-NaN < -inf < ... < -0
// < +0 < ... < +inf < +NaN).
template <typename U>
__global__ void k_key_map(U* __restrict__ k, size_t n, int kind, bool inverse) {
  constexpr U SIGN = U(1) << (sizeof(U) * 8 - 1);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const U x = k[i];
    U y;
    if (kind == 0) y = x ^ SIGN;                                    // two's complement
    else if (!inverse) y = (x & SIGN) ? U(~x) : U(x | SIGN);         // float -> ordered
    else y = (x & SIGN) ? U(x ^ SIGN) : U(~x);                      // ordered -> float
    k[i] = y;
  }
}

template <typename U>
int mapped_entry(U* keys, size_t n, uint64_t seed, void* stream, int kind) {
  return guarded([&] {
    if (n <= 1) return;
    need(keys != nullptr, "keys is NULL");
    need(n <= (sizeof(U) == 4 ? (size_t(1) << 30) : (size_t(1) << 28)), "n exceeds the supported maximum");
    check_device();
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t g = (uint32_t)std::min<size_t>((n + 1023) / 1024, size_t(num_sms()) * 8);
    k_key_map<U><<<g, 256, 0, st>>>(keys, n, kind, false);
    check_launch("k_key_map");
    sort_device<U, false>(keys, nullptr, n, seed, st);
    k_key_map<U><<<g, 256, 0, st>>>(keys, n, kind, true);
    check_launch("k_key_map");
    SQ_CUDA(cudaStreamSynchronize(st));
  });
}

// Pipelined batch of host sorts (sq_sort_*_host_batch): item i's sort on `st`
// overlaps the H2D copy of item i+1 and the D2H copy of item i-1, each on a
// library-owned non-blocking copy stream.  Three device buffers rotate, so a
// buffer's copy-in -> sort -> copy-out cycle (~2 copies + 1 sort) spans three
// items and the steady state is bound by the copies alone.
template <typename K>
int batch_entry(const K* const* in, K* const* out, size_t n, size_t count, uint64_t seed, void* stream) {
  struct Res {
    cudaStream_t st = nullptr, cs[2] = {nullptr, nullptr};
    cudaEvent_t ev[10] = {};
    K* buf[3] = {nullptr, nullptr, nullptr};
    ~Res() {
      for (auto s : cs)
        if (s) cudaStreamSynchronize(s);
      cudaStreamSynchronize(st);
      for (auto b : buf)  // back to the pool (kept, release threshold = max)
        if (b) cudaFreeAsync(b, st);
      cudaStreamSynchronize(st);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
      for (auto s : cs)
        if (s) cudaStreamDestroy(s);
    }
  };
  return guarded([&] {
    if (count == 0) return;
    need(in != nullptr && out != nullptr, "in/out is NULL");
    need(n <= (sizeof(K) == 4 ? (size_t(1) << 30) : (size_t(1) << 28)), "n exceeds the supported maximum");
    const size_t bytes = n * sizeof(K);
    for (size_t i = 0; i < count; ++i) {
      need(in[i] != nullptr && out[i] != nullptr, "in[i]/out[i] is NULL");
      for (size_t j = i + 1; j < count && count <= 4096; ++j)
        need(!overlap(out[i], bytes, in[j], bytes), "out[i] overlaps in[j] with j > i");
    }
    if (n <= 1) {
      for (size_t i = 0; i < count; ++i)
        if (n == 1 && out[i] != in[i]) out[i][0] = in[i][0];
      return;
    }
    check_device();
    cudaStream_t st = (cudaStream_t)stream;
    Res r;
    r.st = st;
    for (auto& s : r.cs) SQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& e : r.ev) SQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int b = 0; b < int(std::min<size_t>(count, 3)); b++) SQ_CUDA(cudaMallocFromPoolAsync((void**)&r.buf[b], bytes, lib_pool(), st));
    cudaStream_t h2d = r.cs[0], d2h = r.cs[1];
    SQ_CUDA(cudaEventRecord(r.ev[9], st));  // the buffers exist
    SQ_CUDA(cudaStreamWaitEvent(h2d, r.ev[9], 0));
    cudaEvent_t* in_done = r.ev;        // [3]: buffer b holds item i's input
    cudaEvent_t* sorted = r.ev + 3;     // [3]: item in buffer b is sorted
    cudaEvent_t* out_done = r.ev + 6;   // [3]: buffer b has been copied out
    auto copy_in = [&](size_t i) {
      const int b = int(i % 3);
      if (i >= 3) SQ_CUDA(cudaStreamWaitEvent(h2d, out_done[b], 0));
      SQ_CUDA(cudaMemcpyAsync(r.buf[b], in[i], bytes, cudaMemcpyHostToDevice, h2d));
      SQ_CUDA(cudaEventRecord(in_done[b], h2d));
    };
    copy_in(0);
    for (size_t i = 0; i < count; ++i) {
      const int b = int(i % 3);
      if (i + 1 < count) copy_in(i + 1);  // enqueued before the sort's host waits
      SQ_CUDA(cudaStreamWaitEvent(st, in_done[b], 0));
      sort_device<K, false>(r.buf[b], nullptr, n, seed, st);
      SQ_CUDA(cudaEventRecord(sorted[b], st));
      SQ_CUDA(cudaStreamWaitEvent(d2h, sorted[b], 0));
      SQ_CUDA(cudaMemcpyAsync(out[i], r.buf[b], bytes, cudaMemcpyDeviceToHost, d2h));
      SQ_CUDA(cudaEventRecord(out_done[b], d2h));
    }
    SQ_CUDA(cudaStreamSynchronize(d2h));
    SQ_CUDA(cudaStreamSynchronize(h2d));
    SQ_CUDA(cudaStreamSynchronize(st));
  });
}

}  // namespace sq
