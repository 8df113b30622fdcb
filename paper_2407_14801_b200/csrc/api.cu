// api.cu -- host level scheduler and the C ABI of libsquaresort.so.
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
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/squaresort.h"
#include "level.cuh"

namespace sq {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
static thread_local std::string g_errmsg;
static thread_local sq_stats g_stats;

#define SQ_CUDA(call)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      if (e_ == cudaErrorMemoryAllocation) throw Error(SQ_ERR_OUT_OF_MEMORY, cudaGetErrorString(e_)); \
      throw Error(SQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    }                                                                                        \
  } while (0)

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(SQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_stats.kernel_launches++;
}

// ------------------------------------------------------------------ per-kernel timing
// When enabled (sq_profile), every launch is bracketed by CUDA events on its
// stream; elapsed times accumulate per kernel role after the call's final sync.
struct ProfEntry {
  const char* name;
  cudaEvent_t a, b;
};
static std::atomic<bool> g_prof{false};
static thread_local std::vector<ProfEntry> g_prof_pending;
static thread_local std::vector<cudaEvent_t> g_event_pool;
static std::mutex g_prof_mu;
static std::map<std::string, std::pair<uint64_t, double>> g_prof_acc;
static thread_local const char* g_role = "blocksort";

static cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  SQ_CUDA(cudaEventCreate(&e));
  return e;
}

struct ProfScope {
  cudaStream_t st;
  const char* name;
  cudaEvent_t a = nullptr;
  ProfScope(const char* n, cudaStream_t s) : st(s), name(n) {
    if (g_prof.load()) {
      a = pool_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = pool_event();
      cudaEventRecord(b, st);
      g_prof_pending.push_back({name, a, b});
    }
  }
};

static void prof_collect() {  // after a stream sync
  if (g_prof_pending.empty()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_prof_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) {
      auto& v = g_prof_acc[e.name];
      v.first++;
      v.second += ms;
    }
    g_event_pool.push_back(e.a);
    g_event_pool.push_back(e.b);
  }
  g_prof_pending.clear();
}

// ------------------------------------------------------------------ options
static uint32_t g_max_tile = 0;  // 0 = default

// ------------------------------------------------------------------ device check
static void check_device() {
  int dev = 0;
  SQ_CUDA(cudaGetDevice(&dev));
  static int checked[64] = {0};  // 1 ok, 2 bad
  if (dev >= 0 && dev < 64 && checked[dev] == 1) return;
  cudaDeviceProp p;
  SQ_CUDA(cudaGetDeviceProperties(&p, dev));
  const bool ok = p.major == 10 && p.minor == 0;
  if (dev >= 0 && dev < 64) checked[dev] = ok ? 1 : 2;
  if (!ok) throw Error(SQ_ERR_UNSUPPORTED_DEVICE, "device is sm_" + std::to_string(p.major) +
                                                      std::to_string(p.minor) + ", need sm_100 (B200)");
  // Keep freed scratch in the default pool between calls (stream-ordered reuse).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
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
};
static thread_local PinnedPool g_pinned;

struct Arena {
  cudaStream_t st;
  std::vector<void*> dev;
  bool used_host = false;
  explicit Arena(cudaStream_t s) : st(s) {}
  void* alloc(size_t bytes) {
    void* p = nullptr;
    SQ_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, st));
    dev.push_back(p);
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
    used_host = true;
    return g_pinned.get(bytes);
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* d = (T*)alloc(v.size() * sizeof(T));
    if (!v.empty()) {
      T* h = (T*)pinned(v.size() * sizeof(T));
      memcpy(h, v.data(), v.size() * sizeof(T));
      SQ_CUDA(cudaMemcpyAsync(d, h, v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
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

// ------------------------------------------------------------------ size classes
// Tiles (NT x V) for 32-bit keys and for 64-bit keys / pair composites.
static const uint32_t kTiles[] = {64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768};

template <typename K> constexpr uint32_t key_max_tile() { return sizeof(K) == 4 ? 32768u : 16384u; }

static uint32_t tile_for(uint32_t len) {
  for (uint32_t t : kTiles)
    if (len <= t) return t;
  return 0;
}

template <typename F>
static void set_smem(F f, size_t bytes) {
  SQ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <typename K, int NT, int V>
static void launch_bs(uint32_t nseg, const SegDesc* d, const K* src, K* dst, cudaStream_t st) {
  using BS = BlockSort<K, NT, V>;
  static bool init = false;
  if (!init) { set_smem(k_blocksort<K, NT, V>, BS::SMEM_BYTES); init = true; }
  ProfScope ps(g_role, st);
  k_blocksort<K, NT, V><<<nseg, NT, BS::SMEM_BYTES, st>>>(d, src, dst);
  check_launch("k_blocksort");
}

template <int NT, int V>
static void launch_bsp(uint32_t nseg, const SegDesc* d, const uint32_t* ks, const uint32_t* vs, uint32_t* kd,
                       uint32_t* vd, cudaStream_t st) {
  using BS = BlockSort<uint64_t, NT, V>;
  const size_t smem = BS::SMEM_BYTES + size_t(BS::TILE) * 4;
  static bool init = false;
  if (!init) { set_smem(k_blocksort_pairs<NT, V>, smem); init = true; }
  ProfScope ps(g_role, st);
  k_blocksort_pairs<NT, V><<<nseg, NT, smem, st>>>(d, ks, vs, kd, vd);
  check_launch("k_blocksort_pairs");
}

template <typename K, int NT, int V>
static void launch_sample(uint32_t ntask, const LevelSeg* segs, const TaskDesc* tasks, const K* data,
                          const K* segmin, K* cand, uint8_t* flags, uint32_t R, cudaStream_t st) {
  using BS = BlockSort<K, NT, V>;
  static bool init = false;
  if (!init) { set_smem(k_sample<K, NT, V>, BS::SMEM_BYTES); init = true; }
  ProfScope ps("sample", st);
  k_sample<K, NT, V><<<ntask, NT, BS::SMEM_BYTES, st>>>(segs, tasks, data, segmin, cand, flags, R);
  check_launch("k_sample");
}

// keys-only block sort dispatch
template <typename K>
static void blocksort_keys(uint32_t tile, uint32_t nseg, const SegDesc* d, const K* src, K* dst, cudaStream_t st) {
  if constexpr (sizeof(K) == 4) {
    switch (tile) {
      case 64: return launch_bs<K, 32, 2>(nseg, d, src, dst, st);
      case 128: return launch_bs<K, 32, 4>(nseg, d, src, dst, st);
      case 256: return launch_bs<K, 32, 8>(nseg, d, src, dst, st);
      case 512: return launch_bs<K, 64, 8>(nseg, d, src, dst, st);
      case 1024: return launch_bs<K, 128, 8>(nseg, d, src, dst, st);
      case 2048: return launch_bs<K, 128, 16>(nseg, d, src, dst, st);
      case 4096: return launch_bs<K, 256, 16>(nseg, d, src, dst, st);
      case 8192: return launch_bs<K, 512, 16>(nseg, d, src, dst, st);
      case 16384: return launch_bs<K, 512, 32>(nseg, d, src, dst, st);
      case 32768: return launch_bs<K, 1024, 32>(nseg, d, src, dst, st);
    }
  } else {
    switch (tile) {
      case 64: return launch_bs<K, 32, 2>(nseg, d, src, dst, st);
      case 128: return launch_bs<K, 32, 4>(nseg, d, src, dst, st);
      case 256: return launch_bs<K, 32, 8>(nseg, d, src, dst, st);
      case 512: return launch_bs<K, 64, 8>(nseg, d, src, dst, st);
      case 1024: return launch_bs<K, 128, 8>(nseg, d, src, dst, st);
      case 2048: return launch_bs<K, 256, 8>(nseg, d, src, dst, st);
      case 4096: return launch_bs<K, 256, 16>(nseg, d, src, dst, st);
      case 8192: return launch_bs<K, 512, 16>(nseg, d, src, dst, st);
      case 16384: return launch_bs<K, 1024, 16>(nseg, d, src, dst, st);
    }
  }
  throw Error(SQ_ERR_CUDA, "no block sort class for tile " + std::to_string(tile));
}

static void blocksort_pairs(uint32_t tile, uint32_t nseg, const SegDesc* d, const uint32_t* ks, const uint32_t* vs,
                            uint32_t* kd, uint32_t* vd, cudaStream_t st) {
  switch (tile) {
    case 64: return launch_bsp<32, 2>(nseg, d, ks, vs, kd, vd, st);
    case 128: return launch_bsp<32, 4>(nseg, d, ks, vs, kd, vd, st);
    case 256: return launch_bsp<32, 8>(nseg, d, ks, vs, kd, vd, st);
    case 512: return launch_bsp<64, 8>(nseg, d, ks, vs, kd, vd, st);
    case 1024: return launch_bsp<128, 8>(nseg, d, ks, vs, kd, vd, st);
    case 2048: return launch_bsp<256, 8>(nseg, d, ks, vs, kd, vd, st);
    case 4096: return launch_bsp<256, 16>(nseg, d, ks, vs, kd, vd, st);
    case 8192: return launch_bsp<512, 16>(nseg, d, ks, vs, kd, vd, st);
    case 16384: return launch_bsp<1024, 16>(nseg, d, ks, vs, kd, vd, st);
  }
  throw Error(SQ_ERR_CUDA, "no pair sort class for tile " + std::to_string(tile));
}

template <typename K>
static void sample_dispatch(uint32_t tile, uint32_t ntask, const LevelSeg* segs, const TaskDesc* tasks,
                            const K* data, const K* segmin, K* cand, uint8_t* flags, uint32_t R, cudaStream_t st) {
  if constexpr (sizeof(K) == 4) {
    switch (tile) {
      case 64: return launch_sample<K, 32, 2>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 128: return launch_sample<K, 32, 4>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 256: return launch_sample<K, 32, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 512: return launch_sample<K, 64, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 1024: return launch_sample<K, 128, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 2048: return launch_sample<K, 128, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 4096: return launch_sample<K, 256, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 8192: return launch_sample<K, 512, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 16384: return launch_sample<K, 512, 32>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 32768: return launch_sample<K, 1024, 32>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
    }
  } else {
    switch (tile) {
      case 64: return launch_sample<K, 32, 2>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 128: return launch_sample<K, 32, 4>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 256: return launch_sample<K, 32, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 512: return launch_sample<K, 64, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 1024: return launch_sample<K, 128, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 2048: return launch_sample<K, 256, 8>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 4096: return launch_sample<K, 256, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 8192: return launch_sample<K, 512, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
      case 16384: return launch_sample<K, 1024, 16>(ntask, segs, tasks, data, segmin, cand, flags, R, st);
    }
  }
  throw Error(SQ_ERR_CUDA, "no sampler class for tile " + std::to_string(tile));
}

// count kernel configuration per key type
template <typename K> struct CountCfg;
template <> struct CountCfg<uint32_t> { static constexpr int NT = 512, STAGE = 16384, KSMEM = 16384; };
template <> struct CountCfg<uint64_t> { static constexpr int NT = 512, STAGE = 8192, KSMEM = 16384; };

// transpose configuration per (key type, pairs)
template <typename K, bool PAIRS> struct TrCfg;
template <> struct TrCfg<uint32_t, false> { static constexpr int NT = 256, S = 4096, G = 256; };
template <> struct TrCfg<uint32_t, true> { static constexpr int NT = 256, S = 4096, G = 256; };
template <> struct TrCfg<uint64_t, false> { static constexpr int NT = 256, S = 4096, G = 256; };

// per-bucket single-value flag: bucket b >= 1 with P[b-1] == P[b]
template <typename K>
__global__ void k_bflags(const LevelSeg* __restrict__ segs, const K* __restrict__ piv, uint8_t* __restrict__ flag) {
  const LevelSeg s = segs[blockIdx.x];
  const K* P = piv + s.piv_base;
  for (uint32_t b = threadIdx.x; b < s.k; b += blockDim.x)
    flag[s.buck_base + b] = (b >= 1 && b + 1 < s.k && P[b - 1] == P[b]) ? 1 : 0;
}

// ------------------------------------------------------------------ the engine
struct Seg {
  uint32_t off, len;
  uint64_t node;
};

struct DebugOut {  // sq_debug_level_u32
  uint32_t* pivots;
  uint32_t* bucend;
  uint32_t* info;
};

template <typename K, bool PAIRS>
struct Engine {
  cudaStream_t st;
  Arena& ar;
  K* kb[2];
  uint32_t* vb[2];
  size_t n;
  uint32_t cap;

  Engine(cudaStream_t s, Arena& a, K* keys, uint32_t* vals, size_t n_) : st(s), ar(a), n(n_) {
    kb[0] = keys;
    kb[1] = nullptr;
    vb[0] = vals;
    vb[1] = nullptr;
    cap = key_max_tile<typename std::conditional<PAIRS, uint64_t, K>::type>();
    if (g_max_tile && g_max_tile < cap) cap = g_max_tile;
  }

  void ensure_scratch() {
    if (!kb[1]) kb[1] = (K*)ar.alloc(n * sizeof(K));
    if (PAIRS && !vb[1]) vb[1] = (uint32_t*)ar.alloc(n * sizeof(uint32_t));
  }

  void copy_ranges(const std::vector<SegDesc>& r, int src, int dst) {
    if (r.empty() || src == dst) return;
    const SegDesc* d = ar.upload(r);
    ProfScope ps("copy", st);
    k_copy_ranges<K><<<(uint32_t)r.size(), 256, 0, st>>>(d, kb[src], kb[dst], PAIRS ? vb[src] : nullptr,
                                                         PAIRS ? vb[dst] : nullptr);
    check_launch("k_copy_ranges");
  }

  void sort_batch(const std::vector<Seg>& segs, int src, int dst, int depth, const char* role) {
    if (depth > 48) throw Error(SQ_ERR_CUDA, "recursion too deep");
    std::map<uint32_t, std::vector<SegDesc>> cls;
    std::vector<Seg> big;
    for (const Seg& s : segs) {
      if (s.len == 0) continue;
      if (s.len > cap) big.push_back(s);
      else cls[tile_for(s.len)].push_back({s.off, s.len});
    }
    for (auto& kv : cls) {
      const SegDesc* d = ar.upload(kv.second);
      g_role = role;
      if constexpr (PAIRS)
        blocksort_pairs(kv.first, (uint32_t)kv.second.size(), d, kb[src], vb[src], kb[dst], vb[dst], st);
      else
        blocksort_keys<K>(kv.first, (uint32_t)kv.second.size(), d, kb[src], kb[dst], st);
    }
    if (!big.empty()) {
      uint64_t ok = 0;
      for (auto& b : big) ok += b.len;
      if (depth > 0) g_stats.oversize_keys += ok;
      run_level(big, src, dst, depth, nullptr);
    }
  }

  // One SquareSort level for a batch of segments living in buffer X; the
  // sorted result goes to buffer `dst`.  The SkewTranspose writes into the
  // other buffer T (each segment's range there is free).
  void run_level(const std::vector<Seg>& segs, int X, int dst, int depth, DebugOut* dbg) {
    ensure_scratch();
    g_stats.levels++;
    const int T = 1 - X;
    const uint32_t ns = (uint32_t)segs.size();
    const uint32_t R = ns == 1 ? kCap : (ns <= 16 ? 4 : 2);
    std::vector<LevelSeg> L(ns);
    std::vector<Seg> cols;
    std::vector<TaskDesc> ctasks, stasks, ttasks;
    uint64_t piv_tot = 0, buck_tot = 0, segmat_tot = 0, cand_tot = 0, totcols = 0;
    uint32_t maxnp = 0;
    for (uint32_t s = 0; s < ns; s++) totcols += ceil_sqrt(segs[s].len);
    const uint64_t cg = std::max<uint64_t>(1, (totcols + 295) / 296);
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
      cand_tot += uint64_t(R + 1) * np;
      for (uint32_t c = 0; c < m; c++) {
        const uint64_t a = uint64_t(c) * m;
        if (a < g.len) cols.push_back({uint32_t(g.off + a), uint32_t(std::min<uint64_t>(m, g.len - a)),
                                       child_key(g.node, 0, c)});
      }
      for (uint32_t j = 0; j < R; j++) stasks.push_back({s, j, 0});
      for (uint32_t c0 = 0; c0 < m; c0 += (uint32_t)cg) ctasks.push_back({s, c0, (uint32_t)std::min<uint64_t>(m, c0 + cg)});
      for (uint32_t bt = 0; bt < l.nbt; bt++) ttasks.push_back({s, bt, 0});
    }
    if (maxnp > key_max_tile<K>()) throw Error(SQ_ERR_INVALID_ARGUMENT, "pivot sample too large for one CTA");

    // 1. sort every column in place
    sort_batch(cols, X, X, depth + 1, "colsort");

    LevelSeg* dL = ar.upload(L);
    // 2. min(D) from the column heads
    K* segmin = (K*)ar.alloc(ns * sizeof(K));
    {
      ProfScope ps("colmin", st);
      k_colmin<K><<<ns, 256, 0, st>>>(dL, kb[X], segmin);
      check_launch("k_colmin");
    }
    // 3. pivots
    K* cand = (K*)ar.alloc(std::max<uint64_t>(cand_tot, 1) * sizeof(K));
    uint8_t* flags = (uint8_t*)ar.alloc(uint64_t(ns) * kCap);
    SQ_CUDA(cudaMemsetAsync(flags, 0, uint64_t(ns) * kCap, st));
    TaskDesc* dS = ar.upload(stasks);
    sample_dispatch<K>(std::max<uint32_t>(64, tile_for(std::max<uint32_t>(maxnp, 1))), (uint32_t)stasks.size(), dL, dS,
                       kb[X], segmin, cand, flags, R, st);
    K* piv = (K*)ar.alloc(std::max<uint64_t>(piv_tot, 1) * sizeof(K));
    uint32_t* info = (uint32_t*)ar.alloc(ns * sizeof(uint32_t));
    {
      ProfScope ps("select", st);
      k_select<K><<<ns, 256, 0, st>>>(dL, cand, flags, piv, info, R);
      check_launch("k_select");
    }
    ar.release(cand);
    // 4. bucket sizes and tile boundaries
    uint32_t* segmat = (uint32_t*)ar.alloc(std::max<uint64_t>(segmat_tot, 1) * sizeof(uint32_t));
    uint32_t* cnt = (uint32_t*)ar.alloc(buck_tot * sizeof(uint32_t));
    SQ_CUDA(cudaMemsetAsync(cnt, 0, buck_tot * sizeof(uint32_t), st));
    TaskDesc* dC = ar.upload(ctasks);
    {
      using CC = CountCfg<K>;
      const size_t smem = CC::STAGE * sizeof(K) + CC::KSMEM * 4;
      static bool init = false;
      if (!init) { set_smem(k_count<K, CC::NT, CC::STAGE, CC::KSMEM>, smem); init = true; }
      ProfScope ps("count", st);
      k_count<K, CC::NT, CC::STAGE, CC::KSMEM><<<(uint32_t)ctasks.size(), CC::NT, smem, st>>>(dL, dC, kb[X], piv,
                                                                                              segmat, cnt);
      check_launch("k_count");
    }
    uint8_t* bflag = (uint8_t*)ar.alloc(buck_tot);
    {
      ProfScope ps("bflags", st);
      k_bflags<K><<<ns, 256, 0, st>>>(dL, piv, bflag);
      check_launch("k_bflags");
    }
    // 5. read the sizes back and plan (one host sync per level)
    uint32_t* hcnt = (uint32_t*)ar.pinned(buck_tot * 4);
    uint8_t* hflag = (uint8_t*)ar.pinned(buck_tot);
    uint32_t* hinfo = (uint32_t*)ar.pinned(ns * 4);
    SQ_CUDA(cudaMemcpyAsync(hcnt, cnt, buck_tot * 4, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaMemcpyAsync(hflag, bflag, buck_tot, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaMemcpyAsync(hinfo, info, ns * 4, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaStreamSynchronize(st));
    g_stats.host_syncs++;
    SQ_CUDA(cudaGetLastError());
    if (depth == 0) {
      g_stats.top_round = hinfo[0] & 0x7fffffffu;
      g_stats.top_degenerate = hinfo[0] >> 31;
      g_stats.top_m = L[0].k;
    }
    std::vector<uint32_t> bstart(buck_tot);
    std::vector<Seg> buckets;
    std::vector<SegDesc> copies;
    for (uint32_t s = 0; s < ns; s++) {
      uint64_t pre = L[s].off;
      for (uint32_t b = 0; b < L[s].k; b++) {
        const uint64_t i = L[s].buck_base + b;
        bstart[i] = (uint32_t)pre;
        const uint32_t c = hcnt[i];
        if (c) {
          if (hflag[i]) copies.push_back({(uint32_t)pre, c});  // single-value bucket: no recursion
          else buckets.push_back({(uint32_t)pre, c, child_key(L[s].node, 1, b)});
        }
        pre += c;
      }
      if (pre != uint64_t(L[s].off) + L[s].len) throw Error(SQ_ERR_CUDA, "bucket sizes do not add up");
    }
    uint32_t* dstart = ar.upload(bstart);
    // 6. SkewTranspose X -> T
    {
      using TC = TrCfg<K, PAIRS>;
      using CF = TransposeCfg<K, PAIRS, TC::NT, TC::S, TC::G>;
      auto f = k_transpose<K, PAIRS, TC::NT, TC::S, TC::G>;
      static bool init = false;
      if (!init) { set_smem(f, CF::SMEM); init = true; }
      TaskDesc* dT = ar.upload(ttasks);
      ProfScope ps("transpose", st);
      f<<<(uint32_t)ttasks.size(), TC::NT, CF::SMEM, st>>>(dL, dT, kb[X], kb[T], PAIRS ? vb[X] : nullptr,
                                                           PAIRS ? vb[T] : nullptr, piv, segmat, dstart);
      check_launch("k_transpose");
    }
    if (dbg) {
      SQ_CUDA(cudaMemcpyAsync(dbg->pivots, piv, piv_tot * sizeof(K), cudaMemcpyDeviceToDevice, st));
      std::vector<uint32_t> be(buck_tot), inf = {hinfo[0] & 0x7fffffffu, hinfo[0] >> 31};
      for (uint64_t i = 0; i < buck_tot; i++) be[i] = bstart[i] + hcnt[i];
      uint32_t* dbe = ar.upload(be);
      uint32_t* dinf = ar.upload(inf);
      SQ_CUDA(cudaMemcpyAsync(dbg->bucend, dbe, buck_tot * 4, cudaMemcpyDeviceToDevice, st));
      SQ_CUDA(cudaMemcpyAsync(dbg->info, dinf, 8, cudaMemcpyDeviceToDevice, st));
      return;
    }
    for (void* p : {(void*)segmat, (void*)cnt, (void*)piv, (void*)segmin, (void*)flags, (void*)info, (void*)bflag})
      ar.release(p);
    // 7. buckets: single-value ones are copied, the rest sorted from T into dst
    copy_ranges(copies, T, dst);
    sort_batch(buckets, T, dst, depth + 1, "bucketsort");
  }
};

// ------------------------------------------------------------------ ABI helpers
static int fail(const Error& e) {
  g_errmsg = e.what();
  return e.code;
}

template <typename Fn>
static int guarded(Fn&& fn) {
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

static void need(bool cond, const char* msg) {
  if (!cond) throw Error(SQ_ERR_INVALID_ARGUMENT, msg);
}

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

template <typename K, bool PAIRS>
static void sort_device(K* keys, uint32_t* vals, size_t n, uint64_t seed, cudaStream_t st) {
  Arena ar(st);
  Engine<K, PAIRS> eng(st, ar, keys, vals, n);
  std::vector<Seg> top = {{0, (uint32_t)n, root_key(seed)}};
  eng.sort_batch(top, 0, 0, 0, "smallsort");
  SQ_CUDA(cudaGetLastError());
}

template <typename K, bool PAIRS>
static int sort_entry(K* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream, bool host) {
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

}  // namespace sq

using namespace sq;

extern "C" {

int sq_sort_u32(uint32_t* keys, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint32_t, false>(keys, nullptr, n, seed, stream, false);
}
int sq_sort_u64(uint64_t* keys, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint64_t, false>(keys, nullptr, n, seed, stream, false);
}
int sq_sort_pairs_u32_u32(uint32_t* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint32_t, true>(keys, vals, n, seed, stream, false);
}
int sq_sort_u32_host(uint32_t* keys, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint32_t, false>(keys, nullptr, n, seed, stream, true);
}
int sq_sort_u64_host(uint64_t* keys, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint64_t, false>(keys, nullptr, n, seed, stream, true);
}
int sq_sort_pairs_u32_u32_host(uint32_t* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint32_t, true>(keys, vals, n, seed, stream, true);
}

int sq_skew_transpose(const uint32_t* src, uint32_t* dst, size_t rows, size_t cols, const sq_skew_params* p,
                      void* stream) {
  return guarded([&] {
    need(p != nullptr, "params is NULL");
    need(p->k >= 1, "k must be >= 1");
    need(p->naive_threshold >= 2, "naive_threshold must be >= 2");
    need(rows == 0 || cols <= SIZE_MAX / rows, "rows*cols overflows");
    const size_t cap = rows * cols;
    const size_t n = p->n ? p->n : cap;
    need(n <= cap, "n > rows*cols");
    need(n < (size_t(1) << 32), "n must be < 2^32");
    need(p->k == 1 || p->pivots != nullptr, "pivots is NULL");
    need(p->buc_out != nullptr, "buc_out is NULL");
    need(cols <= 0xffffffffu && rows <= 0xffffffffu, "rows/cols too large");
    need(p->k - 1 <= 0xffffffffu, "k too large");
    if (n > 0) {
      need(src != nullptr && dst != nullptr, "src/dst is NULL");
      need(!overlap(src, n * 4, dst, n * 4), "src and dst overlap");
    }
    check_device();
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar(st);
    if (p->flags & SQ_FLAG_VALIDATE) {
      uint32_t* bad = (uint32_t*)ar.alloc(4);
      SQ_CUDA(cudaMemsetAsync(bad, 0, 4, st));
      if (n > 0 || p->k > 2) {
        k_validate<<<592, 256, 0, st>>>(src, std::max<size_t>(rows, 1), n, p->pivots, p->k - 1, bad);
        check_launch("k_validate");
      }
      uint32_t hb = 0;
      SQ_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
      SQ_CUDA(cudaStreamSynchronize(st));
      if (hb) throw Error(SQ_ERR_PRECONDITION, hb & 1 ? "a column is not sorted" : "pivots decrease");
    }
    const uint32_t k = p->k;
    const uint32_t nbt = (k + kTB - 1) / kTB;
    LevelSeg l{};
    l.off = 0;
    l.len = (uint32_t)n;
    l.rows = (uint32_t)rows;
    l.ncols = (uint32_t)cols;
    l.k = k;
    l.nbt = nbt;
    LevelSeg* dL = ar.upload(std::vector<LevelSeg>{l});
    // pivots: the user's array (k-1 entries); an empty list gets a dummy buffer
    const uint32_t* piv = p->pivots;
    if (k == 1) piv = (uint32_t*)ar.alloc(4);
    uint32_t* segmat = (uint32_t*)ar.alloc(std::max<uint64_t>(uint64_t(cols) * (nbt + 1), 1) * 4);
    uint32_t* cnt = (uint32_t*)ar.alloc(uint64_t(k) * 4);
    SQ_CUDA(cudaMemsetAsync(cnt, 0, uint64_t(k) * 4, st));
    std::vector<TaskDesc> ct, tt;
    const uint64_t cg = std::max<uint64_t>(1, (cols + 295) / 296);
    for (uint64_t c0 = 0; c0 < cols; c0 += cg) ct.push_back({0, (uint32_t)c0, (uint32_t)std::min<uint64_t>(cols, c0 + cg)});
    for (uint32_t bt = 0; bt < nbt; bt++) tt.push_back({0, bt, 0});
    if (!ct.empty()) {
      using CC = CountCfg<uint32_t>;
      const size_t smem = CC::STAGE * 4 + CC::KSMEM * 4;
      static bool init = false;
      if (!init) { set_smem(k_count<uint32_t, CC::NT, CC::STAGE, CC::KSMEM>, smem); init = true; }
      TaskDesc* dC = ar.upload(ct);
      ProfScope ps("count", st);
      k_count<uint32_t, CC::NT, CC::STAGE, CC::KSMEM><<<(uint32_t)ct.size(), CC::NT, smem, st>>>(dL, dC, src, piv,
                                                                                                 segmat, cnt);
      check_launch("k_count");
    }
    std::vector<uint32_t> hcnt(k), start(k);
    SQ_CUDA(cudaMemcpyAsync(hcnt.data(), cnt, uint64_t(k) * 4, cudaMemcpyDeviceToHost, st));
    if (p->buc_in) SQ_CUDA(cudaMemcpyAsync(start.data(), p->buc_in, uint64_t(k) * 4, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaStreamSynchronize(st));
    g_stats.host_syncs++;
    if (!p->buc_in) {
      uint64_t pre = 0;
      for (uint32_t b = 0; b < k; b++) {
        start[b] = (uint32_t)pre;
        pre += hcnt[b];
      }
    } else {
      for (uint32_t b = 0; b < k; b++)
        need(uint64_t(start[b]) + hcnt[b] <= n, "buc_in[j] + size_j exceeds n");
    }
    uint32_t* dstart = ar.upload(start);
    if (n > 0) {
      using TC = TrCfg<uint32_t, false>;
      using CF = TransposeCfg<uint32_t, false, TC::NT, TC::S, TC::G>;
      auto f = k_transpose<uint32_t, false, TC::NT, TC::S, TC::G>;
      static bool init = false;
      if (!init) { set_smem(f, CF::SMEM); init = true; }
      TaskDesc* dT = ar.upload(tt);
      ProfScope ps("transpose", st);
      f<<<(uint32_t)tt.size(), TC::NT, CF::SMEM, st>>>(dL, dT, src, dst, nullptr, nullptr, piv, segmat, dstart);
      check_launch("k_transpose");
    }
    std::vector<uint32_t> out(k);
    for (uint32_t b = 0; b < k; b++) out[b] = start[b] + hcnt[b];
    uint32_t* dout = ar.upload(out);
    SQ_CUDA(cudaMemcpyAsync(p->buc_out, dout, uint64_t(k) * 4, cudaMemcpyDeviceToDevice, st));
    SQ_CUDA(cudaStreamSynchronize(st));
  });
}

const char* sq_status_string(int s) {
  switch (s) {
    case SQ_OK: return "SQ_OK";
    case SQ_ERR_INVALID_ARGUMENT: return "SQ_ERR_INVALID_ARGUMENT";
    case SQ_ERR_OUT_OF_MEMORY: return "SQ_ERR_OUT_OF_MEMORY";
    case SQ_ERR_CUDA: return "SQ_ERR_CUDA";
    case SQ_ERR_PRECONDITION: return "SQ_ERR_PRECONDITION";
    case SQ_ERR_UNSUPPORTED_DEVICE: return "SQ_ERR_UNSUPPORTED_DEVICE";
  }
  return "unknown sq_status";
}

const char* sq_last_error_message(void) { return g_errmsg.c_str(); }

void sq_get_stats(sq_stats* out) {
  if (out) *out = g_stats;
}

int sq_profile(int enable) {
  g_prof.store(enable != 0);
  return SQ_OK;
}

int sq_profile_read(char* buf, size_t cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::string out = "{";
  bool first = true;
  for (auto& kv : g_prof_acc) {
    if (!first) out += ",";
    first = false;
    char tmp[256];
    snprintf(tmp, sizeof tmp, "\"%s\":[%llu,%.6f]", kv.first.c_str(), (unsigned long long)kv.second.first,
             kv.second.second);
    out += tmp;
  }
  out += "}";
  g_prof_acc.clear();
  if (!buf || cap == 0) return SQ_ERR_INVALID_ARGUMENT;
  snprintf(buf, cap, "%s", out.c_str());
  return out.size() < cap ? SQ_OK : SQ_ERR_INVALID_ARGUMENT;
}

int sq_set_max_tile(uint32_t t) {
  if (t == 0) {
    g_max_tile = 0;
    return SQ_OK;
  }
  if (t < 64 || t > 32768 || (t & (t - 1))) return SQ_ERR_INVALID_ARGUMENT;
  g_max_tile = t;
  return SQ_OK;
}

int sq_debug_level_u32(const uint32_t* src, uint32_t* dst, size_t n, uint64_t seed, uint32_t* pivots_out,
                       uint32_t* bucend_out, uint32_t* info_out, void* stream) {
  return guarded([&] {
    need(n >= 5 && n <= (size_t(1) << 30), "n must be in [5, 2^30]");
    need(src && dst && pivots_out && bucend_out && info_out, "NULL pointer");
    need(!overlap(src, n * 4, dst, n * 4), "src and dst overlap");
    check_device();
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar(st);
    uint32_t* work = (uint32_t*)ar.alloc(n * 4);
    SQ_CUDA(cudaMemcpyAsync(work, src, n * 4, cudaMemcpyDeviceToDevice, st));
    Engine<uint32_t, false> eng(st, ar, work, nullptr, n);
    eng.kb[1] = dst;
    DebugOut dbg{pivots_out, bucend_out, info_out};
    std::vector<Seg> top = {{0, (uint32_t)n, root_key(seed)}};
    eng.run_level(top, 0, 0, 0, &dbg);
    SQ_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
