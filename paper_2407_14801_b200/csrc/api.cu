// api.cu -- the C ABI of libsquaresort.so (include/squaresort.h).
//
// Each call validates its arguments (SQ_ERR_INVALID_ARGUMENT), checks the
// device (SQ_ERR_UNSUPPORTED_DEVICE) and runs the engine (engine.cuh, compiled
// per key type in inst_*.cu) or the standalone SkewTranspose (below).  No
// exception crosses the ABI.
#include "engine.cuh"


namespace sq {

// The standalone SkewTranspose (sq_skew_transpose / _u64): count -> cursors (device
// scan, or the caller's cursors checked on the device) -> transpose -> final cursors.
// The host blocks once, at the end (and once after the optional validation).
template <typename K>
void skew_entry(const K* src, K* dst, size_t rows, size_t cols, const K* pivots, uint32_t k, uint64_t pn,
                const uint32_t* buc_in, uint32_t* buc_out, uint32_t threshold, uint32_t flags, cudaStream_t st) {
  need(k >= 1, "k must be >= 1");
  need(threshold >= 2, "naive_threshold must be >= 2");
  need(rows == 0 || cols <= SIZE_MAX / rows, "rows*cols overflows");
  const size_t cap = rows * cols;
  const size_t n = pn ? pn : cap;
  need(n <= cap, "n > rows*cols");
  need(n < (size_t(1) << 32), "n must be < 2^32");
  need(k == 1 || pivots != nullptr, "pivots is NULL");
  need(buc_out != nullptr, "buc_out is NULL");
  need(cols <= 0xffffffffu && rows <= 0xffffffffu, "rows/cols too large");
  if (n > 0) {
    need(src != nullptr && dst != nullptr, "src/dst is NULL");
    need(!overlap(src, n * sizeof(K), dst, n * sizeof(K)), "src and dst overlap");
  }
  check_device();
  Arena ar(st);
  uint32_t* bad = (uint32_t*)ar.alloc(4);
  SQ_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  if (flags & SQ_FLAG_VALIDATE) {
    if (n > 0 || k > 2) {
      k_validate<K><<<592, 256, 0, st>>>(src, std::max<size_t>(rows, 1), n, pivots, k - 1, bad);
      check_launch("k_validate");
    }
    uint32_t hb = 0;
    SQ_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    SQ_CUDA(cudaStreamSynchronize(st));
    g_stats.host_syncs++;
    if (hb) throw Error(SQ_ERR_PRECONDITION, hb & 1 ? "a column is not sorted" : "pivots decrease");
  }
  const uint32_t nbt = (k + kTB - 1) / kTB;
  LevelSeg l{};
  l.off = 0;
  l.len = (uint32_t)n;
  l.rows = (uint32_t)rows;
  l.ncols = (uint32_t)cols;
  l.k = k;
  l.nbt = nbt;
  // pivots: the user's array (k-1 entries); an empty list gets a dummy buffer
  const K* piv = pivots;
  if (k == 1) piv = (const K*)ar.alloc(sizeof(K));
  uint32_t* segmat = (uint32_t*)ar.alloc(std::max<uint64_t>(uint64_t(cols) * (nbt + 1), 1) * 4);
  // column ranges of 64 columns: the count runs one CTA per range, the transpose one CTA
  // per (bucket tile, range), each range's cursors offset by the ranges before it
  std::vector<TaskDesc> ct, tt;
  const uint64_t cg = std::max<uint64_t>(64, (cols + 1023) / 1024);
  for (uint64_t c0 = 0; c0 < cols; c0 += cg) ct.push_back({0, (uint32_t)c0, (uint32_t)std::min<uint64_t>(cols, c0 + cg)});
  for (uint32_t bt = 0; bt < nbt; bt++) tt.push_back({0, bt, 0});
  const uint32_t nr = std::max<uint32_t>(1, (uint32_t)ct.size());
  uint32_t* cnt = (uint32_t*)ar.alloc(uint64_t(nr) * k * 4);  // (range, bucket) counts, then prefixes
  uint32_t* tot = (uint32_t*)ar.alloc(uint64_t(k) * 4);
  uint32_t* start = (uint32_t*)ar.alloc(uint64_t(k) * 4);
  SQ_CUDA(cudaMemsetAsync(cnt, 0, uint64_t(nr) * k * 4, st));
  if (ct.empty()) ct.push_back({0, 0, 0});
  const std::vector<void*> up = ar.upload_all({Arena::part(std::vector<LevelSeg>{l}), Arena::part(ct), Arena::part(tt)});
  const LevelSeg* dL = (const LevelSeg*)up[0];
  if (cols) {
    using CC = CountCfg<K>;
    const size_t smem = CC::STAGE * sizeof(K) + CC::KSMEM * 4;
    set_smem(k_count<K, CC::NT, CC::STAGE, CC::KSMEM>, smem);
    ProfScope ps("count", st);
    k_count<K, CC::NT, CC::STAGE, CC::KSMEM><<<nr, CC::NT, smem, st>>>(dL, (const TaskDesc*)up[1], src, piv, segmat,
                                                                     cnt);
    check_launch("k_count");
  }
  k_skew_range_prefix<<<std::max<uint32_t>(1, std::min<uint32_t>((k + 255) / 256, 1184)), 256, 0, st>>>(cnt, nr, k, tot);
  check_launch("k_skew_range_prefix");
  k_skew_cursors<<<1, 1024, 0, st>>>(tot, k, n, buc_in, start, bad);
  check_launch("k_skew_cursors");
  if (n > 0) {
    using TC = TrCfg<K, false>;
    using CF = TransposeCfg<K, false, TC::NT, TC::S, TC::G>;
    auto f = k_transpose<K, false, TC::NT, TC::S, TC::G>;
    set_smem(f, CF::SMEM);
    ProfScope ps("transpose", st);
    f<<<dim3((uint32_t)tt.size(), nr), TC::NT, CF::SMEM, st>>>(dL, (const TaskDesc*)up[2], src, dst, nullptr, nullptr,
                                                               piv, segmat, start, bad, (const TaskDesc*)up[1], cnt);
    check_launch("k_transpose");
  }
  k_skew_finish<<<std::max<uint32_t>(1, std::min<uint32_t>((k + 255) / 256, 1184)), 256, 0, st>>>(start, tot, k,
                                                                                                  buc_out);
  check_launch("k_skew_finish");
  uint32_t* hb = (uint32_t*)ar.pinned(4);
  xfer(hb, bad, 4, st);
  SQ_CUDA(cudaStreamSynchronize(st));
  g_stats.host_syncs++;
  if (*hb & 4) throw Error(SQ_ERR_INVALID_ARGUMENT, "buc_in[j] + size_j exceeds n");
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
int sq_sort_pairs_u64_u32(uint64_t* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint64_t, true>(keys, vals, n, seed, stream, false);
}
int sq_sort_pairs_u64_u32_host(uint64_t* keys, uint32_t* vals, size_t n, uint64_t seed, void* stream) {
  return sort_entry<uint64_t, true>(keys, vals, n, seed, stream, true);
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
int sq_sort_i32(int32_t* keys, size_t n, uint64_t seed, void* stream) {
  return mapped_entry<uint32_t>(reinterpret_cast<uint32_t*>(keys), n, seed, stream, 0);
}
int sq_sort_i64(int64_t* keys, size_t n, uint64_t seed, void* stream) {
  return mapped_entry<uint64_t>(reinterpret_cast<uint64_t*>(keys), n, seed, stream, 0);
}
int sq_sort_f32(float* keys, size_t n, uint64_t seed, void* stream) {
  return mapped_entry<uint32_t>(reinterpret_cast<uint32_t*>(keys), n, seed, stream, 1);
}
int sq_sort_f64(double* keys, size_t n, uint64_t seed, void* stream) {
  return mapped_entry<uint64_t>(reinterpret_cast<uint64_t*>(keys), n, seed, stream, 1);
}
int sq_sort_u32_host_batch(const uint32_t* const* in, uint32_t* const* out, size_t n, size_t count, uint64_t seed,
                           void* stream) {
  return batch_entry<uint32_t>(in, out, n, count, seed, stream);
}
int sq_sort_u64_host_batch(const uint64_t* const* in, uint64_t* const* out, size_t n, size_t count, uint64_t seed,
                           void* stream) {
  return batch_entry<uint64_t>(in, out, n, count, seed, stream);
}

int sq_skew_transpose(const uint32_t* src, uint32_t* dst, size_t rows, size_t cols, const sq_skew_params* p,
                      void* stream) {
  return guarded([&] {
    need(p != nullptr, "params is NULL");
    skew_entry<uint32_t>(src, dst, rows, cols, p->pivots, p->k, p->n, p->buc_in, p->buc_out, p->naive_threshold,
                         p->flags, (cudaStream_t)stream);
  });
}

int sq_skew_transpose_u64(const uint64_t* src, uint64_t* dst, size_t rows, size_t cols,
                          const sq_skew_params_u64* p, void* stream) {
  return guarded([&] {
    need(p != nullptr, "params is NULL");
    skew_entry<uint64_t>(src, dst, rows, cols, p->pivots, p->k, p->n, p->buc_in, p->buc_out, p->naive_threshold,
                         p->flags, (cudaStream_t)stream);
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

uint64_t sq_root_key(uint64_t seed) { return root_key(seed); }

int sq_draw_positions(uint64_t node, uint32_t rounds, uint32_t count, uint64_t n, uint64_t* out) {
  if (!out && rounds && count) return SQ_ERR_INVALID_ARGUMENT;
  if (n == 0 && rounds && count) return SQ_ERR_INVALID_ARGUMENT;
  for (uint32_t r = 0; r < rounds; r++)
    for (uint32_t i = 0; i < count; i++) out[uint64_t(r) * count + i] = draw_index_host(draw(node, r, i), n);
  return SQ_OK;
}

int sq_trim_memory(void) {
  return guarded([&] {
    check_device();
    graph_clear_all();
    SQ_CUDA(cudaMemPoolTrimTo(lib_pool(), 0));
  });
}

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

int sq_set_big_bucket_mode(int mode) {
  if (mode < 0 || mode > 4) return SQ_ERR_INVALID_ARGUMENT;
  g_big_mode = mode;
  return SQ_OK;
}

int sq_set_base_case(int which) {
  if (which < 0 || which > 1) return SQ_ERR_INVALID_ARGUMENT;
  g_base_case = which;
  return SQ_OK;
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
    debug_level_u32(src, dst, n, seed, pivots_out, bucend_out, info_out, (cudaStream_t)stream);
  });
}

int sq_debug_level_u64(const uint64_t* src, uint64_t* dst, size_t n, uint64_t seed, uint64_t* pivots_out,
                       uint32_t* bucend_out, uint32_t* info_out, void* stream) {
  return guarded([&] {
    need(n >= 5 && n <= (size_t(1) << 28), "n must be in [5, 2^28]");
    need(src && dst && pivots_out && bucend_out && info_out, "NULL pointer");
    need(!overlap(src, n * 8, dst, n * 8), "src and dst overlap");
    check_device();
    debug_level_engine<uint64_t, false>(src, dst, n, seed, pivots_out, bucend_out, info_out, (cudaStream_t)stream);
  });
}

}  // extern "C"
