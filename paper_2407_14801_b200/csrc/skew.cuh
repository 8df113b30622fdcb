// skew.cuh -- the sort path's SkewTranspose (Alg 2/3): warp-specialised,
// counter-ranked, one piece per ring buffer, persistent grid.
//
// A piece is up to S consecutive keys of one bucket tile's column-major stream
// (the runs of kTB = 32 buckets of up to F consecutive columns), planned by
// k_piece_plan2.  Its image in the output is the stable bucket-major order of those
// keys (column order, then row order, within each bucket: the order Alg 3 writes,
// P:438-449); a bucket of the tile is the concatenation of its sub-chunk in every
// piece, in piece order (L21).  Per piece (k_transpose_ws):
//  * a producer warp loads the piece descriptor, the tile's thresholds and the run
//    bounds before waiting for its ring buffer, then copies every run (16-byte
//    cp.async around its misalignment) into the slot array, marks the slot words
//    that hold keys in a bitmap, and signals the buffer's mbarrier;
//  * pass 1 (eight consumer warps): each thread owns KT consecutive slot words; a
//    key's bucket is found by a branch-free 5-step search over the tile's 31
//    thresholds (held one per lane, read with shuffles; equal-pivot rule L4) and
//    ranked among the thread's keys of that bucket by a shared atomic counter;
//  * scan: the counters in bucket-major, thread-minor order (= stream order within
//    a bucket) give every (bucket, thread) group its first image position;
//  * pass 2: every key goes to its image position; one bulk store (plus per-thread
//    head and tail) writes the image, the bucket prefix goes to ppre and the
//    piece's bucket counts are added to the level's bucket sizes.
#pragma once
#include "level2.cuh"

namespace sq {

// Meta slots of a staged piece.
enum { kMxPiece = 0, kMxNch, kMxPn, kMxOut, kMxNb, kMxBmax, kMxValid, kMxBbase };

// ------------------------------------------------------------------------------
// Consumer word layout: thread t owns KT consecutive words of the staged slot
// array (KT/VW 16-byte vectors, an odd number, so LDS.128 is conflict-free without
// padding); a slot holds S keys plus the alignment padding of up to F runs.
template <typename K, bool PAIRS, int NT, int S, int F>
struct CtCfg {
  static constexpr int NB = 2;  // staging buffers (2: the next piece is staged during this one)
  static constexpr int NW = NT / 32;
  static constexpr int EB = sizeof(K);
  static constexpr int VW = 16 / EB;  // words per 16-byte vector
  static constexpr int SLOTW = S + F * (2 * VW - 2) + VW;
  static constexpr int VPT0 = (SLOTW + NT * VW - 1) / (NT * VW);
  static constexpr int VPT = VPT0 | 1;  // vectors per thread (odd: conflict-free LDS.128)
  static constexpr int KT = VPT * VW;    // words per thread
  static constexpr int WORDS = NT * KT;
  __host__ __device__ static constexpr size_t al(size_t x) { return (x + 127) & ~size_t(127); }
  static constexpr size_t SLOT_B = al(size_t(WORDS) * EB);
  static constexpr size_t VSLOT_B = PAIRS ? al(size_t(WORDS) * 4) : 0;
  static constexpr size_t BITS_B = al((WORDS / 32 + 2) * 4);
  static constexpr size_t THR_B = al(32 * 16 + 32 * 4 + 16 * 4);  // Thr<K>[32], thr32[32], meta[16]
  static constexpr size_t off_slot = 0;
  static constexpr size_t off_vslot = off_slot + NB * SLOT_B;
  static constexpr size_t off_bits = off_vslot + NB * VSLOT_B;
  static constexpr size_t off_thr = off_bits + NB * BITS_B;
  static constexpr size_t off_out = off_thr + NB * THR_B;  // S keys + shift
  static constexpr size_t off_vout = off_out + al((S + 16 / EB) * EB);
  static constexpr size_t off_cnt = off_vout + (PAIRS ? al((S + 4) * 4) : 0);  // 33 x NT u32
  static constexpr size_t off_misc = off_cnt + al(33 * NT * 4);
  static constexpr size_t SMEM = off_misc + al(128 * 4);
};

// counter entry e = bucket * NT + thread -> word: 16-byte chunks XOR-swizzled by
// (e / 32) % 8, so both the per-thread scan reads (32 consecutive entries) and the
// per-warp atomics (32 consecutive entries of one bucket) are conflict-free
__device__ __forceinline__ uint32_t cswz(uint32_t e) { return e ^ (((e >> 5) & 7) << 2); }

// ------------------------------------------------------------------------------
// Warp-specialised SkewTranspose (the sort path's transpose): one producer warp
// stages pieces (descriptor, fragment table via warp scans, bitmap, thresholds,
// 16-byte cp.async per run vector) into a ring of NS buffers and signals each with
// an mbarrier (cp.async.mbarrier.arrive); eight consumer warps run the per-thread
// counter passes of k_transpose_ct on the staged piece, synchronising among
// themselves with a named barrier only, and release the buffer after pass 2.  The
// consumers never wait on global metadata loads or staging work.
template <typename K, bool PAIRS, int S, int F>
struct WsCfg {
  static constexpr int NC = 256;      // consumer threads
  static constexpr int NS = 2;        // ring buffers, one producer warp each
  static constexpr int NT = NC + 32 * NS;
  using CC = CtCfg<K, PAIRS, NC, S, F>;  // per-thread word layout of the consumers
  static constexpr int KT = CC::KT, VW = CC::VW, WORDS = CC::WORDS;
  __host__ __device__ static constexpr size_t al(size_t x) { return (x + 127) & ~size_t(127); }
  static constexpr size_t SLOT_B = CC::SLOT_B, VSLOT_B = CC::VSLOT_B, BITS_B = CC::BITS_B, THR_B = CC::THR_B;
  static constexpr size_t off_slot = 0;
  static constexpr size_t off_vslot = off_slot + NS * SLOT_B;
  static constexpr size_t off_bits = off_vslot + NS * VSLOT_B;
  static constexpr size_t off_thr = off_bits + NS * BITS_B;
  static constexpr size_t off_out = off_thr + NS * THR_B;
  static constexpr size_t off_vout = off_out + al((S + 16 / sizeof(K)) * sizeof(K));
  static constexpr size_t off_cnt = off_vout + (PAIRS ? al((S + 4) * 4) : 0);  // 33 x NC u32
  static constexpr size_t off_misc = off_cnt + al(33 * NC * 4);
  static constexpr size_t off_bar = off_misc + al(128 * 4);                    // full[NS], empty[NS]
  static constexpr size_t SMEM = off_bar + 128;
};

__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

// exclusive sum over the 256 consumer threads (named barrier 1)
__device__ __forceinline__ uint32_t cons_excl_sum(uint32_t v, uint32_t* misc, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  cons_bar();
  if (lane == 31) misc[w] = x;
  cons_bar();
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint32_t m = misc[i];
    pre += i < w ? m : 0u;
    tot += m;
  }
  *total = tot;
  return x - v + pre;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t* total) {
  const int lane = threadIdx.x & 31;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// cache operator of the producer's 16-byte copies (.ca: the two 16-byte halves of a
// 32-byte sector are one L2 request; .cg: two)
#ifndef SQ_TR_CACHE
#define SQ_TR_CACHE "cg"
#endif
// runs of at least this many staged bytes are copied by the whole producer warp
#ifndef SQ_COOP_RUN_BYTES
#define SQ_COOP_RUN_BYTES 1024
#endif
constexpr uint32_t kCoopRunBytes = SQ_COOP_RUN_BYTES;
template <typename K, bool PAIRS, int S, int F>
__global__ void __launch_bounds__(WsCfg<K, PAIRS, S, F>::NT, 2)
k_transpose_ws(const PieceDesc* __restrict__ pieces, const uint32_t* __restrict__ pcount, const K* __restrict__ src,
               K* __restrict__ dst, const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst,
               const K* __restrict__ piv, const uint32_t* __restrict__ segmat, uint16_t* __restrict__ ppre,
               uint32_t* __restrict__ bsize) {
  using C = WsCfg<K, PAIRS, S, F>;
  constexpr int EB = sizeof(K), NC = C::NC, KT = C::KT, VW = C::VW, NS = C::NS;
  static_assert(F <= 128 && F % 32 == 0 && S <= 65535 && kTB == 32 && KT < 64, "shape");
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::off_bar);
  uint64_t* empty = full + NS;
  const int t = threadIdx.x, lane = t & 31;
  const uint32_t npieces = *pcount;
  if (t == 0) {
    for (int b = 0; b < NS; b++) {
      mbar_init(&full[b], 64);    // 32 producer lanes: async (cp.async done) + plain (stores done)
      mbar_init(&empty[b], NC);   // every consumer thread
    }
    fence_proxy_async();
  }
  __syncthreads();

  if (t >= NC) {  // ================= producer warps: warp b stages pieces k = b, b+NS, ... into buffer b
    const int b = (t - NC) >> 5;
    uint32_t k = b;
    PieceDesc pdn;  // the next piece's descriptor, prefetched one iteration ahead
    if (blockIdx.x + b * gridDim.x < npieces) pdn = pieces[blockIdx.x + b * gridDim.x];
    for (uint32_t i = blockIdx.x + b * gridDim.x; i < npieces; i += NS * gridDim.x, k += NS) {
      // the piece's metadata is loaded before waiting for the buffer: the loads
      // overlap the consumers' work on the buffer's previous piece
      const PieceDesc pd = pdn;
      if (i + NS * gridDim.x < npieces) pdn = pieces[i + NS * gridDim.x];
      const uint32_t nb = pd.nb, Pn = pd.pn, nf = pd.nf;
      const K* P = piv + pd.thr0;
      const bool real = lane < (int)nb - 1;
      const K pj = real ? P[lane] : K(0);
      const K pprev = (real && pd.bt * kTB + lane >= 1) ? P[lane - 1] : K(0);
      uint32_t ra[F / 32], rb[F / 32];  // all run bounds loaded at once (one latency)
#pragma unroll
      for (int r = 0; r < F / 32; r++) {
        const uint32_t f = 32 * r + lane;
        if (f < nf) {
          const uint32_t* row = segmat + pd.row0 + f;  // tile-major segmat: coalesced over f
          ra[r] = row[0];
          rb[r] = row[pd.rstride];
        }
      }
      if (k >= NS) mbar_wait(&empty[b], ((k / NS) - 1) & 1);
      K* slot = reinterpret_cast<K*>(sm + C::off_slot + b * C::SLOT_B);
      uint32_t* vslot = reinterpret_cast<uint32_t*>(sm + C::off_vslot + b * C::VSLOT_B);
      uint32_t* bits = reinterpret_cast<uint32_t*>(sm + C::off_bits + b * C::BITS_B);
      Thr<K>* thr = reinterpret_cast<Thr<K>*>(sm + C::off_thr + b * C::THR_B);
      uint32_t* thr32 = reinterpret_cast<uint32_t*>(sm + C::off_thr + b * C::THR_B + 32 * 16);
      uint32_t* meta = thr32 + 32;
      {  // thresholds (lane = boundary)
        const bool dup = real && pd.bt * kTB + lane >= 1 && pprev == pj;
        thr[lane] = Thr<K>::make(pj, dup, !real);
        uint32_t cntmax = 0;
        if constexpr (sizeof(K) == 4) {
          const uint64_t t64 = real ? uint64_t(pj) + (dup ? 1u : 0u) : (1ull << 32);
          thr32[lane] = t64 > 0xffffffffull ? 0xffffffffu : (uint32_t)t64;
          cntmax = __popc(__ballot_sync(0xffffffffu, t64 <= 0xffffffffull));
        }
        if (lane == 0) {
          meta[kMxPiece] = pd.slot;
          meta[kMxPn] = Pn;
          meta[kMxOut] = pd.out;
          meta[kMxNb] = nb;
          meta[kMxBmax] = cntmax;
          meta[kMxBbase] = pd.bbase;
        }
      }
      for (uint32_t q = lane; q < C::BITS_B / 4; q += 32) bits[q] = 0;
      __syncwarp();
      uint32_t carry_len = 0, carry_sb = 0;
#pragma unroll
      for (int r = 0; r < F / 32; r++) {
        const uint32_t f = 32 * r + lane;
        if (32 * r >= nf) break;
        uint32_t len = 0, srcpos = 0;
        if (f < nf) {
          const uint32_t a = ra[r] + (f == 0 ? pd.off : 0), e = rb[r];
          len = e - a;
          srcpos = pd.src0 + f * pd.rows + a;
        }
        uint32_t tl;
        const uint32_t ex = warp_excl_scan(len, &tl) + carry_len;
        carry_len += tl;
        const uint32_t flen = f < nf ? min(ex + len, Pn) - min(ex, Pn) : 0;
        uint32_t mis = 0, sbytes = 0;
        if (flen) {
          mis = (uint32_t)(reinterpret_cast<uintptr_t>(src + srcpos) & 15);
          sbytes = (mis + flen * EB + 15) & ~15u;
        }
        uint32_t ts;
        const uint32_t so = warp_excl_scan(sbytes, &ts) + carry_sb;
        carry_sb += ts;
        // long runs (sorted or clustered input: a column's keys fall into a few buckets,
        // so a run is hundreds of keys): the warp copies each run together instead of
        // one lane walking it (warp-uniform choice)
        const bool coop = __reduce_max_sync(0xffffffffu, sbytes) >= kCoopRunBytes;
        if (coop) {
          uint32_t live = __ballot_sync(0xffffffffu, flen != 0);
          const uint32_t my_e0 = (so + mis) / EB;
          const unsigned long long my_g =
              (unsigned long long)(reinterpret_cast<uintptr_t>(src + srcpos) - mis);
          while (live) {
            const int L = __ffs(live) - 1;
            live &= live - 1;
            const uint32_t e0 = __shfl_sync(0xffffffffu, my_e0, L), fl = __shfl_sync(0xffffffffu, flen, L);
            const uint32_t sb = __shfl_sync(0xffffffffu, sbytes, L), so_l = __shfl_sync(0xffffffffu, so, L);
            const uint32_t sp = __shfl_sync(0xffffffffu, srcpos, L);
            const unsigned char* g = reinterpret_cast<const unsigned char*>((uintptr_t)__shfl_sync(0xffffffffu, my_g, L));
            const uint32_t e1 = e0 + fl;
            for (uint32_t wd = (e0 >> 5) + lane; wd <= (e1 - 1) >> 5; wd += 32) {
              const uint32_t lo = max(e0, wd * 32) - wd * 32, hi = min(e1, wd * 32 + 32) - wd * 32;
              const uint32_t m = (hi == 32 ? 0xffffffffu : ((1u << hi) - 1)) & ~((1u << lo) - 1);
              atomicOr(&bits[wd], m);
            }
            const uint32_t sdst = smem_addr(slot) + so_l;
            for (uint32_t v = 16 * lane; v < sb; v += 512)
              asm volatile("cp.async." SQ_TR_CACHE ".shared.global [%0], [%1], 16;\n" ::"r"(sdst + v), "l"(g + v));
            if (PAIRS) {
              const uint32_t* gv = vsrc + sp;
              for (uint32_t kk = lane; kk < fl; kk += 32) cp_async_elem(&vslot[e0 + kk], &gv[kk]);
            }
          }
        } else if (flen) {
          const uint32_t e0 = (so + mis) / EB, e1 = e0 + flen;
          for (uint32_t wd = e0 >> 5; wd <= (e1 - 1) >> 5; wd++) {
            const uint32_t lo = max(e0, wd * 32) - wd * 32, hi = min(e1, wd * 32 + 32) - wd * 32;
            const uint32_t m = (hi == 32 ? 0xffffffffu : ((1u << hi) - 1)) & ~((1u << lo) - 1);
            atomicOr(&bits[wd], m);
          }
          const uint32_t sdst = smem_addr(slot) + so;
          const unsigned char* g = reinterpret_cast<const unsigned char*>(src + srcpos) - mis;
          for (uint32_t v = 0; v < sbytes; v += 16)
            asm volatile("cp.async." SQ_TR_CACHE ".shared.global [%0], [%1], 16;\n" ::"r"(sdst + v), "l"(g + v));
          if (PAIRS) {
            const uint32_t* gv = vsrc + srcpos;
            for (uint32_t kk = 0; kk < flen; kk++) cp_async_elem(&vslot[e0 + kk], &gv[kk]);
          }
        }
      }
      if (lane == 0) meta[kMxNch] = carry_sb / EB;  // slot words in use
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(&full[b])) : "memory");
      mbar_arrive(&full[b]);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }

  // ================= consumer warps
  unsigned char* outraw = sm + C::off_out;
  unsigned char* voutraw = sm + C::off_vout;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + C::off_cnt);  // [bucket][thread], + a dummy row
  uint32_t* misc = reinterpret_cast<uint32_t*>(sm + C::off_misc);
  uint32_t* poff = misc + 64;
  // cswz(bucket * NC + t) == bucket * NC + (t ^ (warp << 2)) since NC is a multiple of 256
  static_assert(NC % 256 == 0, "swizzle");
  const uint32_t tsw = t ^ (((t >> 5) & 7) << 2);
  uint32_t k = 0;
  for (uint32_t i = blockIdx.x; i < npieces; i += gridDim.x, k++) {
    const int b = k % NS;
    for (int q = t; q < 33 * NC / 4; q += NC)  // 32 bucket rows + the dummy row
      reinterpret_cast<uint4*>(cnt)[q] = make_uint4(0u, 0u, 0u, 0u);
    mbar_wait(&full[b], (k / NS) & 1);
    cons_bar();
    const K* slot = reinterpret_cast<const K*>(sm + C::off_slot + b * C::SLOT_B);
    const uint32_t* vslot = reinterpret_cast<const uint32_t*>(sm + C::off_vslot + b * C::VSLOT_B);
    const uint32_t* bits = reinterpret_cast<const uint32_t*>(sm + C::off_bits + b * C::BITS_B);
    const Thr<K>* thr = reinterpret_cast<const Thr<K>*>(sm + C::off_thr + b * C::THR_B);
    const uint32_t* thr32 = reinterpret_cast<const uint32_t*>(sm + C::off_thr + b * C::THR_B + 32 * 16);
    const uint32_t* meta = thr32 + 32;
    const uint32_t nwords = meta[kMxNch], Pn = meta[kMxPn], oc = meta[kMxOut], bmax = meta[kMxBmax];
    const uint32_t nb = meta[kMxNb], pslot = meta[kMxPiece], bbase = meta[kMxBbase];
    const uint32_t thr_r = sizeof(K) == 4 ? thr32[lane] : 0u;
    // ---- pass 1: buckets and thread-local ranks
    const uint32_t w0 = t * KT;
    uint32_t vb;  // validity of the thread's KT words
    {
      const uint32_t bw = w0 >> 5, sh = w0 & 31;
      vb = __funnelshift_r(bits[bw], bits[bw + 1], sh);
      if (KT < 32) vb &= (1u << KT) - 1;
      if (w0 >= nwords) vb = 0;
    }
    K xs[KT];
    uint32_t cdp[(KT + 1) / 2];  // per key: bucket | thread-local rank << 6, two per word
    // warps whose words all lie past the staged runs (the slot is sized for the
    // worst-case alignment padding; ~1 warp in 8 usually) skip pass 1
    if (!__any_sync(0xffffffffu, vb != 0)) {
#pragma unroll
      for (int q = 0; q < (KT + 1) / 2; q++) cdp[q] = 32u | (32u << 16);
    } else {
#pragma unroll
    for (int q = 0; q < KT / VW; q++) {
      const uint4 v4 = reinterpret_cast<const uint4*>(slot)[t * (KT / VW) + q];
      if constexpr (sizeof(K) == 4) {
        xs[4 * q] = v4.x; xs[4 * q + 1] = v4.y; xs[4 * q + 2] = v4.z; xs[4 * q + 3] = v4.w;
      } else {
        xs[2 * q] = (uint64_t(v4.y) << 32) | v4.x;
        xs[2 * q + 1] = (uint64_t(v4.w) << 32) | v4.z;
      }
    }
    uint32_t E_r = 0;
    if constexpr (sizeof(K) == 4) {
      const uint32_t l = lane ? lane : 1, d = 31 - __clz(l);
      E_r = __shfl_sync(0xffffffffu, thr_r, ((2 * (l - (1u << d)) + 1) << (4 - d)) - 1);
    }
    const uint32_t E1 = __shfl_sync(0xffffffffu, E_r, 1), E2 = __shfl_sync(0xffffffffu, E_r, 2),
                   E3 = __shfl_sync(0xffffffffu, E_r, 3);
#pragma unroll
    for (int j = 0; j < KT; j++) {
      const K x = xs[j];
      uint32_t bk = 0;
      if constexpr (sizeof(K) == 4) {
        const uint32_t p1 = uint32_t(x) >= E1 ? 1u : 0u;
        uint32_t ii = 2 + p1;
        ii = 2 * ii + (uint32_t(x) >= (p1 ? E3 : E2) ? 1u : 0u);
#pragma unroll
        for (int st = 0; st < 3; st++) ii = 2 * ii + (uint32_t(x) >= __shfl_sync(0xffffffffu, E_r, ii) ? 1u : 0u);
        bk = min(ii - 32, bmax);
      } else {
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) bk += thr[bk + st - 1].passed(x) ? st : 0;
      }
      bk = ((vb >> j) & 1) ? bk : 32u;
      const uint32_t r = atomicAdd(&cnt[bk * NC + tsw], 1u);
      const uint32_t c = bk | (r << 6);
      if (j & 1) cdp[j / 2] |= c << 16;
      else cdp[j / 2] = c;
    }
    }
    cons_bar();
    {  // exclusive scan of the counters, bucket-major
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(&cnt[cswz(32 * t + 4 * q)]);
        sum += v4.x + v4.y + v4.z + v4.w;
      }
      uint32_t tot;
      uint32_t run = cons_excl_sum(sum, misc, &tot);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        uint4* p4 = reinterpret_cast<uint4*>(&cnt[cswz(32 * t + 4 * q)]);
        const uint4 v4 = *p4;
        uint4 o;
        o.x = run; run += v4.x;
        o.y = run; run += v4.y;
        o.z = run; run += v4.z;
        o.w = run; run += v4.w;
        *p4 = o;
      }
    }
    cons_bar();
    if (t < 32) poff[t] = t < (int)nb ? cnt[cswz(t * NC)] : Pn;
    if (t == 32) poff[kTB] = Pn;
    if (t == 0) bulk_wait_read0();  // previous piece's image has been read out
    cons_bar();
    // ---- pass 2: scatter into the piece image (shifted for the bulk store)
    const uint32_t oshift = (uint32_t)((reinterpret_cast<uintptr_t>(dst + oc) & 15) / EB);
    K* outb = reinterpret_cast<K*>(outraw) + oshift;
    const uint32_t vshift = PAIRS ? (uint32_t)((reinterpret_cast<uintptr_t>(vdst + oc) & 15) / 4) : 0;
    uint32_t* vout = reinterpret_cast<uint32_t*>(voutraw) + vshift;
#pragma unroll
    for (int j = 0; j < KT; j++) {
      const uint32_t c = (cdp[j / 2] >> (16 * (j & 1))) & 0xffffu;
      const uint32_t bk = c & 63;
      if (bk < 32) {
        const uint32_t dpos = cnt[bk * NC + tsw] + (c >> 6);
        SQ_CHECK(dpos < Pn);
        outb[dpos] = xs[j];
        if (PAIRS) vout[dpos] = vslot[w0 + j];
      }
    }
    mbar_arrive(&empty[b]);  // the producer may refill this buffer
    fence_proxy_async();
    cons_bar();
    {
      const uintptr_t g0 = reinterpret_cast<uintptr_t>(dst + oc);
      const uintptr_t g1 = g0 + uintptr_t(Pn) * EB;
      const uintptr_t a0 = (g0 + 15) & ~uintptr_t(15), a1 = g1 & ~uintptr_t(15);
      if (a1 > a0) {
        if (t == 0)
          bulk_s2g(reinterpret_cast<void*>(a0), reinterpret_cast<unsigned char*>(outb) + (a0 - g0),
                   (uint32_t)(a1 - a0));
        const uint32_t nh = (uint32_t)((a0 - g0) / EB), nt0 = (uint32_t)((a1 - g0) / EB);
        if (t < (int)nh) dst[oc + t] = outb[t];
        if (t < (int)(Pn - nt0)) dst[oc + nt0 + t] = outb[nt0 + t];
      } else {
        for (uint32_t q = t; q < Pn; q += NC) dst[oc + q] = outb[q];
      }
      if (PAIRS) {
        const uintptr_t h0 = reinterpret_cast<uintptr_t>(vdst + oc);
        const uintptr_t h1 = h0 + uintptr_t(Pn) * 4;
        const uintptr_t c0 = (h0 + 15) & ~uintptr_t(15), c1 = h1 & ~uintptr_t(15);
        if (c1 > c0) {
          if (t == 0)
            bulk_s2g(reinterpret_cast<void*>(c0), reinterpret_cast<unsigned char*>(vout) + (c0 - h0),
                     (uint32_t)(c1 - c0));
          const uint32_t nh = (uint32_t)((c0 - h0) / 4), nt0 = (uint32_t)((c1 - h0) / 4);
          if (t < (int)nh) vdst[oc + t] = vout[t];
          if (t < (int)(Pn - nt0)) vdst[oc + nt0 + t] = vout[nt0 + t];
        } else {
          for (uint32_t q = t; q < Pn; q += NC) vdst[oc + q] = vout[q];
        }
      }
      if (t == 0) bulk_commit();
    }
    if (t <= kTB) ppre[uint64_t(pslot) * kPP + t] = (uint16_t)poff[t];
    // bucket sizes of the level: this piece's count of every bucket of its tile
    if (t < (int)nb && poff[t + 1] > poff[t]) atomicAdd(&bsize[bbase + t], poff[t + 1] - poff[t]);
    cons_bar();
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace sq
