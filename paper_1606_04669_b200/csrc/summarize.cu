// summarize.cu -- K1: per-partition Space Saving summaries (Algorithm 1 lines 3-5, PAPER.md:92-96;
// update rules PAPER.md:82) on sm_100a.
//
// One warp owns one partition at a time (persistent 1-warp CTAs pull partition ids from a queue).
// The warp streams its block of A through a shared-memory ring filled by the TMA engine
// (cp.async.bulk + mbarrier) and applies Space Saving to 32 consecutive items per step with an
// exact batched rule:
//   1. each lane looks its item up in a two-choice, two-way bucketed cuckoo index
//      (entry = fingerprint | slot in 16 bits for k <= 4094; a lookup reads both candidate
//      buckets with two independent loads, selects the first fingerprint match without branches
//      and verifies its key; a fingerprint match with another key takes a slow re-check);
//   2. __match_any_sync groups equal keys; the first lane of a group is its leader, multiplicity =
//      popcount of the group restricted to the processed prefix;
//   3. leaders that miss are ranked in stream order; during the fill phase they take slots
//      size, size+1, ... (R2); once all k counters are occupied they take the lowest-index slots of
//      B_m = {slots with count == m, the current minimum} in ascending order (R1). B_m is a bitmap
//      consumed left to right through a cursor; at the start of every step, in parallel with the
//      lookups, lane j fetches the j-th next victim slot and the index entry of its item;
//   4. the step processes the longest prefix [0, c) of the 32 items for which this equals the
//      sequential algorithm: c stops before the first miss that finds no victim left (B_m empty
//      or beyond the fetched words) or the counters full, and before the first hazard where a
//      victim slot is also hit in the window;
//   5. hits add their multiplicity; misses evict (count m + mult, err m), free the victim's index
//      entry and write their own entry into a free way of their buckets; a read-back settles lanes
//      that picked the same entry, and the rare leftovers take a serial cuckoo-kick path.
// Every step consumes >= 1 item, so the result is bit-identical to sequential Space Saving.
// When the block length allows, count and error share one 32-bit word (count in the low cb bits).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace pss {

#ifdef PSS_STATS  // debug build only (tools/k1_stats.py): event counters of the batched rule
__device__ unsigned long long g_ss_stats[16];
#define SS_STAT(i, v)                                                      \
  do {                                                                     \
    const unsigned long long _v = (unsigned long long)(v);                 \
    if (lane == 0) atomicAdd(&g_ss_stats[i], _v);                          \
  } while (0)
}  // namespace pss
extern "C" int pss_debug_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pss::g_ss_stats, sizeof(pss::g_ss_stats));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(pss::g_ss_stats, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
namespace pss {
// step-phase timing (debug build): wait for a value, then read the SM clock
#define SS_TICK(acc, t, val)                                         \
  do {                                                               \
    uint32_t _d;                                                     \
    asm volatile("mov.b32 %0, %1;" : "=r"(_d) : "r"((uint32_t)(val))); \
    const long long _t = clock64() + (_d & 0);                       \
    acc += _t - t;                                                   \
    t = _t;                                                          \
  } while (0)
#else
#define SS_STAT(i, v) \
  do {                \
  } while (0)
#define SS_TICK(acc, t, val) \
  do {                       \
  } while (0)
#endif

// per-warp TMA ring: 3 stages of 512 bytes (a step spans at most two stages; one more in flight)
#ifndef PSS_SS_NSTAGE
#define PSS_SS_NSTAGE 3
#endif
constexpr uint32_t SS_NSTAGE = PSS_SS_NSTAGE;
#ifndef PSS_SS_STAGE_BYTES
#define PSS_SS_STAGE_BYTES 512
#endif
constexpr uint32_t SS_STAGE_BYTES = PSS_SS_STAGE_BYTES;
constexpr uint32_t SS_BAR_BYTES = 32;  // the ring's mbarriers (3 x 8 bytes)
constexpr uint32_t SS_RING_BYTES = SS_NSTAGE * SS_STAGE_BYTES;
// the bypass kernel's ring: 6 stages of which 4 stay resident behind the newest one waited for
// (its classification runs up to 3 stages ahead of the oldest queued item), 2 in flight
#ifndef PSS_SS_BYP_NSTAGE
#define PSS_SS_BYP_NSTAGE 6
#endif
#ifndef PSS_SS_BYP_KEEP
#define PSS_SS_BYP_KEEP 4
#endif
constexpr uint32_t SS_BYP_NSTAGE = PSS_SS_BYP_NSTAGE, SS_BYP_KEEP = PSS_SS_BYP_KEEP;
constexpr uint32_t SS_BYP_RING_BYTES = SS_BYP_NSTAGE * SS_STAGE_BYTES;
constexpr uint32_t SS_BYP_BAR_BYTES = 64;
static_assert(SS_BYP_NSTAGE * 8 <= SS_BYP_BAR_BYTES && SS_BYP_KEEP >= 2 && SS_BYP_KEEP < SS_BYP_NSTAGE, "ring");
constexpr size_t SS_SMEM_STATE_MAX = 100 * 1024;  // bigger per-warp state lives in global memory
constexpr uint32_t SS_K_SMALL = 4094;             // 16-bit index entries up to this k
constexpr double SS_LOAD = 0.24;  // index load factor (live keys / entries), before the slack fill
constexpr int SS_MAX_KICKS = 200;

// Index entry layout (runtime): slot in the low sb bits, fingerprint above. A slot field of all
// ones is never a slot (sb is chosen so that k - 1 < 2^sb - 1) and a fingerprint is never all ones,
// so the EMPTY entry (all ones) matches no fingerprint.
template <typename ET>
struct Ent {
  static constexpr ET EMPTY = (ET)~(ET)0;
  uint32_t sb;     // slot bits
  uint32_t fmask;  // fingerprint field mask (after >> sb)
  __device__ __forceinline__ ET make(uint32_t fp, uint32_t v) const {
    return (ET)(((ET)fp << sb) | (ET)v);
  }
  __device__ __forceinline__ uint32_t slot(ET e) const {
    return (uint32_t)(e & (ET)(((ET)1 << sb) - 1));
  }
  __device__ __forceinline__ bool fp_eq(ET e, uint32_t fp) const {
    return (uint32_t)(e >> sb) == fp;
  }
  __device__ __forceinline__ uint32_t fp_of(uint32_t h) const { return min(h & fmask, fmask - 1); }
};

// both entries of bucket b
__device__ __forceinline__ void load_bucket(const uint16_t* T, uint32_t b, uint16_t& e0,
                                            uint16_t& e1) {
  const uint32_t v = reinterpret_cast<const uint32_t*>(T)[b];
  e0 = (uint16_t)v;
  e1 = (uint16_t)(v >> 16);
}
__device__ __forceinline__ void load_bucket(const uint64_t* T, uint32_t b, uint64_t& e0,
                                            uint64_t& e1) {
  const ulonglong2 v = reinterpret_cast<const ulonglong2*>(T)[b];
  e0 = v.x;
  e1 = v.y;
}

__device__ __forceinline__ uint32_t fold32(uint32_t x) { return x; }
__device__ __forceinline__ uint32_t fold32(uint64_t x) {
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32) ^ (uint32_t)x;
}

// bucket pair + fingerprint of a key (seeded so that a failed build can rehash). b1 == b2 is
// allowed: the key then has two candidate entries instead of four.
template <typename ET, typename KT>
__device__ __forceinline__ void key_hash(const Ent<ET>& en, KT x, uint32_t seed, uint32_t NB,
                                         uint32_t& b1, uint32_t& b2, uint32_t& fp) {
  const uint32_t ha = (fold32(x) ^ seed) * 0x9E3779B1u;
  const uint32_t hb = (ha ^ (ha >> 16)) * 0x85EBCA6Bu;
  b1 = __umulhi(ha, NB);
  b2 = __umulhi(hb, NB);
  fp = en.fp_of(hb);
}

// insert target among the entries (e0, e1) of bucket b1 and (e2, e3) of b2: a free entry of the
// bucket with more free entries (b1 on ties), so that both buckets of a key rarely fill up
// (balanced two-choice allocation); 0xffffffff if all four are occupied
template <typename ET>
__device__ __forceinline__ uint32_t free_entry(ET e0, ET e1, ET e2, ET e3, uint32_t b1,
                                               uint32_t b2) {
  constexpr ET EMPTY = Ent<ET>::EMPTY;
  uint32_t fa = e1 == EMPTY ? 2 * b1 + 1 : 0xffffffffu;
  fa = e0 == EMPTY ? 2 * b1 : fa;
  uint32_t fb = e3 == EMPTY ? 2 * b2 + 1 : 0xffffffffu;
  fb = e2 == EMPTY ? 2 * b2 : fb;
  const bool pickb = (uint32_t)(e2 == EMPTY) + (uint32_t)(e3 == EMPTY) >
                     (uint32_t)(e0 == EMPTY) + (uint32_t)(e1 == EMPTY);
  return pickb ? fb : fa;
}

struct SSLayout {
  size_t keys, cnt, err, pos, bm, vic, hc, cq, cqp, T, total;
  uint32_t NB;
};

// test hook: crowd the index (a 2-way, 2-choice cuckoo table holds up to ~0.89); 0 = unset
static double ss_debug_load() {
  const char* s = std::getenv("PSS_DEBUG_INDEX_LOAD");
  if (s) {
    double v = std::atof(s);
    if (v > 0.05 && v <= 0.85) return v;
  }
  return 0.0;
}
static uint32_t ss_buckets(uint32_t k, double load) {
  return (uint32_t)std::max<double>(2.0, std::ceil(k / (2.0 * load)));
}

// level-pinned bypass: the cold queue's capacity (items), a power of two >= 64
constexpr uint32_t SS_CQ = 128;

static SSLayout ss_layout(uint32_t k, int kb, int eb, bool packed, uint32_t NB, bool byp = false) {
  SSLayout L;
  const size_t KP = align_up(k, 32);
  L.NB = NB;
  Bump b;
  b.al = 16;  // every slot-indexed array holds exactly k entries (slots are < k)
  L.keys = b.take<unsigned char>((size_t)k * kb);
  L.cnt = b.take<uint32_t>(k);
  L.err = packed ? L.cnt : b.take<uint32_t>(k);
  // packed counters carry their index position in the top two bits (bucket choice, way)
  L.pos = packed ? L.cnt : b.take<unsigned char>((size_t)k * (eb == 2 ? 2 : 4));
  L.bm = b.take<uint32_t>(KP / 32 + 2);
  L.vic = b.take<uint32_t>(32);
  // bypass: counts of the pinned hot keys, the queue of cold items and their positions
  L.hc = byp ? b.take<uint32_t>(HOT_MAX) : 0;
  L.cq = byp ? b.take<unsigned char>((size_t)SS_CQ * kb) : 0;
  L.cqp = byp ? b.take<uint16_t>(SS_CQ) : 0;  // positions < 2^16 (blocks of <= 2^16 items)
  L.T = b.take<unsigned char>((size_t)2 * L.NB * eb);
  L.total = b.bytes();  // a multiple of 16
  return L;
}

struct SumArgs {
  const void* A;
  uint64_t n;
  uint32_t k, P;
  uint32_t r0, r1;  // this launch summarizes partitions [r0, r1) of the P-way decomposition
  uint32_t T;       // > 1: P = Pp * T leaves of the two-level decomposition (f4)
  uint32_t* leaf_flags;  // non-null: leaf_flags[r] = 1 (release) once leaf r is written
  int pdl;               // let the tree kernel launch now (it waits on leaf_flags)
  void* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
  uint32_t* queue;
  const unsigned char* skip;  // non-null: only leaves r with skip[r] != 0 (flagged by hist.cu)
  unsigned char* gstate;  // per-CTA state when it does not fit shared memory
  size_t gstride;
  size_t o_cnt, o_err, o_pos, o_bm, o_vic, o_T;
  size_t o_hc, o_cq, o_cqp;
  const uint32_t* hot;    // non-null: the frequent-key table of this launch's range (hot.cu)
  uint32_t NB;
  uint32_t cb;            // PACKED: count in the low cb bits, error above
  uint32_t sb, fmask;     // index entry layout
};

// SB, CB > 0: the index entry's slot bits and the counter word's count bits as compile-time
// constants (shifts and masks become immediates and free registers: 4.5 % at H); 0: runtime
// BYP: the level-pinned bypass (below, "level-pinned bypass"), u32 keys with packed counters
template <typename KT, typename ET, bool GSTATE, bool PACKED, int SB = 0, int CB = 0,
          bool BYP = false>
// 1-warp CTAs: __launch_bounds__(32) measured 12-15 % faster than any multi-warp bound (CTAs of
// several independent warps, sharing the per-CTA reserved shared memory, lost more than the
// extra residency gained)
__global__ void __launch_bounds__(32) ss_summarize_kernel(const SumArgs a) {
  using PT = typename std::conditional<sizeof(ET) == 2, uint16_t, uint32_t>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = threadIdx.x;
  const uint32_t ltm = lanemask_lt();
  constexpr uint32_t ST = SS_STAGE_BYTES / sizeof(KT);  // items per stage
  // ring: NST stages, KEEP of them resident up to the newest one waited for, NST - KEEP in flight
  constexpr uint32_t NST = BYP ? SS_BYP_NSTAGE : SS_NSTAGE, KEEP = BYP ? SS_BYP_KEEP : 2u;
  constexpr uint32_t NFL = NST - KEEP;
  constexpr uint32_t RING_BYTES = BYP ? SS_BYP_RING_BYTES : SS_RING_BYTES;
  constexpr uint32_t BAR_BYTES = BYP ? SS_BYP_BAR_BYTES : SS_BAR_BYTES;
  constexpr uint32_t RING = NST * ST;  // ring capacity in items
  constexpr uint32_t E = 16 / sizeof(KT);  // items per 16 bytes
  constexpr ET EMPTY = Ent<ET>::EMPTY;
  const Ent<ET> en{SB ? (uint32_t)SB : a.sb, SB ? (1u << (16 - SB)) - 1u : a.fmask};

  KT* ring = reinterpret_cast<KT*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RING_BYTES);
  unsigned char* st = GSTATE ? a.gstate + (size_t)blockIdx.x * a.gstride : smem + RING_BYTES + BAR_BYTES;
  KT* keys = reinterpret_cast<KT*>(st);
  // count; if PACKED also err << cb and the index position of the slot's entry in bits 30-31
  uint32_t* cnt = reinterpret_cast<uint32_t*>(st + a.o_cnt);
  PT* pos = reinterpret_cast<PT*>(st + a.o_pos);               // index entry of each slot
  uint32_t* err = reinterpret_cast<uint32_t*>(st + a.o_err);
  uint32_t* bm = reinterpret_cast<uint32_t*>(st + a.o_bm);
  uint32_t* vic = reinterpret_cast<uint32_t*>(st + a.o_vic);
  ET* T = reinterpret_cast<ET*>(st + a.o_T);

  const KT* __restrict__ A = reinterpret_cast<const KT*>(a.A);
  const uint64_t n = a.n;
  const uint32_t k = a.k, P = a.P, NB = a.NB;
  const uint32_t NE = 2 * NB;
  const uint32_t kw = (k + 31u) / 32u;
  const uint32_t cb = CB ? (uint32_t)CB : a.cb;
  const uint32_t CM = PACKED ? ((1u << cb) - 1u) : 0xffffffffu;
  constexpr uint32_t POSM = 3u << 30;
  // index position bits of entry fi of a key whose first bucket is b1: (fi in b2) << 31 | way << 30
  auto pos_bits = [](uint32_t fi, uint32_t b1) -> uint32_t {
    return fi == 0xffffffffu ? 0u : (((fi >> 1) != b1 ? 2u : 0u) | (fi & 1u)) << 30;
  };
  auto set_pos = [&](uint32_t cv, uint32_t idx, uint32_t b1) {
    if (PACKED)
      cnt[cv] = (cnt[cv] & ~POSM) | pos_bits(idx, b1);
    else
      pos[cv] = (PT)idx;
  };
  const bool aligned = (reinterpret_cast<uintptr_t>(A) & 15u) == 0;
  const uint64_t nfloor = aligned ? (n & ~(uint64_t)(E - 1)) : 0;

  if (lane == 0) {
    for (uint32_t j = 0; j < NST; ++j) mbar_init(&bars[j], 1);
    fence_mbar_init();
  }
  for (uint32_t i = kw + lane; i < kw + 2; i += 32) bm[i] = 0;  // guard words
  __syncwarp();
  uint32_t phasebits = 0;
  if (a.pdl) pdl_launch_dependents();
  // level-pinned bypass: the launch's frequent keys (lane j keeps keys j and j + 32)
  uint32_t nhot = 0, hseed = 0, hk0 = 0, hk1 = 0;
  const uint32_t* htab = nullptr;
  if constexpr (BYP) {
    nhot = a.hot[0];
    hseed = a.hot[1];
    htab = a.hot + 4 + HOT_MAX;
    hk0 = lane < nhot ? a.hot[4 + lane] : 0u;
    hk1 = lane + 32 < nhot ? a.hot[4 + 32 + lane] : 0u;
    if (nhot == 0) return;  // no table for this range: the plain kernel (launched next) runs
  } else {
    if (a.hot && a.hot[0] != 0) return;  // the bypass kernel (launched before) took the range
  }
  uint32_t* const hc = reinterpret_cast<uint32_t*>(st + a.o_hc);
  KT* const cq = reinterpret_cast<KT*>(st + a.o_cq);
  uint16_t* const cqp = reinterpret_cast<uint16_t*>(st + a.o_cqp);

  while (true) {
    uint32_t r = 0;
    if (lane == 0) r = a.r0 + atomicAdd(a.queue, 1u);
    r = __shfl_sync(PSS_FULL, r, 0);
    if (r >= a.r1) break;
    if (a.skip && !a.skip[r]) continue;  // leaf written by the histogram kernel (hist.cu)
    uint64_t lo, hi;
    if (a.T <= 1) {
      lo = (uint64_t)r * n / P;  // Alg. 1 l.3-4: r*n < 2^63 as n <= 2^31
      hi = (uint64_t)(r + 1) * n / P;
    } else {  // two-level (hybrid) decomposition: process p = r / T, thread t = r % T
      const uint64_t Pp = P / a.T, p = r / a.T, t = r % a.T;
      const uint64_t b0 = p * n / Pp, Lp = (p + 1) * n / Pp - b0;
      lo = b0 + t * Lp / a.T;
      hi = b0 + (t + 1) * Lp / a.T;
    }
    const uint32_t L = (uint32_t)(hi - lo);

    // ---- reset the summary
    for (uint32_t i = lane; i < NE; i += 32) T[i] = EMPTY;
    uint32_t size = 0, m = 0, bmcount = 0, cur = 0, seed = 0;
    if constexpr (BYP) {
      hc[lane] = 0;
      hc[lane + 32] = 0;
    }
    __syncwarp();

    auto new_level = [&]() {  // m = min count, B_m = {slots with count m}, cursor at slot 0
      uint32_t mn = 0xffffffffu;
      for (uint32_t t = lane; t < k; t += 32) mn = min(mn, cnt[t] & CM);
      m = __reduce_min_sync(PSS_FULL, mn);
      uint32_t tot = 0;
      for (uint32_t w = 0; w < kw; ++w) {
        const uint32_t t = w * 32 + lane;
        const uint32_t bits = __ballot_sync(PSS_FULL, t < k && (cnt[t] & CM) == m);
        if (lane == 0) bm[w] = bits;
        tot += __popc(bits);
      }
      bmcount = tot;
      cur = 0;
      __syncwarp();
    };

    // serial insert of (cx -> slot cv) by the calling lane, cuckoo kicks; false if homeless
    auto slow_insert = [&](KT cx, uint32_t cv) -> bool {
      uint32_t prev = 0xffffffffu;
      for (int step = 0; step < SS_MAX_KICKS; ++step) {
        uint32_t b1, b2, fp;
        key_hash<ET>(en, cx, seed, NB, b1, b2, fp);
        ET f0, f1, f2, f3;
        load_bucket(T, b1, f0, f1);
        load_bucket(T, b2, f2, f3);
        const uint32_t fi = free_entry(f0, f1, f2, f3, b1, b2);
        if (fi != 0xffffffffu) {
          T[fi] = en.make(fp, cv);
          set_pos(cv, fi, b1);
          return true;
        }
        const uint32_t kb = (b1 != prev) ? b1 : b2;
        const uint32_t idx = 2 * kb + ((step ^ (cv & 1)) & 1);
        const ET e = T[idx];
        T[idx] = en.make(fp, cv);
        set_pos(cv, idx, b1);
        cv = en.slot(e);
        cx = keys[cv];
        prev = kb;
      }
      return false;
    };
    auto rehash = [&](uint32_t nslots) {  // rebuild the whole index under a new seed (all lanes)
      bool ok = false;
      while (!ok) {
        ++seed;
        for (uint32_t i = lane; i < NE; i += 32) T[i] = EMPTY;
        __syncwarp();
        uint32_t okl = 1;
        if (lane == 0)
          for (uint32_t t = 0; t < nslots && okl; ++t) okl = slow_insert(keys[t], t);
        ok = __shfl_sync(PSS_FULL, okl, 0) != 0;
        __syncwarp();
      }
    };
    // Fast insert of x -> slot v into the snapshot's free entry `fi`, then read back;
    // lanes that lost a race (or had no free entry) insert serially. `nslots` bounds a rehash.
    auto insert_all = [&](bool ins, KT x, uint32_t v, uint32_t fi, uint32_t fp, uint32_t nslots) {
      const ET mine = en.make(fp, v);
      const bool tryfi = ins && fi != 0xffffffffu;
      // lanes that picked the same free entry: write, then read back (a match instruction here
      // measured 12 % slower: __match_any_sync is the costliest instruction of a step)
      ET* const tp = T + (tryfi ? fi : 0u);
      if (tryfi) *tp = mine;
      __syncwarp();
      const bool won = tryfi && *tp == mine;
      if (!PACKED) {  // packed counters were written with the position bits of fi
        PT* const pp = pos + v;
        if (won) *pp = (PT)fi;
      }
      uint32_t need = __ballot_sync(PSS_FULL, ins && !won);
      SS_STAT(2, __popc(need));
      SS_STAT(10, __popc(__ballot_sync(PSS_FULL, ins && fi == 0xffffffffu)));
      if (need) {
        __syncwarp();  // the serial inserts see every fast-path write and deletion
        bool failed = false;
        while (need) {
          const uint32_t l = __ffs(need) - 1;
          uint32_t okl = 1;
          if (lane == l) okl = slow_insert(x, v);
          failed |= __shfl_sync(PSS_FULL, okl, l) == 0;
          __syncwarp();
          need &= need - 1;
        }
        if (failed) {
          SS_STAT(3, 1);
          rehash(nslots);
        }
      }
    };

    if (L) {
      const uint64_t gbase = aligned ? (lo & ~(uint64_t)(E - 1)) : lo;
      const uint32_t roff = (uint32_t)(lo - gbase);  // ring offset of item lo
      const uint32_t total = (roff + L + ST - 1) / ST;
      auto issue = [&](uint32_t g, uint32_t sl) {  // stage g into ring slot sl (= g % NSTAGE)
        const uint64_t a0 = gbase + (uint64_t)g * ST;
        KT* dst = ring + sl * ST;
        if (a0 + ST <= hi && a0 + ST <= nfloor) {  // an interior stage: one full bulk copy
          if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(&bars[sl], SS_STAGE_BYTES);
            bulk_g2s(dst, A + a0, SS_STAGE_BYTES, &bars[sl]);
          }
          return;
        }
        const uint64_t b0 = min(a0 + ST, hi);
        uint64_t be = (b0 + E - 1) & ~(uint64_t)(E - 1);
        if (be > nfloor) be = nfloor;
        if (be < a0) be = a0;
        const uint32_t bytes = (uint32_t)((be - a0) * sizeof(KT));
        if (lane == 0) {
          fence_proxy_async();
          if (bytes) {
            mbar_arrive_expect_tx(&bars[sl], bytes);
            bulk_g2s(dst, A + a0, bytes, &bars[sl]);
          } else {
            mbar_arrive(&bars[sl]);
          }
        }
        for (uint64_t t = be + lane; t < b0; t += 32) dst[t - a0] = A[t];  // unaligned tail
      };
      // stages 0..NFL in flight; waiting for stage g frees the slot of stage g-KEEP (a window
      // spans at most two stages), which is refilled with stage g+NSTAGE-2
      for (uint32_t g = 0; g < min(total, NFL + 1); ++g) issue(g, g);
      uint32_t ready = 0;      // stages waited for
      uint32_t rsl = 0;        // ring slot of stage `ready`
      uint32_t ready_end = 0;  // items of the partition available in the ring: [0, ready_end)
      auto ensure = [&](uint32_t end) {  // items [0, end) resident in the ring
        if (end > ready_end) {
          __syncwarp();
          while (end > ready_end) {
            mbar_wait(&bars[rsl], (phasebits >> rsl) & 1u);
            phasebits ^= 1u << rsl;
            // stage ready + NFL goes into the slot of stage ready - KEEP (consumed)
            const uint32_t nx = ready + NFL;
            uint32_t nsl = rsl + NFL;
            if (nsl >= NST) nsl -= NST;
            if (nx >= NFL + 1 && nx < total) issue(nx, nsl);
            ++ready;
            rsl = rsl + 1 == NST ? 0u : rsl + 1;
            ready_end = min(L, ready * ST - roff);
          }
          __syncwarp();
        }
      };

      // lookup of x: slot s (-1 if not monitored), its packed count ce, the first free entry fi
      // of its buckets (insert target) and its fingerprint fp
      auto lookup = [&](KT x, bool act, int32_t& s, uint32_t& ce, uint32_t& fi, uint32_t& fp,
                        uint32_t& fbits) {
        uint32_t b1, b2;
        key_hash<ET>(en, x, seed, NB, b1, b2, fp);
        ET e0, e1, e2, e3;
        bool q0, q1, q2, q3;
        if constexpr (sizeof(ET) == 2 && SB > 0) {  // a bucket word's two entries at once
          const uint32_t v1 = reinterpret_cast<const uint32_t*>(T)[b1];
          const uint32_t v2 = reinterpret_cast<const uint32_t*>(T)[b2];
          e0 = (ET)v1;
          e1 = (ET)(v1 >> 16);
          e2 = (ET)v2;
          e3 = (ET)(v2 >> 16);
          const uint32_t fm = (en.fmask << en.sb) * 0x10001u;  // fingerprint fields
          const uint32_t tg = (fp << en.sb) * 0x10001u;
          const uint32_t d1 = (v1 ^ tg) & fm, d2 = (v2 ^ tg) & fm;
          q0 = (d1 & 0xffffu) == 0;
          q1 = (d1 >> 16) == 0;
          q2 = (d2 & 0xffffu) == 0;
          q3 = (d2 >> 16) == 0;
        } else {
          load_bucket(T, b1, e0, e1);
          load_bucket(T, b2, e2, e3);
          q0 = en.fp_eq(e0, fp);
          q1 = en.fp_eq(e1, fp);
          q2 = en.fp_eq(e2, fp);
          q3 = en.fp_eq(e3, fp);
        }
        ET sel = q3 ? e3 : EMPTY;
        sel = q2 ? e2 : sel;
        sel = q1 ? e1 : sel;
        sel = q0 ? e0 : sel;
        const uint32_t t0 = sel == EMPTY ? 0u : en.slot(sel);
        const KT kx = keys[t0];
        ce = cnt[t0];
        const bool hit = act && sel != EMPTY && kx == x;
        s = hit ? (int32_t)t0 : -1;
        // a fingerprint match whose key differs: check the other matches in order
        bool amb = act && !hit && sel != EMPTY;
        while (__ballot_sync(PSS_FULL, amb)) {
          SS_STAT(4, 1);
          if (amb) {
            // drop the first remaining match and take the next one
            if (q0) q0 = false;
            else if (q1) q1 = false;
            else if (q2) q2 = false;
            else q3 = false;
            ET nx = q3 ? e3 : EMPTY;
            nx = q2 ? e2 : nx;
            nx = q1 ? e1 : nx;
            nx = q0 ? e0 : nx;
            if (nx == EMPTY) {
              amb = false;
            } else {
              const uint32_t t = en.slot(nx);
              if (keys[t] == x) {
                s = (int32_t)t;
                ce = cnt[t];
                amb = false;
              }
            }
          }
        }
        fi = free_entry(e0, e1, e2, e3, b1, b2);
        fbits = PACKED ? pos_bits(fi, b1) : 0u;
      };

      uint32_t q = 0;       // items consumed
      // The specialized kernel (SB > 0) keeps the ring position of item q, (roff + q) % RING,
      // incrementally and compares both fingerprints of a bucket word at once; the same two
      // changes measured 2-5 % slower in the runtime-layout kernel (k = 2000), which keeps the
      // modulo and the per-entry compares.
      uint32_t rq = roff;
      auto ring_at = [&](uint32_t lane_off) -> KT {
        if constexpr (SB > 0) {
          const uint32_t i = rq + lane_off;
          return ring[i < RING ? i : i - RING];
        } else {
          return ring[(roff + q + lane_off) % RING];
        }
      };
      auto advance = [&](uint32_t c) {
        q = q + c;
        if constexpr (SB > 0) {
          rq += c;
          if (rq >= RING) rq -= RING;
        }
      };
      // ---- fill phase: free counters are taken in slot order (R2)
      while (q < L && size < k) {
        const uint32_t nv = min(32u, L - q);
        ensure(q + nv);
        const bool act = lane < nv;
        const uint32_t amask = nv >= 32 ? PSS_FULL : ((1u << nv) - 1u);
        const KT x = ring_at(lane);
        const uint32_t grp = __match_any_sync(PSS_FULL, x) & amask;
        int32_t s;
        uint32_t ce, fi, fp, fbits;
        lookup(x, act, s, ce, fi, fp, fbits);
        const bool hit = s >= 0;
        const bool leader = act && (grp & ltm) == 0;
        const uint32_t missL = __ballot_sync(PSS_FULL, leader && !hit);
        uint32_t c = nv;
        const uint32_t freec = k - size;
        if ((uint32_t)__popc(missL) > freec) c = nth_set(missL, freec);
        const uint32_t pm = c >= 32 ? PSS_FULL : ((1u << c) - 1u);
        const bool inpre = leader && lane < c;
        const uint32_t mult = __popc(grp & pm);
        if (inpre && hit) cnt[s] = ce + mult;
        const bool ins = inpre && !hit;
        const uint32_t v = size + __popc(missL & ltm);
        if (ins) {
          keys[v] = x;
          cnt[v] = mult | fbits;
          if (!PACKED) err[v] = 0;
        }
        const uint32_t grow = __popc(missL & pm);
        insert_all(ins, x, v, fi, fp, size + grow);
        size += grow;
        advance(c);
        SS_STAT(8, 1);
        SS_STAT(1, c);
        __syncwarp();
      }
      // ---- level-pinned bypass (BYP). While the minimum level is m, a counter with count > m
      // is never evicted (P:82 evicts a counter with the least count) and a hit only raises it, so
      // the hits of such a key commute with every other update of the level: they change no
      // decision (victims are the slots at count m, in slot order) and can be counted aside. At
      // the start of a level the launch's frequent keys (hot.cu) that are monitored with count > m
      // are *pinned* for the level: the raw items are classified 32 at a time, occurrences of
      // pinned keys add to hc[] and the others (cold) are queued, with their positions, for the
      // exact rule, which takes its windows from the queue. Classification runs ahead of the
      // exact cursor, so when a level ends (after the exact step that emptied B_m) the pinned
      // occurrences at or after the oldest queued item are taken back, hc[] is added to the
      // counters (now the true counts at that position), the next level and its pins are found,
      // and classification restarts from that position. Exact for any table of keys.
      uint32_t R = q, qh = 0, qt = 0;  // raw cursor; cold queue [qh, qt)
      uint32_t rR = 0;                 // ring position of raw item R
      uint32_t limR = 0;               // a classified window must end at or before this position
      uint32_t pm0 = 0, pm1 = 0;       // pinned keys (bit = rank in the table)
      uint32_t ps0 = 0, ps1 = 0;       // the slots of this lane's pinned keys (lane, lane + 32)
      const uint32_t hc_addr = smem_u32(hc);
      // table entry of x and its hash; rank of x from them (>= HOT_MAX: not in the table)
      auto hot_hash = [&](KT x) -> uint32_t { return (uint32_t)x * hseed; };
      auto hot_entry = [&](uint32_t ha) -> uint32_t { return __ldg(htab + (ha >> (32 - HOT_LOG))); };
      auto hot_rank = [&](uint32_t e, uint32_t ha) -> uint32_t {
        return __funnelshift_l(e ^ ha, e ^ ha, HOT_LOG);
      };
      auto is_pinned = [&](uint32_t hr) -> bool {  // bit hr of pm1:pm0, 0 for hr >= 64
        uint32_t r;
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%1, %2};\n\tshr.b64 t, t, %3;\n\t"
            "cvt.u32.u64 %0, t;\n\t}"
            : "=r"(r)
            : "r"(pm0), "r"(pm1), "r"(hr));
        return r & 1u;
      };
      auto raw_at = [&](uint32_t t) -> KT { return ring[(roff + t) % RING]; };
      auto set_R = [&](uint32_t t) {
        R = t;
        rR = (roff + t) % RING;
      };
      // The window [R, R + nv) may be classified if its last stage is at most one past the stage
      // of the oldest queued item (waiting for a stage refills the slot KEEP stages back).
      auto upd_lim = [&]() {
        const uint32_t hp = qt != qh ? cqp[qh & (SS_CQ - 1)] : R;
        limR = ((roff + hp) / ST + KEEP) * ST - roff;
      };
      // second half of a window's classification (x at lane, its table entry and hash loaded
      // earlier): count pinned occurrences, queue the others
      auto classify_tail = [&](KT x, uint32_t e, uint32_t ha, bool act, uint32_t nv) {
        const uint32_t hr = hot_rank(e, ha);
        const bool pin = act && is_pinned(hr);
        if (pin) asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hc_addr + 4 * hr) : "memory");
        const bool cold = act && !pin;
        const uint32_t cm = __ballot_sync(PSS_FULL, cold);
        const uint32_t o = (qt + __popc(cm & ltm)) & (SS_CQ - 1);
        if (cold) {
          cq[o] = x;
          cqp[o] = (uint16_t)(R + lane);
        }
        qt += __popc(cm);
        R += nv;
        rR += nv;
        if (rR >= RING) rR -= RING;
        SS_STAT(14, 1);
      };
      auto ring_raw = [&](uint32_t off) -> KT {  // raw item R + off + lane (off + lane < RING)
        const uint32_t i = rR + off + lane;
        return ring[i < RING ? i : i - RING];
      };
      auto classify = [&]() {
        const uint32_t nv = min(32u, L - R);
        ensure(R + nv);
        const KT x = ring_raw(0);
        const uint32_t ha = hot_hash(x);
        classify_tail(x, hot_entry(ha), ha, lane < nv, nv);
        __syncwarp();
      };
      // a level ended (or the fill phase did): true counts at the oldest queued item, the next
      // level, its pins; classification restarts there
      auto level_b = [&]() {
        if constexpr (BYP) {
          __syncwarp();
          const uint32_t p = qt != qh ? cqp[qh & (SS_CQ - 1)] : R;
          for (uint32_t t0 = p; t0 < R; t0 += 32) {  // take the look-ahead back
            const uint32_t t = t0 + lane;
            if (t < R) {
              const uint32_t ha = hot_hash(raw_at(t));
              const uint32_t hr = hot_rank(hot_entry(ha), ha);
              if (is_pinned(hr)) atomicSub(&hc[hr], 1u);
            }
          }
          __syncwarp();
          if ((pm0 >> lane) & 1u) cnt[ps0] += hc[lane];
          if ((pm1 >> lane) & 1u) cnt[ps1] += hc[lane + 32];
          hc[lane] = 0;
          hc[lane + 32] = 0;
          __syncwarp();
          new_level();
          int32_t s;
          uint32_t ce, fi, fp, fbits;
          lookup((KT)hk0, lane < nhot, s, ce, fi, fp, fbits);
          const bool p0 = s >= 0 && (ce & CM) > m;
          ps0 = p0 ? (uint32_t)s : 0u;
          pm0 = __ballot_sync(PSS_FULL, p0);
          lookup((KT)hk1, lane + 32 < nhot, s, ce, fi, fp, fbits);
          const bool p1 = s >= 0 && (ce & CM) > m;
          ps1 = p1 ? (uint32_t)s : 0u;
          pm1 = __ballot_sync(PSS_FULL, p1);
          set_R(p);
          qt = qh;
          upd_lim();
        }
      };
      if (size == k) {
        if (BYP && nhot)
          level_b();
        else
          new_level();
      }

      // ---- all k counters occupied: misses evict the lowest slots of B_m (R1)
#ifdef PSS_STATS
      long long tk = 0, ph1 = 0, ph2 = 0, ph3 = 0, ph4 = 0, ph5 = 0;
#endif
      // one step; F: a full 32-item window (every step but the block's last), compiled separately
      // so that the window-length predicates fold away
      auto full_step = [&](auto full, auto fromq) {
        constexpr bool F = decltype(full)::value;
        constexpr bool Q = decltype(fromq)::value;  // the window is the head of the cold queue
        const uint32_t nv = F ? 32u : (Q ? qt - qh : min(32u, L - q));
        if constexpr (!Q) ensure(q + nv);
#ifdef PSS_STATS
        tk = clock64();
#endif
        const bool act = F || lane < nv;
        const uint32_t amask = F || nv >= 32 ? PSS_FULL : ((1u << nv) - 1u);
        KT x;
        if constexpr (Q)
          x = cq[(qh + lane) & (SS_CQ - 1)];
        else
          x = ring_at(lane);
        // bypass: up to two raw windows are classified inside a full step -- their loads are
        // issued here, their results are consumed after the step's updates, so the
        // classification's latencies overlap the step's dependent chain
        bool doA = false, doB = false;
        KT xA = 0, xB = 0;
        uint32_t hA = 0, hB = 0, eA = 0, eB = 0;
        if constexpr (Q && F) {
          const uint32_t room = SS_CQ - (qt - qh);
          const uint32_t lim = min(L, limR);
          doA = R + 32u <= lim && room >= 32u;
          doB = R + 64u <= lim && room >= 64u;
          if (doA) ensure(R + (doB ? 64u : 32u));
          xA = ring_raw(0);
          xB = ring_raw(32);
          hA = hot_hash(xA);
          hB = hot_hash(xB);
          eA = hot_entry(hA);
          eB = hot_entry(hB);
        }
        // the match is issued first and its result first used after the lookups, so that its
        // latency (it grows with the number of distinct keys) overlaps them
        const uint32_t grp_all = __match_any_sync(PSS_FULL, x);

        // victims for this step (independent of the lookups): lane j holds the j-th next slot
        // of B_m at or after the cursor (two bitmap words) and the index entry of its item
        uint32_t w0 = cur >> 5;
        uint32_t wa = bm[w0] & (0xffffffffu << (cur & 31u));
        while (wa == 0) wa = bm[++w0];  // bmcount >= 1: some later word has a bit
        const uint32_t wb = bm[w0 + 1];
        const uint32_t ca = __popc(wa);
        const uint32_t navail = min(32u, ca + __popc(wb));
        const uint32_t ra = __popc(wa & ltm), rb = ca + __popc(wb & ltm);
        if ((wa >> lane) & 1u) vic[ra] = w0 * 32 + lane;
        if (((wb >> lane) & 1u) && rb < 32) vic[rb] = w0 * 32 + 32 + lane;
        __syncwarp();
        const uint32_t myvic = vic[lane];
        uint32_t myop;
        if (PACKED) {  // the victim's entry: its key's bucket pair and the position bits
          const uint32_t tv = lane < navail ? myvic : 0;
          const KT vk = keys[tv];
          const uint32_t vc = cnt[tv];
          uint32_t vb1, vb2, vfp;
          key_hash<ET>(en, vk, seed, NB, vb1, vb2, vfp);
          myop = 2 * ((vc >> 31) ? vb2 : vb1) + ((vc >> 30) & 1u);
        } else {
          myop = pos[lane < navail ? myvic : 0];
        }

        int32_t s;
        uint32_t ce, fi, fp, fbits;
        lookup(x, act, s, ce, fi, fp, fbits);
        SS_TICK(ph2, tk, ce ^ (uint32_t)s ^ myop);
        const uint32_t grp = grp_all & amask;
        const bool hit = s >= 0;
        const uint32_t cs = ce & CM;
        const bool leader = act && (grp & ltm) == 0;
        const uint32_t missL = __ballot_sync(PSS_FULL, leader && !hit);
        const uint32_t rank = __popc(missL & ltm);
        const uint32_t M = __popc(missL);
        const uint32_t Ms = min(M, navail);
        const uint32_t vmax = __shfl_sync(PSS_FULL, myvic, (Ms ? Ms : 1) - 1);
        uint32_t c = nv;
        if (Ms < M) {
          c = nth_set(missL, Ms);  // no victim left for this miss
          SS_STAT(5, 1);
        }
        // hazard: a victim slot whose item is also hit in the window
        const bool conf = leader && hit && Ms && cs == m && (uint32_t)s <= vmax;
        if (__ballot_sync(PSS_FULL, conf)) {
          uint32_t cpos = 32;
          if (conf) {
            uint32_t rr = 0;
            while (vic[rr] != (uint32_t)s) ++rr;
            uint32_t mm = missL;
            for (uint32_t i = 0; i < rr; ++i) mm &= mm - 1u;
            const uint32_t pr = (uint32_t)(__ffs(mm) - 1);
            cpos = max(lane, pr);
          }
          c = min(c, __reduce_min_sync(PSS_FULL, cpos));
          SS_STAT(6, 1);
        }
        const uint32_t pm = c >= 32 ? PSS_FULL : ((1u << c) - 1u);
        const bool inpre = leader && lane < c;
        const uint32_t mult = __popc(grp & pm);
        SS_TICK(ph3, tk, mult ^ vmax);
        // hits: count += multiplicity; a hit counter leaves B_m
        const bool hup = inpre && hit;
        const bool hitm = hup && cs == m;
        uint32_t* const cptr = cnt + (hit ? (uint32_t)s : 0u);
        const uint32_t cnew = ce + mult;
        if (hup) *cptr = cnew;
        if (hitm) atomicAnd(&bm[(uint32_t)s >> 5], ~(1u << ((uint32_t)s & 31u)));
        // misses: the victim takes the item, count m + multiplicity ("incremented by one" then
        // further hits in the window), error m; its old item leaves the index
        const bool ev = inpre && !hit;
        const uint32_t v = __shfl_sync(PSS_FULL, myvic, rank & 31u);
        const uint32_t op = __shfl_sync(PSS_FULL, myop, rank & 31u);
        const uint32_t vnew = PACKED ? ((m + mult) | (m << cb) | fbits) : (m + mult);
        ET* const tdel = T + op;
        KT* const kptr = keys + v;
        uint32_t* const vptr = cnt + v;
        if (ev) {
          *tdel = EMPTY;
          *kptr = x;
          *vptr = vnew;
          if (!PACKED) err[v] = m;
        }
        insert_all(ev, x, v, fi, fp, size);
        SS_TICK(ph4, tk, v);
        const uint32_t Mp = __popc(missL & pm);
        const uint32_t last = __shfl_sync(PSS_FULL, myvic, (Mp ? Mp : 1) - 1);
        if (Mp) cur = last + 1;
        bmcount -= __popc(__ballot_sync(PSS_FULL, hitm)) + Mp;
        if constexpr (Q) {
          qh += c;
          if constexpr (F) {
            if (doA) classify_tail(xA, eA, hA, true, 32u);
            if (doB) classify_tail(xB, eB, hB, true, 32u);
          }
          __syncwarp();
          upd_lim();
        } else {
          advance(c);
        }
        SS_STAT(0, 1);
        SS_STAT(9, Mp);
        SS_STAT(1, c);
        if (bmcount == 0) {
          SS_STAT(7, 1);
          if constexpr (Q)
            level_b();
          else
            new_level();
        }
        __syncwarp();
        SS_TICK(ph5, tk, bmcount);
      };
      if (BYP && nhot) {
        if constexpr (BYP) {
          while (size == k) {
            while (qt - qh < 32u && R < L && R + min(32u, L - R) <= limR) classify();
            upd_lim();
            if (qt == qh) {
              if (R >= L) break;
              continue;  // an empty queue never blocks classification
            }
            if (qt - qh >= 32u)
              full_step(std::true_type{}, std::true_type{});
            else
              full_step(std::false_type{}, std::true_type{});
          }
          // the block's end: nothing is queued or ahead, the pinned counts are final
          if ((pm0 >> lane) & 1u) cnt[ps0] += hc[lane];
          if ((pm1 >> lane) & 1u) cnt[ps1] += hc[lane + 32];
          __syncwarp();
        }
      } else {
        while (q + 32 <= L) full_step(std::true_type{}, std::false_type{});
        while (q < L) full_step(std::false_type{}, std::false_type{});
      }
#ifdef PSS_STATS
      SS_STAT(11, ph1);
      SS_STAT(12, ph2);
      SS_STAT(13, ph3);
      SS_STAT(14, ph4);
      SS_STAT(15, ph5);
#endif
    }

    // ---- dump the leaf in slot order
    KT* oi = reinterpret_cast<KT*>(a.items) + (size_t)r * k;
    uint32_t* oc = a.counts + (size_t)r * k;
    uint32_t* oe = a.errs + (size_t)r * k;
    for (uint32_t t = lane; t < size; t += 32) {
      const uint32_t ce = cnt[t];
      oi[t] = keys[t];
      oc[t] = ce & CM;
      oe[t] = PACKED ? (ce & ~POSM) >> cb : err[t];
    }
    if (lane == 0) a.sizes[r] = size;
    if (a.leaf_flags) {  // publish leaf r to the overlapping tree kernel
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release(a.leaf_flags + r, 1u);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------ host side
struct SSPlan {
  bool gstate, packed;
  bool byp;   // level-pinned bypass: u32 keys, packed counters, long blocks (or forced)
  uint32_t cb, sb, fmask;
  SSLayout L;
  size_t smem;
  int grid;   // CTAs of a launch over all P partitions
  int slots;  // resident CTAs the device holds
};

template <typename KT, typename ET, bool G, bool PK, bool BY = false>
static int ss_blocks_per_sm(size_t smem, const DevInfo& d) {
  auto kern = ss_summarize_kernel<KT, ET, G, PK, 0, 0, BY>;
  if (smem > (size_t)d.smem_optin || allow_max_smem(kern, d) != cudaSuccess) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return nb;  // 0: does not fit
}

// PSS_BYPASS: 0 = never use the level-pinned bypass, 2 = use it whenever the kernel supports the
// shape and keep any table (test hook: small blocks, few hot keys); unset/1 = the default gate
static int ss_bypass_mode() {
  const char* s = std::getenv("PSS_BYPASS");
  return s ? std::atoi(s) : 1;
}

static SSPlan ss_plan(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d,
                      bool want_byp = true) {
  SSPlan p;
  // count + error in one word: counts <= Lmax need cb bits, errors <= Lmax / k the rest
  const uint64_t Lmax = (n + P - 1) / P;
  p.cb = 1;
  while (p.cb < 32 && (1ull << p.cb) <= Lmax) ++p.cb;
  p.packed = p.cb < 30 && (Lmax / k) < (1ull << (30 - p.cb));  // bits 30-31: index position
  // 16-bit entries: the slot field's all-ones value must exceed k - 1
  uint32_t sb = 1;
  while ((1u << sb) - 1u < k) ++sb;
  const double dl = ss_debug_load();
  uint32_t NB = ss_buckets(k, dl > 0 ? dl : SS_LOAD);
  const int bm = ss_bypass_mode();
  p.byp = want_byp && kb == 4 && p.packed && bm != 0 && Lmax <= 65536 &&
          (bm == 2 || (Lmax >= 8192 && k >= 128));
  SSLayout Ls = ss_layout(k, kb, 2, p.packed, NB, p.byp);
  p.gstate = k > SS_K_SMALL || Ls.total > SS_SMEM_STATE_MAX;
  if (p.gstate) p.byp = false;
  if (!p.gstate) {
    p.sb = sb;
    p.fmask = (1u << (16 - sb)) - 1u;
    size_t pad = 0;
    if (const char* ps = std::getenv("PSS_DEBUG_SMEM_PAD"))  // experiment hook: fewer warps/SM
      pad = (size_t)std::atoll(ps);
    const size_t ringb = p.byp ? SS_BYP_RING_BYTES + SS_BYP_BAR_BYTES : SS_RING_BYTES + SS_BAR_BYTES;
    auto smem_of = [&](const SSLayout& L) { return ringb + L.total + pad; };
    auto blocks = [&](size_t smem) {
      if (p.byp) return ss_blocks_per_sm<uint32_t, uint16_t, false, true, true>(smem, d);
      if (p.packed)
        return kb == 4 ? ss_blocks_per_sm<uint32_t, uint16_t, false, true>(smem, d)
                       : ss_blocks_per_sm<uint64_t, uint16_t, false, true>(smem, d);
      return kb == 4 ? ss_blocks_per_sm<uint32_t, uint16_t, false, false>(smem, d)
                     : ss_blocks_per_sm<uint64_t, uint16_t, false, false>(smem, d);
    };
    // occupancy of the layout without the bypass arrays at the default load; the bypass keeps it
    // by giving up index entries (down to load 0.36) rather than a warp per SM
    int nb = blocks(SS_RING_BYTES + SS_BAR_BYTES + ss_layout(k, kb, 2, p.packed, NB, false).total + pad);
    // The shared memory left over at this occupancy goes to the index: the largest bucket count
    // that keeps `nb` warps per SM (fewer fingerprint collisions and serial inserts).
    if (dl == 0 && nb > 0) {
      uint32_t lo = p.byp ? ss_buckets(k, 0.36) : NB, hi = 2 * NB;
      const int nlo = blocks(smem_of(ss_layout(k, kb, 2, p.packed, lo, p.byp)));
      if (nlo < nb) nb = nlo;
      while (lo < hi && nb > 0) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (blocks(smem_of(ss_layout(k, kb, 2, p.packed, mid, p.byp))) >= nb)
          lo = mid;
        else
          hi = mid - 1;
      }
      NB = lo;
      Ls = ss_layout(k, kb, 2, p.packed, NB, p.byp);
    } else {
      nb = blocks(smem_of(Ls));
    }
    p.L = Ls;
    p.smem = smem_of(Ls);
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)std::max(nb, 1) * d.sms);
    p.slots = (int)std::min<uint64_t>((uint64_t)nb * d.sms, 1u << 30);
  } else {
    p.packed = false;
    p.sb = 32;
    p.fmask = 0xffffffffu;
    p.L = ss_layout(k, kb, 8, false, ss_buckets(k, dl > 0 ? dl : 0.32));
    p.smem = SS_RING_BYTES + SS_BAR_BYTES;
    // Warps per SM of the global-state kernel. It is bound by the latency of its L2/DRAM accesses
    // (IPC 0.68 at 8 warps per SM), so it takes all 32 CTA slots of an SM (C4-k5000 without K1h:
    // 8.6 -> 3.6 ms, C4-k20000 9.5 -> 4.0 ms) as long as the states fit a 4 GiB workspace.
    const uint64_t budget = 4ull << 30;
    int gw = (int)std::min<uint64_t>(32, std::max<uint64_t>(8, budget / (p.L.total * (uint64_t)d.sms)));
    if (const char* gs = std::getenv("PSS_DEBUG_GSTATE_WARPS")) gw = std::max(1, std::atoi(gs));
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)gw * d.sms);
    p.slots = gw * d.sms;
  }
  if (p.grid < 1) p.grid = 1;
  return p;
}

// workspace: K1's partition queues, the histogram kernel's queues and per-leaf flags, K1's
// global-memory states (large k)
struct SumWs {
  size_t q, hq, flagged, hot, g, total;
};
static SumWs sum_ws(const SSPlan& p, uint32_t P) {
  SumWs w;
  Bump b;
  w.q = b.take<uint32_t>(SS_MAX_RANGES);
  w.hq = b.take<uint32_t>(SS_MAX_RANGES);
  w.flagged = b.take<unsigned char>(P);
  w.hot = p.byp ? b.take<uint32_t>((size_t)HOT_WORDS * SS_MAX_RANGES) : 0;
  w.g = p.gstate ? b.take<unsigned char>(p.L.total * (size_t)p.grid) : 0;
  w.total = b.bytes();
  return w;
}

size_t summarize_ws(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  return sum_ws(ss_plan(n, kb, k, P, d), P).total;
}

cudaError_t summarize_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P,
                             void* items, uint32_t* counts, uint32_t* errs, uint32_t* sizes,
                             void* ws, cudaStream_t s, const DevInfo& d, uint32_t r0,
                             uint32_t r1, uint32_t qi, uint32_t T, uint32_t* leaf_flags,
                             bool pdl) {
  SSPlan p = ss_plan(n, kb, k, P, d);
  if (r1 > P) r1 = P;
  if (r0 >= r1 || qi >= SS_MAX_RANGES) return cudaErrorInvalidValue;
  int grid = (int)std::min<uint64_t>(r1 - r0, (uint64_t)p.grid);
  const SumWs W = sum_ws(p, P);
  unsigned char* w = static_cast<unsigned char*>(ws);
  // blocks with at most k distinct keys: the histogram kernel; K1 takes the others
  const bool hist = hist_used(n, kb, k, P, d);
  if (hist) {
    cudaError_t e = hist_launch(A, n, kb, k, P, items, counts, errs, sizes,
                                reinterpret_cast<uint32_t*>(w + W.hq) + qi, w + W.flagged, s, d,
                                r0, r1, T, leaf_flags);
    if (e != cudaSuccess) return e;
  }
  if (epoch_used(n, kb, k, P, d))
    return epoch_launch(A, n, k, P, items, counts, errs, sizes,
                        reinterpret_cast<uint32_t*>(w + W.q) + qi, hist ? w + W.flagged : nullptr,
                        s, d, r0, r1, T, leaf_flags, pdl);
  SumArgs a;
  a.skip = hist ? w + W.flagged : nullptr;
  a.A = A;
  a.n = n;
  a.k = k;
  a.P = P;
  a.T = T;
  a.leaf_flags = leaf_flags;
  a.pdl = pdl ? 1 : 0;
  a.r0 = r0;
  a.r1 = r1;
  a.items = items;
  a.counts = counts;
  a.errs = errs;
  a.sizes = sizes;
  a.queue = reinterpret_cast<uint32_t*>(w + W.q) + qi;
  a.gstate = p.gstate ? w + W.g : nullptr;
  a.gstride = p.L.total;
  a.o_cnt = p.L.cnt;
  a.o_err = p.L.err;
  a.o_pos = p.L.pos;
  a.o_bm = p.L.bm;
  a.o_vic = p.L.vic;
  a.o_T = p.L.T;
  a.NB = p.L.NB;
  a.cb = p.cb;
  a.sb = p.sb;
  a.fmask = p.fmask;
  a.o_hc = p.L.hc;
  a.o_cq = p.L.cq;
  a.o_cqp = p.L.cqp;
  a.hot = nullptr;
  cudaError_t e = cudaMemsetAsync(a.queue, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  if (p.byp) {  // K0: the frequent keys of the launch's range of A (hot.cu)
    auto bound = [&](uint64_t r) -> uint64_t {  // first item of partition r (the kernel's bounds)
      if (T <= 1) return (uint64_t)((unsigned __int128)r * n / P);
      const uint64_t Pp = P / T, pr = r / T, t = r % T;
      if (pr >= Pp) return n;
      const uint64_t b0 = pr * n / Pp, Lp = (pr + 1) * n / Pp - b0;
      return b0 + t * Lp / T;
    };
    const uint64_t lo = bound(r0), hi = bound(r1);
    uint32_t* hot = reinterpret_cast<uint32_t*>(w + W.hot) + (size_t)qi * HOT_WORDS;
    if (hi > lo) {
      e = hot_sample_launch(A, lo, hi, hot, ss_bypass_mode() == 2, s);
      if (e != cudaSuccess) return e;
      a.hot = hot;
    }
  }
  if (a.hot) {
    // Whether the range has a table is known on the device only: the bypass kernel is launched
    // first and returns at once without one; the plain kernel (its own layout: no queue, a
    // larger index) follows and returns at once if the bypass kernel took the range.
    const int spec = p.cb == 17 && p.sb == 10 ? 10 : 0;
    SumArgs ab = a;
    ab.pdl = 0;
    if (spec == 10) {
      allow_max_smem(ss_summarize_kernel<uint32_t, uint16_t, false, true, 10, 17, true>, d);
      ss_summarize_kernel<uint32_t, uint16_t, false, true, 10, 17, true><<<grid, 32, p.smem, s>>>(ab);
    } else {
      ss_summarize_kernel<uint32_t, uint16_t, false, true, 0, 0, true><<<grid, 32, p.smem, s>>>(ab);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    p = ss_plan(n, kb, k, P, d, false);
    grid = (int)std::min<uint64_t>(r1 - r0, (uint64_t)p.grid);
    a.gstride = p.L.total;
    a.o_cnt = p.L.cnt;
    a.o_err = p.L.err;
    a.o_pos = p.L.pos;
    a.o_bm = p.L.bm;
    a.o_vic = p.L.vic;
    a.o_T = p.L.T;
    a.NB = p.L.NB;
  }
  if (!p.gstate) {
    if (p.packed) {
      // the common shape compiled with its layout constants: k in [512, 1023] (slot bits 10) and
      // blocks of 2^16 .. 2^17 - 1 keys (count bits 17). (Slot bits 11, k in [1024, 2047], was
      // measured too: 3 % faster on evicting inputs, 4-7 % slower on the fill-heavy C3 s >= 1.5.)
      const int spec = p.cb == 17 && p.sb == 10 ? 10 : 0;
      if (spec == 10)
        allow_max_smem(kb == 4 ? ss_summarize_kernel<uint32_t, uint16_t, false, true, 10, 17>
                               : ss_summarize_kernel<uint64_t, uint16_t, false, true, 10, 17>, d);
      if (kb == 4) {
        if (spec == 10)
          ss_summarize_kernel<uint32_t, uint16_t, false, true, 10, 17><<<grid, 32, p.smem, s>>>(a);
        else
          ss_summarize_kernel<uint32_t, uint16_t, false, true><<<grid, 32, p.smem, s>>>(a);
      } else {
        if (spec == 10)
          ss_summarize_kernel<uint64_t, uint16_t, false, true, 10, 17><<<grid, 32, p.smem, s>>>(a);
        else
          ss_summarize_kernel<uint64_t, uint16_t, false, true><<<grid, 32, p.smem, s>>>(a);
      }
    } else {
      if (kb == 4)
        ss_summarize_kernel<uint32_t, uint16_t, false, false><<<grid, 32, p.smem, s>>>(a);
      else
        ss_summarize_kernel<uint64_t, uint16_t, false, false><<<grid, 32, p.smem, s>>>(a);
    }
  } else {
    if (kb == 4)
      ss_summarize_kernel<uint32_t, uint64_t, true, false><<<grid, 32, p.smem, s>>>(a);
    else
      ss_summarize_kernel<uint64_t, uint64_t, true, false><<<grid, 32, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace pss
