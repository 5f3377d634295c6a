// summarize.cu -- K1: per-partition Space Saving summaries (Algorithm 1 lines 3-5, PAPER.md:92-96;
// update rules PAPER.md:82) on sm_100a.
//
// One warp owns one partition at a time (persistent 1-warp CTAs pull partition ids from a queue).
// The warp streams its block of A through a shared-memory ring filled by the TMA engine
// (cp.async.bulk + mbarrier) and applies Space Saving to 32 consecutive items per step with an
// exact batched rule (K1):
//   1. each lane looks its item up in a two-choice, two-way bucketed cuckoo index
//      (entry = fingerprint | slot in 16 bits for k <= 4094; a lookup reads both candidate
//      buckets with two independent loads, selects the first fingerprint match without branches
//      and verifies its key; a fingerprint match with another key takes a slow re-check);
//   2. __match_any_sync groups equal keys; the first lane of a group is its leader, multiplicity =
//      popcount of the group restricted to the processed prefix;
//   3. leaders that miss are ranked in stream order; during the fill phase they take slots
//      size, size+1, ... (R2); once all k counters are occupied they take the lowest-index slots of
//      B_m = {slots with count == m, the current minimum} in ascending order (R1). B_m is kept as
//      a list of slot indices in ascending order (refilled 256 at a time from a scan of the
//      counters); a slot stays in B_m exactly while its count is m, so stale list entries (slots
//      hit since the list was built) are recognised by a load of the count and skipped. At the
//      start of every step, in parallel with the lookups, lane j loads the j-th next list entry
//      and its counter word (which also holds the position of the slot's index entry);
//   4. the step processes the longest prefix [0, c) of the 32 items for which this equals the
//      sequential algorithm: c stops before the first miss that finds no victim among the fetched
//      entries or past the last free counter, and at the later of the two positions when a
//      victim slot is also hit in the window;
//   5. hits add their multiplicity; misses evict (count m + mult, err m), free the victim's index
//      entry and write their own entry into a free way of their buckets; a read-back settles lanes
//      that picked the same entry, and the rare leftovers take a serial cuckoo-kick path.
// Every step consumes >= 1 item, so the result is bit-identical to sequential Space Saving.
// When the block length allows (blocks < 2^17 keys), a counter word holds the count in its low cb
// bits and the position of the slot's index entry above them; errors live in their own array.
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
#else
#define SS_STAT(i, v) \
  do {                \
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
constexpr size_t SS_SMEM_STATE_MAX = 100 * 1024;  // bigger per-warp state lives in global memory
constexpr uint32_t SS_K_SMALL = 4094;             // 16-bit index entries up to this k
constexpr double SS_LOAD = 0.30;  // index load factor (live keys / entries), before the slack fill
constexpr int SS_MAX_KICKS = 200;
// capacity of the B_m list (slot indices) for windows of R rows of 32 items
__host__ __device__ constexpr uint32_t ss_vq(uint32_t R) { return R <= 2 ? 256u : 512u; }
constexpr uint32_t SS_PB = 15;    // index-position bits of a packed counter word (entries < 2^15)

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
                                               uint32_t b2, uint32_t pref) {
  constexpr ET EMPTY = Ent<ET>::EMPTY;
  // within a bucket the key's preferred way first (pref = a bit of its hash), so that two keys
  // choosing one bucket in the same step take different ways half of the time
  const uint32_t w0 = pref & 1u, w1 = w0 ^ 1u;
  const bool f0 = (w0 ? e1 : e0) == EMPTY, f1 = (w0 ? e0 : e1) == EMPTY;
  const bool f2 = (w0 ? e3 : e2) == EMPTY, f3 = (w0 ? e2 : e3) == EMPTY;
  uint32_t fa = f1 ? 2 * b1 + w1 : 0xffffffffu;
  fa = f0 ? 2 * b1 + w0 : fa;
  uint32_t fb = f3 ? 2 * b2 + w1 : 0xffffffffu;
  fb = f2 ? 2 * b2 + w0 : fb;
  const bool pickb = (uint32_t)f2 + (uint32_t)f3 > (uint32_t)f0 + (uint32_t)f1;
  return pickb ? fb : fa;
}

// one summary's state (shared memory, or global memory for large k); every slot-indexed array
// holds exactly k entries (slots are < k)
struct SSLayout {
  size_t keys, cw, err, pos, vq, vic, T, total;
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
// experiment hook: target index load before the slack fill (sets the occupancy)
static double ss_target_load() {
  if (const char* s = std::getenv("PSS_SS_LOAD")) {
    double v = std::atof(s);
    if (v > 0.1 && v < 0.8) return v;
  }
  return SS_LOAD;
}
static uint32_t ss_buckets(uint32_t k, double load) {
  return (uint32_t)std::max<double>(2.0, std::ceil(k / (2.0 * load)));
}

// kb: key bytes; eb: index entry bytes (2 or 8); errb: error bytes; packed: the entry position
// lives in the counter word (else a pos array of 2- or 4-byte entries)
static SSLayout ss_layout(uint32_t k, int kb, int eb, int errb, bool packed, uint32_t NB,
                          uint32_t R) {
  SSLayout L;
  const int pb = eb == 2 ? 2 : 4;  // pos / list entry bytes
  L.NB = NB;
  Bump b;
  b.al = 16;
  L.keys = b.take<unsigned char>((size_t)k * kb);
  L.cw = b.take<uint32_t>(k);
  L.err = b.take<unsigned char>((size_t)k * errb);
  L.pos = packed ? L.cw : b.take<unsigned char>((size_t)k * pb);
  L.vq = b.take<unsigned char>((size_t)ss_vq(R) * pb);
  L.vic = b.take<uint2>(32 * R);
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
  unsigned char* gstate;  // per-CTA state when it does not fit shared memory
  size_t gstride;
  size_t o_cw, o_err, o_pos, o_vq, o_vic, o_T;
  uint32_t NB;
  uint32_t cb;            // PACKED: count in the low cb bits, index position above
  uint32_t sb, fmask;     // index entry layout
};

// SB, CB > 0: the index entry's slot bits and the counter word's count bits as compile-time
// constants (shifts and masks become immediates); 0: runtime. ERRT: the error array's type
// (errors are <= the block length / k).
template <typename KT, typename ET, bool GSTATE, bool PACKED, typename ERRT, int SB = 0, int CB = 0,
          uint32_t R = 1>
// 1-warp CTAs: __launch_bounds__(32) measured 12-15 % faster than any multi-warp bound (round 1)
__global__ void __launch_bounds__(32) ss_summarize_kernel(const SumArgs a) {
  using PT = typename std::conditional<sizeof(ET) == 2, uint16_t, uint32_t>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = threadIdx.x;
  const uint32_t ltm = lanemask_lt();
  constexpr uint32_t ST = SS_STAGE_BYTES / sizeof(KT);  // items per stage
  constexpr uint32_t RING = SS_NSTAGE * ST;  // ring capacity in items
  constexpr uint32_t E = 16 / sizeof(KT);  // items per 16 bytes
  constexpr ET EMPTY = Ent<ET>::EMPTY;
  constexpr uint32_t VQ = ss_vq(R);
  const Ent<ET> en{SB ? (uint32_t)SB : a.sb, SB ? (1u << (16 - SB)) - 1u : a.fmask};

  KT* ring = reinterpret_cast<KT*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SS_RING_BYTES);
  unsigned char* st = GSTATE ? a.gstate + (size_t)blockIdx.x * a.gstride : smem + SS_RING_BYTES + SS_BAR_BYTES;
  KT* keys = reinterpret_cast<KT*>(st);
  // count; if PACKED also the position of the slot's index entry above the low cb bits
  uint32_t* cw = reinterpret_cast<uint32_t*>(st + a.o_cw);
  ERRT* err = reinterpret_cast<ERRT*>(st + a.o_err);
  PT* pos = reinterpret_cast<PT*>(st + a.o_pos);  // index entry of each slot (unpacked)
  PT* vq = reinterpret_cast<PT*>(st + a.o_vq);    // B_m list: slot indices, ascending
  uint2* vic = reinterpret_cast<uint2*>(st + a.o_vic);  // this step's victims: (slot, entry)
  ET* T = reinterpret_cast<ET*>(st + a.o_T);

  const KT* __restrict__ A = reinterpret_cast<const KT*>(a.A);
  const uint64_t n = a.n;
  const uint32_t k = a.k, P = a.P, NB = a.NB;
  const uint32_t NE = 2 * NB;
  const uint32_t cb = CB ? (uint32_t)CB : a.cb;
  const uint32_t CM = PACKED ? ((1u << cb) - 1u) : 0xffffffffu;
  auto set_pos = [&](uint32_t v, uint32_t idx) {
    if (PACKED)
      cw[v] = (cw[v] & CM) | (idx << cb);
    else
      pos[v] = (PT)idx;
  };
  const bool aligned = (reinterpret_cast<uintptr_t>(A) & 15u) == 0;
  const uint64_t nfloor = aligned ? (n & ~(uint64_t)(E - 1)) : 0;

  if (lane == 0) {
    for (uint32_t j = 0; j < SS_NSTAGE; ++j) mbar_init(&bars[j], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phasebits = 0;
  if (a.pdl) pdl_launch_dependents();

  while (true) {
    uint32_t r = 0;
    if (lane == 0) r = a.r0 + atomicAdd(a.queue, 1u);
    r = __shfl_sync(PSS_FULL, r, 0);
    if (r >= a.r1) break;
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
    uint32_t size = 0, m = 0, seed = 0;
    uint32_t cur = 0, vlen = 0, vscan = 0;  // B_m list: next entry, length, next slot to scan
    __syncwarp();

    // append to the list the slots t in [vscan, size) with count m, 32 at a time, until it holds
    // more than VQ - 32 entries (the next word always fits) or every slot was scanned
    auto scan_level = [&]() {
      const uint32_t kw = (size + 31u) >> 5;
      uint32_t w = vscan >> 5;
      while (w < kw && vlen <= VQ - 32) {
        const uint32_t t = w * 32 + lane;
        const bool at = t < size && (cw[t] & CM) == m;
        const uint32_t b = __ballot_sync(PSS_FULL, at);
        if (at) vq[vlen + __popc(b & ltm)] = (PT)t;
        vlen += __popc(b);
        ++w;
      }
      vscan = w * 32;
    };
    // B_m is exhausted: the next minimum is m + 1 if any counter has it (every count is > m
    // now), otherwise a full minimum scan
    auto new_level = [&](bool first) {
      cur = 0;
      vlen = 0;
      vscan = 0;
      if (!first) {
        ++m;
        scan_level();
        SS_STAT(7, 1);
      }
      if (first || vlen == 0) {
        uint32_t mn = 0xffffffffu;
        for (uint32_t t = lane; t < size; t += 32) mn = min(mn, cw[t] & CM);
        m = __reduce_min_sync(PSS_FULL, mn);
        vscan = 0;
        scan_level();
      }
      __syncwarp();
    };
    // fewer than a window of entries left and more slots to scan: move the rest to the front,
    // append
    auto refill = [&]() {
      const uint32_t rem = vlen - cur;  // < 32 R
      PT t[R];
#pragma unroll
      for (uint32_t j = 0; j < R; ++j) t[j] = 32 * j + lane < rem ? vq[cur + 32 * j + lane] : (PT)0;
      __syncwarp();
#pragma unroll
      for (uint32_t j = 0; j < R; ++j)
        if (32 * j + lane < rem) vq[32 * j + lane] = t[j];
      vlen = rem;
      cur = 0;
      scan_level();
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
        const uint32_t fi = free_entry(f0, f1, f2, f3, b1, b2, fp >> 1);
        if (fi != 0xffffffffu) {
          T[fi] = en.make(fp, cv);
          set_pos(cv, fi);
          return true;
        }
        const uint32_t kb = (b1 != prev) ? b1 : b2;
        const uint32_t idx = 2 * kb + ((step ^ (cv & 1)) & 1);
        const ET e = T[idx];
        T[idx] = en.make(fp, cv);
        set_pos(cv, idx);
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
      // measured 12 % slower in round 1)
      ET* const tp = T + (tryfi ? fi : 0u);
      if (tryfi) *tp = mine;
      __syncwarp();
      const bool won = tryfi && *tp == mine;
      if (!PACKED) {  // packed counters were written with the position fi
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
      // stages 0..NSTAGE-2 in flight; waiting for stage g frees the slot of stage g-2 (a window
      // spans at most two stages), which is refilled with stage g+NSTAGE-2
      for (uint32_t g = 0; g < min(total, SS_NSTAGE - 1); ++g) issue(g, g);
      uint32_t ready = 0;      // stages waited for
      uint32_t rsl = 0;        // ring slot of stage `ready`
      uint32_t ready_end = 0;  // items of the partition available in the ring: [0, ready_end)
      auto ensure = [&](uint32_t end) {  // items [0, end) resident in the ring
        if (end > ready_end) {
          __syncwarp();
          while (end > ready_end) {
            mbar_wait(&bars[rsl], (phasebits >> rsl) & 1u);
            phasebits ^= 1u << rsl;
            // stage ready + NSTAGE - 2 goes into the slot of stage ready - 2 (consumed)
            const uint32_t nx = ready + SS_NSTAGE - 2;
            uint32_t nsl = rsl + SS_NSTAGE - 2;
            if (nsl >= SS_NSTAGE) nsl -= SS_NSTAGE;
            if (nx >= SS_NSTAGE - 1 && nx < total) issue(nx, nsl);
            ++ready;
            rsl = rsl + 1 == SS_NSTAGE ? 0u : rsl + 1;
            ready_end = min(L, ready * ST - roff);
          }
          __syncwarp();
        }
      };

      // lookup of x: slot s (-1 if not monitored), its counter word ce, the free entry fi of its
      // buckets (insert target) and its fingerprint fp
      auto lookup = [&](KT x, bool act, int32_t& s, uint32_t& ce, uint32_t& fi, uint32_t& fp) {
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
        ce = cw[t0];
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
                ce = cw[t];
                amb = false;
              }
            }
          }
        }
        fi = free_entry(e0, e1, e2, e3, b1, b2, fp >> 1);
      };

      // lookup of x with the first two fingerprint matches checked at once (their keys are
      // loaded together): slot s and counter word ce if hit; amb if neither matched and a third
      // fingerprint match remains (the caller then runs `lookup`)
      auto lookup2 = [&](KT x, bool act, uint32_t& s, uint32_t& ce, uint32_t& fi, uint32_t& fp,
                         bool& hit, bool& amb) {
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
        const ET r3 = q3 ? e3 : EMPTY;
        const ET r23 = q2 ? e2 : r3;
        const ET r123 = q1 ? e1 : r23;
        const ET m1 = q0 ? e0 : r123;
        const ET m2 = q0 ? r123 : (q1 ? r23 : (q2 ? r3 : EMPTY));
        const uint32_t t1 = m1 == EMPTY ? 0u : en.slot(m1);
        const uint32_t t2 = m2 == EMPTY ? 0u : en.slot(m2);
        const KT k1 = keys[t1], k2 = keys[t2];
        const uint32_t c1 = cw[t1], c2 = cw[t2];
        const bool h1 = m1 != EMPTY && k1 == x;
        const bool h2 = m2 != EMPTY && k2 == x;
        hit = act && (h1 || h2);
        s = h1 ? t1 : t2;
        ce = h1 ? c1 : c2;
        amb = act && !hit && (uint32_t)q0 + (uint32_t)q1 + (uint32_t)q2 + (uint32_t)q3 >= 3u;
        fi = free_entry(e0, e1, e2, e3, b1, b2, fp >> 1);
      };

      uint32_t q = 0;  // items consumed
      // The specialized kernel (SB > 0) keeps the ring position of item q, (roff + q) % RING,
      // incrementally and compares both fingerprints of a bucket word at once (round 1: the same
      // two changes measured 2-5 % slower in the runtime-layout kernel).
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
        uint32_t ce, fi, fp;
        lookup(x, act, s, ce, fi, fp);
        const bool hit = s >= 0;
        const bool leader = act && (grp & ltm) == 0;
        const uint32_t missL = __ballot_sync(PSS_FULL, leader && !hit);
        uint32_t c = nv;
        const uint32_t freec = k - size;
        if ((uint32_t)__popc(missL) > freec) c = nth_set(missL, freec);
        const uint32_t pm = c >= 32 ? PSS_FULL : ((1u << c) - 1u);
        const bool inpre = leader && lane < c;
        const uint32_t mult = __popc(grp & pm);
        if (inpre && hit) cw[s] = ce + mult;
        const bool ins = inpre && !hit;
        const uint32_t v = size + __popc(missL & ltm);
        if (ins) {
          keys[v] = x;
          cw[v] = PACKED ? (mult | (fi << cb)) : mult;
          err[v] = (ERRT)0;
        }
        const uint32_t grow = __popc(missL & pm);
        insert_all(ins, x, v, fi, fp, size + grow);
        size += grow;
        advance(c);
        SS_STAT(8, 1);
        SS_STAT(1, c);
        __syncwarp();
      }
      if (size == k) new_level(true);

      // ---- all k counters occupied: misses evict the lowest slots of B_m (R1)
      // A step takes a window of W = 32 R consecutive items, R rows of 32 (item p = 32 j + lane
      // in row j), loaded by the previous step as soon as it knows its length.
      constexpr uint32_t W = 32u * R;
      static_assert(W <= ST, "a window spans at most two ring stages");
      KT x[R];
#pragma unroll
      for (uint32_t j = 0; j < R; ++j) x[j] = 0;
      auto next_window = [&]() {
        if (q < L) {
          ensure(q + min(W, L - q));
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) x[j] = ring_at(32u * j + lane);
        }
      };
      next_window();
      // one step; F: a full window (every step but the block's last), compiled separately so that
      // the window-length predicates fold away
      auto full_step = [&](auto full) {
        constexpr bool F = decltype(full)::value;
        const uint32_t nv = F ? W : min(W, L - q);
        bool act[R];
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) act[j] = F || 32u * j + lane < nv;

        // victim candidates (independent of the lookups): lane j of row r takes list entry
        // cur + 32 r + lane; it is still in B_m iff its count is m. The valid ones are compacted
        // into vic[] in list order: (slot | list index << 16, index entry).
        uint32_t navail = 0;
#pragma unroll
        for (uint32_t r = 0; r < R; ++r) {
          const uint32_t vi = cur + 32u * r + lane;
          const bool inq = vi < vlen;
          const uint32_t vs = inq ? (uint32_t)vq[vi] : 0u;
          const uint32_t vc = cw[vs];
          const bool valid = inq && (vc & CM) == m;
          const uint32_t vmask = __ballot_sync(PSS_FULL, valid);
          if (valid)
            vic[navail + __popc(vmask & ltm)] =
                make_uint2(vs | (vi << 16), PACKED ? vc >> cb : (uint32_t)pos[vs]);
          navail += __popc(vmask);
        }

        // lookups of every row, then one test for the rare third fingerprint match
        uint32_t s[R], ce[R], fi[R], fp[R];
        bool hit[R];
        bool amb = false;
        if constexpr (R == 1) {  // one row: the first fingerprint match, rare re-checks inside
          int32_t ss;
          lookup(x[0], act[0], ss, ce[0], fi[0], fp[0]);
          hit[0] = ss >= 0;
          s[0] = hit[0] ? (uint32_t)ss : 0u;
        } else {
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) {
            bool am;
            lookup2(x[j], act[j], s[j], ce[j], fi[j], fp[j], hit[j], am);
            amb |= am;
          }
        }
        if (R > 1 && __ballot_sync(PSS_FULL, amb)) {
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) {
            int32_t ss;
            uint32_t c2, f2, p2;
            lookup(x[j], act[j], ss, c2, f2, p2);  // the full check (every fingerprint match)
            hit[j] = ss >= 0;
            s[j] = hit[j] ? (uint32_t)ss : 0u;
            ce[j] = c2;
          }
          SS_STAT(4, 1);
        }
        __syncwarp();  // vic[] written

        // every miss is ranked in stream order (a key that misses twice is found below)
        uint32_t missL[R], base[R];
        uint32_t M = 0;
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) {
          missL[j] = __ballot_sync(PSS_FULL, act[j] && !hit[j]);
          base[j] = M;
          M += __popc(missL[j]);
        }
        const uint32_t Ms = min(M, navail);
        uint32_t c = nv;
        if (M > navail) {  // the first miss without a fetched victim
          uint32_t jr = 0;
#pragma unroll
          for (uint32_t j = 1; j < R; ++j)
            if (base[j] <= navail) jr = j;
          uint32_t mj = missL[0], bj = base[0];
#pragma unroll
          for (uint32_t j = 1; j < R; ++j)
            if (jr == j) {
              mj = missL[j];
              bj = base[j];
            }
          c = 32u * jr + nth_set(mj, navail - bj);
          SS_STAT(5, 1);
        }
        // hazard: a victim slot whose item is also hit in the window. A hit slot with count m is
        // at or after the cursor (every slot passed by the cursor was evicted or had left B_m),
        // so it is among this step's victims iff it is <= the last one.
        const uint32_t vmax = vic[Ms ? Ms - 1 : 0].x & 0xffffu;
        bool conf = false;
#pragma unroll
        for (uint32_t j = 0; j < R; ++j)
          conf |= hit[j] && Ms && (ce[j] & CM) == m && s[j] <= vmax;
        if (__ballot_sync(PSS_FULL, conf)) {
          uint32_t cpos = W;
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) {
            if (hit[j] && Ms && (ce[j] & CM) == m && s[j] <= vmax) {
              uint32_t rr = 0;  // s is victim rr, taken by the miss of rank rr
              while ((vic[rr].x & 0xffffu) != s[j]) ++rr;
              uint32_t jr = 0;
#pragma unroll
              for (uint32_t i = 1; i < R; ++i)
                if (base[i] <= rr) jr = i;
              uint32_t mm = 0, bb = 0;
#pragma unroll
              for (uint32_t i = 0; i < R; ++i)
                if (jr == i) {
                  mm = missL[i];
                  bb = base[i];
                }
              for (uint32_t i = bb; i < rr; ++i) mm &= mm - 1u;
              const uint32_t prr = 32u * jr + (uint32_t)(__ffs(mm) - 1);
              // hit first (t < p): the hit is processed and the eviction waits; eviction first
              // (t > p): the eviction is processed and the item at t becomes a miss
              cpos = min(cpos, max(32u * j + lane, prr));
            }
          }
          c = min(c, __reduce_min_sync(PSS_FULL, cpos));
          SS_STAT(6, 1);
        }
        // Misses of [0, c) claim the free entry of their buckets for (fingerprint, victim slot)
        // and read it back. Two misses of one key pick the same entry (same buckets, same
        // snapshot): if every claim holds, no key misses twice in the window.
        uint2 vv[R];
        bool ev[R], won[R];
        ET* tp[R];
        ET mine[R];
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) {
          const uint32_t rank = base[j] + __popc(missL[j] & ltm);
          vv[j] = vic[min(rank, W - 1)];
          vv[j].x &= 0xffffu;
          ev[j] = act[j] && !hit[j] && 32u * j + lane < c;
          const bool tryfi = ev[j] && fi[j] != 0xffffffffu;
          mine[j] = en.make(fp[j], vv[j].x);
          tp[j] = T + (tryfi ? fi[j] : 0u);
          if (tryfi) *tp[j] = mine[j];
        }
        __syncwarp();
        bool anylost = false;
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) {
          won[j] = ev[j] && fi[j] != 0xffffffffu && *tp[j] == mine[j];
          anylost |= ev[j] && !won[j];
        }
        const uint32_t lostb = __ballot_sync(PSS_FULL, anylost);
        if (lostb) {
          // a claim did not hold: two misses picked one entry (one key twice, or two keys
          // sharing a bucket) or a miss found no free entry. Every key that misses more than once
          // has a losing occurrence: for each losing miss, any other miss of its key ends the
          // step before that key's second occurrence (which is a hit on the first one's slot).
          uint32_t cd = c;
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) {
            uint32_t lm = __ballot_sync(PSS_FULL, ev[j] && !won[j]);
            while (lm) {
              const uint32_t l = __ffs(lm) - 1;
              lm &= lm - 1;
              const KT xl = __shfl_sync(PSS_FULL, x[j], l);
              uint32_t first = W, second = W;
#pragma unroll
              for (uint32_t i = 0; i < R; ++i) {
                const uint32_t same = __ballot_sync(PSS_FULL, ev[i] && x[i] == xl);
                if (same) {
                  const uint32_t p0 = 32u * i + (uint32_t)(__ffs(same) - 1);
                  const uint32_t rest = same & (same - 1);
                  if (p0 < first) {
                    second = first;
                    first = p0;
                  } else if (p0 < second) {
                    second = p0;
                  }
                  if (rest) second = min(second, 32u * i + (uint32_t)(__ffs(rest) - 1));
                }
              }
              cd = min(cd, second);
            }
          }
          if (cd < c) {  // undo the claims at or after the new end; those before keep theirs
            c = cd;
#pragma unroll
            for (uint32_t j = 0; j < R; ++j) {
              const bool out = 32u * j + lane >= c;
              if (won[j] && out) *tp[j] = EMPTY;
              ev[j] = ev[j] && !out;
              won[j] = won[j] && !out;
            }
            SS_STAT(13, 1);
          }
          __syncwarp();
          SS_STAT(12, 1);
        }
        // hits: count + 1 per occurrence (occurrences of one key add to one counter; a hit
        // counter at m leaves B_m and its list entry goes stale)
#pragma unroll
        for (uint32_t j = 0; j < R; ++j)
          if (hit[j] && 32u * j + lane < c) atomicAdd(cw + s[j], 1u);
        // misses: the victim takes the item, count m + 1 ("incremented by one"), error m; its old
        // item leaves the index
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) {
          ET* const tdel = T + vv[j].y;
          KT* const kptr = keys + vv[j].x;
          uint32_t* const vptr = cw + vv[j].x;
          ERRT* const eptr = err + vv[j].x;
          if (ev[j]) {
            *tdel = EMPTY;
            *kptr = x[j];
            *vptr = PACKED ? ((m + 1u) | (fi[j] << cb)) : (m + 1u);
            *eptr = (ERRT)m;
            if (!PACKED) pos[vv[j].x] = (PT)fi[j];
          }
        }
        if (lostb) {  // the misses whose claim did not hold insert serially (cuckoo kicks)
          __syncwarp();
#pragma unroll
          for (uint32_t j = 0; j < R; ++j) {
            uint32_t need = __ballot_sync(PSS_FULL, ev[j] && !won[j]);
            SS_STAT(2, __popc(need));
            bool failed = false;
            while (need) {
              const uint32_t l = __ffs(need) - 1;
              uint32_t okl = 1;
              if (lane == l) okl = slow_insert(x[j], vv[j].x);
              failed |= __shfl_sync(PSS_FULL, okl, l) == 0;
              __syncwarp();
              need &= need - 1;
            }
            if (failed) {
              SS_STAT(3, 1);
              rehash(size);
            }
          }
        }
        uint32_t Mp = 0;
#pragma unroll
        for (uint32_t j = 0; j < R; ++j) {
          const uint32_t pj = c >= 32u * (j + 1) ? PSS_FULL
                              : (c <= 32u * j ? 0u : ((1u << (c - 32u * j)) - 1u));
          Mp += __popc(missL[j] & pj);
        }
        // the cursor moves past the last victim taken (stale entries before it are skipped); a
        // window of stale entries only is skipped as a whole
        if (Mp)
          cur = (vic[Mp - 1].x >> 16) + 1u;
        else if (navail == 0)
          cur = min(cur + W, vlen);
        advance(c);
        next_window();
        SS_STAT(0, 1);
        SS_STAT(9, Mp);
        SS_STAT(1, c);
        if (vlen - cur < W && vscan < size) {
          refill();
          SS_STAT(11, 1);
        }
        if (cur >= vlen && vscan >= size) new_level(false);
        __syncwarp();
      };
      while (q + W <= L) full_step(std::true_type{});
      while (q < L) full_step(std::false_type{});
    }

    // ---- dump the leaf in slot order
    KT* oi = reinterpret_cast<KT*>(a.items) + (size_t)r * k;
    uint32_t* oc = a.counts + (size_t)r * k;
    uint32_t* oe = a.errs + (size_t)r * k;
    for (uint32_t t = lane; t < size; t += 32) {
      oi[t] = keys[t];
      oc[t] = cw[t] & CM;
      oe[t] = (uint32_t)err[t];
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
using SSKernel = void (*)(const SumArgs);

struct SSPlan {
  bool gstate, packed;
  int spec;   // 10: the kernel compiled for slot bits 10 / count bits 17
  int errb;   // bytes per error
  uint32_t R; // rows of 32 items per step
  uint32_t cb, sb, fmask;
  SSLayout L;
  size_t smem;
  int grid;   // CTAs of a launch over all P partitions
  int slots;  // resident CTAs the device holds
};

template <typename KT>
static SSKernel ss_kernel_of(bool gstate, bool packed, int spec, uint32_t R) {
  if (gstate) return ss_summarize_kernel<KT, uint64_t, true, false, uint32_t>;
  if (!packed) return ss_summarize_kernel<KT, uint16_t, false, false, uint32_t>;
  if (spec == 10) {
    if constexpr (sizeof(KT) == 4) {
      if (R == 4) return ss_summarize_kernel<KT, uint16_t, false, true, uint8_t, 10, 17, 4>;
    }
    if (R == 2) return ss_summarize_kernel<KT, uint16_t, false, true, uint8_t, 10, 17, 2>;
    return ss_summarize_kernel<KT, uint16_t, false, true, uint8_t, 10, 17, 1>;
  }
  return ss_summarize_kernel<KT, uint16_t, false, true, uint16_t>;
}
static SSKernel ss_kernel_of(int kb, const SSPlan& p) {
  return kb == 4 ? ss_kernel_of<uint32_t>(p.gstate, p.packed, p.spec, p.R)
                 : ss_kernel_of<uint64_t>(p.gstate, p.packed, p.spec, p.R);
}

// rows of 32 items per step of the specialized kernel (experiment hook PSS_SS_ROWS: 1, 2, 4)
static uint32_t ss_rows(int kb) {
  uint32_t R = 2;
  if (const char* s = std::getenv("PSS_SS_ROWS")) R = (uint32_t)std::atoi(s);
  if (R != 1 && R != 2 && R != 4) R = 2;
  if (kb == 8 && R > 2) R = 2;  // a window spans at most two 64-key ring stages
  return R;
}

static int ss_blocks_per_sm(SSKernel kern, size_t smem, const DevInfo& d) {
  if (smem > (size_t)d.smem_optin || allow_max_smem(kern, d) != cudaSuccess) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return nb;  // 0: does not fit
}

static SSPlan ss_plan(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  SSPlan p;
  // counts <= Lmax need cb bits; the index position takes SS_PB bits above them when they fit
  const uint64_t Lmax = (n + P - 1) / P;
  p.cb = 1;
  while (p.cb < 32 && (1ull << p.cb) <= Lmax) ++p.cb;
  p.packed = p.cb + SS_PB <= 32;
  // 16-bit entries: the slot field's all-ones value must exceed k - 1
  uint32_t sb = 1;
  while ((1u << sb) - 1u < k) ++sb;
  p.spec = p.packed && p.cb == 17 && sb == 10 ? 10 : 0;  // errors <= Lmax / k < 2^17 / 512
  p.errb = p.spec ? 1 : (p.packed ? 2 : 4);               // packed: Lmax / k < 2^16
  p.R = p.spec ? ss_rows(kb) : 1;
  const double dl = ss_debug_load();
  uint32_t NB = ss_buckets(k, dl > 0 ? dl : ss_target_load());
  if (p.packed) NB = std::min(NB, ((1u << SS_PB) - 1u) / 2u);  // packed words address < 2^SS_PB entries
  SSLayout Ls = ss_layout(k, kb, 2, p.errb, p.packed, NB, p.R);
  p.gstate = k > SS_K_SMALL || Ls.total > SS_SMEM_STATE_MAX;
  if (!p.gstate) {
    p.sb = sb;
    p.fmask = (1u << (16 - sb)) - 1u;
    size_t pad = 0;
    if (const char* ps = std::getenv("PSS_DEBUG_SMEM_PAD"))  // experiment hook: fewer warps/SM
      pad = (size_t)std::atoll(ps);
    auto smem_of = [&](const SSLayout& L) { return SS_RING_BYTES + SS_BAR_BYTES + L.total + pad; };
    const SSKernel kern = ss_kernel_of(kb, p);
    const int nb = ss_blocks_per_sm(kern, smem_of(Ls), d);
    // The shared memory left over at this occupancy goes to the index: the largest bucket count
    // that keeps `nb` warps per SM (fewer fingerprint collisions and serial inserts); packed
    // counter words address at most 2^SS_PB entries.
    const uint32_t nb_max = p.packed ? ((1u << SS_PB) - 1u) / 2u : 0x7fffffffu;
    if (dl == 0 && nb > 0) {
      uint32_t lo = NB, hi = std::min(2 * NB, nb_max);
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (ss_blocks_per_sm(kern, smem_of(ss_layout(k, kb, 2, p.errb, p.packed, mid, p.R)), d) >= nb)
          lo = mid;
        else
          hi = mid - 1;
      }
      NB = lo;
      Ls = ss_layout(k, kb, 2, p.errb, p.packed, NB, p.R);
    }
    p.L = Ls;
    p.smem = smem_of(Ls);
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)std::max(nb, 1) * d.sms);
    p.slots = (int)std::min<uint64_t>((uint64_t)nb * d.sms, 1u << 30);
  } else {
    p.packed = false;
    p.spec = 0;
    p.R = 1;
    p.errb = 4;
    p.sb = 32;
    p.fmask = 0xffffffffu;
    p.L = ss_layout(k, kb, 8, 4, false, ss_buckets(k, dl > 0 ? dl : 0.32), 1);
    p.smem = SS_RING_BYTES + SS_BAR_BYTES;
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)8 * d.sms);
    p.slots = 8 * d.sms;
  }
  if (p.grid < 1) p.grid = 1;
  return p;
}

size_t summarize_ws(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  SSPlan p = ss_plan(n, kb, k, P, d);
  Bump b;
  b.take<uint32_t>(SS_MAX_RANGES);
  if (p.gstate) b.take<unsigned char>(p.L.total * (size_t)p.grid);
  return b.bytes();
}

cudaError_t summarize_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P,
                             void* items, uint32_t* counts, uint32_t* errs, uint32_t* sizes,
                             void* ws, cudaStream_t s, const DevInfo& d, uint32_t r0,
                             uint32_t r1, uint32_t qi, uint32_t T, uint32_t* leaf_flags,
                             bool pdl) {
  SSPlan p = ss_plan(n, kb, k, P, d);
  if (r1 > P) r1 = P;
  if (r0 >= r1 || qi >= SS_MAX_RANGES) return cudaErrorInvalidValue;
  const int grid = (int)std::min<uint64_t>(r1 - r0, (uint64_t)p.grid);
  Bump b;
  const size_t oq = b.take<uint32_t>(SS_MAX_RANGES);
  const size_t og = p.gstate ? b.take<unsigned char>(p.L.total * (size_t)p.grid) : 0;
  SumArgs a;
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
  a.queue = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(ws) + oq) + qi;
  a.gstate = p.gstate ? static_cast<unsigned char*>(ws) + og : nullptr;
  a.gstride = p.L.total;
  a.o_cw = p.L.cw;
  a.o_err = p.L.err;
  a.o_pos = p.L.pos;
  a.o_vq = p.L.vq;
  a.o_vic = p.L.vic;
  a.o_T = p.L.T;
  a.NB = p.L.NB;
  a.cb = p.cb;
  a.sb = p.sb;
  a.fmask = p.fmask;
  cudaError_t e = cudaMemsetAsync(a.queue, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const SSKernel kern = ss_kernel_of(kb, p);
  if (!p.gstate) allow_max_smem(kern, d);
  kern<<<grid, 32, p.smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace pss
