// summarize.cu -- K1: per-partition Space Saving summaries (Algorithm 1 lines 3-5, PAPER.md:92-96;
// update rules PAPER.md:82) on sm_100a.
//
// One warp owns one partition at a time (persistent 1-warp CTAs pull partition ids from a queue).
// The warp streams its block of A through a shared-memory ring filled by the TMA engine
// (cp.async.bulk + mbarrier) and applies Space Saving to 32 consecutive items per step with an
// exact batched rule:
//   1. each lane looks its item up in a linear-probing hash index (key -> slot);
//   2. __match_any_sync groups equal keys; the first lane of a group is its leader, multiplicity =
//      popcount of the group restricted to the processed prefix;
//   3. leaders that miss are ranked in stream order; during the fill phase they take slots
//      size, size+1, ... (R2); once all k counters are occupied they take the lowest-index slots of
//      B_m = {slots with count == m, the current minimum} in ascending order (R1). B_m is a bitmap.
//   4. the step processes the longest prefix [0, c) of the 32 items for which this equals the
//      sequential algorithm: c stops before the first miss that finds B_m empty or the counters
//      full, and before the first hazard where a victim slot is also hit in the window.
//   5. hits add their multiplicity; misses evict (count m + mult, err m) and re-index the hash.
// Every step consumes >= 1 item, so the result is bit-identical to sequential Space Saving.
#include "common.cuh"

namespace pss {

constexpr uint32_t SS_RING_BYTES = 8192;  // per-warp TMA ring
constexpr uint32_t SS_NSTAGE = 4;
constexpr uint32_t SS_STAGE_BYTES = SS_RING_BYTES / SS_NSTAGE;
constexpr size_t SS_SMEM_STATE_MAX = 100 * 1024;  // bigger per-warp state lives in global memory

template <typename HT>
struct HTag {
  static constexpr HT EMPTY = (HT)~(HT)0;
  static constexpr HT TOMB = (HT)(~(HT)0 - 1);
};

struct SSLayout {
  size_t keys, cnt, err, bm, vic, ht, total;
  uint32_t logH;
};

static SSLayout ss_layout(uint32_t k, int kb, int htb) {
  SSLayout L;
  const size_t KP = align_up(k, 32);
  L.logH = ceil_log2(4ull * k);  // load factor of live keys <= 1/4
  L.keys = 0;
  L.cnt = L.keys + KP * kb;
  L.err = L.cnt + KP * 4;
  L.bm = L.err + KP * 4;
  L.vic = L.bm + KP / 32 * 4;
  L.ht = L.vic + 32 * 4;
  L.total = align_up(L.ht + ((size_t)1 << L.logH) * htb, 128);
  return L;
}

struct SumArgs {
  const void* A;
  uint64_t n;
  uint32_t k, P;
  void* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
  uint32_t* queue;
  unsigned char* gstate;  // per-CTA state when it does not fit shared memory
  size_t gstride;
  size_t o_cnt, o_err, o_bm, o_vic, o_ht;
  uint32_t logH;
};

template <typename KT, typename HT>
__device__ __forceinline__ int32_t ht_find(const HT* ht, const KT* keys, KT x, uint32_t logH) {
  const uint32_t mask = (1u << logH) - 1u;
  uint32_t h = hslot(x, logH);
  while (true) {
    const HT e = ht[h];
    if (e == HTag<HT>::EMPTY) return -1;
    if (e != HTag<HT>::TOMB && keys[e] == x) return (int32_t)e;
    h = (h + 1u) & mask;
  }
}

// insert slot v for key x (x absent); returns true if an EMPTY entry was consumed
template <typename KT, typename HT>
__device__ __forceinline__ bool ht_insert(HT* ht, KT x, uint32_t v, uint32_t logH) {
  const uint32_t mask = (1u << logH) - 1u;
  uint32_t h = hslot(x, logH);
  volatile HT* vh = ht;
  while (true) {
    const HT e = vh[h];
    if (e == HTag<HT>::EMPTY || e == HTag<HT>::TOMB) {
      const HT old = atomicCAS(&ht[h], e, (HT)v);
      if (old == e) return e == HTag<HT>::EMPTY;
      continue;
    }
    h = (h + 1u) & mask;
  }
}

template <typename KT, typename HT>
__device__ __forceinline__ void ht_delete(HT* ht, KT y, uint32_t v, uint32_t logH) {
  const uint32_t mask = (1u << logH) - 1u;
  uint32_t h = hslot(y, logH);
  while (ht[h] != (HT)v) h = (h + 1u) & mask;
  ht[h] = HTag<HT>::TOMB;
}

template <typename KT, typename HT, bool GSTATE>
__global__ void __launch_bounds__(32) ss_summarize_kernel(const SumArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = threadIdx.x;
  const uint32_t ltm = lanemask_lt();
  constexpr uint32_t ST = SS_STAGE_BYTES / sizeof(KT);  // items per stage
  constexpr uint32_t RING = SS_NSTAGE * ST;
  constexpr uint32_t E = 16 / sizeof(KT);  // items per 16 bytes

  KT* ring = reinterpret_cast<KT*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SS_RING_BYTES);
  unsigned char* st = GSTATE ? a.gstate + (size_t)blockIdx.x * a.gstride : smem + SS_RING_BYTES + 64;
  KT* keys = reinterpret_cast<KT*>(st);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(st + a.o_cnt);
  uint32_t* err = reinterpret_cast<uint32_t*>(st + a.o_err);
  uint32_t* bm = reinterpret_cast<uint32_t*>(st + a.o_bm);
  uint32_t* vic = reinterpret_cast<uint32_t*>(st + a.o_vic);
  HT* ht = reinterpret_cast<HT*>(st + a.o_ht);

  const KT* __restrict__ A = reinterpret_cast<const KT*>(a.A);
  const uint64_t n = a.n;
  const uint32_t k = a.k, P = a.P, logH = a.logH;
  const uint32_t H = 1u << logH;
  const uint32_t kw = (k + 31u) / 32u;
  const bool aligned = (reinterpret_cast<uintptr_t>(A) & 15u) == 0;
  const uint64_t nfloor = aligned ? (n & ~(uint64_t)(E - 1)) : 0;

  if (lane == 0) {
    for (uint32_t j = 0; j < SS_NSTAGE; ++j) mbar_init(&bars[j], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phasebits = 0;

  while (true) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(a.queue, 1u);
    r = __shfl_sync(PSS_FULL, r, 0);
    if (r >= P) break;
    const uint64_t lo = (uint64_t)r * n / P;  // Alg. 1 l.3-4: r*n < 2^63 as n <= 2^31
    const uint64_t hi = (uint64_t)(r + 1) * n / P;

    // ---- reset the summary
    for (uint32_t i = lane; i < H; i += 32) ht[i] = HTag<HT>::EMPTY;
    uint32_t size = 0, m = 0, bmcount = 0, bmf = 0, nempty = H;
    bool full = false;
    __syncwarp();

    auto new_level = [&]() {  // m = min count, B_m = {slots with count m}
      uint32_t mn = 0xffffffffu;
      for (uint32_t t = lane; t < k; t += 32) mn = min(mn, cnt[t]);
      m = __reduce_min_sync(PSS_FULL, mn);
      uint32_t tot = 0;
      for (uint32_t w = 0; w < kw; ++w) {
        const uint32_t t = w * 32 + lane;
        const uint32_t bits = __ballot_sync(PSS_FULL, t < k && cnt[t] == m);
        if (lane == 0) bm[w] = bits;
        tot += __popc(bits);
      }
      bmcount = tot;
      bmf = 0;
      __syncwarp();
    };
    auto ht_rebuild = [&]() {  // drop tombstones
      for (uint32_t i = lane; i < H; i += 32) ht[i] = HTag<HT>::EMPTY;
      __syncwarp();
      for (uint32_t t = lane; t < size; t += 32) ht_insert<KT, HT>(ht, keys[t], t, logH);
      __syncwarp();
      nempty = H - size;
    };

    if (lo < hi) {
      const uint64_t gbase = aligned ? (lo & ~(uint64_t)(E - 1)) : lo;
      const uint32_t total = (uint32_t)((hi - gbase + ST - 1) / ST);
      uint32_t issued = 0, ready = 0;
      auto issue = [&](uint32_t g) {
        const uint64_t a0 = gbase + (uint64_t)g * ST;
        const uint64_t b0 = min(a0 + ST, hi);
        uint64_t be = (b0 + E - 1) & ~(uint64_t)(E - 1);
        if (be > nfloor) be = nfloor;
        if (be < a0) be = a0;
        const uint32_t sl = g % SS_NSTAGE;
        KT* dst = ring + sl * ST;
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
      while (issued < total && issued < SS_NSTAGE) issue(issued++);

      uint64_t pos = lo;
      while (pos < hi) {
        const uint32_t nv = (uint32_t)min((uint64_t)32, hi - pos);
        const uint32_t gf = (uint32_t)((pos - gbase) / ST);
        const uint32_t gl = (uint32_t)((pos + nv - 1 - gbase) / ST);
        if (issued < total && issued < gf + SS_NSTAGE) {
          __syncwarp();
          do {
            issue(issued);
            ++issued;
          } while (issued < total && issued < gf + SS_NSTAGE);
        }
        while (ready <= gl) {
          const uint32_t sl = ready % SS_NSTAGE;
          mbar_wait(&bars[sl], (phasebits >> sl) & 1u);
          phasebits ^= 1u << sl;
          ++ready;
        }
        __syncwarp();

        // ---- one step over the window [pos, pos + nv)
        const bool act = lane < nv;
        const uint32_t amask = nv >= 32 ? PSS_FULL : ((1u << nv) - 1u);
        const KT x = act ? ring[(uint32_t)(pos - gbase + lane) & (RING - 1)] : (KT)0;
        const int32_t s = act ? ht_find<KT, HT>(ht, keys, x, logH) : -1;
        __syncwarp();
        const uint32_t grp = __match_any_sync(PSS_FULL, x) & amask;
        const bool leader = act && (grp & ltm) == 0;
        const uint32_t missL = __ballot_sync(PSS_FULL, leader && s < 0);
        const uint32_t cs = (leader && s >= 0) ? cnt[s] : 0u;
        uint32_t c = nv;

        if (!full) {
          // fill phase: free counters are taken in slot order (R2)
          const uint32_t freec = k - size;
          if ((uint32_t)__popc(missL) > freec) c = nth_set(missL, freec);
          const uint32_t pm = c >= 32 ? PSS_FULL : ((1u << c) - 1u);
          const bool inpre = leader && lane < c;
          const uint32_t mult = __popc(grp & pm);
          if (inpre && s >= 0) cnt[s] = cs + mult;
          bool took = false;
          if (inpre && s < 0) {
            const uint32_t v = size + __popc(missL & ltm);
            keys[v] = x;
            cnt[v] = mult;
            err[v] = 0;
            took = ht_insert<KT, HT>(ht, x, v, logH);
          }
          nempty -= __popc(__ballot_sync(PSS_FULL, took));
          size += __popc(missL & pm);
          __syncwarp();
          if (size == k) {
            full = true;
            new_level();
          }
        } else {
          // all k counters occupied: misses evict the lowest slots of B_m (R1)
          const uint32_t M = __popc(missL);
          const uint32_t Ms = min(M, bmcount);  // bmcount >= 1 here
          uint32_t vmax = 0;
          if (Ms) {
            uint32_t base = 0, w = bmf;
            while (base < Ms) {
              const uint32_t word = bm[w];
              const uint32_t pc = __popc(word);
              if (base == 0 && pc == 0) bmf = w + 1;
              const uint32_t rr = base + __popc(word & ltm);
              if (((word >> lane) & 1u) && rr < Ms) vic[rr] = w * 32 + lane;
              base += pc;
              ++w;
            }
            __syncwarp();
            vmax = vic[Ms - 1];
          }
          if (Ms < M) c = nth_set(missL, Ms);  // B_m runs out at this miss
          // hazard: a victim slot whose item is also hit in the window
          const bool conf = leader && s >= 0 && Ms && cs == m && (uint32_t)s <= vmax;
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
          }
          const uint32_t pm = c >= 32 ? PSS_FULL : ((1u << c) - 1u);
          const bool inpre = leader && lane < c;
          const uint32_t mult = __popc(grp & pm);
          const bool hitm = inpre && s >= 0 && cs == m;
          if (inpre && s >= 0) {
            cnt[s] = cs + mult;
            if (cs == m) atomicAnd(&bm[(uint32_t)s >> 5], ~(1u << ((uint32_t)s & 31u)));
          }
          const bool ev = inpre && s < 0;
          uint32_t v = 0;
          if (ev) {
            v = vic[__popc(missL & ltm)];
            ht_delete<KT, HT>(ht, keys[v], v, logH);
          }
          __syncwarp();
          bool took = false;
          if (ev) {
            keys[v] = x;
            cnt[v] = m + mult;  // "incremented by one" then further hits in the window
            err[v] = m;
            atomicAnd(&bm[v >> 5], ~(1u << (v & 31u)));
            took = ht_insert<KT, HT>(ht, x, v, logH);
          }
          bmcount -= __popc(__ballot_sync(PSS_FULL, hitm)) + __popc(missL & pm);
          nempty -= __popc(__ballot_sync(PSS_FULL, took));
          __syncwarp();
          if (bmcount == 0) new_level();
          if (nempty < (H >> 1)) ht_rebuild();
        }
        pos += c;
      }
    }

    // ---- dump the leaf in slot order
    KT* oi = reinterpret_cast<KT*>(a.items) + (size_t)r * k;
    uint32_t* oc = a.counts + (size_t)r * k;
    uint32_t* oe = a.errs + (size_t)r * k;
    for (uint32_t t = lane; t < size; t += 32) {
      oi[t] = keys[t];
      oc[t] = cnt[t];
      oe[t] = err[t];
    }
    if (lane == 0) a.sizes[r] = size;
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------ host side
struct SSPlan {
  bool gstate;
  SSLayout L;
  size_t smem;
  int grid;
};

template <typename KT, typename HT, bool G>
static int ss_blocks_per_sm(size_t smem) {
  auto kern = ss_summarize_kernel<KT, HT, G>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32, smem);
  return nb > 0 ? nb : 1;
}

static SSPlan ss_plan(int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  SSPlan p;
  SSLayout Ls = ss_layout(k, kb, 2);
  p.gstate = Ls.total > SS_SMEM_STATE_MAX || k >= 65000u;
  if (!p.gstate) {
    p.L = Ls;
    p.smem = SS_RING_BYTES + 64 + Ls.total;
    int nb = kb == 4 ? ss_blocks_per_sm<uint32_t, uint16_t, false>(p.smem)
                     : ss_blocks_per_sm<uint64_t, uint16_t, false>(p.smem);
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)nb * d.sms);
  } else {
    p.L = ss_layout(k, kb, 4);
    p.smem = SS_RING_BYTES + 64;
    p.grid = (int)std::min<uint64_t>(P, (uint64_t)8 * d.sms);
  }
  if (p.grid < 1) p.grid = 1;
  return p;
}

size_t summarize_ws(uint64_t, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  SSPlan p = ss_plan(kb, k, P, d);
  Bump b;
  b.take<uint32_t>(1);
  if (p.gstate) b.take<unsigned char>(p.L.total * (size_t)p.grid);
  return b.bytes();
}

cudaError_t summarize_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P,
                             void* items, uint32_t* counts, uint32_t* errs, uint32_t* sizes,
                             void* ws, cudaStream_t s, const DevInfo& d) {
  SSPlan p = ss_plan(kb, k, P, d);
  Bump b;
  const size_t oq = b.take<uint32_t>(1);
  const size_t og = p.gstate ? b.take<unsigned char>(p.L.total * (size_t)p.grid) : 0;
  SumArgs a;
  a.A = A;
  a.n = n;
  a.k = k;
  a.P = P;
  a.items = items;
  a.counts = counts;
  a.errs = errs;
  a.sizes = sizes;
  a.queue = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(ws) + oq);
  a.gstate = p.gstate ? static_cast<unsigned char*>(ws) + og : nullptr;
  a.gstride = p.L.total;
  a.o_cnt = p.L.cnt;
  a.o_err = p.L.err;
  a.o_bm = p.L.bm;
  a.o_vic = p.L.vic;
  a.o_ht = p.L.ht;
  a.logH = p.L.logH;
  cudaError_t e = cudaMemsetAsync(a.queue, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  if (!p.gstate) {
    if (kb == 4)
      ss_summarize_kernel<uint32_t, uint16_t, false><<<p.grid, 32, p.smem, s>>>(a);
    else
      ss_summarize_kernel<uint64_t, uint16_t, false><<<p.grid, 32, p.smem, s>>>(a);
  } else {
    if (kb == 4)
      ss_summarize_kernel<uint32_t, uint32_t, true><<<p.grid, 32, p.smem, s>>>(a);
    else
      ss_summarize_kernel<uint64_t, uint32_t, true><<<p.grid, 32, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace pss
