// verify.cu -- K4/K5: the off-line verification scan ("a parallel scan of the input
// can be used to determine the actual frequent items") and the final k-majority report
// (PAPER.md:47, :80).
//
// K4 streams A once with 128-bit read-only loads, software-pipelined (the next loads are in flight
// while the current ones are counted). The candidate list is a static set, so a setup kernel
// builds a two-choice cuckoo table (key, candidate index) sized for the actual number of
// candidates; every CTA copies it to shared memory and each item is looked up with two
// independent loads and no probing loop. Counting, by the candidate count nc (decided on the
// device, as nc is only known there):
//   - small nc: every lane owns a private 16-bit counter per candidate, laid out [cand][lane] so
//     a warp's increments hit 32 different banks: no atomics, no grouping;
//   - larger nc: equal indices of a warp instruction are grouped with __match_any_sync and the
//     leader adds the group size to a per-warp 32-bit counter;
//   - beyond shared memory: the same grouping with 64-bit global atomics.
// Per-CTA sums are flushed into 64-bit global accumulators at the end. K5 keeps the candidates
// whose exact count reaches floor(n/k) + 1 and ranks them by (count desc, item asc).
#include "common.cuh"

namespace pss {

#ifndef PSS_VT_THREADS
#define PSS_VT_THREADS 128
#endif
#ifndef PSS_VT_EXP
#define PSS_VT_EXP 0
#endif
#ifndef PSS_VT_U
#define PSS_VT_U 4
#endif
#ifndef PSS_VT_TAGPAD  // experiment: extra shared memory of the tagged kernel (fewer CTAs per SM)
#define PSS_VT_TAGPAD 0
#endif
#ifndef PSS_VT_TAGMINB
#define PSS_VT_TAGMINB 8
#endif
#ifndef PSS_VT_FILTER
#define PSS_VT_FILTER 0
#endif
constexpr int VTHREADS = PSS_VT_THREADS;
constexpr int VWARPS = VTHREADS / 32;
constexpr uint32_t VT_SMEM = 2048;       // table entries staged in shared memory
// shared-memory counter bytes per warp: the general kernel's, and a smaller one for up to 75
// candidates (per-lane counters only) that fits more CTAs per SM -- K4 is latency-bound, so the
// occupancy pays (H, 72 candidates: 580 -> 504 us). The candidate count is known on the device
// only: both kernels are launched when it may exceed 75 and the one that does not fit exits.
constexpr uint32_t VCW_BIG = 8192, VCW_SMALL = 4864;
__host__ __device__ constexpr uint32_t vlane_max(uint32_t vcw) { return vcw / (32 * 2); }
__host__ __device__ constexpr uint32_t vwarp_max(uint32_t vcw) { return vcw / 4; }

// table entry: (key, candidate index); index all-ones = empty
template <typename KT>
struct VEnt;
template <>
struct VEnt<uint32_t> {
  using T = unsigned long long;  // idx << 32 | key
  __device__ static __forceinline__ T make(uint32_t key, uint32_t idx) {
    return ((T)idx << 32) | key;
  }
  __device__ static __forceinline__ uint32_t key(T e) { return (uint32_t)e; }
  __device__ static __forceinline__ uint32_t idx(T e) { return (uint32_t)(e >> 32); }
  __device__ static __forceinline__ bool empty(T e) { return (uint32_t)(e >> 32) == 0xffffffffu; }
  __device__ static __forceinline__ T none() { return ~0ull; }
};
template <>
struct VEnt<uint64_t> {
  using T = ulonglong2;  // {key, idx}
  __device__ static __forceinline__ T make(uint64_t key, uint32_t idx) {
    return make_ulonglong2(key, idx);
  }
  __device__ static __forceinline__ uint64_t key(T e) { return e.x; }
  __device__ static __forceinline__ uint32_t idx(T e) { return (uint32_t)e.y; }
  __device__ static __forceinline__ bool empty(T e) { return e.y == ~0ull; }
  __device__ static __forceinline__ T none() { return make_ulonglong2(0ull, ~0ull); }
};

__device__ __forceinline__ uint32_t vfold(uint32_t x) { return x; }
__device__ __forceinline__ uint32_t vfold(uint64_t x) {
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32) ^ (uint32_t)x;
}
template <typename KT>
__device__ __forceinline__ void vhash(KT x, uint32_t seed, uint32_t logT, uint32_t& h1,
                                      uint32_t& h2) {
  const uint32_t a = vfold(x) ^ seed;
  const uint32_t ha = a * 0x9E3779B1u;
  const uint32_t hb = (ha ^ (ha >> 15)) * 0x85EBCA6Bu;
  h1 = ha >> (32u - logT);
  h2 = hb >> (32u - logT);
  h2 = h2 == h1 ? (h2 ^ 1u) : h2;  // two distinct entries per key
}

__host__ __device__ static uint32_t v_logT(uint32_t nc) {
  uint32_t l = ceil_log2(4ull * (nc ? nc : 1));
  return l < 6 ? 6 : l;
}

struct VLayout {
  size_t acc, tab, tab32, ctl, total;
};

// perfect (collision-free, one probe) tables for up to PH_MAX distinct candidates
constexpr uint32_t PH_MAX = 80;
constexpr uint32_t PH_LOG = 11;  // 2048 entries
constexpr int PH_TRIES = 64;
// Tagged one-probe table for u32 keys (K4's common case: a few dozen candidates, per-lane
// counters). ha = x * mult (mult odd: a bijection of the key); its top PH_LOG bits h are the entry,
// so the low 21 bits identify the key inside it. Entry h holds (f ^ h) << 21 | ha's low bits, f the
// key's counter code: e ^ ha is then f << 21 exactly for that key, and any other key leaves low
// bits set. Rotated left by 11 this is f for a match and >= 2048 otherwise, so min(., PH_FDUMMY)
// maps every non-candidate to the dummy counter without a compare. f = word | half << 10 of the
// 16-bit counter [word][lane]; the dummy is the upper half of word 37, above every valid code
// (at most 74 candidates). Empty entries hold the dummy's code with low bits 0. One 32-bit
// shared-memory load and 12 instructions per key instead of a 64-bit load and 18.
constexpr uint32_t PH_TAG_MAXC = 74;
constexpr uint32_t PH_FDUMMY = 1024u + 37u;
__host__ __device__ constexpr uint32_t ph_fcode(uint32_t idx) {
  return (idx >> 1) | ((idx & 1u) << 10);
}
static_assert(ph_fcode(PH_TAG_MAXC - 1) < PH_FDUMMY && PH_TAG_MAXC <= PH_MAX, "tagged entry");
static_assert((PH_FDUMMY - 1024u + 1u) * 128u <= VCW_SMALL, "tagged counters fit the small area");
// u64 keys: the same with 64-bit entries and ha = key * (a 64-bit odd multiplier derived from the
// 32-bit one): the low 53 bits identify the key (a 64-bit shared load instead of a 128-bit one).
template <typename KT>
struct VTag;
template <>
struct VTag<uint32_t> {
  using TE = uint32_t;
  static constexpr uint32_t BITS = 32 - PH_LOG;
  __host__ __device__ static __forceinline__ TE hash(uint32_t x, uint32_t mult) { return x * mult; }
};
template <>
struct VTag<uint64_t> {
  using TE = unsigned long long;
  static constexpr uint32_t BITS = 64 - PH_LOG;
  __host__ __device__ static __forceinline__ TE hash(uint64_t x, uint32_t mult) {
    return x * (((unsigned long long)mult * 0x9E3779B97F4A7C15ull) | 1ull);
  }
};
// entry of the table position h for the counter code f and the hash ha / for no key
template <typename KT>
__device__ __forceinline__ typename VTag<KT>::TE vtag_entry(uint32_t f, uint32_t h,
                                                            typename VTag<KT>::TE ha) {
  using TE = typename VTag<KT>::TE;
  return ((TE)(f ^ h) << VTag<KT>::BITS) | (ha & (((TE)1 << VTag<KT>::BITS) - 1));
}
// counter code of a key from its entry e and hash ha
template <typename KT>
__device__ __forceinline__ uint32_t vtag_code(typename VTag<KT>::TE e,
                                              typename VTag<KT>::TE ha) {
  const typename VTag<KT>::TE t = e ^ ha;
  if constexpr (sizeof(KT) == 4) {
    return min(__funnelshift_l(t, t, PH_LOG), PH_FDUMMY);
  } else {
    const unsigned long long v = (t << PH_LOG) | (t >> (64 - PH_LOG));
    return (uint32_t)min(v, (unsigned long long)PH_FDUMMY);
  }
}

static VLayout v_layout(int kb, uint32_t cap) {
  VLayout L;
  Bump b;
  L.acc = b.take<unsigned long long>(cap ? cap : 1);
  L.tab = b.take<unsigned char>(((size_t)1 << std::max(v_logT(cap), PH_LOG)) * (kb == 4 ? 8 : 16));
  L.tab32 = b.take<unsigned long long>((size_t)1 << PH_LOG);  // tagged one-probe table
  // [0] seed, [1] logT, [2] 1 = perfect table, [3] multiplier of the tagged table (0 = none)
  L.ctl = b.take<uint32_t>(4);
  L.total = b.bytes();
  return L;
}

__device__ __forceinline__ uint32_t eff_count(uint32_t cap, const uint32_t* d_n) {
  return d_n ? min(cap, *d_n) : cap;
}

// candidate index of x in the table, or 0xffffffff (perfect: one entry per key)
template <typename KT>
__device__ __forceinline__ uint32_t vlookup(const typename VEnt<KT>::T* tab, KT x, uint32_t seed,
                                            uint32_t logT, bool perfect) {
  uint32_t h1, h2;
  vhash(x, seed, logT, h1, h2);
  // an empty entry's index is 0xffffffff, so a key equal to its filler still finds nothing
  const typename VEnt<KT>::T a = tab[h1];
  const uint32_t ia = VEnt<KT>::key(a) == x ? VEnt<KT>::idx(a) : 0xffffffffu;
  if (perfect) return ia;
  const typename VEnt<KT>::T b = tab[h2];
  const uint32_t ib = VEnt<KT>::key(b) == x ? VEnt<KT>::idx(b) : 0xffffffffu;
  return min(ia, ib);
}
template <typename KT>
__device__ __forceinline__ uint32_t vlookup(const typename VEnt<KT>::T* tab, KT x, uint32_t seed,
                                            uint32_t logT) {
  return vlookup<KT>(tab, x, seed, logT, false);
}

// builds the cuckoo table of the (deduplicated) candidates, sized for the actual count; zeroes
// the accumulators
template <typename KT>
__global__ void verify_setup_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                                    unsigned long long* acc, typename VEnt<KT>::T* tab,
                                    void* tab32v, uint32_t* ctl) {
  using VT = typename VEnt<KT>::T;
  using TE = typename VTag<KT>::TE;
  TE* const tab32 = static_cast<TE*>(tab32v);
  const uint32_t nc = eff_count(cap, d_n);
  for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) acc[j] = 0;
  // perfect table: find a seed under which the (distinct) candidates occupy distinct entries
  __shared__ uint32_t occ[(1u << PH_LOG) / 32];
  __shared__ uint32_t clash;
  if (nc > 0 && nc <= PH_MAX) {
    const uint32_t TP = 1u << PH_LOG;
    for (int tr = 0; tr < PH_TRIES; ++tr) {
      const uint32_t seed = (uint32_t)tr * 0x9E3779B9u + 0x7F4A7C15u;
      for (uint32_t i = threadIdx.x; i < TP / 32; i += blockDim.x) occ[i] = 0;
      if (threadIdx.x == 0) clash = 0;
      __syncthreads();
      uint32_t h = 0, h2;
      if (threadIdx.x < nc) {
        vhash(cand[threadIdx.x], seed, PH_LOG, h, h2);
        const uint32_t old = atomicOr(&occ[h >> 5], 1u << (h & 31));
        if (old & (1u << (h & 31))) clash = 1;  // also catches duplicate candidates
      }
      __syncthreads();
      if (!clash) {
        for (uint32_t e = threadIdx.x; e < TP; e += blockDim.x) tab[e] = VEnt<KT>::none();
        __syncthreads();
        if (threadIdx.x < nc) tab[h] = VEnt<KT>::make(cand[threadIdx.x], threadIdx.x);
        if (threadIdx.x == 0) {
          ctl[0] = seed;
          ctl[1] = PH_LOG;
          ctl[2] = 1;
          ctl[3] = 0;
        }
        // the tagged table: its own multiplier search; ctl[3] = multiplier, 0 = none
        if (nc <= PH_TAG_MAXC) {
          for (int t2 = 0; t2 < PH_TRIES; ++t2) {
            const uint32_t mult = ((uint32_t)t2 * 0x9E3779B9u + 0x85EBCA6Bu) | 1u;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < TP / 32; i += blockDim.x) occ[i] = 0;
            if (threadIdx.x == 0) clash = 0;
            __syncthreads();
            TE ha = 0;
            uint32_t hh = 0;
            if (threadIdx.x < nc) {
              ha = VTag<KT>::hash(cand[threadIdx.x], mult);
              hh = (uint32_t)(ha >> VTag<KT>::BITS);
              if (atomicOr(&occ[hh >> 5], 1u << (hh & 31)) & (1u << (hh & 31))) clash = 1;
            }
            __syncthreads();
            if (clash) continue;
            for (uint32_t e = threadIdx.x; e < TP; e += blockDim.x)
              tab32[e] = vtag_entry<KT>(PH_FDUMMY, e, 0);
            __syncthreads();
            if (threadIdx.x < nc) tab32[hh] = vtag_entry<KT>(ph_fcode(threadIdx.x), hh, ha);
            if (threadIdx.x == 0) ctl[3] = mult;
            break;
          }
        }
        return;
      }
      __syncthreads();
    }
  }
  // two-choice cuckoo table (duplicates allowed: the first occurrence owns the entry)
  const uint32_t logT = v_logT(nc);
  const uint32_t T = 1u << logT;
  for (uint32_t h = threadIdx.x; h < T; h += blockDim.x) tab[h] = VEnt<KT>::none();
  __syncthreads();
  if (threadIdx.x != 0) return;
  ctl[2] = 0;
  ctl[3] = 0;
  for (uint32_t seed = 0;; seed += 0x9E3779B9u) {
    if (seed)
      for (uint32_t h = 0; h < T; ++h) tab[h] = VEnt<KT>::none();
    bool ok = true;
    for (uint32_t j = 0; j < nc && ok; ++j) {
      KT x = cand[j];
      if (vlookup<KT>(tab, x, seed, logT) != 0xffffffffu) continue;  // duplicate: first wins
      uint32_t idx = j;
      uint32_t prev = 0xffffffffu;
      ok = false;
      for (int step = 0; step < 500; ++step) {
        uint32_t h1, h2;
        vhash(x, seed, logT, h1, h2);
        if (VEnt<KT>::empty(tab[h1])) {
          tab[h1] = VEnt<KT>::make(x, idx);
          ok = true;
          break;
        }
        if (VEnt<KT>::empty(tab[h2])) {
          tab[h2] = VEnt<KT>::make(x, idx);
          ok = true;
          break;
        }
        const uint32_t h = (h1 != prev) ? h1 : h2;
        const VT e = tab[h];
        tab[h] = VEnt<KT>::make(x, idx);
        x = VEnt<KT>::key(e);
        idx = VEnt<KT>::idx(e);
        prev = h;
      }
    }
    if (ok) {
      ctl[0] = seed;
      ctl[1] = logT;
      return;
    }
  }
}

// fire-and-forget shared-memory add (no return value, so no scoreboard wait on the result)
__device__ __forceinline__ void red_shared_add(uint32_t* p, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// One warp's scan of its share of A. MODE 0: per-lane 16-bit counters, two per 32-bit word laid
// out [cand / 2][lane] (a warp's adds hit 32 banks and never the same word), added with
// red.shared so successive increments do not wait on each other; MODE 1: __match_any_sync groups
// + per-warp 32-bit counters; MODE 2: groups + 64-bit global atomics. PERF: one-probe table.
template <typename KT, int MODE, bool PERF, bool TAG = false>
__device__ __forceinline__ void verify_scan(const KT* __restrict__ A, uint64_t n,
                                            const typename VEnt<KT>::T* tab, uint32_t seed,
                                            uint32_t logT, uint32_t* lw, uint32_t* wc,
                                            unsigned long long* acc, uint64_t wid,
                                            uint64_t nwarps, uint32_t nc, uint32_t fw = 0) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t ltm = lanemask_lt();
  uint32_t* const lwl = lw + lane;
  const uint32_t lwl_addr = smem_u32(lwl);
  (void)lwl_addr;
#if PSS_VT_EXP == 2 || PSS_VT_EXP == 3  // timing experiment: no table lookup
  auto look = [&](KT x) { return (uint32_t)x & 31u; };
#elif PSS_VT_FILTER
  // one-probe table behind a 1024-bit filter held one word per lane (bit b: an occupied entry
  // whose index is b modulo 1024): a non-candidate usually costs a shuffle, not a table read
  auto look = [&](KT x) -> uint32_t {
    if (!PERF) return vlookup<KT>(tab, x, seed, logT, PERF);
    uint32_t h1, h2;
    vhash(x, seed, logT, h1, h2);
    const uint32_t fb = h1 & 1023u;
    const uint32_t w = __shfl_sync(PSS_FULL, fw, fb >> 5);
    if (!((w >> (fb & 31u)) & 1u)) return 0xffffffffu;
    const typename VEnt<KT>::T a = tab[h1];
    return VEnt<KT>::key(a) == x ? VEnt<KT>::idx(a) : 0xffffffffu;
  };
#else
  auto look = [&](KT x) -> uint32_t {
    if constexpr (TAG) {  // tagged entries: the counter code, PH_FDUMMY for no candidate
      using TE = typename VTag<KT>::TE;
      const TE ha = VTag<KT>::hash(x, seed);  // seed = the table's multiplier
      const TE e = reinterpret_cast<const TE*>(tab)[(uint32_t)(ha >> VTag<KT>::BITS)];
      return vtag_code<KT>(e, ha);
    } else {
      return vlookup<KT>(tab, x, seed, logT, PERF);
    }
  };
#endif
#if PSS_VT_EXP == 1 || PSS_VT_EXP == 3  // timing experiment: no counting
  uint32_t sink = 0;
  auto count1 = [&](uint32_t j) { sink += j; };
#else
  auto count1 = [&](uint32_t j) {
    if (TAG) {  // j = counter code: word | half << 10 (0xffffffff: an item outside A)
      const uint32_t f = min(j, PH_FDUMMY);
      uint32_t ad;  // lwl + word * 32 words, as one multiply-add
      asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(ad) : "r"(f & 1023u), "r"(lwl_addr));
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ad), "r"((f >> 10) * 65535u + 1u)
                   : "memory");
    } else if (MODE == 0) {  // no candidate: counted in the dummy counter nc (no branch)
      const uint32_t jj = min(j, nc);
      red_shared_add(lwl + (jj >> 1) * 32, 1u << ((jj & 1u) << 4));
    } else {
      const uint32_t g = __match_any_sync(PSS_FULL, j);
      if ((g & ltm) == 0 && j != 0xffffffffu) {
        if (MODE == 1)
          wc[j] += __popc(g);
        else
          atomicAdd(&acc[j], (unsigned long long)__popc(g));
      }
    }
  };
#endif

  constexpr uint32_t E = 16 / sizeof(KT);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(A);
  uint64_t head = ((16u - (addr & 15u)) & 15u) / sizeof(KT);
  if ((addr % sizeof(KT)) != 0) head = n;  // not naturally aligned: scalar path only
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / E;
  const uint64_t tail0 = head + nvec * E;
  // scalar head and tail (warp-uniform loops)
  for (uint64_t base = wid * 32; base < head; base += nwarps * 32) {
    const uint64_t i = base + lane;
    const uint32_t j = look(i < head ? A[i] : KT(0));  // every lane looks (shuffles inside)
    count1(i < head ? j : 0xffffffffu);
  }
  const uint4* V = reinterpret_cast<const uint4*>(A + head);
  const uint64_t stride = nwarps * 32;
  // software pipeline over U 16-byte loads per lane; all lanes of a warp take the same trip count
  constexpr int U = PSS_VT_U;
  uint4 q[U], nq[U];
  uint64_t vb = wid * 32;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t va = vb + u * stride + lane;
    q[u] = va < nvec ? __ldg(V + va) : make_uint4(0, 0, 0, 0);
  }
  // steady state, two batches per trip (q and nq alternate, no register copies): the batches
  // being loaded lie entirely inside A, no bounds checks
  auto process = [&](const uint4(&b)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const KT* xs = reinterpret_cast<const KT*>(&b[u]);
#pragma unroll
      for (uint32_t e = 0; e < E; ++e) count1(look(xs[e]));
    }
  };
  for (; vb + 3 * U * stride <= nvec; vb += 2 * U * stride) {
    const uint4* p = V + vb + lane;
#pragma unroll
    for (int u = 0; u < U; ++u) nq[u] = __ldg(p + (U + u) * stride);
    process(q);
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = __ldg(p + (2 * U + u) * stride);
    process(nq);
  }
  for (; vb < nvec; vb += U * stride) {
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = vb + u * stride + lane < nvec;
      const uint64_t vn = vb + (U + u) * stride + lane;
      nq[u] = vn < nvec ? __ldg(V + vn) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const KT* xs = reinterpret_cast<const KT*>(&q[u]);
#pragma unroll
      for (uint32_t e = 0; e < E; ++e) {
        const uint32_t j = look(xs[e]);
        count1(ok[u] ? j : 0xffffffffu);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = nq[u];
  }
  for (uint64_t base = tail0 + wid * 32; base < n; base += nwarps * 32) {
    const uint64_t i = base + lane;
    const uint32_t j = look(i < n ? A[i] : KT(0));
    count1(i < n ? j : 0xffffffffu);
  }
#if PSS_VT_EXP == 1 || PSS_VT_EXP == 3
  if (sink == 0x12345678u) acc[0] = sink;
#endif
}

// lane_ok: per-lane 16-bit counters cannot overflow for this launch (host-checked).
// The VCW_SMALL kernel of u32 keys is the tagged one (TAG): it takes the launches whose candidates
// sit in a one-probe table (perf) and fit per-lane counters; everything else goes to VCW_BIG.
template <typename KT, uint32_t VCW>
struct VKern {
  static constexpr bool TAG = VCW == VCW_SMALL;
  static constexpr size_t TAB_BYTES =
      TAG ? (sizeof(typename VTag<KT>::TE) << PH_LOG) : (size_t)VT_SMEM * sizeof(typename VEnt<KT>::T);
  static constexpr size_t SMEM = TAB_BYTES + (size_t)VWARPS * VCW + (TAG ? PSS_VT_TAGPAD : 0);
  // CTAs per SM the registers must allow
  static constexpr int MINB = TAG ? (sizeof(KT) == 4 ? PSS_VT_TAGMINB : 6) : 1;
};

template <typename KT, uint32_t VCW>
__global__ void __launch_bounds__(VTHREADS, VKern<KT, VCW>::MINB) verify_kernel(const KT* __restrict__ A, uint64_t n,
                                                          uint32_t cap, const uint32_t* d_n,
                                                          unsigned long long* acc,
                                                          const typename VEnt<KT>::T* gtab,
                                                          const void* gtab32v,
                                                          const uint32_t* ctl, uint32_t lane_ok) {
  using VT = typename VEnt<KT>::T;
  constexpr bool TAG = VKern<KT, VCW>::TAG;
  extern __shared__ __align__(16) unsigned char vsm[];
  const uint32_t nc = eff_count(cap, d_n);
  if (nc == 0) return;
  const uint32_t seed = TAG ? ctl[3] : ctl[0], logT = ctl[1];
  const bool perf = ctl[2] != 0;
  const uint32_t T = 1u << logT;
  const uint32_t warp = threadIdx.x >> 5;
  // counting mode (uniform): 0 per-lane u16, 1 per-warp u32 + match, 2 global + match
  const bool small_fits = lane_ok && perf && ctl[3] != 0 && nc <= PH_TAG_MAXC;
  if (small_fits != (VCW == VCW_SMALL)) return;  // the other kernel's case
  const int mode = (lane_ok && nc < vlane_max(VCW) && T <= VT_SMEM) ? 0
                   : (nc <= vwarp_max(VCW) ? 1 : 2);
  VT* stab = reinterpret_cast<VT*>(vsm);
  unsigned char* carea = vsm + VKern<KT, VCW>::TAB_BYTES;
  // words per lane in mode 0 (nc counters + the dummy; the tagged kernel's dummy is fixed)
  const uint32_t ncw = TAG ? PH_FDUMMY - 1024u + 1u : (nc + 2) / 2;
  uint32_t* lw = reinterpret_cast<uint32_t*>(carea) + (size_t)warp * ncw * 32;  // [cand/2][lane]
  uint32_t* wc = reinterpret_cast<uint32_t*>(carea) + (size_t)warp * nc;        // [cand]
  const bool tab_smem = T <= VT_SMEM;
  if (TAG) {
    using TE = typename VTag<KT>::TE;
    for (uint32_t h = threadIdx.x; h < (1u << PH_LOG); h += VTHREADS)
      reinterpret_cast<TE*>(vsm)[h] = static_cast<const TE*>(gtab32v)[h];
  } else
  if (tab_smem)
    for (uint32_t h = threadIdx.x; h < T; h += VTHREADS) stab[h] = gtab[h];
  if (mode == 0)
    for (uint32_t i = threadIdx.x; i < VWARPS * ncw * 32; i += VTHREADS)
      reinterpret_cast<uint32_t*>(carea)[i] = 0;
  else if (mode == 1)
    for (uint32_t i = threadIdx.x; i < VWARPS * nc; i += VTHREADS)
      reinterpret_cast<uint32_t*>(carea)[i] = 0;
  __syncthreads();
  const uint64_t wid = (uint64_t)blockIdx.x * VWARPS + warp;
  const uint64_t nwarps = (uint64_t)gridDim.x * VWARPS;
  if (mode == 0) {
    uint32_t fw = 0;
#if PSS_VT_FILTER
    if (perf) {  // this lane's word of the filter: entries 32*lane + i and 1024 + 32*lane + i
      const uint32_t lane = threadIdx.x & 31u;
      for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t h = 32 * lane + i;
        const bool occ = !VEnt<KT>::empty(stab[h]) || (h + 1024 < T && !VEnt<KT>::empty(stab[h + 1024]));
        fw |= (occ ? 1u : 0u) << i;
      }
    }
#endif
    if (TAG)
      verify_scan<KT, 0, true, TAG>(A, n, stab, seed, logT, lw, wc, acc, wid, nwarps, nc, fw);
    else if (perf)
      verify_scan<KT, 0, true>(A, n, stab, seed, logT, lw, wc, acc, wid, nwarps, nc, fw);
    else
      verify_scan<KT, 0, false>(A, n, stab, seed, logT, lw, wc, acc, wid, nwarps, nc);
  } else {
    const VT* tab = tab_smem ? stab : gtab;
    if (mode == 1)
      verify_scan<KT, 1, false>(A, n, tab, seed, logT, lw, wc, acc, wid, nwarps, nc);
    else
      verify_scan<KT, 2, false>(A, n, tab, seed, logT, lw, wc, acc, wid, nwarps, nc);
  }
  if (mode != 2) {
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < nc; c += VTHREADS) {
      unsigned long long t = 0;
      if (mode == 0) {
        const uint32_t* base = reinterpret_cast<const uint32_t*>(carea);
        const uint32_t sh = (c & 1u) << 4;
        for (uint32_t w = 0; w < VWARPS; ++w)
          for (uint32_t l = 0; l < 32; ++l)
            t += (base[((size_t)w * ncw + (c >> 1)) * 32 + l] >> sh) & 0xffffu;
      } else {
        const uint32_t* base = reinterpret_cast<const uint32_t*>(carea);
        for (uint32_t w = 0; w < VWARPS; ++w) t += base[(size_t)w * nc + c];
      }
      if (t) atomicAdd(&acc[c], t);
    }
  }
}

// exact[j] = the count accumulated for the first position holding cand[j] (duplicates share it)
template <typename KT>
__global__ void verify_finalize_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                                       const unsigned long long* acc,
                                       const typename VEnt<KT>::T* tab, const uint32_t* ctl,
                                       uint64_t* exact) {
  const uint32_t nc = eff_count(cap, d_n);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const uint32_t f = vlookup<KT>(tab, cand[j], ctl[0], ctl[1], ctl[2] != 0);
  exact[j] = acc[f];
}

size_t verify_ws(int kb, uint32_t cap, const DevInfo&) { return v_layout(kb, cap).total; }

template <typename KT>
static cudaError_t verify_run(const KT* A, uint64_t n, const KT* cand, uint32_t cap,
                              const uint32_t* d_n, uint64_t* exact, void* ws, cudaStream_t s,
                              const DevInfo& d) {
  using VT = typename VEnt<KT>::T;
  VLayout L = v_layout(sizeof(KT), cap);
  unsigned char* w = static_cast<unsigned char*>(ws);
  auto* acc = reinterpret_cast<unsigned long long*>(w + L.acc);
  auto* tab = reinterpret_cast<VT*>(w + L.tab);
  auto* ctl = reinterpret_cast<uint32_t*>(w + L.ctl);
  void* tab32 = w + L.tab32;
  if (cap == 0) return cudaSuccess;
  verify_setup_kernel<KT><<<1, 1024, 0, s>>>(cand, cap, d_n, acc, tab, tab32, ctl);
  // per-lane 16-bit counters cannot overflow: a lane counts at most n / (CTAs * VTHREADS) + the
  // head/tail items; checked against the smaller of the two grids (the big kernel's)
  int nb_big = 0;
  allow_max_smem(verify_kernel<KT, VCW_BIG>, d);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb_big, verify_kernel<KT, VCW_BIG>, VTHREADS,
                                                VKern<KT, VCW_BIG>::SMEM);
  const uint64_t want0 = (n + (uint64_t)VTHREADS * 64 - 1) / ((uint64_t)VTHREADS * 64);
  const uint64_t grid_min = std::max<uint64_t>(1, std::min<uint64_t>(want0, (uint64_t)std::max(nb_big, 1) * d.sms));
  const uint32_t lane_ok = n / (grid_min * VTHREADS) + 64 < 65535u;
  auto launch = [&](auto kern, size_t smem) {
    allow_max_smem(kern, d);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, VTHREADS, smem);
    if (nb < 1) nb = 1;
    const uint64_t want = (n + (uint64_t)VTHREADS * 64 - 1) / ((uint64_t)VTHREADS * 64);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)nb * d.sms));
    // items one lane counts: at most ceil(n / (grid * VTHREADS)) + the head/tail; both
    // kernels must agree on it (the small kernel's grid is the larger one)
    kern<<<grid, VTHREADS, smem, s>>>(A, n, cap, d_n, acc, tab, tab32, ctl, lane_ok);
  };
  launch(verify_kernel<KT, VCW_SMALL>, VKern<KT, VCW_SMALL>::SMEM);
  // the small kernel takes tagged one-probe tables only, so the general one is always launched
  // (it exits at once when the case is the small kernel's)
  launch(verify_kernel<KT, VCW_BIG>, VKern<KT, VCW_BIG>::SMEM);
  verify_finalize_kernel<KT><<<(cap + 255) / 256, 256, 0, s>>>(cand, cap, d_n, acc, tab, ctl, exact);
  return cudaGetLastError();
}

cudaError_t verify_launch(const void* A, uint64_t n, int kb, const void* cand, uint32_t cap,
                          const uint32_t* d_n_cand, uint64_t* exact, void* ws, cudaStream_t s,
                          const DevInfo& d) {
  if (kb == 4)
    return verify_run<uint32_t>(static_cast<const uint32_t*>(A), n,
                                static_cast<const uint32_t*>(cand), cap, d_n_cand, exact, ws, s, d);
  return verify_run<uint64_t>(static_cast<const uint64_t*>(A), n,
                              static_cast<const uint64_t*>(cand), cap, d_n_cand, exact, ws, s, d);
}

// ---- K5: {(x, f(x)) : f(x) >= floor(n/k) + 1}, ranked by (f desc, x asc). Internal: the
// candidates come from pss_prune, i.e. distinct root items.
template <typename KT>
__global__ void result_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                              const uint64_t* exact, uint64_t thr, KT* out_items,
                              uint64_t* out_counts, uint32_t* out_len) {
  const uint32_t nc = eff_count(cap, d_n);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) {
    uint32_t len = 0;
    for (uint32_t i = 0; i < nc; ++i) len += exact[i] >= thr;
    *out_len = len;
  }
  if (j >= nc || exact[j] < thr) return;
  const KT x = cand[j];
  const uint64_t f = exact[j];
  uint32_t rank = 0;
  for (uint32_t i = 0; i < nc; ++i)
    rank += exact[i] >= thr && (exact[i] > f || (exact[i] == f && cand[i] < x));
  out_items[rank] = x;
  out_counts[rank] = f;
}

cudaError_t result_launch(int kb, uint32_t cap, const void* cand, const uint32_t* d_n_cand,
                          const uint64_t* exact, uint64_t n, uint32_t k, void* out_items,
                          uint64_t* out_counts, uint32_t* out_len, cudaStream_t s) {
  const uint64_t thr = n / k + 1;
  const int grid = (int)((cap + 255) / 256 + (cap == 0));
  if (kb == 4)
    result_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(cand), cap,
                                                 d_n_cand, exact, thr,
                                                 static_cast<uint32_t*>(out_items), out_counts,
                                                 out_len);
  else
    result_kernel<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(cand), cap,
                                                 d_n_cand, exact, thr,
                                                 static_cast<uint64_t*>(out_items), out_counts,
                                                 out_len);
  return cudaGetLastError();
}

}  // namespace pss
