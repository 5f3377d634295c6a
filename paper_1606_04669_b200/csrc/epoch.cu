// epoch.cu -- K1e: per-partition Space Saving summaries (Algorithm 1 lines 3-5, PAPER.md:92-96;
// update rules PAPER.md:82) computed one *epoch* at a time by a whole CTA.
//
// Sequential Space Saving with R1/R2 restated per epoch (K1e):
// an epoch begins when a minimum level m forms; its members are B = {slots with count m} in slot
// order, r = 0..b-1 (the fill phase is the epoch m = 0 whose members are the k free slots).
//  * During the epoch only members can leave the summary, and only by being the lowest
//    unconsumed member when a miss arrives. So a key that is monitored with count > m (S), or
//    that entered during the epoch (count m + 1), is hit by every occurrence in the epoch.
//  * An *event* is the first occurrence in the epoch of a key that was unmonitored (U) or a
//    member (V) at the epoch start. A U event is a miss and pops the lowest unconsumed member; a V
//    event either hits its member (which is consumed) or, if that member was popped already, is a
//    miss that pops the lowest unconsumed one. Every event consumes exactly one member, so the
//    epoch ends right after its b-th event, and the new minimum is m + 1.
//  * With v = event index (time order) and r = member index (slot order), the V event of member r
//    is a hit iff  v - r <= |{hit V events y : r_y > r, v_y < v}|  (the pointer of pops lags the
//    event count by the hits ahead of it). The j-th miss in time order pops the j-th member that
//    is not hit, in slot order. A popped member takes the miss's key, count m + (occurrences of
//    that key in the epoch), error m; hit members and S keys add their occurrences.
// tools/epoch_model.py runs exactly this formulation on the host and equals sequential Space
// Saving there; the GPU parity tests (tests/test_epoch.py) compare K1e's leaves bit for bit.
//
// The CTA streams its block in windows of NT * R items (registers, prefetched one window ahead).
// Per window: (1) every item is looked up in the epoch-start index (a two-choice table of 4-way
// buckets holding the keys, rebuilt at every epoch end with a member flag per entry), S items are
// classified at once, V items lower their member's first-occurrence time (atomicMin), U items are
// found in or inserted into the epoch's U table (64-bit entries key << 32 | first time:
// atomicCAS, then atomicMin); (2) after a barrier an item is an event iff its time is its key's
// first time; events are ranked in time order by ballots and a scan of per-warp counts; (3) items
// up to the epoch's b-th event add their occurrence (red.shared) to their slot or U entry and
// write their event. When the b-th event is in the window, the epoch is resolved (one warp finds
// the V hits by the closed form, 32 events at a time; all threads rank misses and pops, then
// apply), the index is rebuilt for level m + 1, and the rest of the window is processed again
// under the new state. No step is speculative: every item is applied exactly once, in its epoch.
#include <cstdlib>

#include "common.cuh"

namespace pss {

constexpr uint32_t EP_E16 = 0xffffu;  // empty index entry (slot field)
constexpr unsigned long long EP_UEMPTY = ~0ull;  // empty U-table entry (a time is never 2^32-1)
constexpr uint32_t EP_VFLAG = 0x8000u;  // index entry / event code: a member (V)
constexpr uint32_t EP_KMAX = 2048;      // slots fit 15 bits with the flag, member bitmaps 64 words
constexpr uint32_t EP_KW = EP_KMAX / 32;
constexpr uint32_t EP_HIT = 0xffffu;    // event code of a V hit (after resolution)
constexpr uint32_t EP_OVF = 64;         // homeless keys a rebuild places by cuckoo kicks
#ifndef PSS_EP_MIN_CTAS
#define PSS_EP_MIN_CTAS 4
#endif
constexpr int EP_MIN_CTAS = PSS_EP_MIN_CTAS;

struct EpArgs {
  const uint32_t* A;
  uint64_t n;
  uint32_t k, P;
  uint32_t r0, r1;
  uint32_t T;                  // > 1: two-level (hybrid) decomposition
  uint32_t* leaf_flags;        // non-null: leaf_flags[r] = 1 (release) once leaf r is written
  int pdl;
  uint32_t* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
  uint32_t* queue;
  const unsigned char* skip;   // non-null: only leaves r with skip[r] != 0
  uint32_t cb;                 // counter word: count in the low cb bits, error above
  uint32_t NB;                 // index buckets (4 ways)
  uint32_t UC;                 // U-table entries
  uint32_t o_cw, o_vft, o_ml, o_tk, o_ts, o_fill, o_ut, o_uo, o_ev, o_vl, o_bits;
  volatile unsigned* hb;  // debug heartbeat (PSS_EP_HB builds): host-mapped, 8 words per CTA
};

#ifdef PSS_EP_HB
#define EPHB(ph)                                                        \
  do {                                                                  \
    if (tid == 0 && a.hb) {                                             \
      volatile unsigned* _h = a.hb + 8 * blockIdx.x;                   \
      _h[0] = r; _h[1] = q_dbg; _h[2] = eseq; _h[3] = m; _h[4] = b;    \
      _h[5] = ecount; _h[6] = (ph); _h[7] = _h[7] + 1;                  \
    }                                                                   \
  } while (0)
__device__ __forceinline__ uint32_t ep_idx(uint32_t i, uint32_t n, uint32_t code,
                                           volatile unsigned* hb, uint32_t r, uint32_t eseq) {
  if (i < n) return i;
  if (hb && atomicCAS((unsigned*)(hb + 8 * 4000), 0u, code) == 0u) {
    hb[8 * 4000 + 1] = i;
    hb[8 * 4000 + 2] = n;
    hb[8 * 4000 + 3] = r;
    hb[8 * 4000 + 4] = eseq;
    hb[8 * 4000 + 5] = blockIdx.x;
    hb[8 * 4000 + 6] = threadIdx.x;
  }
  return 0;
}
#define EPIDX(i, n, code) ep_idx((i), (n), (code), a.hb, r, eseq)
#else
#define EPHB(ph) \
  do {           \
  } while (0)
#define EPIDX(i, n, code) (i)
#endif

#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)  // debug builds only (tools/epoch_debug.py): the first broken invariant
__device__ unsigned int g_ep_dbg[16];
#define EPREC(cond, code, a0, a1, a2)                                              \
  do {                                                                             \
    if (!(cond) && atomicCAS(&g_ep_dbg[0], 0u, (unsigned)(code)) == 0u) {          \
      g_ep_dbg[1] = r;                                                             \
      g_ep_dbg[2] = m;                                                             \
      g_ep_dbg[3] = b;                                                             \
      g_ep_dbg[4] = ecount;                                                        \
      g_ep_dbg[5] = (unsigned)(a0);                                                \
      g_ep_dbg[6] = (unsigned)(a1);                                                \
      g_ep_dbg[7] = (unsigned)(a2);                                                \
      g_ep_dbg[8] = eseq;                                                          \
      g_ep_dbg[9] = size;                                                          \
    }                                                                              \
  } while (0)
#ifdef PSS_EP_DUMP  // per-epoch snapshots of leaf 0: [epoch][0..3] = m, ne, nvv, nh; then keys, cw
constexpr int EP_DUMP_E = 96;
__device__ unsigned int g_ep_dump[EP_DUMP_E][4 + 2 * EP_KMAX];
#endif
}  // namespace pss
extern "C" int pss_debug_epoch_dump(unsigned* out) {
#ifdef PSS_EP_DUMP
  cudaMemcpyFromSymbol(out, pss::g_ep_dump, sizeof(pss::g_ep_dump));
#endif
  return (int)cudaGetLastError();
}
extern "C" int pss_debug_epoch(unsigned* out, int reset) {
  cudaMemcpyFromSymbol(out, pss::g_ep_dbg, sizeof(pss::g_ep_dbg));
  if (reset) {
    unsigned z[16] = {};
    cudaMemcpyToSymbol(pss::g_ep_dbg, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
namespace pss {
#else
#define EPREC(cond, code, a0, a1, a2) \
  do {                                \
  } while (0)
#endif
#ifdef PSS_EP_DEBUG  // invariant checks (extra reads); guards (loop caps) in both debug builds
#define EPCHK(cond, code, a0, a1, a2) EPREC(cond, code, a0, a1, a2)
#else
#define EPCHK(cond, code, a0, a1, a2) \
  do {                                \
  } while (0)
#endif
#define EPWATCH(cond, code, a0, a1, a2) EPREC(cond, code, a0, a1, a2)

#ifdef PSS_EP_TIMING  // debug build: cycles per stage, summed over CTAs (tid 0's view)
__device__ unsigned long long g_ep_tm[16];
}  // namespace pss
extern "C" int pss_debug_epoch_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pss::g_ep_tm, sizeof(pss::g_ep_tm));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(pss::g_ep_tm, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
namespace pss {
#define EPTM(i)                                         \
  do {                                                  \
    if (tid == 0) {                                     \
      const long long _n = clock64();                   \
      atomicAdd(&g_ep_tm[i], (unsigned long long)(_n - tm0)); \
      tm0 = _n;                                         \
    }                                                   \
  } while (0)
#else
#define EPTM(i) \
  do {          \
  } while (0)
#endif

// block barrier entered by converged warps only: bar.sync counts a warp as arrived when any of its
// lanes executes it, so lanes that diverged (the U-table claim loop) must reconverge first
__device__ __forceinline__ void ep_bar() {
  __syncwarp();
  __syncthreads();
}

// index hash (seeded: a failed rebuild reseeds)
__device__ __forceinline__ void ep_hash(uint32_t x, uint32_t seed, uint32_t NB, uint32_t& b1,
                                        uint32_t& b2) {
  const uint32_t ha = (x ^ seed) * 0x9E3779B1u;
  const uint32_t hb = (ha ^ (ha >> 16)) * 0x85EBCA6Bu;
  b1 = __umulhi(ha, NB);
  b2 = __umulhi(hb, NB);
}
__device__ __forceinline__ uint32_t ep_uhash(uint32_t x, uint32_t UC) {
  const uint32_t h = (x ^ (x >> 15)) * 0x2C1B3C6Du;
  return __umulhi(h ^ (h >> 12), UC);
}

template <int NT, int R>
__global__ void __launch_bounds__(NT, EP_MIN_CTAS) ep_kernel(const EpArgs a) {
  constexpr uint32_t NW = NT / 32;
  constexpr uint32_t SW = NT * R;  // items per window
  static_assert(R * NW <= 32, "one warp scans the per-warp counts");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t cbuf[R * NW];  // per (row, warp): events | V events << 16
  // [0] leaf id, [1] V events of an ended epoch, [2] rebuild failed, [3] b, [4] hits,
  // [5] time of the epoch's last item, [6] homeless keys of a rebuild
  __shared__ uint32_t s_misc[8];
  __shared__ uint32_t s_ovf[EP_OVF];  // keys whose two buckets were full in a rebuild
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t ltm = lanemask_lt();
#ifdef PSS_EP_TIMING
  long long tm0 = clock64();
#endif

  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
  uint32_t* cw = reinterpret_cast<uint32_t*>(smem + a.o_cw);     // count | err << cb
  uint32_t* vft = reinterpret_cast<uint32_t*>(smem + a.o_vft);   // member first time (stamped)
  uint16_t* ml = reinterpret_cast<uint16_t*>(smem + a.o_ml);     // misses in time order
  uint32_t* tk = reinterpret_cast<uint32_t*>(smem + a.o_tk);     // index keys [NB][4]
  uint16_t* ts = reinterpret_cast<uint16_t*>(smem + a.o_ts);     // index slot | VFLAG [NB][4]
  uint32_t* fill = reinterpret_cast<uint32_t*>(smem + a.o_fill); // 16-bit fill counts, 2 per word
  unsigned long long* ut = reinterpret_cast<unsigned long long*>(smem + a.o_ut);
  uint32_t* uo = reinterpret_cast<uint32_t*>(smem + a.o_uo);     // U-key occurrences
  uint16_t* ev = reinterpret_cast<uint16_t*>(smem + a.o_ev);     // events: uid | VFLAG | slot
  uint16_t* vl = reinterpret_cast<uint16_t*>(smem + a.o_vl);     // V event indices (time order)
  uint32_t* memb = reinterpret_cast<uint32_t*>(smem + a.o_bits); // member bitmap (slots)
  uint32_t* wpre = memb + EP_KW;   // exclusive prefix of popc(memb) per word
  uint32_t* hsl = wpre + EP_KW;    // hit members (slots)
  uint32_t* hr = hsl + EP_KW;      // hit members (member index)
  uint32_t* hc = hr + EP_KW;       // hits per 32 events
  uint32_t* hcp = hc + EP_KW;      // exclusive prefix of hc
  uint32_t* aux = hcp + EP_KW;     // H suffix counts (65) / popped members before each word
  const uint4* tk4 = reinterpret_cast<const uint4*>(tk);
  const uint2* ts2 = reinterpret_cast<const uint2*>(ts);

  const uint32_t k = a.k, UC = a.UC, UB = a.UC / 4, cb = a.cb;
#ifdef PSS_EP_NBDIV  // debug: a crowded index (frequent rebuild overflows)
  const uint32_t NB = max(1u, a.NB * 2 / PSS_EP_NBDIV);
#else
  const uint32_t NB = a.NB;
#endif
  const uint32_t KW = (k + 31u) / 32u;
  const uint32_t CM = (1u << cb) - 1u;
  const uint32_t* __restrict__ A = a.A;
  if (tid == 0) s_misc[6] = 0;
  if (a.pdl) pdl_launch_dependents();

  auto clear_index = [&](uint32_t t0, uint32_t stride) {
    uint4* t4 = reinterpret_cast<uint4*>(ts);
    const uint4 e4 = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (uint32_t i = t0; i < NB / 2; i += stride) t4[i] = e4;  // two buckets per 16 bytes
    if ((NB & 1u) && t0 == 0) reinterpret_cast<uint2*>(ts)[NB - 1] = make_uint2(~0u, ~0u);
    for (uint32_t i = t0; i < (NB + 1) / 2; i += stride) fill[i] = 0;
  };

  while (true) {
    if (tid == 0) s_misc[0] = a.r0 + atomicAdd(a.queue, 1u);
    ep_bar();
    const uint32_t r = s_misc[0];
    if (r >= a.r1) break;
    if (a.skip && !a.skip[r]) {
      ep_bar();  // s_misc[0] is rewritten by the next iteration
      continue;
    }
    uint64_t lo, hi;
    if (a.T <= 1) {
      lo = (uint64_t)r * a.n / a.P;  // Alg. 1 l.3-4
      hi = (uint64_t)(r + 1) * a.n / a.P;
    } else {  // two-level (hybrid) decomposition
      const uint64_t Pp = a.P / a.T, p = r / a.T, t = r % a.T;
      const uint64_t b0 = p * a.n / Pp, Lp = (p + 1) * a.n / Pp - b0;
      lo = b0 + t * Lp / a.T;
      hi = b0 + (t + 1) * Lp / a.T;
    }
    const uint32_t L = (uint32_t)(hi - lo);
    const uint32_t* __restrict__ Ab = A + lo;

    // ---- empty summary; the fill epoch: m = 0, members = all k slots, empty index.
    // First-time stamps: member v = eseq << 20 | (2^20 - 1 - t) (atomicMax), U entry
    // key << 32 | eseq << 20 | t (atomicMin); entries of earlier epochs are stale by their eseq.
    clear_index(tid, NT);
    for (uint32_t i = tid; i < k; i += NT) {
      cw[i] = 0;
      vft[i] = 0;
    }
    for (uint32_t i = tid; i < UC; i += NT) ut[i] = EP_UEMPTY;
    for (uint32_t w = tid; w < EP_KW; w += NT) {
      const uint32_t base = w * 32;
      memb[w] = base >= k ? 0u : (k - base >= 32 ? 0xffffffffu : (1u << (k - base)) - 1u);
      wpre[w] = min(base, k);
      hsl[w] = 0;
      hr[w] = 0;
      hc[w] = 0;
    }
    uint32_t m = 0, b = k, size = 0, seed = 0, ecount = 0, nv = 0, eseq = 1;
    uint32_t q_dbg = 0;
    (void)q_dbg;
    ep_bar();

    // ---- epoch end: resolve the ne events, apply, and (full) form level m + 1
    auto epoch_end = [&](bool full) {
      ep_bar();  // events, V list and occurrence counts of the epoch are complete
      EPHB(10);
      EPTM(4);
      const uint32_t ne = ecount;
      const uint32_t nvv = full ? s_misc[1] : nv;
      // (1) warp 0: which V events hit (closed form, in time order, 32 at a time). A hit marks
      // its event EP_HIT; a V miss copies its key and occurrences aside (into the index key
      // array, rebuilt below) and points its event there. The other warps clear the index.
      if (wid == 0) {
        uint32_t nvm = 0;
        for (uint32_t c0 = 0; c0 < nvv; c0 += 32) {
          {  // aux[w] = hit members in words >= w (words lane, lane + 32)
            const uint32_t pa = __popc(hr[lane]), pb = __popc(hr[lane + 32]);
            uint32_t sa = pa, sb = pb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t ta = __shfl_down_sync(PSS_FULL, sa, o);
              const uint32_t tb = __shfl_down_sync(PSS_FULL, sb, o);
              if (lane + o < 32) {
                sa += ta;
                sb += tb;
              }
            }
            aux[lane] = sa + __shfl_sync(PSS_FULL, sb, 0);
            aux[lane + 32] = sb;
            if (lane == 0) aux[64] = 0;
            __syncwarp();
          }
          const uint32_t j = c0 + lane;
          const bool act = j < nvv;
          const uint32_t v = act ? vl[EPIDX(j, k, 101)] : 0u;
          const uint32_t evv = act ? ev[EPIDX(v, k, 102)] : (uint32_t)EP_VFLAG;
#ifdef PSS_EP_HB
          if (act && (!(evv & EP_VFLAG) || evv == EP_HIT) && a.hb &&
              atomicCAS((unsigned*)(a.hb + 8 * 4000), 0u, 130u) == 0u) {
            a.hb[8 * 4000 + 1] = evv;
            a.hb[8 * 4000 + 2] = v;
            a.hb[8 * 4000 + 3] = r;
            a.hb[8 * 4000 + 4] = eseq;
            a.hb[8 * 4000 + 5] = j;
            a.hb[8 * 4000 + 6] = nvv;
            a.hb[8 * 4000 + 7] = ne;
          }
#endif
          const uint32_t s = act ? EPIDX(evv & 0x7fffu, k, 131) : 0u;
          EPCHK(!act || (v < ne && (ev[v] & EP_VFLAG) && ((memb[s >> 5] >> (s & 31u)) & 1u)), 7,
                v, ev[v], nvv);
          const uint32_t rr = wpre[s >> 5] + __popc(memb[s >> 5] & ((1u << (s & 31u)) - 1u));
          const int d = (int)v - (int)rr;
          const uint32_t rw = rr >> 5, rb = rr & 31u;
          const int lo_c = (int)(aux[EPIDX(rw + 1, 65, 103)] + __popc((hr[EPIDX(rw, 64, 104)] >> rb) >> 1));
          const bool hitl = act && d <= lo_c;
          const bool missl = act && d > lo_c + (int)lane;
          uint32_t hb = __ballot_sync(PSS_FULL, hitl);
          uint32_t um = __ballot_sync(PSS_FULL, act && !hitl && !missl);
          while (um) {  // near the pointer: decide in time order with the chunk's earlier hits
            const uint32_t u = __ffs(um) - 1;
            const uint32_t ru = __shfl_sync(PSS_FULL, rr, u);
            const int du = __shfl_sync(PSS_FULL, d, u);
            const int lu = __shfl_sync(PSS_FULL, lo_c, u);
            const uint32_t gt = __ballot_sync(PSS_FULL, rr > ru);
            if (du <= lu + __popc(hb & gt & ((1u << u) - 1u))) hb |= 1u << u;
            um &= um - 1;
          }
          const uint32_t am = __ballot_sync(PSS_FULL, act);
          if (act) {
            if ((hb >> lane) & 1u) {
              atomicOr(&hr[rw], 1u << rb);
              atomicOr(&hsl[s >> 5], 1u << (s & 31u));
              atomicAdd(&hc[EPIDX(v >> 5, 64, 105)], 1u);
              ev[v] = (uint16_t)EP_HIT;
            } else {
              const uint32_t idx = nvm + __popc(am & ~hb & ltm);
              tk[EPIDX(2 * idx, 4 * NB, 106)] = keys[EPIDX(s, k, 107)];
              tk[EPIDX(2 * idx + 1, 4 * NB, 108)] = (cw[s] & CM) - m;
              ev[v] = (uint16_t)(EP_VFLAG | idx);
            }
          }
          nvm += __popc(am & ~hb);
          __syncwarp();
        }
        // hcp: exclusive prefix of the per-chunk hit counts; aux: popped members before word w
        const uint32_t ha = hc[lane], hb2 = hc[lane + 32];
        const uint32_t pa = __popc(memb[lane] & ~hsl[lane]);
        const uint32_t pb = __popc(memb[lane + 32] & ~hsl[lane + 32]);
        uint32_t sa = pa, sb = pb, qa = ha, qb = hb2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t ta = __shfl_up_sync(PSS_FULL, sa, o);
          const uint32_t tb = __shfl_up_sync(PSS_FULL, sb, o);
          const uint32_t ua = __shfl_up_sync(PSS_FULL, qa, o);
          const uint32_t ub = __shfl_up_sync(PSS_FULL, qb, o);
          if (lane >= (uint32_t)o) {
            sa += ta;
            sb += tb;
            qa += ua;
            qb += ub;
          }
        }
        aux[lane] = sa - pa;
        aux[lane + 32] = __shfl_sync(PSS_FULL, sa, 31) + sb - pb;
        hcp[lane] = qa - ha;
        hcp[lane + 32] = __shfl_sync(PSS_FULL, qa, 31) + qb - hb2;
        if (lane == 31) s_misc[4] = qa + qb;
        hc[lane] = 0;
        hc[lane + 32] = 0;
        hr[lane] = 0;
        hr[lane + 32] = 0;
      } else if (full) {
        clear_index(tid - 32, NT - 32);
      }
      ep_bar();
      EPHB(11);
      EPTM(5);
      const uint32_t nmiss = ne - s_misc[4];
      EPCHK(s_misc[4] <= nvv && nvv <= ne, 9, s_misc[4], nvv, ne);
      // (2) misses in time order: event i's rank is i minus the hits before it
      for (uint32_t base = wid * 32; base < ne; base += NT) {
        const uint32_t i = base + lane;
        const uint32_t code = i < ne ? ev[i] : EP_HIT;
        const uint32_t hm = __ballot_sync(PSS_FULL, code == EP_HIT);
        EPCHK(code == EP_HIT || i - hcp[base >> 5] - __popc(hm & ltm) < nmiss, 5, i, ne, nmiss);
        if (code != EP_HIT) ml[EPIDX(i - hcp[base >> 5] - __popc(hm & ltm), k, 109)] = (uint16_t)code;
      }
      ep_bar();
      EPTM(6);
      // (3) pops: the j-th unhit member (slot order) takes miss j: key, count m + occurrences,
      // error m. Sources are the U table or the V misses' copies, so slots are written in place.
      for (uint32_t s = tid; s < KW * 32; s += NT) {
        const uint32_t w = s >> 5;
        const uint32_t pw = memb[w] & ~hsl[w];
        if (s < k && ((pw >> (s & 31u)) & 1u)) {
          const uint32_t j = aux[w] + __popc(pw & ((1u << (s & 31u)) - 1u));
          if (j < nmiss) {
            const uint32_t code = ml[EPIDX(j, k, 110)];
            uint32_t key, occ;
            EPCHK((code & EP_VFLAG) ? (code & 0x7fffu) < nvv : code < UC, 2, j, code, nmiss);
            if (code & EP_VFLAG) {
              key = tk[EPIDX(2 * (code & 0x7fffu), 4 * NB, 111)];
              occ = tk[2 * (code & 0x7fffu) + 1];
            } else {
              key = (uint32_t)(ut[EPIDX(code, UC, 112)] >> 32);
              occ = uo[code];
            }
            keys[s] = key;
            cw[s] = (m + occ) | (m << cb);
          }
        }
        __syncwarp();
        if (lane == 0) hsl[w] = 0;
      }
      if (size < k) size = full ? k : nmiss;  // the fill epoch pops slots 0, 1, ... in order
      ep_bar();
#ifdef PSS_EP_DUMP
      if (r == 0 && full && eseq - 1 < EP_DUMP_E) {
        unsigned* dd = g_ep_dump[eseq - 1];
        if (tid == 0) {
          dd[0] = m;
          dd[1] = ne;
          dd[2] = nvv;
          dd[3] = s_misc[4];
        }
        for (uint32_t s = tid; s < k; s += NT) {
          dd[4 + s] = keys[s];
          dd[4 + EP_KMAX + s] = cw[s];
        }
      }
#endif
      if (!full) return;
      EPTM(7);
      // (4) level m + 1: members = slots with count m + 1; rebuild the index with member flags
      ++m;
      ++eseq;
      while (true) {
        EPHB(20);
        for (uint32_t s = tid; s < KW * 32; s += NT) {  // whole warps: the ballot is word s >> 5
          const bool in = s < k;
          const uint32_t x = in ? keys[s] : 0u;
          const bool mem = in && (cw[s] & CM) == m;
          const uint32_t bits = __ballot_sync(PSS_FULL, mem);
          if (lane == 0) memb[s >> 5] = bits;
          if (in) {
            uint32_t b1, b2;
            ep_hash(x, seed, NB, b1, b2);
            const uint32_t f1 = (fill[b1 >> 1] >> ((b1 & 1u) * 16)) & 0xffffu;
            const uint32_t f2 = (fill[b2 >> 1] >> ((b2 & 1u) * 16)) & 0xffffu;
            const uint32_t ba = f2 < f1 ? b2 : b1, bz = f2 < f1 ? b1 : b2;
            const uint32_t sha = (ba & 1u) * 16, shz = (bz & 1u) * 16;
            uint32_t bk = ba;
            uint32_t way = (atomicAdd(&fill[ba >> 1], 1u << sha) >> sha) & 0xffffu;
            if (way >= 4) {
              bk = bz;
              way = (atomicAdd(&fill[bz >> 1], 1u << shz) >> shz) & 0xffffu;
            }
            if (way < 4) {
              tk[bk * 4 + way] = x;
              ts[bk * 4 + way] = (uint16_t)(s | (mem ? EP_VFLAG : 0u));
            } else {  // both buckets full: placed below by cuckoo kicks
              const uint32_t o = atomicAdd(&s_misc[6], 1u);
              if (o < EP_OVF) s_ovf[o] = s;
            }
          }
        }
        ep_bar();
        const uint32_t novf = s_misc[6];
        if (novf == 0) break;
        ep_bar();  // every thread has read novf before thread 0 resets it
        EPHB(21);
        // cuckoo kicks (one thread): a homeless key displaces an entry of one of its buckets,
        // which moves to its other bucket, ... (bounded; failing that, a new hash)
        if (tid == 0) {
          bool ok = novf <= EP_OVF;
          for (uint32_t o = 0; o < novf && ok; ++o) {
            uint32_t cs = EPIDX(s_ovf[o], k, 113);
            uint32_t cx = keys[cs];
            uint32_t cv = cs | ((cw[cs] & CM) == m ? EP_VFLAG : 0u);
            uint32_t from = 0xffffffffu;
            ok = false;
            for (int step = 0; step < 256 && !ok; ++step) {
              uint32_t b1, b2;
              ep_hash(cx, seed, NB, b1, b2);
              for (uint32_t w = 0; w < 8 && !ok; ++w) {
                const uint32_t bk = w < 4 ? b1 : b2;
                if (ts[bk * 4 + (w & 3u)] == (uint16_t)EP_E16) {
                  tk[bk * 4 + (w & 3u)] = cx;
                  ts[bk * 4 + (w & 3u)] = (uint16_t)cv;
                  ok = true;
                }
              }
              if (ok) break;
              const uint32_t bk = (b1 != from) ? b1 : b2;  // not back where it came from
              const uint32_t e = bk * 4 + ((step + cs) & 3u);
              const uint32_t nx = tk[e], nv2 = ts[e];
              tk[e] = cx;
              ts[e] = (uint16_t)cv;
              cx = nx;
              cv = nv2;
              from = bk;
            }
          }
          s_misc[2] = ok ? 0u : 1u;
          s_misc[6] = 0;
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
          atomicAdd(&g_ep_dbg[15], novf);
          if (!ok) atomicAdd(&g_ep_dbg[14], 1u);
#endif
        }
        ep_bar();
        if (s_misc[2] == 0) break;
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
        EPWATCH(seed < 64, 11, seed, novf, 0);
        if (seed >= 64) break;
#endif
        ++seed;  // kicks failed: rebuild the whole index under a new hash (rare)
        clear_index(tid, NT);
        ep_bar();
      }
      if (wid == 0) {
        const uint32_t pa = __popc(memb[lane]), pb = __popc(memb[lane + 32]);
        uint32_t sa = pa, sb = pb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t ta = __shfl_up_sync(PSS_FULL, sa, o);
          const uint32_t tb = __shfl_up_sync(PSS_FULL, sb, o);
          if (lane >= (uint32_t)o) {
            sa += ta;
            sb += tb;
          }
        }
        const uint32_t tota = __shfl_sync(PSS_FULL, sa, 31);
        wpre[lane] = sa - pa;
        wpre[lane + 32] = tota + sb - pb;
        if (lane == 31) s_misc[3] = tota + sb;
      }
      ep_bar();
      b = s_misc[3];
      EPTM(8);
      EPWATCH(b >= 1, 3, ne, nvv, 0);
      ecount = 0;
      nv = 0;
    };

    // ---- the block, window by window
    uint32_t xn[R];
    auto load = [&](uint32_t q, uint32_t* dst) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint32_t p = q + j * NT + tid;
        dst[j] = p < L ? __ldcs(Ab + p) : 0u;
      }
    };
    load(0, xn);
    for (uint32_t q = 0; q < L; q += SW) {
      uint32_t x[R];
      uint32_t pend = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        x[j] = xn[j];
        if (q + j * NT + tid < L) pend |= 1u << j;
      }
      if (q + SW < L) load(q + SW, xn);
      const uint32_t wend = min(q + SW, L);  // one past the window's last item
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
      uint32_t npass = 0;
#endif
      while (true) {
#ifdef PSS_EP_BAR3
        ep_bar();
#endif
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
        EPWATCH(++npass < 600, 12, q, npass, b);
        if (npass >= 600) break;
#endif
        EPTM(0);
        // (1) classify against the epoch-start index; first times of V and U keys
        uint32_t cls[R], id[R];  // cls 0: S, 1: V, 2: U; id: slot or U entry
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t xx = x[j];
          uint32_t b1, b2;
          ep_hash(xx, seed, NB, b1, b2);
          const uint4 k1 = tk4[b1], k2 = tk4[b2];
          const uint2 s1 = ts2[b1], s2 = ts2[b2];
          uint32_t e = EP_E16;
          auto pick = [&](uint32_t kk, uint32_t sv) {
            e = (kk == xx && sv != EP_E16) ? sv : e;
          };
          pick(k1.x, s1.x & 0xffffu);
          pick(k1.y, s1.x >> 16);
          pick(k1.z, s1.y & 0xffffu);
          pick(k1.w, s1.y >> 16);
          pick(k2.x, s2.x & 0xffffu);
          pick(k2.y, s2.x >> 16);
          pick(k2.z, s2.y & 0xffffu);
          pick(k2.w, s2.y >> 16);
          id[j] = e & 0x7fffu;
          cls[j] = e == EP_E16 ? 2u : (e >> 15);
        }
        EPTM(9);
#ifdef PSS_EP_TIMING
        if (tid == 0) atomicAdd(&g_ep_tm[12], 1ull);
        if (lane == 0) {
          uint32_t nu = 0;
          for (int j = 0; j < R; ++j) nu += __popc(__ballot_sync(1u, 0) | 0);
          (void)nu;
        }
#endif
        const uint32_t estamp = eseq << 20;
        uint32_t utodo = 0;  // rows whose U key still has to be found or claimed
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t t = q + j * NT + tid;
          if (((pend >> j) & 1u) && cls[j] == 1)
            atomicMax(&vft[EPIDX(id[j], k, 118)], estamp | (0xfffffu - t));
          if (((pend >> j) & 1u) && cls[j] == 2) {
            utodo |= 1u << j;
            id[j] = ep_uhash(x[j], UB);  // the bucket to look in next
          }
        }
        // U keys: find or claim their entry in the epoch's U table (buckets of 4 64-bit entries
        // key << 32 | eseq << 20 | t, read whole; linear probing over buckets). One warp-uniform
        // loop serves every row, one probe per lane per trip, so that warps reach the barrier
        // converged. Entries change only by 64-bit CAS (claims, and lowering the first time).
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
        uint32_t probes = 0;
#endif
        while (__any_sync(PSS_FULL, utodo != 0)) {
#ifdef PSS_EP_TIMING
          if (tid == 0) atomicAdd(&g_ep_tm[11], 1ull);
#endif
          if (utodo) {
            const uint32_t j = __ffs(utodo) - 1;
            uint32_t xx = x[0], ub = id[0];
#pragma unroll
            for (int jj = 1; jj < R; ++jj)
              if (j == (uint32_t)jj) {
                xx = x[jj];
                ub = id[jj];
              }
            const uint32_t lo_m = estamp | (q + j * NT + tid);
            const uint4 w01 = reinterpret_cast<const uint4*>(ut)[2 * ub];
            const uint4 w23 = reinterpret_cast<const uint4*>(ut)[2 * ub + 1];
            // entry w = (lo, hi) = (eseq << 20 | t, key): current iff (lo ^ estamp) < 2^20;
            // t = 2^20 - 1 marks an entry being claimed (its key not yet written)
            const uint32_t busyv = estamp | 0xfffffu;
            const uint32_t cur = ((w01.x ^ estamp) < 0x100000u ? 1u : 0u) |
                                 ((w01.z ^ estamp) < 0x100000u ? 2u : 0u) |
                                 ((w23.x ^ estamp) < 0x100000u ? 4u : 0u) |
                                 ((w23.z ^ estamp) < 0x100000u ? 8u : 0u);
            const uint32_t busy = (w01.x == busyv ? 1u : 0u) | (w01.z == busyv ? 2u : 0u) |
                                  (w23.x == busyv ? 4u : 0u) | (w23.z == busyv ? 8u : 0u);
            const uint32_t hit = cur & ~busy &
                                 ((w01.y == xx ? 1u : 0u) | (w01.w == xx ? 2u : 0u) |
                                  (w23.y == xx ? 4u : 0u) | (w23.w == xx ? 8u : 0u));
            // the way to use: x's entry, else (no claim in flight here) the first free one
            const uint32_t sel = hit ? hit : (busy ? 0u : (~cur & 15u));
            bool done = false;
            uint32_t h = 0;
            if (sel) {
              const uint32_t w = __ffs(sel) - 1;
              h = 4 * ub + w;
              uint32_t elo = w01.x;
              elo = w == 1 ? w01.z : elo;
              elo = w == 2 ? w23.x : elo;
              elo = w == 3 ? w23.z : elo;
              uint32_t* const lop = reinterpret_cast<uint32_t*>(ut) + 2 * h;
              if (hit) {  // found: keep the earliest time (native 32-bit min on the low word)
                if (elo > lo_m) atomicMin(lop, lo_m);
                done = true;
              } else if (atomicCAS(lop, elo, busyv) == elo) {  // claimed: publish key and time
                *reinterpret_cast<uint2*>(lop) = make_uint2(lo_m, xx);
                uo[h] = 0;
                done = true;
              }  // else: raced, look at the bucket again
            } else if (busy) {
              // a claim in flight in this bucket (maybe of x): look again
            } else {  // bucket full of other keys of this epoch: next bucket
              ub = ub + 1 == UB ? 0u : ub + 1;
#if defined(PSS_EP_DEBUG) || defined(PSS_EP_GUARD)
              if (++probes >= UB) {
                EPWATCH(false, 1, xx, q + j * NT + tid, UB);
                done = true;
              }
#endif
            }
#pragma unroll
            for (int jj = 0; jj < R; ++jj)
              if (j == (uint32_t)jj) id[jj] = done ? h : ub;
            if (done) utodo &= utodo - 1;
          }
        }
        EPTM(10);
        ep_bar();
        EPTM(1);
        // (2) events: first occurrences of V and U keys; per-warp counts for the time-order scan
        uint32_t evb[R], vb[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t t = q + j * NT + tid;
          bool isev = false;
          if ((pend >> j) & 1u) {
            if (cls[j] == 1) isev = vft[EPIDX(id[j], k, 122)] == ((eseq << 20) | (0xfffffu - t));
            else if (cls[j] == 2) isev = (uint32_t)ut[EPIDX(id[j], UC, 123)] == ((eseq << 20) | t);
          }
          evb[j] = __ballot_sync(PSS_FULL, isev);
          vb[j] = __ballot_sync(PSS_FULL, isev && cls[j] == 1);
          if (lane == 0) cbuf[j * NW + wid] = __popc(evb[j]) | (__popc(vb[j]) << 16);
        }
        ep_bar();
        EPTM(2);
        // (3) time-order ranks (a shuffle scan of the R * NW counts); items up to the epoch's
        // b-th event are applied
        const uint32_t cv = lane < R * NW ? cbuf[lane] : 0u;
        uint32_t inc = cv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t tv = __shfl_up_sync(PSS_FULL, inc, o);
          if (lane >= (uint32_t)o) inc += tv;
        }
        const uint32_t run = __shfl_sync(PSS_FULL, inc, R * NW - 1);
        const uint32_t need = b - ecount;
        const uint32_t tot_e = run & 0xffffu, tot_v = run >> 16;
        const bool ended = tot_e >= need;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const uint32_t pre = __shfl_sync(PSS_FULL, inc - cv, j * NW + wid);
          if (!((pend >> j) & 1u)) continue;
          const bool isev = (evb[j] >> lane) & 1u;
          const uint32_t ee = (pre & 0xffffu) + __popc(evb[j] & ltm);
          if (ended && ee >= need) continue;  // after the epoch's last event: next epoch
          pend &= ~(1u << j);
          if (cls[j] == 2) atomicAdd(&uo[EPIDX(id[j], UC, 114)], 1u);
          else atomicAdd(&cw[EPIDX(id[j], k, 115)], 1u);
          EPCHK(ecount + ee < b || !isev, 10, ee, need, tot_e);
          if (isev) {
            const uint32_t isv = cls[j] == 1;
            ev[EPIDX(ecount + ee, k, 116)] = (uint16_t)(isv ? (EP_VFLAG | id[j]) : id[j]);
#ifdef PSS_EP_HB
            if (a.hb && ecount + ee == 0) {  // log: writes of event 0
              const unsigned li = atomicAdd((unsigned*)(a.hb + 8 * 4000 + 16), 1u);
              if (li < 4096) {
                volatile unsigned* lg = a.hb + 8 * 4100 + 8 * li;
                lg[0] = r; lg[1] = eseq; lg[2] = ecount; lg[3] = ee; lg[4] = isv ? (EP_VFLAG | id[j]) : id[j];
                lg[5] = tid; lg[6] = q + j * NT + tid; lg[7] = need;
              }
            }
#endif
            const uint32_t ve = (pre >> 16) + __popc(vb[j] & ltm);
            if (isv) vl[EPIDX(nv + ve, k, 117)] = (uint16_t)(ecount + ee);
            if (ended && ee == need - 1) {
              s_misc[1] = nv + ve + isv;
              s_misc[5] = q + j * NT + tid;
            }
          }
        }
        EPTM(3);
        if (!ended) {
          ecount += tot_e;
          nv += tot_v;
          break;
        }
        ecount = b;
        epoch_end(true);
        if (s_misc[5] + 1 >= wend) break;  // nothing of the window is left
      }
    }
    epoch_end(false);  // the block's last (partial) epoch

    EPHB(30);
    // ---- dump the leaf in slot order
    uint32_t* oi = a.items + (size_t)r * k;
    uint32_t* oc = a.counts + (size_t)r * k;
    uint32_t* oe = a.errs + (size_t)r * k;
    for (uint32_t s = tid; s < EPIDX(size, k + 1, 119); s += NT) {
      const uint32_t c = cw[s];
      oi[s] = keys[s];
      oc[s] = c & CM;
      oe[s] = c >> cb;
    }
    if (tid == 0) a.sizes[r] = size;
    if (a.leaf_flags) {  // publish leaf r to the overlapping tree kernel
      __threadfence();
      ep_bar();
      if (tid == 0) st_release(a.leaf_flags + r, 1u);
    }
    ep_bar();
  }
}

// ------------------------------------------------------------------------------ host side
#ifndef PSS_EP_NT
#define PSS_EP_NT 256
#endif
#ifndef PSS_EP_R
#define PSS_EP_R 2
#endif
constexpr int EP_NT = PSS_EP_NT;
constexpr int EP_R = PSS_EP_R;
constexpr uint32_t EP_KMIN = 64;
#ifndef PSS_EP_DEFAULT_ON
#define PSS_EP_DEFAULT_ON 0
#endif
constexpr bool EP_DEFAULT_ON = PSS_EP_DEFAULT_ON;  // below this, epochs are short and K1 is used

struct EpPlan {
  bool ok = false;
  uint32_t cb = 0, NB = 0, UC = 0;
  uint32_t o_cw, o_vft, o_ml, o_tk, o_ts, o_fill, o_ut, o_uo, o_ev, o_vl, o_bits;
  size_t smem = 0;
  int grid = 0;
};

static EpPlan ep_plan(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  EpPlan p;
  // routing: PSS_EPOCH=1 / 0 forces K1e on / off; otherwise EP_DEFAULT_ON decides
  if (const char* e = std::getenv("PSS_EPOCH")) {
    if (e[0] == '0') return p;
  } else if (!EP_DEFAULT_ON || std::getenv("PSS_NO_EPOCH")) {
    return p;
  }
  if (kb != 4 || k < EP_KMIN || k > EP_KMAX || P == 0) return p;
  const uint64_t Lmax = (n + P - 1) / P;
  uint32_t cb = 1;
  while (cb < 32 && (1ull << cb) <= Lmax) ++cb;
  uint32_t eb = 0;
  while (eb < 32 && (1ull << eb) <= Lmax / k) ++eb;
  // stamps: block times below 2^20, epochs (at most Lmax / k + 2) below 2^12 - 1
  if (cb + eb > 32 || Lmax >= (1ull << 20) || Lmax / k + 2 >= 4095) return p;
  p.cb = cb;
#ifdef PSS_EP_BIGTABLE
  p.NB = k;
#else
  p.NB = std::max<uint32_t>(1, (k + 1) / 2);
#endif
  const uint32_t SW = EP_NT * EP_R;
  // distinct U keys of an epoch <= b + one window; buckets of 4 entries at load <= ~0.7
  p.UC = 4 * ((((k + SW) * 10 + 6) / 7 + 3) / 4);
  if (p.UC >= EP_VFLAG) return p;
  Bump b;
  b.al = 16;
  b.take<uint32_t>(k);  // keys
  p.o_cw = (uint32_t)b.take<uint32_t>(k);
  p.o_vft = (uint32_t)b.take<uint32_t>(k);
  p.o_ml = (uint32_t)b.take<uint16_t>(k);
  p.o_tk = (uint32_t)b.take<uint32_t>(4 * (size_t)p.NB);
  p.o_ts = (uint32_t)b.take<uint16_t>(4 * (size_t)p.NB);
  p.o_fill = (uint32_t)b.take<uint32_t>((p.NB + 1) / 2);
  b.al = 32;
  p.o_ut = (uint32_t)b.take<unsigned long long>(p.UC);  // 32-byte buckets
  b.al = 16;
  p.o_uo = (uint32_t)b.take<uint32_t>(p.UC);
  p.o_ev = (uint32_t)b.take<uint16_t>(k);
  p.o_vl = (uint32_t)b.take<uint16_t>(k);
  p.o_bits = (uint32_t)b.take<uint32_t>(7 * EP_KW + 1);
  p.smem = b.bytes();
  auto kern = ep_kernel<EP_NT, EP_R>;
  if (p.smem > (size_t)d.smem_optin || allow_max_smem(kern, d) != cudaSuccess) return p;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, EP_NT, p.smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return p;
  }
  if (nb < 1) return p;
  p.grid = (int)std::min<uint64_t>(P, (uint64_t)nb * d.sms);
  p.ok = true;
  return p;
}

bool epoch_used(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  return ep_plan(n, kb, k, P, d).ok;
}

cudaError_t epoch_launch(const void* A, uint64_t n, uint32_t k, uint32_t P, void* items,
                         uint32_t* counts, uint32_t* errs, uint32_t* sizes, uint32_t* queue,
                         const unsigned char* skip, cudaStream_t s, const DevInfo& d, uint32_t r0,
                         uint32_t r1, uint32_t T, uint32_t* leaf_flags, bool pdl) {
  const EpPlan p = ep_plan(n, 4, k, P, d);
  if (!p.ok) return cudaErrorInvalidValue;
  EpArgs a;
  a.A = static_cast<const uint32_t*>(A);
  a.n = n;
  a.k = k;
  a.P = P;
  a.r0 = r0;
  a.r1 = r1;
  a.T = T;
  a.leaf_flags = leaf_flags;
  a.pdl = pdl ? 1 : 0;
  a.items = static_cast<uint32_t*>(items);
  a.counts = counts;
  a.errs = errs;
  a.sizes = sizes;
  a.queue = queue;
  a.skip = skip;
  a.cb = p.cb;
  a.NB = p.NB;
  a.UC = p.UC;
  a.o_cw = p.o_cw;
  a.o_vft = p.o_vft;
  a.o_ml = p.o_ml;
  a.o_tk = p.o_tk;
  a.o_ts = p.o_ts;
  a.o_fill = p.o_fill;
  a.o_ut = p.o_ut;
  a.o_uo = p.o_uo;
  a.o_ev = p.o_ev;
  a.o_vl = p.o_vl;
  a.o_bits = p.o_bits;
  a.hb = nullptr;
#ifdef PSS_EP_HB
  if (const char* hp = std::getenv("PSS_EP_HB_PTR")) a.hb = (volatile unsigned*)std::strtoull(hp, nullptr, 0);
#endif
  const int grid = (int)std::min<uint64_t>(r1 - r0, (uint64_t)p.grid);
  cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  ep_kernel<EP_NT, EP_R><<<grid, EP_NT, p.smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace pss
