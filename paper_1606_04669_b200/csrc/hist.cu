// hist.cu -- K1h: the leaf summaries of blocks that never fill their k counters, computed as an
// exact histogram in first-occurrence order by a whole CTA (Algorithm 1 lines 3-5).
//
// Space Saving evicts only when an unmonitored item arrives while all k counters are
// occupied. A block with D <= k distinct keys therefore never evicts: its summary holds every
// distinct key with its exact frequency and error 0, in the slots the keys took when they first
// arrived (R2: slots fill in order), i.e. in first-occurrence order. That summary is computed here
// without the sequential rule: the CTA's threads count the block's keys into one shared-memory
// hash table (linear probing, entries claimed with atomicCAS on the first-position word, counts by
// atomicAdd, first positions by atomicMin), then rank the keys by first position through a bitmap
// over the block's positions. As soon as the block shows more than min(k, 3/4 of the table)
// distinct keys the CTA gives up on it and flags it; K1 (summarize.cu) then runs the sequential
// rule on the flagged blocks only. Both produce the same leaf bit for bit (the GPU parity tests
// compare every leaf with sequential Space Saving run on the CPU).
#include <cstdlib>

#include "common.cuh"

namespace pss {

constexpr uint32_t H_EMPTY = 0xffffffffu;  // first-position word of an unclaimed entry
constexpr uint32_t H_READY = 0x80000000u;  // count word: the entry's key is written
constexpr int H_NT = 512;                  // threads per CTA (one block per CTA at a time)

struct HistArgs {
  const void* A;
  uint64_t n;
  uint32_t k, P, T;
  uint32_t r0, r1;
  uint32_t* queue;
  unsigned char* flagged;  // flagged[r] = 1: leaf r left to K1
  uint32_t* leaf_flags;    // non-null: release leaf r to the overlapping tree kernel
  void* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
  uint32_t logtc;  // table capacity 2^logtc
  uint32_t dmax;   // give up beyond this many distinct keys (min(k, 3/4 of the table))
  uint32_t bw;     // bitmap words (>= max block length / 32)
};

__device__ __forceinline__ uint32_t ldv(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ uint32_t hkey(uint32_t x) { return x * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t hkey(uint64_t x) {
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32);
}

template <typename KT>
__global__ void __launch_bounds__(H_NT) hist_kernel(const HistArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t TC = 1u << a.logtc, mask = TC - 1u;
  KT* keys = reinterpret_cast<KT*>(smem);
  uint32_t* st = reinterpret_cast<uint32_t*>(smem + (size_t)TC * sizeof(KT));  // first position
  uint32_t* cnt = st + TC;                                                     // READY | count
  uint32_t* bm = cnt + TC;                     // positions that are first occurrences
  uint32_t* tp = bm + a.bw;                    // per-thread prefix of the bitmap popcounts
  uint32_t* sc = tp + H_NT;                    // [0] distinct, [1] give up, [2] leaf id
  const uint32_t tid = threadIdx.x;
  const KT* __restrict__ A = reinterpret_cast<const KT*>(a.A);
  constexpr uint32_t V = 16 / sizeof(KT);     // keys per 16-byte load

  while (true) {
    if (tid == 0) sc[2] = a.r0 + atomicAdd(a.queue, 1u);
    for (uint32_t i = tid; i < TC; i += H_NT) {
      st[i] = H_EMPTY;
      cnt[i] = 0;
    }
    for (uint32_t i = tid; i < a.bw; i += H_NT) bm[i] = 0;
    if (tid == 0) {
      sc[0] = 0;
      sc[1] = 0;
    }
    __syncthreads();
    const uint32_t r = sc[2];
    if (r >= a.r1) break;
    uint64_t lo, hi;
    if (a.T <= 1) {
      lo = (uint64_t)r * a.n / a.P;  // Alg. 1 l.3-4
      hi = (uint64_t)(r + 1) * a.n / a.P;
    } else {  // two-level (hybrid) decomposition, as K1
      const uint64_t Pp = a.P / a.T, p = r / a.T, t = r % a.T;
      const uint64_t b0 = p * a.n / Pp, Lp = (p + 1) * a.n / Pp - b0;
      lo = b0 + t * Lp / a.T;
      hi = b0 + (t + 1) * Lp / a.T;
    }
    const uint32_t L = (uint32_t)(hi - lo);

    // count: item at position p (0-based in the block) into the table
    auto insert = [&](KT x, uint32_t p) {
      uint32_t h = hkey(x) & mask;
      while (true) {
        uint32_t s = ldv(st + h);
        if (s == H_EMPTY) {
          const uint32_t old = atomicCAS(st + h, H_EMPTY, p);
          if (old == H_EMPTY) {  // a new key: publish it, then count it
            keys[h] = x;
            __threadfence_block();
            atomicAdd(cnt + h, H_READY + 1u);
            if (atomicAdd(sc, 1u) >= a.dmax) sc[1] = 1;
            return;
          }
          s = old;
        }
        while ((ldv(cnt + h) & H_READY) == 0) {
        }
        __threadfence_block();
        if (*reinterpret_cast<const volatile KT*>(keys + h) == x) {
          atomicAdd(cnt + h, 1u);
          if (p < s) atomicMin(st + h, p);
          return;
        }
        if (ldv(sc + 1)) return;  // given up: the table may be full
        h = (h + 1) & mask;
      }
    };
    const KT* B = A + lo;
    const bool vec = (reinterpret_cast<uintptr_t>(B) & 15u) == 0;
    // the next trip's 16 bytes are loaded before this trip's keys are counted (the counting is a
    // chain of shared-memory round trips; one load in flight per thread left HBM idle)
    uint4 pre = make_uint4(0, 0, 0, 0);
    if (vec && tid * V + V <= L) pre = *reinterpret_cast<const uint4*>(B + tid * V);
    for (uint32_t base = 0; base < L; base += H_NT * V) {
      // Give up early on blocks whose distinct keys grow too fast to stay within k: more than
      // k sqrt(f) after a fraction f of the block (heuristics: a block given up on wrongly is
      // still summarized exactly, by K1)
      if (tid == 0 && base) {
        const uint64_t dd = ldv(sc);
        if (dd * dd * L > (uint64_t)a.k * a.k * base) sc[1] = 1;
        // Zipf streams around s = 1.5 grow like f^(1/s): from 1/8 of the block on, also give up
        // if the count extrapolated with exponent 0.6 exceeds k (C3-s1.5: given up at 1/8 instead
        // of 1/2 of the block)
        if (base * 8 >= L && (float)dd * __powf((float)L / (float)base, 0.6f) > (float)a.k) sc[1] = 1;
      }
      if (ldv(sc + 1)) break;
      const uint32_t p0 = base + tid * V;
      KT x[V];
      if (vec && p0 + V <= L) {
        const uint4 v = pre;
        const uint32_t pn = p0 + H_NT * V;
        if (pn + V <= L) pre = *reinterpret_cast<const uint4*>(B + pn);
        if constexpr (V == 4) {
          x[0] = v.x;
          x[1] = v.y;
          x[2] = v.z;
          x[3] = v.w;
        } else {
          x[0] = ((uint64_t)v.y << 32) | v.x;
          x[1] = ((uint64_t)v.w << 32) | v.z;
        }
#pragma unroll
        for (uint32_t j = 0; j < V; ++j) insert(x[j], p0 + j);
      } else {
        for (uint32_t j = 0; j < V; ++j)
          if (p0 + j < L) insert(B[p0 + j], p0 + j);
      }
    }
    __syncthreads();
    const uint32_t D = sc[0];
    const bool gave_up = sc[1] != 0;
    __syncthreads();  // sc[] is reset by the next block's start
    if (tid == 0) a.flagged[r] = gave_up ? 1 : 0;
    if (gave_up) continue;  // uniform: K1 takes this block

    // slot of a key = its rank by first position: bitmap of first positions, prefix popcounts
    for (uint32_t i = tid; i < TC; i += H_NT) {
      const uint32_t s = st[i];
      if (s != H_EMPTY) atomicOr(bm + (s >> 5), 1u << (s & 31u));
    }
    __syncthreads();
    const uint32_t wpt = (a.bw + H_NT - 1) / H_NT;  // bitmap words per thread
    uint32_t mine = 0;
    for (uint32_t w = tid * wpt; w < min(a.bw, (tid + 1) * wpt); ++w) mine += __popc(bm[w]);
    // exclusive scan of the per-thread sums over the CTA
    const uint32_t lane = tid & 31u, warp = tid >> 5;
    uint32_t incl = mine;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(PSS_FULL, incl, o);
      if (lane >= o) incl += t;
    }
    __shared__ uint32_t wsum[H_NT / 32];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = lane < H_NT / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(PSS_FULL, v, o);
        if (lane >= o) v += t;
      }
      if (lane < H_NT / 32) wsum[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    tp[tid] = (warp ? wsum[warp - 1] : 0u) + incl - mine;
    __syncthreads();
    KT* oi = reinterpret_cast<KT*>(a.items) + (size_t)r * a.k;
    uint32_t* oc = a.counts + (size_t)r * a.k;
    uint32_t* oe = a.errs + (size_t)r * a.k;
    for (uint32_t i = tid; i < TC; i += H_NT) {
      const uint32_t s = st[i];
      if (s == H_EMPTY) continue;
      const uint32_t w = s >> 5, own = w / wpt;
      uint32_t rank = tp[own] + __popc(bm[w] & ((1u << (s & 31u)) - 1u));
      for (uint32_t j = own * wpt; j < w; ++j) rank += __popc(bm[j]);
      oi[rank] = keys[i];
      oc[rank] = cnt[i] & ~H_READY;
      oe[rank] = 0;
    }
    if (tid == 0) a.sizes[r] = D;
    if (a.leaf_flags) {  // publish leaf r to the overlapping tree kernel
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(a.leaf_flags + r, 1u);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ host side
struct HistPlan {
  bool use;
  uint32_t logtc, dmax, bw;
  size_t smem;
  int grid;
};

static HistPlan hist_plan(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  HistPlan h{};
  const uint64_t Lmax = (n + P - 1) / P;
  // Used when the counters are many for the block (40 k >= block length: C3, C4 k >= 5000, C5),
  // where blocks that do not fill are common. Blocks with more distinct keys are given up as soon
  // as they show k + 1 of them, but each block costs the kernel a start, so with few counters
  // (H, C2, C4 k <= 1000: every block fills within its first few thousand items) K1 alone is
  // faster (measured at H: 7.77 ms with this kernel first, 7.51 ms without).
  const char* env = std::getenv("PSS_HIST");  // experiment hook: 0 = never, 1 = always
  h.use = Lmax > 0 && Lmax <= (1u << 17) && (40ull * k >= Lmax || (env && env[0] == '1')) &&
          !(env && env[0] == '0');
  if (!h.use) return h;
  const uint32_t tcmax = kb == 4 ? 8192u : 4096u;
  const uint64_t want = std::min<uint64_t>(k, Lmax);
  uint32_t tc = 256;
  while (tc < tcmax && (uint64_t)tc * 3 / 4 < want) tc *= 2;
  h.logtc = 0;
  while ((1u << h.logtc) < tc) ++h.logtc;
  h.dmax = (uint32_t)std::min<uint64_t>(k, (uint64_t)tc * 3 / 4);
  h.bw = (uint32_t)((Lmax + 31) / 32);
  h.smem = (size_t)tc * (kb + 8) + (size_t)h.bw * 4 + H_NT * 4 + 16;
  if (h.smem > (size_t)d.smem_optin) {
    h.use = false;
    return h;
  }
  auto kern = kb == 4 ? hist_kernel<uint32_t> : hist_kernel<uint64_t>;
  allow_max_smem(kern, d);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, H_NT, h.smem) != cudaSuccess ||
      nb < 1) {
    (void)cudaGetLastError();
    h.use = false;
    return h;
  }
  h.grid = (int)std::min<uint64_t>(P, (uint64_t)nb * d.sms);
  return h;
}

bool hist_used(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  return hist_plan(n, kb, k, P, d).use;
}

cudaError_t hist_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P, void* items,
                        uint32_t* counts, uint32_t* errs, uint32_t* sizes, uint32_t* queue,
                        unsigned char* flagged, cudaStream_t s, const DevInfo& d, uint32_t r0,
                        uint32_t r1, uint32_t T, uint32_t* leaf_flags) {
  const HistPlan h = hist_plan(n, kb, k, P, d);
  if (!h.use) return cudaErrorInvalidValue;
  HistArgs a;
  a.A = A;
  a.n = n;
  a.k = k;
  a.P = P;
  a.T = T;
  a.r0 = r0;
  a.r1 = r1;
  a.queue = queue;
  a.flagged = flagged;
  a.leaf_flags = leaf_flags;
  a.items = items;
  a.counts = counts;
  a.errs = errs;
  a.sizes = sizes;
  a.logtc = h.logtc;
  a.dmax = h.dmax;
  a.bw = h.bw;
  cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<uint64_t>(r1 - r0, (uint64_t)h.grid);
  if (kb == 4)
    hist_kernel<uint32_t><<<grid, H_NT, h.smem, s>>>(a);
  else
    hist_kernel<uint64_t><<<grid, H_NT, h.smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace pss
