// hot.cu -- K0: a static table of the frequent keys of a range of A, for K1's level-pinned bypass
// (summarize.cu). Space Saving never evicts a counter whose count exceeds the current minimum
// (the evicted counter is one "with the least hit count"), so the hits of such a key
// commute with every other update until the minimum level changes; K1 counts them aside. Which
// keys are worth that is a performance choice only (K1 stays exact for any table, also an empty or
// a badly chosen one), so one CTA picks them from a sample:
//   1. 8192 items (8 runs of 1024 consecutive items spread over the range; the whole range if it
//      is shorter), 8 per thread kept in registers, are counted into a sketch of 4096 buckets
//      (32768 items took 32 us, mostly same-address shared atomics of the heaviest keys);
//   2. the sample items whose bucket reached a threshold are counted exactly in a small
//      open-addressing table (64-bit entries valid|key claimed by atomicCAS, no sentinel keys);
//   3. the (up to) 64 entries with the greatest counts (ties: smaller key) are ranked;
//   4. an odd multiplier is searched under which they occupy distinct entries of a 2048-entry
//      one-probe table (entry = top 11 bits h of ha = key * multiplier, a bijection of the key);
//      entry h holds (rank ^ h) << 21 | ha's low 21 bits, so that rotl(entry ^ ha, 11) is the
//      rank for that key and >= 2048 for any other key; empty entries hold rank HOT_NONE.
// The table is dropped (n = 0) when the chosen keys cover less than 70 % of the sample: measured
// on B200, the bypass pays only on strongly skewed inputs.
#include "common.cuh"

namespace pss {

constexpr uint32_t HOT_SAMPLE = 8192, HOT_RUN = 1024, HOT_NT = 1024;
constexpr uint32_t HOT_PER = HOT_SAMPLE / HOT_NT;  // sample items per thread
constexpr uint32_t HOT_SK_LOG = 12, HOT_ET = 2048, HOT_LIST = 1024, HOT_TRIES = 256;

__device__ __forceinline__ uint32_t hot_mix(uint32_t x) {
  uint32_t h = x * 0x85EBCA6Bu;
  return (h ^ (h >> 15)) * 0xC2B2AE35u;
}

__global__ void __launch_bounds__(HOT_NT) hot_sample_kernel(const uint32_t* __restrict__ A,
                                                            uint64_t lo, uint64_t hi,
                                                            uint32_t* out, uint32_t force) {
  extern __shared__ __align__(16) unsigned char hsm[];
  uint32_t* const sk = reinterpret_cast<uint32_t*>(hsm);                          // sketch
  unsigned long long* const ek = reinterpret_cast<unsigned long long*>(sk + (1u << HOT_SK_LOG));
  uint32_t* const ec = reinterpret_cast<uint32_t*>(ek + HOT_ET);
  uint32_t* const lkey = sk;              // after pass 2 the sketch is free: list of candidates
  uint32_t* const lcnt = sk + HOT_LIST;
  __shared__ uint32_t occ[(1u << HOT_LOG) / 32];
  __shared__ uint32_t hk[HOT_MAX];
  __shared__ uint32_t nlist, clash, mass;
  const uint32_t tid = threadIdx.x;
  const uint64_t len = hi - lo;
  const uint32_t S = (uint32_t)(len < HOT_SAMPLE ? len : HOT_SAMPLE);
  const uint32_t nrun = HOT_SAMPLE / HOT_RUN;
  const uint64_t stride = len > HOT_SAMPLE ? (len - HOT_RUN) / (nrun - 1) : HOT_RUN;
  auto item = [&](uint32_t j) -> uint32_t {
    return A[lo + (uint64_t)(j / HOT_RUN) * stride + (j % HOT_RUN)];
  };
  for (uint32_t i = tid; i < (1u << HOT_SK_LOG); i += HOT_NT) sk[i] = 0;
  for (uint32_t i = tid; i < HOT_ET; i += HOT_NT) {
    ek[i] = 0;
    ec[i] = 0;
  }
  if (tid == 0) {
    nlist = 0;
    mass = 0;
  }
  // this thread's sample items: all loads in flight together
  uint32_t xs[HOT_PER];
#pragma unroll
  for (uint32_t u = 0; u < HOT_PER; ++u) {
    const uint32_t j = u * HOT_NT + tid;
    xs[u] = j < S ? item(j) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (uint32_t u = 0; u < HOT_PER; ++u)
    if (u * HOT_NT + tid < S) atomicAdd(&sk[hot_mix(xs[u]) >> (32 - HOT_SK_LOG)], 1u);
  __syncthreads();
  const uint32_t thr = max(4u, S >> 11);
#pragma unroll
  for (uint32_t u = 0; u < HOT_PER; ++u) {
    if (u * HOT_NT + tid >= S) continue;
    const uint32_t x = xs[u];
    const uint32_t h = hot_mix(x);
    if (sk[h >> (32 - HOT_SK_LOG)] < thr) continue;
    const unsigned long long mine = (1ull << 32) | x;
    uint32_t e = h & (HOT_ET - 1);
    for (int probe = 0; probe < 64; ++probe) {  // a full neighbourhood drops the item
      const unsigned long long old = atomicCAS(&ek[e], 0ull, mine);
      if (old == 0ull || old == mine) {
        atomicAdd(&ec[e], 1u);
        break;
      }
      e = (e + 1) & (HOT_ET - 1);
    }
  }
  __syncthreads();
  // candidates (keys counted at least thr times), then their ranks by (count desc, key asc)
  for (uint32_t e = tid; e < HOT_ET; e += HOT_NT) {
    const uint32_t c = ec[e];
    if (c >= thr) {
      const uint32_t o = atomicAdd(&nlist, 1u);
      if (o < HOT_LIST) {
        lkey[o] = (uint32_t)ek[e];
        lcnt[o] = c;
      }
    }
  }
  __syncthreads();
  const uint32_t nl = min(nlist, HOT_LIST);
  for (uint32_t i = tid; i < nl; i += HOT_NT) {
    const uint32_t c = lcnt[i], x = lkey[i];
    uint32_t r = 0;
    for (uint32_t u = 0; u < nl; ++u) r += lcnt[u] > c || (lcnt[u] == c && lkey[u] < x);
    if (r < HOT_MAX) {
      hk[r] = x;
      atomicAdd(&mass, c);
    }
  }
  __syncthreads();
  const uint32_t nh = min(nl, HOT_MAX);
  uint32_t* const okeys = out + 4;
  uint32_t* const otab = out + 4 + HOT_MAX;
  if (nh == 0 || (!force && (uint64_t)mass * 10 < (uint64_t)S * 7)) {
    if (tid == 0) out[0] = 0;
    return;
  }
  for (uint32_t tr = 0; tr < HOT_TRIES; ++tr) {
    const uint32_t seed = (tr * 0x9E3779B9u + 0x7F4A7C15u) | 1u;  // the multiplier
    for (uint32_t i = tid; i < (1u << HOT_LOG) / 32; i += HOT_NT) occ[i] = 0;
    if (tid == 0) clash = 0;
    __syncthreads();
    uint32_t ha = 0;
    if (tid < nh) {
      ha = hk[tid] * seed;
      const uint32_t h = ha >> (32 - HOT_LOG);
      if (atomicOr(&occ[h >> 5], 1u << (h & 31u)) & (1u << (h & 31u))) clash = 1;
    }
    __syncthreads();
    if (!clash) {
      for (uint32_t e = tid; e < (1u << HOT_LOG); e += HOT_NT)
        otab[e] = (HOT_NONE ^ e) << (32 - HOT_LOG);
      __syncthreads();
      if (tid < nh) {
        const uint32_t h = ha >> (32 - HOT_LOG);
        otab[h] = ((tid ^ h) << (32 - HOT_LOG)) | (ha & HOT_TAG_MASK);
        okeys[tid] = hk[tid];
      }
      if (tid == 0) {
        out[0] = nh;
        out[1] = seed;
        out[2] = mass;
        out[3] = S;
      }
      return;
    }
    __syncthreads();
  }
  if (tid == 0) out[0] = 0;
}

cudaError_t hot_sample_launch(const void* A, uint64_t lo, uint64_t hi, uint32_t* out, bool force,
                              cudaStream_t s) {
  const size_t smem = ((size_t)4 << HOT_SK_LOG) + (size_t)HOT_ET * 12;
  // per device and process-wide: set on every call (cheap), never cached per process
  cudaError_t e = cudaFuncSetAttribute(hot_sample_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  hot_sample_kernel<<<1, HOT_NT, smem, s>>>(static_cast<const uint32_t*>(A), lo, hi, out,
                                           force ? 1u : 0u);
  return cudaGetLastError();
}

}  // namespace pss
