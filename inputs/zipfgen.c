/*
 * inputs/zipfgen.c -- seeded synthetic workload generator (shared by the oracle side and the
 * CUDA side; holds NONE of the method's arithmetic).
 *
 * The paper's datasets are "synthetic input datasets ... derived from a zipfian distribution
 * with skew 1.1" (PAPER.md:195, also :406, :431); universe, RNG and seed are not stated there.
 * BASELINE.json's configs fix universe, skew and seed; DESIGN.md (section "Input recipe") states
 * the recipe implemented here:
 *
 *   - a counter-based RNG: draw j of position i is splitmix64-finalised
 *     (seed, i, j) -> 64 bits, so any sub-range of the stream can be generated independently and
 *     in parallel with identical results;
 *   - Zipf(s) ranks 1..U by rejection-inversion (Hoermann & Derflinger, 1996), which covers s = 1
 *     through the log1p/expm1 helpers; rank r in [0, U) = sample - 1;
 *   - ids = a fixed bijective mix of the rank (murmur3 fmix32 for u32 keys, fmix64 for u64 keys);
 *   - optional adversarial tail (config C5): with probability tail_frac a position gets a uniform
 *     rank in [0, 2^40) instead of a Zipf rank, then the same mix.
 *
 * Plain C + pthreads; called from Python through ctypes (inputs/__init__.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

static inline uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static inline uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bU;
  h ^= h >> 13;
  h *= 0xc2b2ae35U;
  h ^= h >> 16;
  return h;
}

/* splitmix64 step used as a stateless counter hash */
static inline uint64_t sm64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* draw j of position i under seed: 64 uniform bits */
static inline uint64_t draw64(uint64_t seed, uint64_t i, uint32_t j) {
  return sm64(sm64(seed * 0x2545F4914F6CDD1DULL + 0x1234567ULL) ^ sm64(i * 4ULL + j));
}

static inline double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

uint64_t pssgen_draw64(uint64_t seed, uint64_t i, uint32_t j) { return draw64(seed, i, j); }
uint32_t pssgen_mix32(uint32_t r) { return fmix32(r); }
uint64_t pssgen_mix64(uint64_t r) { return fmix64(r); }

/* ---- rejection-inversion Zipf sampler ---- */
typedef struct {
  double s, N, hx1, hN, sconst;
} zipf_t;

static double helper1(double x) { /* log1p(x)/x */
  return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x));
}
static double helper2(double x) { /* expm1(x)/x */
  return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
}
static double zh(const zipf_t* z, double x) { return exp(-z->s * log(x)); }
static double zH(const zipf_t* z, double x) { /* integral of x^-s: (x^(1-s)-1)/(1-s), log x at s=1 */
  double lx = log(x);
  return helper2((1.0 - z->s) * lx) * lx;
}
static double zHinv(const zipf_t* z, double x) {
  double t = x * (1.0 - z->s);
  if (t < -1.0) t = -1.0;
  return exp(helper1(t) * x);
}
static void zipf_init(zipf_t* z, double s, double N) {
  z->s = s;
  z->N = N;
  z->hx1 = zH(z, 1.5) - 1.0;
  z->hN = zH(z, N + 0.5);
  z->sconst = 2.0 - zHinv(z, zH(z, 2.5) - zh(z, 2.0));
}
/* returns a rank in [1, N]; draws j0, j0+1, ... of position i */
static uint64_t zipf_sample(const zipf_t* z, uint64_t seed, uint64_t i, uint32_t j0) {
  for (uint32_t j = j0;; ++j) {
    double u = z->hN + unit(draw64(seed, i, j)) * (z->hx1 - z->hN);
    double x = zHinv(z, u);
    double kd = floor(x + 0.5);
    if (kd < 1.0) kd = 1.0;
    if (kd > z->N) kd = z->N;
    if (kd - x <= z->sconst || u >= zH(z, kd + 0.5) - zh(z, kd)) return (uint64_t)kd;
  }
}

typedef struct {
  void* out;
  uint64_t offset; /* global position of out[0] */
  uint64_t begin, end;
  int key_bytes;
  double s;
  double U;
  uint64_t seed;
  double tail_frac;
  int hash_ids;
} job_t;

static void* worker(void* arg) {
  job_t* jb = (job_t*)arg;
  zipf_t z;
  zipf_init(&z, jb->s, jb->U);
  for (uint64_t i = jb->begin; i < jb->end; ++i) {
    uint64_t rank;
    if (jb->tail_frac > 0.0 && unit(draw64(jb->seed, i, 0)) < jb->tail_frac) {
      rank = draw64(jb->seed, i, 1) >> 24; /* uniform in [0, 2^40) */
    } else {
      rank = zipf_sample(&z, jb->seed, i, jb->tail_frac > 0.0 ? 2u : 0u) - 1u;
    }
    if (jb->key_bytes == 4) {
      uint32_t r = (uint32_t)rank;
      ((uint32_t*)jb->out)[i - jb->offset] = jb->hash_ids ? fmix32(r) : r;
    } else {
      ((uint64_t*)jb->out)[i - jb->offset] = jb->hash_ids ? fmix64(rank) : rank;
    }
  }
  return NULL;
}

/* Fill out[0..n) with positions [start, start + n) of the Zipf(s) stream over universe U (see
 * header); a range of the stream is identical to the same positions of a longer stream. */
int pssgen_zipf_range(void* out, uint64_t start, uint64_t n, int key_bytes, double s, double U,
                      uint64_t seed, double tail_frac, int hash_ids, int nthreads) {
  if (!out && n) return -1;
  if (key_bytes != 4 && key_bytes != 8) return -1;
  if (!(s > 0.0) || !(U >= 1.0)) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((uint64_t)nthreads > n / 4096 + 1) nthreads = (int)(n / 4096 + 1);
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (job_t){out, start, start + n * (uint64_t)t / nthreads,
                      start + n * (uint64_t)(t + 1) / nthreads, key_bytes, s, U, seed, tail_frac,
                      hash_ids};
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

int pssgen_zipf(void* out, uint64_t n, int key_bytes, double s, double U, uint64_t seed,
                double tail_frac, int hash_ids, int nthreads) {
  return pssgen_zipf_range(out, 0, n, key_bytes, s, U, seed, tail_frac, hash_ids, nthreads);
}
