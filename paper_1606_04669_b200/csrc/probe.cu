// probe.cu -- K6, the read-bandwidth probe: streams the n
// keys of A once with 128-bit loads and folds them into one word, so that the attainable HBM
// read bandwidth of the box is measured on the same array, in the same run, as the hot path it
// is the roofline of (the driver's MEASURED_PEAKS.json figure is a copy: read + write).
#include <algorithm>

#include "common.cuh"

namespace pss {
namespace {

constexpr int PROBE_THREADS = 512;
constexpr int PROBE_UNROLL = 4;

__global__ void __launch_bounds__(PROBE_THREADS) read_probe_kernel(const uint4* __restrict__ v,
                                                                   uint64_t nv,
                                                                   const unsigned char* tail,
                                                                   uint32_t ntail,
                                                                   uint32_t* out) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * PROBE_THREADS;
  uint64_t i = (uint64_t)blockIdx.x * PROBE_THREADS + threadIdx.x;
  // PROBE_UNROLL independent 16-byte loads in flight per thread
  for (; i + (PROBE_UNROLL - 1) * stride < nv; i += PROBE_UNROLL * stride) {
    uint4 x[PROBE_UNROLL];
#pragma unroll
    for (int u = 0; u < PROBE_UNROLL; ++u) x[u] = __ldcs(v + i + u * stride);
#pragma unroll
    for (int u = 0; u < PROBE_UNROLL; ++u) acc ^= x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
  }
  for (; i < nv; i += stride) {
    const uint4 x = __ldcs(v + i);
    acc ^= x.x ^ x.y ^ x.z ^ x.w;
  }
  if (blockIdx.x == 0)  // the last bytes of a length that is not a multiple of 16
    for (uint32_t t = threadIdx.x; t < ntail; t += PROBE_THREADS)
      acc ^= (uint32_t)tail[t] << (8 * (t & 3));
  acc = __reduce_xor_sync(PSS_FULL, acc);
  if ((threadIdx.x & 31) == 0) atomicXor(out, acc);
}

}  // namespace
}  // namespace pss

using namespace pss;

extern "C" {

pss_status pss_read_probe(const void* d_A, uint64_t n, pss_key_type kt, uint32_t* d_out,
                          cudaStream_t stream) {
  const int kb = kt == PSS_KEY_U32 ? 4 : (kt == PSS_KEY_U64 ? 8 : 0);
  if (!kb || (n && !d_A) || !d_out) return PSS_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_A) & 15u) != 0) return PSS_ERR_INVALID_ARG;
  const uint64_t bytes = n * (uint64_t)kb;
  const uint64_t nv = bytes / 16;
  const DevInfo d = dev_info();
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(uint32_t), stream);
  if (e != cudaSuccess) return PSS_ERR_CUDA;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, read_probe_kernel, PROBE_THREADS, 0) !=
          cudaSuccess ||
      nb < 1)
    nb = 1;
  const uint64_t want = (nv + PROBE_THREADS - 1) / PROBE_THREADS;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)nb * d.sms));
  read_probe_kernel<<<grid, PROBE_THREADS, 0, stream>>>(
      static_cast<const uint4*>(d_A), nv, static_cast<const unsigned char*>(d_A) + nv * 16,
      (uint32_t)(bytes - nv * 16), d_out);
  return cudaGetLastError() == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

}  // extern "C"
