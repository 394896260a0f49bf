// k_huffman.cu -- device side of the entropy stage.
//
// vlz_histogram: symbol frequencies of a uint16 code stream (huffman.py:62,
// np.bincount).  Codes cluster tightly around the radius R (delta = code - R
// is small), so each CTA keeps a private shared-memory histogram of the 8192
// bins around R plus a private counter for the outlier sentinel 0; every other
// symbol goes straight to a global atomic.  Grid-stride over 16-byte vectors.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"

namespace vlz {
namespace {

constexpr int HWIN = 8192;

__global__ void __launch_bounds__(512) histogram_kernel(const uint16_t* __restrict__ codes,
                                                        int64_t n, int lo,
                                                        unsigned long long* freqs) {
  __shared__ unsigned int bins[HWIN];
  __shared__ unsigned int zero;
  for (int i = threadIdx.x; i < HWIN; i += blockDim.x) bins[i] = 0;
  if (threadIdx.x == 0) zero = 0;
  __syncthreads();
  auto add = [&](unsigned c) {
    const unsigned k = c - (unsigned)lo;
    if (k < (unsigned)HWIN) atomicAdd(&bins[k], 1u);
    else if (c == 0) atomicAdd(&zero, 1u);
    else atomicAdd(&freqs[c], 1ull);
  };
  const int64_t nvec = n / 8;
  const uint4* v = reinterpret_cast<const uint4*>(codes);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = v[i];
    const unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      add(ws[k] & 0xffffu);
      add(ws[k] >> 16);
    }
  }
  for (int64_t i = nvec * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    add(codes[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < HWIN; i += blockDim.x)
    if (bins[i]) atomicAdd(&freqs[lo + i], (unsigned long long)bins[i]);
  if (threadIdx.x == 0 && zero) atomicAdd(&freqs[0], (unsigned long long)zero);
}

}  // namespace
}  // namespace vlz

extern "C" {

// d_freqs: uint64[65536] (zeroed here); codes must be 16-byte aligned
int vlz_histogram(const uint16_t* d_codes, int64_t n, int32_t radius, uint64_t* d_freqs,
                  void* stream) {
  if (!d_freqs || n < 0 || (n > 0 && !d_codes)) return VLZ_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_freqs, 0, 65536 * sizeof(uint64_t), st);
  if (e != cudaSuccess) return VLZ_E_CUDA;
  if (n == 0) return VLZ_OK;
  int lo = radius - vlz::HWIN / 2;
  if (lo < 1) lo = 1;
  if (lo + vlz::HWIN > 65536) lo = 65536 - vlz::HWIN;
  int64_t grid = (n / 8 + 511) / 512;
  const int64_t cap = (int64_t)vlz::num_sms() * 4;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  vlz::histogram_kernel<<<(unsigned)grid, 512, 0, st>>>(
      d_codes, n, lo, reinterpret_cast<unsigned long long*>(d_freqs));
  vlz::g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

}  // extern "C"
