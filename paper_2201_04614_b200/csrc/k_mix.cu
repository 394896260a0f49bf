// k_mix.cu -- measurement support: arithmetic-free streaming kernels with the
// fused kernels' read : write mixes, so that bench.py can report what HBM
// bandwidth each mix reaches on the box it runs on, next to the 1 : 1 copy
// figure of MEASURED_PEAKS.json.
//   kind 0  copy    f32 -> f32   4 B read, 4 B written per element
//   kind 1  narrow  f32 -> u16   4 read, 2 written (the fused compress mix)
//   kind 2  widen   u16 -> f32   2 read, 4 written (the fused decompress mix)
// 16-byte accesses, persistent grid-stride, ctas_per_sm CTAs of 256 threads per
// SM (the write-heavy mix is sensitive to it: the caller sweeps a few values
// and keeps the best).  Not on any product path.
#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"

namespace vlz {
namespace {

constexpr int MIX_THREADS = 256;

__global__ void __launch_bounds__(MIX_THREADS) mix_copy(const float4* __restrict__ in,
                                                        float4* __restrict__ out, size_t n4) {
  const size_t stride = (size_t)gridDim.x * MIX_THREADS;
  for (size_t i = (size_t)blockIdx.x * MIX_THREADS + threadIdx.x; i < n4; i += stride) out[i] = in[i];
}

__global__ void __launch_bounds__(MIX_THREADS) mix_narrow(const float4* __restrict__ in,
                                                          uint4* __restrict__ out, size_t n8) {
  const size_t stride = (size_t)gridDim.x * MIX_THREADS;
  for (size_t i = (size_t)blockIdx.x * MIX_THREADS + threadIdx.x; i < n8; i += stride) {
    const float4 a = in[2 * i], b = in[2 * i + 1];
    uint4 o;
    o.x = (__float_as_uint(a.x) >> 16) | (__float_as_uint(a.y) & 0xffff0000u);
    o.y = (__float_as_uint(a.z) >> 16) | (__float_as_uint(a.w) & 0xffff0000u);
    o.z = (__float_as_uint(b.x) >> 16) | (__float_as_uint(b.y) & 0xffff0000u);
    o.w = (__float_as_uint(b.z) >> 16) | (__float_as_uint(b.w) & 0xffff0000u);
    out[i] = o;
  }
}

__global__ void __launch_bounds__(MIX_THREADS) mix_widen(const uint4* __restrict__ in,
                                                         float4* __restrict__ out, size_t n8) {
  const size_t stride = (size_t)gridDim.x * MIX_THREADS;
  for (size_t i = (size_t)blockIdx.x * MIX_THREADS + threadIdx.x; i < n8; i += stride) {
    const uint4 c = in[i];
    out[2 * i] = make_float4(__uint_as_float(c.x << 16), __uint_as_float(c.x & 0xffff0000u),
                             __uint_as_float(c.y << 16), __uint_as_float(c.y & 0xffff0000u));
    out[2 * i + 1] = make_float4(__uint_as_float(c.z << 16), __uint_as_float(c.z & 0xffff0000u),
                                 __uint_as_float(c.w << 16), __uint_as_float(c.w & 0xffff0000u));
  }
}

}  // namespace
}  // namespace vlz

extern "C" int vlz_bench_stream(int32_t kind, const void* d_src, void* d_dst, int64_t n_elems,
                                int32_t ctas_per_sm, void* stream) {
  using namespace vlz;
  if (!d_src || !d_dst || n_elems < 8 || (n_elems & 7) || ctas_per_sm < 1 || ctas_per_sm > 8 ||
      (reinterpret_cast<uintptr_t>(d_src) & 15) || (reinterpret_cast<uintptr_t>(d_dst) & 15))
    return VLZ_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)(num_sms() * ctas_per_sm);
  const size_t n = (size_t)n_elems;
  switch (kind) {
    case 0:
      mix_copy<<<grid, MIX_THREADS, 0, st>>>(static_cast<const float4*>(d_src),
                                             static_cast<float4*>(d_dst), n / 4);
      break;
    case 1:
      mix_narrow<<<grid, MIX_THREADS, 0, st>>>(static_cast<const float4*>(d_src),
                                               static_cast<uint4*>(d_dst), n / 8);
      break;
    case 2:
      mix_widen<<<grid, MIX_THREADS, 0, st>>>(static_cast<const uint4*>(d_src),
                                              static_cast<float4*>(d_dst), n / 8);
      break;
    default: return VLZ_E_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}
