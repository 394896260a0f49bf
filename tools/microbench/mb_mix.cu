// Microbenchmark: what HBM bandwidth does a kernel with the dual-quant kernels'
// read : write mix reach on this B200?  MEASURED_PEAKS.json's figure is a 1 : 1
// copy; the fused compress kernel reads 4 B and writes 2 B per element, the
// fused decompress kernel reads 2 B and writes 4 B.  Three streaming kernels
// with no arithmetic to speak of, 16-byte accesses, persistent grid-stride:
//   copy   : f32 -> f32   (4 read, 4 written)
//   narrow : f32 -> u16   (4 read, 2 written: the compress mix)
//   widen  : u16 -> f32   (2 read, 4 written: the decompress mix)
// Prints GB/s (read + written bytes) per kernel, best and median of the runs.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_mix mb_mix.cu && ./mb_mix [elements]
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int THREADS = 256;

__global__ void __launch_bounds__(THREADS) k_copy(const float4* __restrict__ in, float4* __restrict__ out,
                                                  size_t n4) {
  const size_t stride = (size_t)gridDim.x * THREADS;
  for (size_t i = (size_t)blockIdx.x * THREADS + threadIdx.x; i < n4; i += stride) out[i] = in[i];
}

// 8 elements per thread: two 16-byte loads, one 16-byte store
__global__ void __launch_bounds__(THREADS) k_narrow(const float4* __restrict__ in, uint4* __restrict__ out,
                                                    size_t n8) {
  const size_t stride = (size_t)gridDim.x * THREADS;
  for (size_t i = (size_t)blockIdx.x * THREADS + threadIdx.x; i < n8; i += stride) {
    const float4 a = in[2 * i], b = in[2 * i + 1];
    uint4 o;
    o.x = (__float_as_uint(a.x) >> 16) | (__float_as_uint(a.y) & 0xffff0000u);
    o.y = (__float_as_uint(a.z) >> 16) | (__float_as_uint(a.w) & 0xffff0000u);
    o.z = (__float_as_uint(b.x) >> 16) | (__float_as_uint(b.y) & 0xffff0000u);
    o.w = (__float_as_uint(b.z) >> 16) | (__float_as_uint(b.w) & 0xffff0000u);
    out[i] = o;
  }
}

// 8 elements per thread: one 16-byte load, two 16-byte stores
__global__ void __launch_bounds__(THREADS) k_widen(const uint4* __restrict__ in, float4* __restrict__ out,
                                                   size_t n8) {
  const size_t stride = (size_t)gridDim.x * THREADS;
  for (size_t i = (size_t)blockIdx.x * THREADS + threadIdx.x; i < n8; i += stride) {
    const uint4 c = in[i];
    out[2 * i] = make_float4(__uint_as_float(c.x << 16), __uint_as_float(c.x & 0xffff0000u),
                             __uint_as_float(c.y << 16), __uint_as_float(c.y & 0xffff0000u));
    out[2 * i + 1] = make_float4(__uint_as_float(c.z << 16), __uint_as_float(c.z & 0xffff0000u),
                                 __uint_as_float(c.w << 16), __uint_as_float(c.w & 0xffff0000u));
  }
}

// widen variants: store policy SP (0 default, 1 .cs streaming, 2 .wt write-through,
// 3 256-bit st.global.v8), loads through ld.global.cs when LCS, U tiles in flight per thread
template <int SP>
__device__ __forceinline__ void store16(float4* p, float4 v) {
  if constexpr (SP == 1) __stcs(p, v);
  else if constexpr (SP == 2) __stwt(p, v);
  else *p = v;
}
template <int SP, bool LCS, int U>
__global__ void __launch_bounds__(THREADS) k_widen_v(const uint4* __restrict__ in, float4* __restrict__ out,
                                                     size_t n8) {
  const size_t stride = (size_t)gridDim.x * THREADS;
  for (size_t i0 = (size_t)blockIdx.x * THREADS + threadIdx.x; i0 < n8; i0 += stride * U) {
    uint4 c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = i0 + u * stride;
      if (i < n8) c[u] = LCS ? __ldcs(in + i) : in[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= n8) continue;
      const float4 a = make_float4(__uint_as_float(c[u].x << 16), __uint_as_float(c[u].x & 0xffff0000u),
                                   __uint_as_float(c[u].y << 16), __uint_as_float(c[u].y & 0xffff0000u));
      const float4 b = make_float4(__uint_as_float(c[u].z << 16), __uint_as_float(c[u].z & 0xffff0000u),
                                   __uint_as_float(c[u].w << 16), __uint_as_float(c[u].w & 0xffff0000u));
      if constexpr (SP == 3) {
        asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(out + 2 * i),
                     "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                     : "memory");
      } else {
        store16<SP>(out + 2 * i, a);
        store16<SP>(out + 2 * i + 1, b);
      }
    }
  }
}
// the fused kernels' own access pattern without the arithmetic: a warp owns a
// tile = 8 planes x 8 rows x 128 columns (16 blocks of 8x8x8); input rows are
// 512 B, one row pitch apart; codes are 128-byte block planes (block-major).
// `order` maps the warp's k-th tile: 0 grid-stride (the kernels' order),
// 1 contiguous per warp, 2 contiguous per CTA with its warps interleaved,
// 3 grid-stride over a z-fastest tile numbering
__device__ __forceinline__ size_t tile_of(int order, size_t k, size_t w0, size_t nwarps, size_t ntiles,
                                          size_t NW, size_t P1, size_t P0) {
  const size_t per = (ntiles + nwarps - 1) / nwarps;
  size_t t;
  if (order == 1) t = w0 * per + k;
  else if (order == 2) t = (w0 / 4) * per * 4 + k * 4 + (w0 & 3);
  else t = w0 + k * nwarps;
  if (order == 3 && t < ntiles) {  // t = (wx, by) slow, bz fast
    const size_t bz = t % P0, r = t / P0;
    t = (bz * P1 + r / NW) * NW + r % NW;
  }
  return t;
}
template <bool WIDEN>
__global__ void __launch_bounds__(128) k_tiles(uint2* __restrict__ codes, float4* __restrict__ field,
                                               int D0, int D1, int D2, int order) {
  const int lane = threadIdx.x & 31;
  const size_t nwarps = (size_t)gridDim.x * 4, w0 = (size_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const size_t NW = D2 / 128, P1 = D1 / 8, P0 = D0 / 8, ntiles = NW * P1 * P0;
  const size_t per = (ntiles + nwarps - 1) / nwarps;
  for (size_t k = 0; k < per; ++k) {
    const size_t t = tile_of(order, k, w0, nwarps, ntiles, NW, P1, P0);
    if (t >= ntiles) continue;
    const size_t wx = t % NW, by = (t / NW) % P1, bz = t / (NW * P1);
    const size_t cbase = ((bz * P1 + by) * (D2 / 8) + wx * 16) * 512;  // 16 blocks of 512 codes
    for (int zl = 0; zl < 8; ++zl) {
      if (WIDEN) {
        uint2 c[8];
#pragma unroll
        for (int r = 0; r < 8; ++r)  // lane's 4 codes of row r: block lane/2, plane zl
          c[r] = codes[(cbase + (size_t)(lane >> 1) * 512 + zl * 64 + r * 8 + (lane & 1) * 4) / 4];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float4 v = make_float4(__uint_as_float(c[r].x << 16), __uint_as_float(c[r].x & 0xffff0000u),
                                       __uint_as_float(c[r].y << 16), __uint_as_float(c[r].y & 0xffff0000u));
          field[(((bz * 8 + zl) * (size_t)D1 + by * 8 + r) * D2 + wx * 128) / 4 + lane] = v;
        }
      } else {
        float4 v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
          v[r] = field[(((bz * 8 + zl) * (size_t)D1 + by * 8 + r) * D2 + wx * 128) / 4 + lane];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          uint2 c;
          c.x = (__float_as_uint(v[r].x) >> 16) | (__float_as_uint(v[r].y) & 0xffff0000u);
          c.y = (__float_as_uint(v[r].z) >> 16) | (__float_as_uint(v[r].w) & 0xffff0000u);
          codes[(cbase + (size_t)(lane >> 1) * 512 + zl * 64 + r * 8 + (lane & 1) * 4) / 4] = c;
        }
      }
    }
  }
}

template <typename F>
static void timeit(const char* name, double bytes, F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch();
  std::vector<float> ms;
  for (int i = 0; i < 15; ++i) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  std::printf("{\"kernel\": \"%s\", \"best_gbs\": %.1f, \"median_gbs\": %.1f, \"median_ms\": %.4f}\n", name,
              bytes / ms.front() * 1e-6, bytes / ms[ms.size() / 2] * 1e-6, ms[ms.size() / 2]);
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (size_t)1 << 32;  // C5: 2^32 elements
  float* f = nullptr;
  float* g = nullptr;
  uint16_t* h = nullptr;
  if (cudaMalloc(&f, n * 4) != cudaSuccess || cudaMalloc(&g, n * 4) != cudaSuccess ||
      cudaMalloc(&h, n * 2) != cudaSuccess) {
    std::fprintf(stderr, "allocation failed\n");
    return 1;
  }
  cudaMemset(f, 1, n * 4);
  cudaMemset(h, 1, n * 2);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {4, 8}) {
    const int grid = sms * per_sm;
    std::printf("{\"grid\": %d, \"elements\": %zu}\n", grid, n);
    timeit("copy 4r+4w", 8.0 * n, [&] {
      k_copy<<<grid, THREADS>>>(reinterpret_cast<const float4*>(f), reinterpret_cast<float4*>(g), n / 4);
    });
    timeit("narrow 4r+2w (compress mix)", 6.0 * n, [&] {
      k_narrow<<<grid, THREADS>>>(reinterpret_cast<const float4*>(f), reinterpret_cast<uint4*>(h), n / 8);
    });
    timeit("widen 2r+4w (decompress mix)", 6.0 * n, [&] {
      k_widen<<<grid, THREADS>>>(reinterpret_cast<const uint4*>(h), reinterpret_cast<float4*>(g), n / 8);
    });
  }
  if (n == ((size_t)1 << 32)) {
    const uint4* hi = reinterpret_cast<const uint4*>(h);
    float4* go = reinterpret_cast<float4*>(g);
    for (int per_sm : {2, 3, 4, 6}) {
      const int grid = sms * per_sm;
      std::printf("{\"grid\": %d}\n", grid);
      timeit("widen default U1", 6.0 * n, [&] { k_widen_v<0, false, 1><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen st.cs U1", 6.0 * n, [&] { k_widen_v<1, false, 1><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen st.cs ld.cs U1", 6.0 * n, [&] { k_widen_v<1, true, 1><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen st.wt U1", 6.0 * n, [&] { k_widen_v<2, false, 1><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen v8 U1", 6.0 * n, [&] { k_widen_v<3, false, 1><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen default U2", 6.0 * n, [&] { k_widen_v<0, false, 2><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen default U4", 6.0 * n, [&] { k_widen_v<0, false, 4><<<grid, THREADS>>>(hi, go, n / 8); });
      timeit("widen st.cs U4", 6.0 * n, [&] { k_widen_v<1, false, 4><<<grid, THREADS>>>(hi, go, n / 8); });
    }
    for (int per_sm : {4, 5, 8}) {
      const int grid = sms * per_sm;
      std::printf("{\"grid\": %d, \"threads\": 128}\n", grid);
      for (int order = 0; order < 4; ++order) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "widen C5 tiles order %d", order);
        timeit(nm, 6.0 * n, [&] {
          k_tiles<true><<<grid, 128>>>(reinterpret_cast<uint2*>(h), go, 1024, 2048, 2048, order);
        });
        std::snprintf(nm, sizeof nm, "narrow C5 tiles order %d", order);
        timeit(nm, 6.0 * n, [&] {
          k_tiles<false><<<grid, 128>>>(reinterpret_cast<uint2*>(h), reinterpret_cast<float4*>(f), 1024, 2048,
                                        2048, order);
        });
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
