// k_crc.cu -- CRC-32 (zlib: reflected polynomial 0xEDB88320, init and final
// xor 0xFFFFFFFF) of a device byte range, for the VLZ1 container's payload
// CRC (reference container.py:160-163 writes it, :214-217 checks it).
//
// The register update R(c, data) of a CRC is affine in the incoming register:
// R(c, A||B) = R(0, B) ^ c * x^(8|B|) mod P (zlib's crc32_combine).  So:
//   crc_segments  one thread per 4 KiB segment (aligned to the range's 16-byte
//                 floor; the first segment is shorter) computes R(0, segment)
//                 with slicing-by-8 tables in shared memory, 16-byte loads;
//   crc_fold      one CTA folds the segment values left to right in 1024
//                 runs and combines the runs in a tree, each combine being a
//                 GF(2) multiply by x^(8 len(right)) mod P;
// crc32 = ~(R(0, data) ^ 0xFFFFFFFF * x^(8 n) mod P).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"

namespace vlz {
namespace {

constexpr uint32_t CRC_POLY = 0xEDB88320u;
constexpr int64_t CRC_SEG = 4096;
constexpr int CRC_FOLD_THREADS = 1024;

struct CrcTables {
  uint32_t t[8][256];   // slicing-by-8
  uint32_t x2n[32];     // x^(2^k) mod P
};
__constant__ uint32_t c_x2n[32];

// a * b mod P, reflected bit order (zlib multmodp; x^0 is bit 31)
__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t p = 0;
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    if (a & (0x80000000u >> i)) p ^= b;
    b = (b & 1u) ? (b >> 1) ^ CRC_POLY : b >> 1;
  }
  return p;
}

// x^(8 n) mod P: the operator that appends n zero bytes
__device__ uint32_t x8nmodp(uint64_t n) {
  uint32_t p = 0x80000000u;
  int k = 3;
  while (n) {
    if (n & 1) p = multmodp(c_x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

__device__ __forceinline__ uint32_t step8(const uint32_t (*T)[256], uint32_t c, uint64_t w) {
  c ^= (uint32_t)w;
  const uint32_t h = (uint32_t)(w >> 32);
  return T[7][c & 0xff] ^ T[6][(c >> 8) & 0xff] ^ T[5][(c >> 16) & 0xff] ^ T[4][c >> 24] ^
         T[3][h & 0xff] ^ T[2][(h >> 8) & 0xff] ^ T[1][(h >> 16) & 0xff] ^ T[0][h >> 24];
}

__global__ void __launch_bounds__(256) crc_segments(const uint8_t* __restrict__ base, int64_t lo,
                                                    int64_t hi, int64_t nseg,
                                                    const CrcTables* __restrict__ tabs,
                                                    uint32_t* __restrict__ seg_crc) {
  __shared__ uint32_t T[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) T[i >> 8][i & 255] = tabs->t[i >> 8][i & 255];
  __syncthreads();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    // bytes [a, b) of the 16-byte aligned frame that starts at `base`
    const int64_t a = s == 0 ? lo : s * CRC_SEG;
    const int64_t b = (s + 1) * CRC_SEG < hi ? (s + 1) * CRC_SEG : hi;
    uint32_t c = 0;
    int64_t p = a;
    for (; p < b && (p & 15); ++p) c = (c >> 8) ^ T[0][(c ^ base[p]) & 0xff];
    for (; p + 16 <= b; p += 16) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + p));
      c = step8(T, c, ((uint64_t)v.y << 32) | v.x);
      c = step8(T, c, ((uint64_t)v.w << 32) | v.z);
    }
    for (; p < b; ++p) c = (c >> 8) ^ T[0][(c ^ base[p]) & 0xff];
    seg_crc[s] = c;
  }
}

__global__ void __launch_bounds__(CRC_FOLD_THREADS) crc_fold(const uint32_t* __restrict__ seg_crc,
                                                             int64_t lo, int64_t hi, int64_t nseg,
                                                             uint32_t* out) {
  __shared__ uint32_t r[CRC_FOLD_THREADS];
  __shared__ int64_t len[CRC_FOLD_THREADS];
  const int t = threadIdx.x;
  const int64_t per = (nseg + CRC_FOLD_THREADS - 1) / CRC_FOLD_THREADS;
  const int64_t s0 = t * per, s1 = s0 + per < nseg ? s0 + per : nseg;
  const uint32_t full = x8nmodp(CRC_SEG);
  uint32_t acc = 0;
  int64_t n = 0;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t a = s == 0 ? lo : s * CRC_SEG;
    const int64_t b = (s + 1) * CRC_SEG < hi ? (s + 1) * CRC_SEG : hi;
    const int64_t l = b - a;
    acc = (s == s0 ? 0u : multmodp(l == CRC_SEG ? full : x8nmodp(l), acc)) ^ seg_crc[s];
    n += l;
  }
  r[t] = acc;
  len[t] = n;
  __syncthreads();
  for (int w = 1; w < CRC_FOLD_THREADS; w <<= 1) {
    if ((t & (2 * w - 1)) == 0 && len[t + w] > 0)
      r[t] = (len[t] > 0 ? multmodp(x8nmodp(len[t + w]), r[t]) : 0u) ^ r[t + w];
    __syncthreads();
    if ((t & (2 * w - 1)) == 0) len[t] += len[t + w];
    __syncthreads();
  }
  if (t == 0) *out = ~(multmodp(x8nmodp(hi - lo), 0xFFFFFFFFu) ^ r[0]);
}

// host: tables (slicing-by-8) and x^(2^k) mod P, built once
uint32_t h_multmodp(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (int i = 0; i < 32; ++i) {
    if (a & (0x80000000u >> i)) p ^= b;
    b = (b & 1u) ? (b >> 1) ^ CRC_POLY : b >> 1;
  }
  return p;
}

const CrcTables* device_tables(cudaError_t& err) {
  static CrcTables* d = nullptr;
  static cudaError_t e0 = [] {
    CrcTables h;
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ CRC_POLY : c >> 1;
      h.t[0][i] = c;
    }
    for (int s = 1; s < 8; ++s)
      for (int i = 0; i < 256; ++i) h.t[s][i] = (h.t[s - 1][i] >> 8) ^ h.t[0][h.t[s - 1][i] & 0xff];
    h.x2n[0] = 1u << 30;  // x^1
    for (int k = 1; k < 32; ++k) h.x2n[k] = h_multmodp(h.x2n[k - 1], h.x2n[k - 1]);
    cudaError_t e = cudaMalloc(&d, sizeof(CrcTables));
    if (e == cudaSuccess) e = cudaMemcpy(d, &h, sizeof(CrcTables), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_x2n, h.x2n, sizeof(h.x2n));
    return e;
  }();
  err = e0;
  return d;
}

}  // namespace
}  // namespace vlz

extern "C" {

size_t vlz_crc32_ws_size(int64_t n) {
  if (n < 0) return 0;
  return (size_t)((n + 2 * vlz::CRC_SEG) / vlz::CRC_SEG + 1) * 4 + 256;
}

int vlz_crc32_device(const uint8_t* d_data, int64_t n, uint32_t* d_crc, void* d_ws,
                     size_t ws_bytes, void* stream) {
  if (n < 0 || !d_crc || (n > 0 && !d_data) || !d_ws || ws_bytes < vlz_crc32_ws_size(n))
    return VLZ_E_ARG;
  cudaError_t err;
  const vlz::CrcTables* tabs = vlz::device_tables(err);
  if (err != cudaSuccess) return VLZ_E_CUDA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // segment frame: 16-byte aligned base at or below d_data
  const uintptr_t addr = reinterpret_cast<uintptr_t>(d_data);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(addr & ~uintptr_t(15));
  const int64_t lo = (int64_t)(addr & 15), hi = lo + n;
  const int64_t nseg = n == 0 ? 0 : (hi + vlz::CRC_SEG - 1) / vlz::CRC_SEG;
  uint32_t* seg = static_cast<uint32_t*>(d_ws);
  if (nseg > 0) {
    int64_t grid = (nseg + 255) / 256;
    const int64_t cap = (int64_t)vlz::num_sms() * 8;
    if (grid > cap) grid = cap;
    vlz::crc_segments<<<(unsigned)grid, 256, 0, st>>>(base, lo, hi, nseg, tabs, seg);
  }
  vlz::crc_fold<<<1, vlz::CRC_FOLD_THREADS, 0, st>>>(seg, lo, hi, nseg, d_crc);
  vlz::g_launches.fetch_add(nseg > 0 ? 2 : 1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

}  // extern "C"
