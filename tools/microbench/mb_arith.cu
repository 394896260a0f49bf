// Microbenchmark: throughput of the per-element arithmetic candidates for the
// dual-quant prequant + narrowing check on B200 (no memory traffic).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_exact(const float* seed, double y, double eb, int iters, unsigned long long* out) {
  float v = seed[threadIdx.x & 31] + threadIdx.x * 0.001f + blockIdx.x;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    double q = __ddiv_rn((double)v, y);
    double a = fabs(q);
    double fl = floor(__dadd_rn(a, 0.5));
    long long n = (long long)fl;
    n = q < 0 ? -n : n;
    float w = (float)__dmul_rn((double)n, y);
    bool bad = fabs(__dsub_rn((double)w, (double)v)) > eb;
    acc += (unsigned long long)n + bad;
    v = __fadd_rn(v, 0.37f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_mulonly(const float* seed, double iy, double y, double eb, int iters, unsigned long long* out) {
  float v = seed[threadIdx.x & 31] + threadIdx.x * 0.001f + blockIdx.x;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    double q = __dmul_rn((double)v, iy);
    double a = fabs(q);
    double fl = floor(__dadd_rn(a, 0.5));
    long long n = (long long)fl;
    n = q < 0 ? -n : n;
    float w = (float)__dmul_rn((double)n, y);
    bool bad = fabs(__dsub_rn((double)w, (double)v)) > eb;
    acc += (unsigned long long)n + bad;
    v = __fadd_rn(v, 0.37f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// fp32 fast path: magic-number floor, margin test, no conversions.
__global__ void k_fast32(const float* seed, float iy, float margin_k, int iters, unsigned long long* out) {
  float v = seed[threadIdx.x & 31] + threadIdx.x * 0.001f + blockIdx.x;
  unsigned acc = 0, slow = 0;
  for (int i = 0; i < iters; ++i) {
    float q = __fmul_rn(v, iy);
    float a = fabsf(q);
    float t = __fadd_rn(a, 0.5f);
    float r = __fadd_rd(t, 12582912.0f);
    int n = __float_as_int(r) - 0x4B400000;
    float fl = __fsub_rn(r, 12582912.0f);
    float fr = __fsub_rn(t, fl);
    float m = __fmul_rn(a, margin_k);
    bool ok = (fr > m) & (fr < 1.0f - m) & (a < 1048576.0f);
    slow += !ok;
    n = q < 0 ? -n : n;
    acc += n;
    v = __fadd_rn(v, 0.37f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + slow;
}

__global__ void k_cvt(const float* seed, int iters, unsigned long long* out) {
  float v = seed[threadIdx.x & 31] + threadIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += (double)v;  // F2F.F64.F32 + DADD
    v = __fadd_rn(v, 1.0f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned long long)acc;
}

// streaming: read f32, write u16 (the compress traffic shape)
__global__ void k_stream(const float4* __restrict__ in, uint2* __restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = in[i];
    uint2 o;
    o.x = ((unsigned)(int)v.x & 0xffff) | ((unsigned)(int)v.y << 16);
    o.y = ((unsigned)(int)v.z & 0xffff) | ((unsigned)(int)v.w << 16);
    out[i] = o;
  }
}

int main() {
  float* seed; cudaMalloc(&seed, 128); cudaMemset(seed, 0, 128);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  unsigned long long* out; cudaMalloc(&out, sizeof(unsigned long long) * blocks * threads);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double elems = (double)blocks * threads * iters;
  float ms;
  double y = 2.0 * 1.49e-3, eb = 1.49e-3;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_exact<<<blocks, threads>>>(seed, y, eb, iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("exact fp64 div path : %.3f Telem/s\n", elems / ms / 1e9);
    cudaEventRecord(a); k_mulonly<<<blocks, threads>>>(seed, 1.0 / y, y, eb, iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("fp64 mul path       : %.3f Telem/s\n", elems / ms / 1e9);
    cudaEventRecord(a); k_fast32<<<blocks, threads>>>(seed, (float)(1.0 / y), 1e-6f, iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("fp32 fast path      : %.3f Telem/s\n", elems / ms / 1e9);
    cudaEventRecord(a); k_cvt<<<blocks, threads>>>(seed, iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("f32->f64 cvt+dadd   : %.3f Telem/s\n", elems / ms / 1e9);
  }
  size_t n = (size_t)1 << 30;  // 4 GiB in, 2 GiB out
  float4* in; uint2* o2; cudaMalloc(&in, n * 4); cudaMalloc(&o2, n * 2); cudaMemset(in, 0, n * 4);
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a); k_stream<<<g, 512>>>(in, o2, n / 4); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("stream f32->u16 grid %d: %.1f GB/s (6 B/elem)\n", g, n * 6.0 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
