// k_sweep.cu -- test support: exhaustive check of the float32 exact-fast
// prequantizer against the exact float64 one over all 2^32 float bit patterns.
//
// The compress kernels accept quant_fast's n whenever its `ok` test passes
// and re-evaluate the element with
// quant_exact otherwise.  The argument that an accepted n equals the
// reference's round_half_away(fl64(v / (2 eb))) (quantize.py:31-42,66-78)
// and that its float32-narrowed reconstruction passes the bound check
// (vector.py:72-77) is checked here for every pattern, for a given eb:
//   * both forms the kernels use -- the scalar quant_fast (vlz_common.cuh,
//     1-D and generic kernels) and the paired-FP32 form of
//     dq_compress_fast.cuh (FMUL2/FADD2/FFMA2 on two patterns at a time) --
//     must agree on n and on the verdict;
//   * an accepted pattern must be finite, must not overflow the quantizer,
//     must give quant_exact's n and must pass the narrowing check.
// Not on any product path: only tests/test_gpu_sweep.py calls it.
#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "vlz_common.cuh"

namespace vlz {

QP make_qp(const vlz_params* p);

namespace {

// counters: 0 accepted, 1 fallback (finite, rejected), 2 non-finite,
// 3 mismatches (accepted but wrong), 4 form disagreements, 5 first bad pattern
__global__ void __launch_bounds__(256) prequant_sweep_kernel(QP q, unsigned long long* cnt) {
  unsigned long long acc = 0, fb = 0, nf = 0, bad = 0, form = 0;
  unsigned long long first = ~0ull;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (1ull << 31);
       i += stride) {
    const unsigned u0 = (unsigned)(2 * i);
    const float2 v = make_float2(__uint_as_float(u0), __uint_as_float(u0 + 1));
    // paired form, operation for operation as dq_compress_fast.cuh
    const float2 qq = __fmul2_rn(v, make_float2(q.inv32, q.inv32));
    const float2 r = __fadd2_rn(qq, make_float2(12582912.0f, 12582912.0f));
    const float2 rn = __fadd2_rn(r, make_float2(-12582912.0f, -12582912.0f));
    const float2 e = __ffma2_rn(rn, make_float2(-1.0f, -1.0f), qq);
    const float2 lim = __ffma2_rn(make_float2(fabsf(qq.x), fabsf(qq.y)),
                                  make_float2(-q.kq, -q.kq), make_float2(q.lim0, q.lim0));
    const int np[2] = {__float_as_int(r.x) - 0x4B400000, __float_as_int(r.y) - 0x4B400000};
    const bool okp[2] = {fabsf(e.x) < lim.x, fabsf(e.y) < lim.y};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float vk = k ? v.y : v.x;
      bool oks;
      const int ns = quant_fast(vk, q, oks);  // scalar form
      if (oks != okp[k] || (oks && ns != np[k])) {
        ++form;
        first = min(first, (unsigned long long)(u0 + k));
      }
      if (!isfinite(vk)) {
        ++nf;
        if (okp[k]) {
          ++bad;
          first = min(first, (unsigned long long)(u0 + k));
        }
        continue;
      }
      if (!okp[k]) {
        ++fb;
        continue;
      }
      ++acc;
      bool nb, ovf;
      const int ne = quant_exact(vk, q, nb, ovf);
      if (ne != np[k] || nb || ovf) {
        ++bad;
        first = min(first, (unsigned long long)(u0 + k));
      }
    }
  }
  // warp then CTA reduction, one set of atomics per CTA
  for (int o = 16; o; o >>= 1) {
    acc += __shfl_xor_sync(FULL, acc, o);
    fb += __shfl_xor_sync(FULL, fb, o);
    nf += __shfl_xor_sync(FULL, nf, o);
    bad += __shfl_xor_sync(FULL, bad, o);
    form += __shfl_xor_sync(FULL, form, o);
    first = min(first, __shfl_xor_sync(FULL, first, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(cnt + 0, acc);
    atomicAdd(cnt + 1, fb);
    atomicAdd(cnt + 2, nf);
    atomicAdd(cnt + 3, bad);
    atomicAdd(cnt + 4, form);
    atomicMin(cnt + 5, first);
  }
}

__global__ void sweep_init(unsigned long long* cnt) {
  if (threadIdx.x < 6) cnt[threadIdx.x] = threadIdx.x == 5 ? ~0ull : 0ull;
}

}  // namespace
}  // namespace vlz

extern "C" int vlz_test_prequant_sweep(double eb, unsigned long long* d_counts, void* stream) {
  if (!d_counts || !(eb > 0.0)) return VLZ_E_ARG;
  vlz_params p{};
  p.eb = eb;
  p.radius = 512;
  const vlz::QP q = vlz::make_qp(&p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  vlz::sweep_init<<<1, 32, 0, st>>>(d_counts);
  vlz::prequant_sweep_kernel<<<sms * 8, 256, 0, st>>>(q, d_counts);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

// the fast path's enable flag for this eb (make_qp): 1 when quant_fast runs
extern "C" int vlz_test_fast_enabled(double eb) {
  vlz_params p{};
  p.eb = eb;
  return vlz::make_qp(&p).lim0 >= 0.0f ? 1 : 0;
}
