// lookback.cuh -- single-pass chunked exclusive scan (decoupled look-back),
// shared by the entropy-stage kernels.
//
// Chunk order is the dynamic ticket order (a CTA only ever waits on chunks
// that already started), each chunk publishes its aggregate as soon as it is
// known (flag A) and its inclusive prefix once resolved (flag P); warp 0 of a
// chunk walks back 32 descriptors at a time.  Values are 62-bit.
#pragma once

#include <cuda/atomic>

#include <cstdint>

namespace vlz {

constexpr unsigned long long LB_FLAG_A = 1ull << 62;
constexpr unsigned long long LB_FLAG_P = 2ull << 62;
constexpr unsigned long long LB_VAL = (1ull << 62) - 1;

// called by all 32 lanes of ONE warp; returns the exclusive prefix of `tile`
// (all lanes) and publishes its inclusive prefix
__device__ __forceinline__ long long lookback_exclusive(unsigned long long* lb, int64_t tile,
                                                        long long agg, int lane) {
  using ref = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
  ref me(lb[tile]);
  if (lane == 0)
    me.store((tile == 0 ? LB_FLAG_P : LB_FLAG_A) | (unsigned long long)agg,
             cuda::memory_order_release);
  long long excl = 0;
  int64_t pred = tile - 1;
  while (pred >= 0) {
    const int64_t idx = pred - lane;
    unsigned long long w = LB_FLAG_P;  // before chunk 0: prefix 0
    if (idx >= 0) {
      ref r(lb[idx]);
      w = r.load(cuda::memory_order_acquire);
      while ((w >> 62) == 0) w = r.load(cuda::memory_order_acquire);
    }
    const unsigned pm = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    const int stop = pm ? __ffs(pm) - 1 : 31;
    long long val = (lane <= stop && idx >= 0) ? (long long)(w & LB_VAL) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    if (pm) break;
    pred -= 32;
  }
  if (lane == 0 && tile > 0)
    me.store(LB_FLAG_P | (unsigned long long)(excl + agg), cuda::memory_order_release);
  return excl;
}

}  // namespace vlz
