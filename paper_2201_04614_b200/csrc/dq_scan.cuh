// dq_scan.cuh -- single-pass block-count scan + outlier compaction.
//
// Turns the per-block outlier counts (CodeStream.outlier_counts, model.py:
// 253-256) into canonical offsets with a decoupled look-back scan over chunks
// of CH blocks (chunk order = dynamic ticket order, so every chunk only waits
// on chunks that are already running), then copies each block's outliers from
// its block-relative scratch slots into the compact canonical array
// (vector.py:193-202: outliers in block-major, in-block traversal order).
//
// For *:global padding it first resolves the block origins that the fused
// kernel left pending (the origin is the only element whose delta depends on
// the global scalar): it derives s0 from the reduced
// statistics (padding.py:62-69, 72-85), re-quantizes the origin value, writes
// the origin code, and adds the origin to the block's count when it is an
// outlier (its value goes to scratch slot 0).
//
// In OFFSETS mode (decompression) it only writes the exclusive offsets.
#pragma once

#include <cuda/atomic>

#include "vlz_common.cuh"

namespace vlz {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_MIN_CH = SCAN_THREADS;  // smallest chunk (blocks per CTA)

// blocks per thread: 8 for large grids (few look-back steps), fewer when the
// grid is small so that the outlier gather still spreads over >= ~4 CTAs/SM
inline int scan_ipt(int64_t nblocks) {
  int ipt = 1;
  while (ipt < 8 && nblocks > (int64_t)SCAN_THREADS * ipt * 148 * 4) ipt *= 2;
  return ipt;
}
inline int64_t scan_chunks(int64_t nblocks) {
  const int64_t ch = (int64_t)SCAN_THREADS * scan_ipt(nblocks);
  const int64_t n = (nblocks + ch - 1) / ch;
  return n < 1 ? 1 : n;
}

struct ScanArgs {
  Geo g;
  QP q;
  int BZ, BY, BX;
  int fix_origin;  // 1: resolve pending origins (*:global policies)
  int gather;      // 1: compact outliers; 0: write offsets
  const float* in;
  uint16_t* codes;
  int64_t* counts;
  float* scratch;
  float* out;
  int64_t* offsets;
  int64_t* scalars;
  unsigned long long* lb;  // per chunk look-back words
  unsigned int* ticket;
  long long* n_out;
  const long long* gstats;  // sum, count, min, neg_max (reduced)
  // compress status finalisation (done by the chunk holding the last block)
  int* status;
  long long* index;
  const unsigned long long* first_nonfinite;
  const unsigned long long* first_overflow;
  // optional list of rewritten origin codes, (position << 16) | code, for
  // callers that copied the provisional codes out early (host pipeline)
  unsigned long long* patch_list;
  unsigned int* patch_count;
};

__device__ __forceinline__ void block_of(const Geo& g, int64_t bi, int BZ, int BY, int BX,
                                         int64_t& bstart, int64_t& origin) {
  int64_t bx, by, bz;
  if (g.nblocks < 0xffffffffll) {  // 32-bit magic division (the common case)
    const uint32_t t = g.divP2.div((uint32_t)bi);
    bx = (uint32_t)bi - t * (uint32_t)g.P2;
    bz = g.divP1.div(t);
    by = t - (uint32_t)bz * (uint32_t)g.P1;
  } else {
    bx = bi % g.P2;
    const int64_t t = bi / g.P2;
    by = t % g.P1;
    bz = t / g.P1;
  }
  const int64_t ez = imin64(BZ, g.D0 - bz * BZ);
  const int64_t ey = imin64(BY, g.D1 - by * BY);
  bstart = block_start(g, bz, by, bx, BZ, BY, BX, ez, ey);
  origin = ((bz * BZ) * g.D1 + by * BY) * g.D2 + bx * BX;
}

constexpr unsigned long long FLAG_A = 1ull << 62;
constexpr unsigned long long FLAG_P = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

template <int SCAN_IPT>
__global__ void __launch_bounds__(SCAN_THREADS) dq_scan_kernel(ScanArgs a) {
  constexpr int SCAN_CH = SCAN_THREADS * SCAN_IPT;
  __shared__ long long s_src[SCAN_CH];   // scratch source of each block's outliers
  __shared__ long long s_cnt[SCAN_CH];   // counts in, final counts / offsets out
  __shared__ long long s_warp[SCAN_THREADS / 32];
  __shared__ long long s_excl;
  __shared__ unsigned int s_tile;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SCAN_CH;
  const int64_t nb = a.g.nblocks;

  int64_t s0 = 0;
  if (a.fix_origin) {
    const long long* gs = a.gstats;
    s0 = stat_value(a.q.kind, gs[0], gs[1], gs[2], -gs[3]);
  }

  // the chunk's count words move through shared memory so that global loads
  // and stores are coalesced; thread t then owns blocks t*IPT .. t*IPT+IPT-1
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t bi = base + (int64_t)k * SCAN_THREADS + tid;
    s_cnt[k * SCAN_THREADS + tid] = bi < nb ? a.counts[bi] : 0;
  }
  __syncthreads();
  // per-block counts fit 32 bits (<= block volume), so do chunk-local sums
  // (<= SCAN_CH * 2^18); 32-bit state keeps the register count low
  int c[SCAN_IPT];
  int tsum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t bi = base + (int64_t)tid * SCAN_IPT + k;
    c[k] = 0;
    if (bi < nb) {
      const long long rec = s_cnt[tid * SCAN_IPT + k];
      c[k] = (int)rec;
      if (a.fix_origin || (a.gather && c[k] > 0)) {
        int64_t bstart, origin;
        block_of(a.g, bi, a.BZ, a.BY, a.BX, bstart, origin);
        if (a.fix_origin) {
          // pending-origin record written by the fused kernel (pack_origin)
          const int d = (int)(rec >> 32);
          const bool bad = (rec >> 24) & 1;
          c[k] = (int)(rec & 0xffffff);
          const int64_t delta = (int64_t)d - s0;
          const int R = a.q.radius;
          const bool out = bad || delta > (int64_t)(R - 1) || delta < -(int64_t)(R - 1);
          const uint16_t code = out ? (uint16_t)0 : (uint16_t)(delta + R);
          // the fused kernel already stored the s0 = 0 code of the origin;
          // rewrite only when s0 changes it (saves a sector read-modify-write
          // per block when the global scalar is 0)
          const bool out0 = bad || d > R - 1 || d < -(R - 1);
          const uint16_t code0 = out0 ? (uint16_t)0 : (uint16_t)(d + R);
          if (code != code0) {
            a.codes[bstart] = code;
            if (a.patch_list)
              a.patch_list[atomicAdd(a.patch_count, 1u)] =
                  ((unsigned long long)bstart << 16) | (unsigned long long)code;
          }
          if (out) {
            a.scratch[bstart] = a.in[origin];  // verbatim value, read only for outliers
            c[k] += 1;
          }
          s_cnt[tid * SCAN_IPT + k] = c[k];  // final count, stored coalesced below
          s_src[tid * SCAN_IPT + k] = bstart + (out ? 0 : 1);
        } else {
          s_src[tid * SCAN_IPT + k] = bstart + (a.codes[bstart] == 0 ? 0 : 1);
        }
      }
    }
    tsum += c[k];
  }
  // block-wide exclusive scan of the per-thread sums
  int inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  int wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < SCAN_THREADS / 32; ++w) {
    if (w < wid) wbase += (int)s_warp[w];
    agg += (int)s_warp[w];
  }
  const int texcl = wbase + inc - tsum;

  // decoupled look-back (warp 0)
  if (wid == 0) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(a.lb[tile]);
    if (lane == 0) me.store((tile == 0 ? FLAG_P : FLAG_A) | (unsigned long long)agg,
                            cuda::memory_order_relaxed);
    long long excl = 0;
    int64_t pred = tile - 1;
    while (pred >= 0) {
      const int64_t idx = pred - lane;
      unsigned long long w = FLAG_P;
      if (idx >= 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(a.lb[idx]);
        w = r.load(cuda::memory_order_relaxed);
        while ((w >> 62) == 0) w = r.load(cuda::memory_order_relaxed);
      }
      const unsigned pm = __ballot_sync(FULL, (w >> 62) == 2);
      const int stop = pm ? __ffs(pm) - 1 : 31;
      long long val = (lane <= stop) ? (long long)(w & VAL_MASK) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL, val, o);
      excl += val;
      if (pm) break;
      pred -= 32;
    }
    if (lane == 0) {
      if (tile > 0) me.store(FLAG_P | (unsigned long long)(excl + agg), cuda::memory_order_relaxed);
      s_excl = excl;
      if (base + SCAN_CH >= nb) {
        *a.n_out = excl + agg;
        if (a.fix_origin && a.scalars) a.scalars[0] = s0;
        if (a.status) {
          // quantize.py:62-72 precedence: any non-finite value first, then overflow
          const unsigned long long nf = *a.first_nonfinite, ov = *a.first_overflow;
          if (nf != 0x7fffffffffffffffull) {
            *a.status = 1;  // VLZ_ST_NONFINITE
            *a.index = (long long)nf;
          } else if (ov != 0x7fffffffffffffffull) {
            *a.status = 2;  // VLZ_ST_OVERFLOW
            *a.index = (long long)ov;
          }
        }
      }
    }
  }
  __syncthreads();
  const long long cexcl = s_excl;

  // per-block offsets (decompress) or outlier gather (compress): each thread
  // copies the outliers of its own blocks -- all copies of the chunk are in
  // flight at once -- and blocks with >= 32 outliers are copied by the whole
  // warp, coalesced
  int run = texcl;  // chunk-local offset
  unsigned heavy = 0;
  int hdst[SCAN_IPT];
  float* const outc = a.out + cexcl;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    hdst[k] = run;
    if (!a.gather) {
      s_cnt[tid * SCAN_IPT + k] = cexcl + run;  // offset, stored coalesced below
    } else if (c[k] > 0 && c[k] < 32) {
      const float* src = a.scratch + s_src[tid * SCAN_IPT + k];
      for (int t = 0; t < c[k]; ++t) outc[run + t] = src[t];
    } else if (c[k] >= 32) {
      heavy |= 1u << k;
    }
    run += c[k];
  }
  if (!a.gather || a.fix_origin) {  // offsets, or the fixed counts, go out coalesced
    __syncthreads();
    int64_t* dst = a.gather ? a.counts : a.offsets;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      const int64_t bi = base + (int64_t)k * SCAN_THREADS + tid;
      if (bi < nb) dst[bi] = s_cnt[k * SCAN_THREADS + tid];
    }
  }
  if (!a.gather) return;
  unsigned hm = __ballot_sync(FULL, heavy != 0);
  while (hm) {
    const int src_lane = __ffs(hm) - 1;
    hm &= hm - 1;
    const unsigned mk = __shfl_sync(FULL, heavy, src_lane);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      if (!((mk >> k) & 1u)) continue;  // warp-uniform
      const int n = __shfl_sync(FULL, c[k], src_lane);
      const int dst = __shfl_sync(FULL, hdst[k], src_lane);
      const float* src = a.scratch + s_src[(tid - lane + src_lane) * SCAN_IPT + k];
      for (int t0 = 0; t0 < n; t0 += 128) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = t0 + lane + 32 * j;
          if (t < n) v[j] = __ldg(src + t);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = t0 + lane + 32 * j;
          if (t < n) outc[dst + t] = v[j];
        }
      }
    }
  }
}

}  // namespace vlz
