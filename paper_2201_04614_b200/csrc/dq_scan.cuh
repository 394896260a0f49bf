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

#ifndef VLZ_SCAN_LANE_STEP
#define VLZ_SCAN_LANE_STEP 32  // codes a lane reads per regeneration step
#endif
#ifndef VLZ_SCAN_LANE_BATCH
#define VLZ_SCAN_LANE_BATCH 8  // input loads a lane keeps in flight
#endif
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
  const float* origin_vals;  // *:global: verbatim origin value per block (fused kernel)
  uint16_t* codes;
  int64_t* counts;
  float* scratch;
  int scratch_dense;  // 1: one scratch slot per element (vlz_common.cuh)
  float* out;
  int64_t* offsets;
  int64_t* scalars;
  unsigned long long* lb;  // per chunk look-back words
  unsigned int* ticket;
  unsigned long long* flag;  // compress: the call's reset flag, cleared at the end
  InitArgs init;             // decompress: reset done by CTA 0 of the offsets kernel
  long long* n_out;
  const long long* gstats;  // sum, count, min, neg_max per record (nstats records:
  int nstats;               // one reduced record, or one per rank when sharded)
  // compress status finalisation (done by the chunk holding the last block)
  int* status;
  long long* index;
  const unsigned long long* first_nonfinite;
  const unsigned long long* first_overflow;
  // optional list of rewritten origin codes, (position << 16) | code, for
  // callers that copied the provisional codes out early (host pipeline)
  unsigned long long* patch_list;
  unsigned int* patch_count;
  // floats the compact outlier array holds (vlz_dq_compress_capped); stores
  // past it are dropped and the call ends with VLZ_ST_OUTLIER_CAPACITY
  long long out_cap;
};

// element extents of a block along the padded dims
struct BlockExt {
  int ez, ey, ex;
};
__device__ __forceinline__ BlockExt block_of(const Geo& g, int64_t bi, int BZ, int BY, int BX,
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
  return BlockExt{(int)ez, (int)ey, (int)imin64(BX, g.D2 - bx * BX)};
}

constexpr unsigned long long FLAG_A = 1ull << 62;
constexpr unsigned long long FLAG_P = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

// shared-memory padding: element i of a chunk staged as [k][tid] (coalesced
// global side) and read as [tid][k] (IPT consecutive blocks per thread).
// 8-byte words: one pad word per IPT words (thread rows land on distinct
// bank pairs); 4-byte words: one per 32.
template <int IPT>
__device__ __forceinline__ int pad_l(int i) { return i + i / IPT; }
__device__ __forceinline__ int pad_f(int i) { return i + (i >> 5); }

// publish a chunk's aggregate (thread 0) as soon as it is known
__device__ __forceinline__ void publish_aggregate(unsigned long long* lb, int64_t tile,
                                                  long long agg) {
  if (threadIdx.x == 0) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(lb[tile]);
    me.store((tile == 0 ? FLAG_P : FLAG_A) | (unsigned long long)agg, cuda::memory_order_relaxed);
  }
}

// Decoupled look-back with the whole CTA: every round, thread t inspects
// predecessor tile-1-t (SCAN_THREADS flags per L2 round trip instead of 32;
// the other warps would only wait at the barrier otherwise).  Returns the
// chunk's exclusive prefix in every thread and publishes the inclusive one.
__device__ __forceinline__ long long lookback_cta(unsigned long long* lb, int64_t tile,
                                                  long long agg, int* s_first,
                                                  long long* s_wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = SCAN_THREADS / 32;
  long long excl = 0;
  int64_t pred = tile - 1;
  while (pred >= 0) {  // uniform across the CTA
    const int64_t idx = pred - tid;
    unsigned long long w = FLAG_P;  // before chunk 0: an inclusive prefix of 0
    if (idx >= 0) {
      cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> r(lb[idx]);
      w = r.load(cuda::memory_order_relaxed);
      while ((w >> 62) == 0) w = r.load(cuda::memory_order_relaxed);
    }
    const unsigned pm = __ballot_sync(FULL, (w >> 62) == 2);
    if (lane == 0) s_first[wid] = pm ? wid * 32 + __ffs(pm) - 1 : SCAN_THREADS;
    __syncthreads();
    int stop = SCAN_THREADS;
#pragma unroll
    for (int k = 0; k < NW; ++k) stop = min(stop, s_first[k]);
    long long val = (tid <= stop) ? (long long)(w & VAL_MASK) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL, val, o);
    if (lane == 0) s_wsum[wid] = val;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NW; ++k) excl += s_wsum[k];
    __syncthreads();  // s_first / s_wsum are rewritten by the next round
    if (stop < SCAN_THREADS) break;
    pred -= SCAN_THREADS;
  }
  if (tid == 0 && tile > 0) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(lb[tile]);
    me.store(FLAG_P | (unsigned long long)(excl + agg), cuda::memory_order_relaxed);
  }
  return excl;
}

// block-wide exclusive scan of one value per thread; also returns the total
template <typename T>
__device__ __forceinline__ T cta_excl_scan(T v, T* s_warp, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  T wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < SCAN_THREADS / 32; ++w) {
    if (w < wid) wbase += s_warp[w];
    agg += s_warp[w];
  }
  total = agg;
  return wbase + inc - v;
}

// The outliers of NB blocks from position p0 on, in canonical (code) order,
// written to outp[u] by one warp: per block 512 codes per step (16 per lane,
// loaded together), ranks by a byte-packed warp scan of the four 128-code
// groups' zero counts, then the input values at the zero codes' coordinates.
// The NB blocks go through each phase together, so their loads overlap (one
// block at a time left ~3 dependent round trips per block exposed).
template <int NB>
__device__ __forceinline__ void regen_blocks(const ScanArgs& a, const int64_t (&bi)[NB], int nvalid,
                                             int p0, float* const (&outp)[NB],
                                             const int (&olim)[NB], int lane) {
  int64_t origin[NB];
  const uint16_t* cp[NB];
  int nelem[NB], exy[NB], ex[NB], ey[NB], done[NB];
  int nmax = 0;
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    int64_t bstart = 0;
    origin[u] = 0;
    BlockExt e{0, 0, 1};
    if (u < nvalid) e = block_of(a.g, bi[u], a.BZ, a.BY, a.BX, bstart, origin[u]);
    nelem[u] = e.ez * e.ey * e.ex;
    ex[u] = e.ex;
    ey[u] = e.ey > 0 ? e.ey : 1;
    exy[u] = ex[u] * ey[u];
    cp[u] = a.codes + bstart;
    done[u] = 0;
    nmax = nelem[u] > nmax ? nelem[u] : nmax;
  }
  const float* __restrict__ in = a.in;
  for (int i0 = 0; i0 < nmax; i0 += 512) {
    unsigned zm[NB], excl[NB], tot[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      zm[u] = 0;  // bit g*4+j: code (i0 + g*128 + lane*4 + j) is an outlier
#pragma unroll
      for (int g = 0; g < 4; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + g * 128 + lane * 4 + j;
          const unsigned cv = (i >= p0 && i < nelem[u]) ? (unsigned)cp[u][i] : 1u;
          zm[u] |= (cv == 0u) ? (1u << (g * 4 + j)) : 0u;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      // per-group counts packed in bytes (<= 128 each over the warp)
      unsigned cnt = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) cnt |= (unsigned)__popc((zm[u] >> (g * 4)) & 15u) << (8 * g);
      unsigned inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
      }
      tot[u] = __shfl_sync(FULL, inc, 31);
      excl[u] = inc - cnt;
    }
    // all of the step's input loads first (independent), then the stores.
    // A lane's 4 codes of a group are consecutive: their coordinates advance
    // from the first one's (one division pair per group, not per element)
    float val[NB][16];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int ig = i0 + g * 128 + lane * 4;
        const int z0 = ig / exy[u], r0 = ig - z0 * exy[u], y0 = r0 / ex[u];
        int z = z0, y = y0, x = r0 - y0 * ex[u];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          val[u][g * 4 + j] = 0.f;
          if ((zm[u] >> (g * 4 + j)) & 1u)
            val[u][g * 4 + j] = __ldg(in + origin[u] + ((int64_t)z * a.g.D1 + y) * a.g.D2 + x);
          if (++x == ex[u]) {
            x = 0;
            if (++y == ey[u]) {
              y = 0;
              ++z;
            }
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      int gbase = done[u];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        int r = gbase + (int)((excl[u] >> (8 * g)) & 255u);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if ((zm[u] >> (g * 4 + j)) & 1u) {
            if (r < olim[u]) outp[u][r] = val[u][g * 4 + j];
            ++r;
          }
        gbase += (int)((tot[u] >> (8 * g)) & 255u);
      }
      done[u] = gbase;
    }
  }
}

// The same regeneration by ONE thread for its own block: when most lanes of a
// warp own dense blocks (an outlier-heavy field), 32 blocks advance together,
// each lane walking its block 32 codes at a time, instead of one block per
// warp pass (32 passes of ~3 dependent round trips each).
__device__ __forceinline__ void regen_lane(const ScanArgs& a, int64_t bi, int p0, float* outp,
                                           int olim) {
  int64_t bstart, origin;
  const BlockExt e = block_of(a.g, bi, a.BZ, a.BY, a.BX, bstart, origin);
  const int nelem = e.ez * e.ey * e.ex;
  const uint16_t* __restrict__ cp = a.codes + bstart;
  const float* __restrict__ in = a.in;
  const bool al = ((bstart & 7) == 0) && ((reinterpret_cast<uintptr_t>(a.codes) & 15) == 0);  // 16-byte aligned code vectors
  constexpr int STEP = VLZ_SCAN_LANE_STEP;  // codes per step (32 or 64)
  int r = 0, x = 0, y = 0;                  // rank; in-block coordinates of the current position
  const float* pin = in + origin;           // ... and its element of the input
  const int64_t row_skip = a.g.D2 - e.ex, plane_skip = (a.g.D1 - e.ey) * a.g.D2;
  for (int i0 = 0; i0 < nelem; i0 += STEP) {
    unsigned long long zm = 0;  // bit j: code i0 + j is an outlier
    if (al && i0 + STEP <= nelem) {
      uint4 w[STEP / 8];
#pragma unroll
      for (int q = 0; q < STEP / 8; ++q) w[q] = *reinterpret_cast<const uint4*>(cp + i0 + 8 * q);
#pragma unroll
      for (int q = 0; q < STEP / 8; ++q) {
        const unsigned ws[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          zm |= ((ws[t] & 0xffffu) == 0u) ? (1ull << (8 * q + 2 * t)) : 0ull;
          zm |= ((ws[t] >> 16) == 0u) ? (1ull << (8 * q + 2 * t + 1)) : 0ull;
        }
      }
    } else {
#pragma unroll 8
      for (int j = 0; j < STEP; ++j)
        if (i0 + j < nelem && cp[i0 + j] == 0) zm |= 1ull << j;
    }
    if (i0 == 0 && p0) zm &= ~1ull;  // the origin is settled from its record
    // the step's input loads together (VB at a time), then their stores
    constexpr int VB = VLZ_SCAN_LANE_BATCH;
    unsigned long long m = zm;
    int cur = 0;  // codes of this step the coordinates have advanced over
    while (m) {
      float val[VB];
      int n = 0;
#pragma unroll
      for (int u = 0; u < VB; ++u) {
        val[u] = 0.f;
        if (m) {
          const int j = __ffsll((long long)m) - 1;
          m &= m - 1;
          x += j - cur;  // advance by j - cur positions
          pin += j - cur;
          cur = j;
          while (x >= e.ex) {
            x -= e.ex;
            pin += row_skip;
            if (++y == e.ey) {
              y = 0;
              pin += plane_skip;
            }
          }
          val[u] = __ldg(pin);
          n = u + 1;
        }
      }
#pragma unroll
      for (int u = 0; u < VB; ++u)
        if (u < n) {
          if (r < olim) outp[r] = val[u];
          ++r;
        }
    }
    // to the first position of the next step
    x += STEP - cur;
    pin += STEP - cur;
    while (x >= e.ex) {
      x -= e.ex;
      pin += row_skip;
      if (++y == e.ey) {
        y = 0;
        pin += plane_skip;
      }
    }
  }
}

// Compress: origin fix-up (*:global), count scan and outlier gather.  Thread t
// owns blocks t*IPT .. t*IPT+IPT-1 of its chunk.  Order of work:
//  1. counts from the records (shared memory) -> chunk scan -> the aggregate
//     is published at once (successors' look-backs need nothing else);
//  2. the scattered work that does not depend on the chunk's offset -- origin
//     code rewrites, slot-0 probes, the first scratch outlier of every block --
//     is issued, so its latency overlaps the look-back;
//  3. CTA-wide look-back, then the compact stores.
// Under *:global the origin's verbatim value comes from the fused kernel's
// per-block side array (read coalesced) and goes straight into the compact
// array; the other outliers come from the block's scratch slots 1.. (0.. when
// a non-global origin sits in slot 0).
#ifndef VLZ_SCAN_HEAVY
#define VLZ_SCAN_HEAVY 8
#endif
#ifndef VLZ_SCAN_HB
#define VLZ_SCAN_HB 1  // heavy blocks regenerated together by a warp (2: 193 us, 4: 358 us on the
                       // outlier-stress field against 155 us -- the register arrays spill)
#endif
#ifndef VLZ_SCAN_LANE_REGEN
#define VLZ_SCAN_LANE_REGEN 8  // lanes of a warp with dense blocks from which each regenerates its own
#endif
#ifndef VLZ_SCAN_MINB
#define VLZ_SCAN_MINB 3
#endif
template <int SCAN_IPT>
__global__ void __launch_bounds__(SCAN_THREADS, VLZ_SCAN_MINB) dq_scan_kernel(ScanArgs a) {
  pdl_enter();
  constexpr int SCAN_CH = SCAN_THREADS * SCAN_IPT;
  // blocks with >= HEAVY outliers besides a register-held origin: copied by
  // whole warps (dense scratch) or regenerated (compact scratch, whose slots
  // hold at most SCRATCH_SLOTS - 1 of them)
  constexpr int HEAVY = VLZ_SCAN_HEAVY;
  static_assert(HEAVY >= 2 && HEAVY <= SCRATCH_SLOTS, "light blocks must fit the compact scratch slots");
  // padded so that both the coalesced ([k][tid]) and the per-thread
  // ([tid][k]) access patterns are (nearly) bank-conflict free
  __shared__ long long s_rec[SCAN_CH + SCAN_THREADS];  // count records in, final counts out
  __shared__ float s_vo[SCAN_CH + SCAN_CH / 32];       // *:global: origin values
  __shared__ int s_warp[SCAN_THREADS / 32];
  __shared__ int s_first[SCAN_THREADS / 32];
  __shared__ long long s_wsum[SCAN_THREADS / 32];
  __shared__ unsigned int s_tile;

  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SCAN_CH;
  const int64_t nb = a.g.nblocks;
  const float* __restrict__ scratch = a.scratch;
  const bool fix = a.fix_origin != 0;

  int64_t s0 = 0;
  if (fix) {
    // the records of all ranks (or the single reduced one) reduced here, as
    // np.sum / min / max over the whole field (padding.py:62-69): the sum
    // wraps in int64 like the reference's
    const long long* gs = a.gstats;
    unsigned long long sum = (unsigned long long)gs[0];
    long long cnt = gs[1], mn = gs[2], nmx = gs[3];
    for (int r = 1; r < a.nstats; ++r) {
      sum += (unsigned long long)gs[4 * r];
      cnt += gs[4 * r + 1];
      mn = gs[4 * r + 2] < mn ? gs[4 * r + 2] : mn;
      nmx = gs[4 * r + 3] < nmx ? gs[4 * r + 3] : nmx;
    }
    s0 = stat_value(a.q.kind, (long long)sum, cnt, mn, -nmx);
  }

#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t bi = base + (int64_t)k * SCAN_THREADS + tid;
    s_rec[pad_l<SCAN_IPT>(k * SCAN_THREADS + tid)] = bi < nb ? a.counts[bi] : 0;
    if (fix) s_vo[pad_f(k * SCAN_THREADS + tid)] = bi < nb ? a.origin_vals[bi] : 0.f;
  }
  __syncthreads();

  // 1. counts (and, under *:global, the origin verdicts) from the records
  int c[SCAN_IPT];
  unsigned omask = 0;  // *:global: origin is an outlier
  unsigned wmask = 0;  // *:global: origin code must be rewritten
  uint16_t ocode[SCAN_IPT];
  float vo[SCAN_IPT];
  int tsum = 0;
  const int R = a.q.radius;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t bi = base + (int64_t)tid * SCAN_IPT + k;
    const long long rec = s_rec[pad_l<SCAN_IPT>(tid * SCAN_IPT + k)];
    c[k] = 0;
    ocode[k] = 0;
    vo[k] = 0.f;
    if (bi < nb) {
      if (fix) {
        // pending-origin record written by the fused kernel (pack_origin)
        const int d = (int)(rec >> 32);
        const bool bad = (rec >> 24) & 1;
        const int64_t delta = (int64_t)d - s0;
        const bool out = bad || delta > (int64_t)(R - 1) || delta < -(int64_t)(R - 1);
        ocode[k] = out ? (uint16_t)0 : (uint16_t)(delta + R);
        // the fused kernel already stored the s0 = 0 code of the origin;
        // rewrite only when s0 changes it
        const bool out0 = bad || d > R - 1 || d < -(R - 1);
        const uint16_t c0 = out0 ? (uint16_t)0 : (uint16_t)(d + R);
        if (ocode[k] != c0) wmask |= 1u << k;
        if (out) {
          omask |= 1u << k;
          vo[k] = s_vo[pad_f(tid * SCAN_IPT + k)];
        }
        c[k] = (int)(rec & 0xffffff) + (out ? 1 : 0);
        s_rec[pad_l<SCAN_IPT>(tid * SCAN_IPT + k)] = c[k];  // final count (ordered by the scan's barrier)
      } else {
        c[k] = (int)rec;
      }
    }
    tsum += c[k];
  }
  int agg;
  const int texcl = cta_excl_scan<int>(tsum, s_warp, agg);
  publish_aggregate(a.lb, tile, agg);
  if (fix) {
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      const int64_t bi = base + (int64_t)k * SCAN_THREADS + tid;
      if (bi < nb) a.counts[bi] = s_rec[pad_l<SCAN_IPT>(k * SCAN_THREADS + tid)];
    }
  }

  // 2. scattered work that does not need the chunk offset
  int64_t src[SCAN_IPT];  // first scratch slot of the block's remaining outliers
  int rem[SCAN_IPT];      // outliers left after the (register) origin
  float v0[SCAN_IPT];     // first of them, prefetched
  unsigned heavy = 0;
  int tmax = 0;
  if (fix) {
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      const int64_t bi = base + (int64_t)tid * SCAN_IPT + k;
      rem[k] = c[k] - (int)((omask >> k) & 1u);
      src[k] = 0;
      if (((wmask >> k) & 1u) || rem[k] > 0) {
        int64_t bstart = 0, origin;
        if (a.scratch_dense || ((wmask >> k) & 1u))
          block_of(a.g, bi, a.BZ, a.BY, a.BX, bstart, origin);
        src[k] = scratch_base(a.scratch_dense, bstart, bi) + 1;
        if ((wmask >> k) & 1u) {
          a.codes[bstart] = ocode[k];
          if (a.patch_list)
            a.patch_list[atomicAdd(a.patch_count, 1u)] =
                ((unsigned long long)bstart << 16) | (unsigned long long)ocode[k];
        }
      }
    }
  } else {
    uint16_t code0[SCAN_IPT];
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      const int64_t bi = base + (int64_t)tid * SCAN_IPT + k;
      rem[k] = c[k];
      src[k] = 0;
      code0[k] = 1;
      if (c[k] > 0) {
        int64_t bstart, origin;
        block_of(a.g, bi, a.BZ, a.BY, a.BX, bstart, origin);
        src[k] = scratch_base(a.scratch_dense, bstart, bi);
        code0[k] = a.codes[bstart];  // 0: the origin is an outlier in slot 0
      }
    }
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) src[k] += code0[k] == 0 ? 0 : 1;
  }
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    if (rem[k] >= HEAVY) {
      heavy |= 1u << k;
      rem[k] = 0;
    }
    tmax = max(tmax, rem[k]);
    v0[k] = 0.f;
    if (rem[k] > 0) v0[k] = __ldg(scratch + src[k]);
  }

  // 3. look-back, then the compact stores
  const long long cexcl = lookback_cta(a.lb, tile, agg, s_first, s_wsum);
  if (tid == 0 && base + SCAN_CH >= nb) {
    *a.flag = 0ull;  // a graph replay of this call starts from a cleared flag
    *a.n_out = cexcl + agg;
    if (fix && a.scalars) a.scalars[0] = s0;
    if (a.status) {
      // quantize.py:62-72 precedence: any non-finite value first, then overflow
      const unsigned long long nf = *a.first_nonfinite, ov = *a.first_overflow;
      if (nf != 0x7fffffffffffffffull) {
        *a.status = 1;  // VLZ_ST_NONFINITE
        *a.index = (long long)nf;
      } else if (ov != 0x7fffffffffffffffull) {
        *a.status = 2;  // VLZ_ST_OVERFLOW
        *a.index = (long long)ov;
      } else if (cexcl + agg > a.out_cap) {
        *a.status = 8;  // VLZ_ST_OUTLIER_CAPACITY (n_outliers holds the true count)
        *a.index = -1;
      }
    }
  }
  float* const outc = a.out + cexcl;
  // chunk-relative positions below `lim` fit the caller's outlier array
  const long long lim64 = a.out_cap - cexcl;
  const int lim = lim64 > 0x7fffffffll ? 0x7fffffff : (lim64 < 0 ? 0 : (int)lim64);
  int dst[SCAN_IPT];
  int run = texcl;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int first = (omask >> k) & 1u;
    if (first && run < lim) outc[run] = vo[k];
    dst[k] = run + first;
    if (rem[k] > 0 && dst[k] < lim) outc[dst[k]] = v0[k];
    run += c[k];
  }
  for (int t = 1; t < tmax; ++t) {
    float v[SCAN_IPT];
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k)
      if (t < rem[k]) v[k] = __ldg(scratch + src[k] + t);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k)
      if (t < rem[k] && dst[k] + t < lim) outc[dst[k] + t] = v[k];
  }
  // heavy blocks (>= HEAVY outliers).  Dense scratch: whole-warp copies from
  // the block's slots, four blocks per batch so that their loads overlap.
  // Compact scratch (the slots hold 7 + the origin): a warp, or each lane for
  // its own block when most lanes have one, regenerates the values from the
  // codes (0 marks an outlier) and the input, in canonical order.
  if (a.scratch_dense) {
    constexpr int HB = 4;
    int bn[HB], bd[HB];
    int64_t bs[HB];
    int cnt = 0;
    auto flush = [&]() {
      int nmax = 0;
#pragma unroll
      for (int u = 0; u < HB; ++u) nmax = (u < cnt && bn[u] > nmax) ? bn[u] : nmax;
      for (int t0 = 0; t0 < nmax; t0 += 128) {
        float v[HB][4];
#pragma unroll
        for (int u = 0; u < HB; ++u) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + lane + 32 * j;
            if (u < cnt && t < bn[u]) v[u][j] = __ldg(scratch + bs[u] + t);
          }
        }
#pragma unroll
        for (int u = 0; u < HB; ++u) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + lane + 32 * j;
            if (u < cnt && t < bn[u] && bd[u] + t < lim) outc[bd[u] + t] = v[u][j];
          }
        }
      }
      cnt = 0;
    };
    unsigned hmd = __ballot_sync(FULL, heavy != 0);
    while (hmd) {
      const int src_lane = __ffs(hmd) - 1;
      hmd &= hmd - 1;
      const unsigned mk = __shfl_sync(FULL, heavy, src_lane);
#pragma unroll
      for (int k = 0; k < SCAN_IPT; ++k) {
        if (!((mk >> k) & 1u)) continue;  // warp-uniform
        const int first = __shfl_sync(FULL, (int)((omask >> k) & 1u), src_lane);
        const int n = __shfl_sync(FULL, c[k], src_lane) - first;
        const int d0 = __shfl_sync(FULL, dst[k], src_lane);
        const int64_t sb = __shfl_sync(FULL, src[k], src_lane);
#pragma unroll
        for (int u = 0; u < HB; ++u) {
          if (cnt == u) {
            bn[u] = n;
            bd[u] = d0;
            bs[u] = sb;
          }
        }
        if (++cnt == HB) flush();
      }
    }
    if (cnt) flush();
    return;
  }
  constexpr int NB = VLZ_SCAN_HB;
  int64_t hb[NB];
  float* ho[NB];
  int hl[NB];
  int cnt = 0;
  unsigned hm = __ballot_sync(FULL, heavy != 0);
  if (__popc(hm) >= VLZ_SCAN_LANE_REGEN) {
    // most lanes own dense blocks: every lane regenerates its own
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k)
      if ((heavy >> k) & 1u)
        regen_lane(a, base + (int64_t)tid * SCAN_IPT + k, fix ? 1 : 0, outc + dst[k], lim - dst[k]);
    hm = 0;
  }
  while (hm) {
    const int src_lane = __ffs(hm) - 1;
    hm &= hm - 1;
    const unsigned mk = __shfl_sync(FULL, heavy, src_lane);
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
      if (!((mk >> k) & 1u)) continue;  // warp-uniform
      const int d0 = __shfl_sync(FULL, dst[k], src_lane);
      const int64_t bi = base + (int64_t)(tid - lane + src_lane) * SCAN_IPT + k;
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if (cnt == u) {
          hb[u] = bi;
          ho[u] = outc + d0;
          hl[u] = lim - d0;
        }
      }
      // under *:global the origin (position 0) is settled above, from its record
      if (++cnt == NB) {
        regen_blocks<NB>(a, hb, NB, fix ? 1 : 0, ho, hl, lane);
        cnt = 0;
      }
    }
  }
  if (cnt) regen_blocks<NB>(a, hb, cnt, fix ? 1 : 0, ho, hl, lane);
}

// Decompress: exclusive per-block outlier offsets (counts are the stream's
// int64 values, summed in int64).  Reduce-then-scan inside one kernel: the
// CTA holding ticket t owns a contiguous range of OFF_SPAN blocks (tens of KB
// of counts), sums it with 8 independent coalesced loads per thread in
// flight, publishes the sum for the look-back (one look-back per range, so
// the chain is short), then re-reads the range -- an L2 hit -- and writes the
// offsets, 2048 blocks per sweep staged through shared memory.
constexpr int OFF_IPT = 8;
constexpr int OFF_SWEEP = SCAN_THREADS * OFF_IPT;
// `ranges` = the CTAs of this kernel the device holds at once (occupancy x
// SMs, a few per SM): one range per resident CTA, at least one sweep each, so
// that every CTA of the grid is resident and the blockIdx-ordered look-back
// below never waits on a CTA that has not started
inline int64_t offsets_span(int64_t nblocks, int64_t ranges) {
  if (ranges < 1) ranges = 1;
  int64_t span = (nblocks + ranges - 1) / ranges;
  span = (span + OFF_SWEEP - 1) / OFF_SWEEP * OFF_SWEEP;
  return span < OFF_SWEEP ? OFF_SWEEP : span;
}
inline int64_t offsets_chunks(int64_t nblocks, int64_t ranges) {
  const int64_t span = offsets_span(nblocks, ranges);
  const int64_t n = (nblocks + span - 1) / span;
  return n < 1 ? 1 : n;
}

__global__ void __launch_bounds__(SCAN_THREADS) dq_offsets_kernel(ScanArgs a, int64_t span) {
  pdl_enter();
  __shared__ long long s_val[OFF_SWEEP + SCAN_THREADS];  // padded (pad_l)
  __shared__ long long s_warp[SCAN_THREADS / 32];
  __shared__ int s_first[SCAN_THREADS / 32];
  __shared__ long long s_wsum[SCAN_THREADS / 32];
  const int tid = threadIdx.x;
  // first kernel of a decompress call: CTA 0 resets the result block, the
  // header and the look-back words (no init launch).  Ranges go by blockIdx:
  // the grid is sized to the resident CTA count (offsets_span), so every
  // predecessor of a waiting CTA is running; the look-back words are first
  // touched after the range sum, behind the reset flag.
  if (blockIdx.x == 0) ws_reset_cta0(a.init);
  const int64_t tile = blockIdx.x;
  const int64_t nb = a.g.nblocks;
  const int64_t lo = tile * span;
  const int64_t hi = lo + span < nb ? lo + span : nb;
  const int64_t* __restrict__ counts = a.counts;

  long long part = 0;
#pragma unroll 2
  for (int64_t b0 = lo; b0 < hi; b0 += OFF_SWEEP) {
    long long v[OFF_IPT];
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) {
      const int64_t bi = b0 + (int64_t)k * SCAN_THREADS + tid;
      v[k] = bi < hi ? counts[bi] : 0;
    }
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) part += v[k];
  }
  long long agg;
  if (tid == 0) ws_wait(a.init);  // (ordered before the other threads' look-back reads by the scan's barrier)
  cta_excl_scan<long long>(part, s_warp, agg);
  publish_aggregate(a.lb, tile, agg);
  // first sweep of the second pass in flight during the look-back
  long long nxt[OFF_IPT];
#pragma unroll
  for (int k = 0; k < OFF_IPT; ++k) {
    const int64_t bi = lo + (int64_t)k * SCAN_THREADS + tid;
    nxt[k] = bi < hi ? counts[bi] : 0;
  }
  long long carry = lookback_cta(a.lb, tile, agg, s_first, s_wsum);
  if (tid == 0 && hi >= nb) *a.n_out = carry + agg;
  for (int64_t b0 = lo; b0 < hi; b0 += OFF_SWEEP) {
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) s_val[pad_l<OFF_IPT>(k * SCAN_THREADS + tid)] = nxt[k];
    if (b0 + OFF_SWEEP < hi) {  // next sweep in flight during this one
#pragma unroll
      for (int k = 0; k < OFF_IPT; ++k) {
        const int64_t bi = b0 + OFF_SWEEP + (int64_t)k * SCAN_THREADS + tid;
        nxt[k] = bi < hi ? counts[bi] : 0;
      }
    }
    __syncthreads();
    long long v[OFF_IPT];
    long long tsum = 0;
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) {
      v[k] = s_val[pad_l<OFF_IPT>(tid * OFF_IPT + k)];
      tsum += v[k];
    }
    long long sweep;
    long long run = carry + cta_excl_scan<long long>(tsum, s_warp, sweep);
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) {
      s_val[pad_l<OFF_IPT>(tid * OFF_IPT + k)] = run;
      run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < OFF_IPT; ++k) {
      const int64_t bi = b0 + (int64_t)k * SCAN_THREADS + tid;
      if (bi < hi) a.offsets[bi] = s_val[pad_l<OFF_IPT>(k * SCAN_THREADS + tid)];
    }
    carry += sweep;
    __syncthreads();  // s_val and s_warp are reused by the next sweep
  }
}

}  // namespace vlz
