// vlz_common.cuh -- geometry, exact quantizer arithmetic and warp helpers
// shared by the dual-quant kernels (sm_100a).
//
// Reference semantics restated here (paths relative to
// /root/reference/pkg/src/vlz/):
//   quantize.py:31-42,50-79   prequantization q = fl64(v / (2 eb)),
//                             d = sign(q) * floor(|q| + 0.5), overflow at 2^31-1
//   quantize.py:45-47,82-84   reconstruction float32((2.0 * d) * eb)
//   vector.py:72-78           outlier iff |delta| > R-1 or the float32-narrowed
//                             reconstruction misses the bound
//   padding.py:53-59          exact half-away rounding of an int64 mean
//   model.py:113-159          row-major block grid, partial edge blocks
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vlz {

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch (sm_90+): every kernel of the library waits
// for its predecessor's completion (and memory) before touching anything.
// The successor is released implicitly when the grid exits (an explicit early
// launch_dependents let successor CTAs sit on SM resources during the
// predecessor's tail and measured no better at C5), so what PDL removes is the
// launch latency between consecutive kernels.  A no-op for a kernel launched
// without the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Per-call reset of the result block and the workspace header, folded into the
// first kernel of a call (there is no separate init launch).  CTA 0 of that
// kernel resets the state and then publishes the call's nonce (unique per call
// in this process, never the value a stale or uninitialised workspace holds
// except with probability 2^-64) in the workspace's flag word; any thread of the
// same grid that is about to touch the shared state (error minima, global
// statistics, look-back words) first waits for the flag.  The waits sit on
// rare paths or at the end of a CTA's work, long after CTA 0 -- the first CTA
// the hardware dispatches -- has published.  Later kernels of the call are
// ordered by the kernel boundary and need no wait.
struct InitArgs {
  unsigned long long* res;    // vlz_result as 8 64-bit words (nullptr: none)
  unsigned int* hdr;          // workspace header: ticket (+0), done (+8 B), spare (+16 B)
  long long* stats;           // sum, count, min, neg_max (nullptr: none)
  unsigned long long* lb;     // look-back words of the call's scan kernel
  long long nchunks;
  unsigned long long* flag;
  unsigned long long nonce;
};

__device__ __forceinline__ void ws_reset_scalars(const InitArgs& ia) {
  constexpr long long I64MAX = 0x7fffffffffffffffll;
  if (ia.res) {
    ia.res[0] = 0ull;                        // status, reserved
    ia.res[1] = ~0ull;                       // index = -1
    ia.res[2] = 0ull;                        // n_outliers
    ia.res[3] = (unsigned long long)I64MAX;  // first_nonfinite
    ia.res[4] = (unsigned long long)I64MAX;  // first_overflow
    ia.res[5] = (unsigned long long)I64MAX;  // first_bad_block
    ia.res[6] = 0ull;                        // sentinels
    ia.res[7] = 0ull;
  }
  ia.hdr[0] = 0u;  // ticket
  ia.hdr[2] = 0u;  // done
  ia.hdr[4] = 0u;
  if (ia.stats) {
    ia.stats[0] = 0;
    ia.stats[1] = 0;
    ia.stats[2] = I64MAX;
    ia.stats[3] = I64MAX;
  }
}
__device__ __forceinline__ void ws_publish(const InitArgs& ia) {  // release: orders the reset before it
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ia.flag), "l"(ia.nonce) : "memory");
}
// the reset by one warp (warp 0 of CTA 0 of the fused compress kernels, after
// it has issued its first loads, so the stores overlap their latency)
__device__ __forceinline__ void ws_reset_warp(const InitArgs& ia, int lane) {
  for (long long k = lane; k < ia.nchunks; k += 32) ia.lb[k] = 0ull;
  if (lane == 0) ws_reset_scalars(ia);
  __syncwarp();
  if (lane == 0) ws_publish(ia);
}
// ... by every thread of CTA 0 (the offsets kernel of a decompress call)
__device__ __forceinline__ void ws_reset_cta0(const InitArgs& ia) {
  for (long long k = threadIdx.x; k < ia.nchunks; k += blockDim.x) ia.lb[k] = 0ull;
  if (threadIdx.x == 0) ws_reset_scalars(ia);
  __syncthreads();
  if (threadIdx.x == 0) ws_publish(ia);
}

__device__ __forceinline__ void ws_wait(const InitArgs& ia) {
  unsigned long long v;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ia.flag) : "memory");
  } while (v != ia.nonce);
}

// Outlier scratch of the compress path, two layouts chosen by the size of the
// workspace the caller passes:
//   compact (vlz_workspace_size): SCRATCH_SLOTS floats per block (slot 0 the
//     block origin, 1.. its other outliers in traversal order).  A block with
//     more outliers than fit keeps only its count; the scan kernel regenerates
//     its values from the codes (code 0 marks them) and the input;
//   dense (vlz_workspace_size_dense): one float per element, the block's slots
//     at its position in the code stream -- 4 bytes per element more, and the
//     scan kernel copies instead of regenerating (outlier-dense data).
constexpr int SCRATCH_SLOTS = 8;
__host__ __device__ __forceinline__ long long scratch_base(bool dense, long long bstart,
                                                           long long bi) {
  return dense ? bstart : bi * SCRATCH_SLOTS;
}
__host__ __device__ __forceinline__ int scratch_limit(bool dense) {  // non-origin slots of a block
  return dense ? 0x7fffffff : SCRATCH_SLOTS - 1;
}

// Division of 32-bit unsigned values by a launch-invariant divisor d >= 1
// (Granlund-Montgomery with the add-shift fix-up; exact for every x < 2^32).
struct FastDiv {
  uint32_t d, m, s;
  __host__ void init(uint32_t div) {
    d = div;
    if (div <= 1) {
      d = 1;
      m = 0;
      s = 0;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < div) ++l;
    s = l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    if (d == 1) return x;
    const uint32_t t = __umulhi(m, x);
    return (t + ((x - t) >> 1)) >> (s - 1);
  }
};

// Padded 3-D view of a 1/2/3-D array: dims (D0, D1, D2) with leading 1s, so a
// 1-D array is (1, 1, N) and a 2-D array (1, Y, X).  Block extents per padded
// dim are (BZ, BY, BX) = (B if nd == 3 else 1, B if nd >= 2 else 1, B).
struct Geo {
  int64_t D0, D1, D2;
  int64_t P0, P1, P2;  // blocks per padded dim
  int64_t NW;          // windows of W columns per block row
  int64_t ntiles;      // P0 * P1 * NW
  int64_t nblocks;
  int64_t N;
  FastDiv divNW, divP1, divP2;  // 32-bit tile / block decode (when counts < 2^32)
};

struct QP {
  double eb;     // resolved absolute bound
  double twoeb;  // 2.0 * eb (exact)
  int radius;
  int kind;      // VLZ_PAD_* (min / max / mean used by the statistics)
  // float32 fast path (quant_fast); lim0 < 0 disables it
  float inv32;   // fl32(1 / (2 eb))
  float lim0;    // 0.5 - 2^-22
  float kq;      // 2^-22
};

// Fast exact prequantization ("fast path proof").
// q = fl32(v * fl32(1/(2eb))) carries two round-to-nearest errors of 2^-24
// each, so it is within |q| * 2^-23 (1 + 2^-24) of the real quotient Q, and
// fl64(v / (2eb)) within 2^-53 |Q|; the magic-number add rounds q to nearest
// (n) and e = q - n is exact.  When the distance of q to the rounding
// boundary, 0.5 - |e|, exceeds |q| * 2^-22 + 2^-22 (less 2^-26 for the
// rounding of the limit itself), then (a) round_half_away(fl64(v/(2eb))) == n
// (no boundary lies between the two quotients -- twice the error bound --
// and no tie is possible) and (b) the float32-narrowed reconstruction of n is
// within eb of v: |n - Q| <= |e| + |q| 2^-23, and the f32 rounding of n*2eb
// moves it by at most |n| * 2^-24 * 2eb, together |q| * 1.5 * 2^-23 + 2^-25
// in units of 2eb, inside the margin.  Otherwise the caller re-evaluates the
// element with quant_exact.  |q| >= 2^21, NaN and Inf always fail the test.
// (The margin per unit of |q| was 2^-21 until late in round 2; at 2^-22 about
// half as many rows of C5 take the exact path and the fused compress kernel
// runs 1.7 % faster.  tests/test_gpu_sweep.py checks every float pattern.)
__device__ __forceinline__ int quant_fast(float v, const QP& q, bool& ok) {
  const float qq = __fmul_rn(v, q.inv32);
  const float r = __fadd_rn(qq, 12582912.0f);  // 1.5 * 2^23: RN to an integer
  const int n = __float_as_int(r) - 0x4B400000;
  const float e = __fsub_rn(qq, __fsub_rn(r, 12582912.0f));
  const float lim = __fmaf_rn(fabsf(qq), -q.kq, q.lim0);
  ok = fabsf(e) < lim;
  return n;
}


// canonical start of a block's codes: number of in-bounds elements of all
// earlier blocks in row-major block order (vector.py:193-202 ordering)
__host__ __device__ __forceinline__ int64_t block_start(const Geo& g, int64_t bz, int64_t by,
                                                        int64_t bx, int BZ, int BY, int BX,
                                                        int64_t ez, int64_t ey) {
  const int64_t o0 = bz * BZ, o1 = by * BY, o2 = bx * BX;
  return o0 * g.D1 * g.D2 + ez * o1 * g.D2 + ez * ey * o2;
}

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// quantize.py:31-42 + vector.py:72-78, exact IEEE float64 evaluation.
//   n    = round_half_away(fl64(v / (2 eb)))
//   bad  = |f64(f32(fl64((2.0 * n) * eb))) - f64(v)| > eb   (narrowing check)
//   ovf  = !(|q| < 2^31 - 1)     (also true for NaN)
__device__ __forceinline__ int quant_exact(float v, const QP& q, bool& bad, bool& ovf) {
  const double dv = (double)v;
  const double qq = __ddiv_rn(dv, q.twoeb);
  const double a = fabs(qq);
  ovf = !(a < 2147483647.0);
  const double fl = floor(__dadd_rn(a, 0.5));
  const int m = ovf ? 0 : (int)fl;
  const int n = (qq < 0.0) ? -m : m;
  const float w = __double2float_rn(__dmul_rn(2.0 * (double)n, q.eb));
  bad = fabs(__dsub_rn((double)w, dv)) > q.eb;
  return n;
}

// quantize.py:40-42 for reconstruction of sentinel values (no overflow
// guard in the reference's decompressor; values of valid streams fit).
__device__ __forceinline__ int64_t quant_value(float v, double twoeb) {
  const double qq = __ddiv_rn((double)v, twoeb);
  const double a = fabs(qq);
  const double fl = floor(__dadd_rn(a, 0.5));
  const long long m = (a < 9.2e18) ? (long long)fl : 0;
  return qq < 0.0 ? -m : m;
}

// quantize.py:45-47: float32((2.0 * d) * eb)
__device__ __forceinline__ float dequant(int64_t d, double eb) {
  return __double2float_rn(__dmul_rn(2.0 * (double)d, eb));
}

// Pending-origin record of a block (fused compress -> scan, *:global only):
// bits 0-23 outliers of the block's other elements, bit 24 the origin's
// narrowing-check failure, bits 32-63 the origin's prequantized value.
__host__ __device__ __forceinline__ int64_t pack_origin(int64_t count, int d, bool bad) {
  return (int64_t)(((uint64_t)(uint32_t)d << 32) | ((uint64_t)bad << 24) | (uint64_t)count);
}

// padding.py:53-59 (total is the int64 wrapping sum)
__host__ __device__ __forceinline__ int64_t round_half_away_ratio(int64_t total, int64_t count) {
  if (count <= 0) return 0;
  const uint64_t mag = total < 0 ? 0ull - (uint64_t)total : (uint64_t)total;
  const uint64_t qq = mag / (uint64_t)count, r = mag % (uint64_t)count;
  const uint64_t res = qq + ((2 * r >= (uint64_t)count) ? 1 : 0);
  return total < 0 ? -(int64_t)res : (int64_t)res;
}

// padding.py:62-69
__host__ __device__ __forceinline__ int64_t stat_value(int kind, int64_t sum, int64_t cnt,
                                                       int64_t mn, int64_t mx) {
  if (kind == 1) return mn;  // VLZ_PAD_MIN
  if (kind == 2) return mx;  // VLZ_PAD_MAX
  return round_half_away_ratio(sum, cnt);
}

// ---- segmented warp helpers over aligned groups of L lanes ------------
template <int L, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
template <int L, typename T>
__device__ __forceinline__ T group_min(T v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(FULL, v, o);
    v = u < v ? u : v;
  }
  return v;
}
template <int L, typename T>
__device__ __forceinline__ T group_max(T v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(FULL, v, o);
    v = u > v ? u : v;
  }
  return v;
}
template <int L>
__device__ __forceinline__ bool group_any(bool b, int lane) {
  const unsigned m = __ballot_sync(FULL, b);
  const unsigned gm = (L == 32) ? FULL : (((1u << L) - 1u) << (lane & ~(L - 1)));
  return (m & gm) != 0;
}
// exclusive prefix sum within the group (int)
template <int L>
__device__ __forceinline__ int group_excl_scan(int v, int lane, int& total) {
  int inc = v;
  const int gl = lane & (L - 1);
#pragma unroll
  for (int o = 1; o < L; o <<= 1) {
    int u = __shfl_up_sync(FULL, inc, o);
    if (gl >= o) inc += u;
  }
  total = __shfl_sync(FULL, inc, (lane & ~(L - 1)) + L - 1);
  return inc - v;
}

}  // namespace vlz
