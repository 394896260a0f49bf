// dq_compress_fast.cuh -- the production fused compress kernel (sm_100a).
//
// Same tile decomposition and output contract as dq_compress.cuh (one warp per
// tile = one block layer x one block row x a window of W = 32*VPL columns),
// specialised for the throughput-critical shapes (3-D b=8/16, 2-D b=8/16):
//
//  * input planes (BY rows x W floats, 4 KB) stream into a per-warp shared-
//    memory ring with TMA bulk copies (cp.async.bulk + mbarrier complete_tx),
//    FAST_STAGES planes ahead of the compute and across tile boundaries; each
//    lane reads its VPL columns of a row with one vector LDS;
//  * prequantization runs the float32 fast path (vlz_common.cuh quant_fast)
//    and re-evaluates only flagged elements with the exact float64 rules;
//  * the Lorenzo stencil runs in int32 (every |d| of the tile < 2^24); a tile
//    holding a larger |d| commits nothing in the streamed pass and is redone in
//    int64 by the same warp after its loop (compress_redo_tail: no redo launch);
//  * interior tiles (whole window inside the row, full block rows) take a
//    branch-free specialisation with constant code strides;
//  * tile ids are decoded with 32-bit magic division, ring slots advance
//    incrementally -- per-plane overhead is a handful of instructions.
// Origin deferral, padding statistics, outlier slots and error minima are
// identical to dq_compress.cuh.
#pragma once

#include <cuda.h>

#include "dq_compress.cuh"
#include "tma.cuh"

namespace vlz {

constexpr int FAST_STAGES = 2;
#ifndef VLZ_BIG_BATCH_C
#define VLZ_BIG_BATCH_C 1  // 3-D b >= 32 compress: interior stage rows in batches
#endif                     // (512^3 b=64 564 -> 318 us, b=32 193 -> 148 us; 2-D slower: off)
#ifndef VLZ_BATCH_ROWS
#define VLZ_BATCH_ROWS 8  // rows per batch (divides the 8-row stage; 4: b=64 337 us)
#endif
constexpr int FAST_WARPS = 4;

// per-lane vector moves of VPL (2, 4, 8) consecutive 32-bit values
template <typename T>
__device__ __forceinline__ T from_bits(int x) {
  if constexpr (sizeof(T) == 4 && T(0.5f) != T(0)) return __int_as_float(x);  // float
  else return (T)x;
}
template <int N, typename T>
__device__ __forceinline__ void ld_vec(const T* p, T (&v)[N]) {
  static_assert(sizeof(T) == 4, "32-bit lanes");
  int t[N];
  if constexpr (N == 8) {
    const int4 a = *reinterpret_cast<const int4*>(p), b = *reinterpret_cast<const int4*>(p + 4);
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
    t[4 % N] = b.x; t[5 % N] = b.y; t[6 % N] = b.z; t[7 % N] = b.w;
  } else if constexpr (N == 4) {
    const int4 a = *reinterpret_cast<const int4*>(p);
    t[0] = a.x; t[1] = a.y; t[2 % N] = a.z; t[3 % N] = a.w;
  } else {
    const int2 a = *reinterpret_cast<const int2*>(p);
    t[0] = a.x; t[1] = a.y;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = from_bits<T>(t[j]);
}
template <int N>
__device__ __forceinline__ void st_vec(int* p, const int (&v)[N]) {
  if constexpr (N == 8) {
    *reinterpret_cast<int4*>(p) = make_int4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<int4*>(p + 4) = make_int4(v[4], v[5], v[6], v[7]);
  } else if constexpr (N == 4) {
    *reinterpret_cast<int4*>(p) = make_int4(v[0], v[1], v[2], v[3]);
  } else {
    *reinterpret_cast<int2*>(p) = make_int2(v[0], v[1]);
  }
}
// VPL u16 codes (low halves of c, plus `add` per packed pair) with one
// 4/8/16-byte store
template <int N>
__device__ __forceinline__ void st_codes(uint16_t* p, const uint32_t (&c)[N], uint32_t add = 0u) {
  if constexpr (N == 8) {
    *reinterpret_cast<uint4*>(p) =
        make_uint4(__byte_perm(c[0], c[1], 0x5410) + add, __byte_perm(c[2], c[3], 0x5410) + add,
                   __byte_perm(c[4], c[5], 0x5410) + add, __byte_perm(c[6], c[7], 0x5410) + add);
  } else if constexpr (N == 4) {
    *reinterpret_cast<uint2*>(p) =
        make_uint2(__byte_perm(c[0], c[1], 0x5410) + add, __byte_perm(c[2], c[3], 0x5410) + add);
  } else {
    *reinterpret_cast<uint32_t*>(p) = __byte_perm(c[0], c[1], 0x5410) + add;
  }
}

template <int ND, int B, int VPL>
struct FastShape {
  using S = Shape<ND, B, VPL>;
  static constexpr int PLANE_FLOATS = S::BY * S::W;
  static constexpr int PLANE_BYTES = PLANE_FLOATS * 4;
  // a plane streams in SPLIT ring stages of STAGE_ROWS rows each
  static constexpr int SPLIT = S::BY >= 32 ? S::BY / 8 : 1;  // b >= 32: 8-row stages
  static constexpr int STAGE_ROWS = S::BY / SPLIT;
  static constexpr int STAGE_FLOATS = STAGE_ROWS * S::W;
  static constexpr int STAGE_BYTES = STAGE_FLOATS * 4;
  // ring of input planes + the previous plane's Dy Dx d (int32, 3-D only)
  static constexpr int PREV_BYTES = (ND == 3) ? PLANE_BYTES : 0;
  static constexpr int WARP_SMEM = (FAST_STAGES * STAGE_BYTES + PREV_BYTES + 64 + 127) / 128 * 128;
  // CTAs per SM the register budget targets (VPL 8: 24 KB of smem per warp)
  static constexpr int MINB = VPL == 8 ? 2 : 4;
};

template <int ND, int B, int VPL>
__host__ __device__ constexpr int fast_smem_bytes() {
  return FAST_WARPS * FastShape<ND, B, VPL>::WARP_SMEM;
}

struct FastArgs {
  CUtensorMap tmap;  // input viewed as (D2, D1, D0) uint32, box (W, BY, 1)
  CompressArgs c;
};

struct TileXY {
  uint32_t wx, by, bz;
};

__device__ __forceinline__ TileXY decode_tile(const Geo& g, uint32_t tile) {
  TileXY t;
  const uint32_t t2 = g.divNW.div(tile);
  t.wx = tile - t2 * (uint32_t)g.NW;
  t.bz = g.divP1.div(t2);
  t.by = t2 - t.bz * (uint32_t)g.P1;
  return t;
}

// producer side of the per-warp ring: one TMA tensor load per half plane
template <int ND, int B, int VPL>
struct Producer {
  using S = Shape<ND, B, VPL>;
  uint32_t tile;  // current tile (>= ntiles: done)
  int zl, ez, part;
  int x0, y0, z0;
  int stage;

  __device__ __forceinline__ void start(const Geo& g, uint32_t t) {
    tile = t;
    zl = 0;
    part = 0;
    stage = 0;
    setup(g);
  }
  __device__ __forceinline__ void setup(const Geo& g) {
    if (tile >= (uint32_t)g.ntiles) return;
    const TileXY c = decode_tile(g, tile);
    z0 = (int)c.bz * S::BZ;
    y0 = (int)c.by * S::BY;
    x0 = (int)c.wx * S::W;
    ez = (int)imin64(S::BZ, g.D0 - z0);
  }
  // issue the current plane into `stage`, then advance (all lanes call)
  __device__ __forceinline__ void issue(const Geo& g, const CUtensorMap* tmap, float* ring,
                                        uint64_t* bars, int lane, uint32_t nwarps) {
    using F = FastShape<ND, B, VPL>;
    if (tile >= (uint32_t)g.ntiles) return;
    if (lane == 0) {
      uint64_t* bar = &bars[stage];
      mbar_arrive_expect_tx(bar, (uint32_t)F::STAGE_BYTES);
      tma_load_3d(ring + stage * F::STAGE_FLOATS, tmap, x0, y0 + part * F::STAGE_ROWS, z0 + zl,
                  bar);
    }
    if (++stage == FAST_STAGES) stage = 0;
    if (++part < F::SPLIT) return;
    part = 0;
    if (++zl >= ez) {
      zl = 0;
      tile += nwarps;
      setup(g);
    }
  }
};

template <int ND, int B, int VPL, int NST = FAST_STAGES>
struct Consumer {
  int stage;
  uint32_t parity;
  __device__ __forceinline__ void advance() {
    if (++stage == NST) {
      stage = 0;
      parity ^= 1u;
    }
  }
};


// statistic accumulator for a compile-time padding kind K (1 min, 2 max, 3 mean)
template <int K>
struct KAcc {
  long long sum = 0;
  int mn = 0x7fffffff, mx = (int)0x80000000;
  __device__ __forceinline__ void add(int v) {
    if (K == 3) sum += v;
    if (K == 1) mn = v < mn ? v : mn;
    if (K == 2) mx = v > mx ? v : mx;
  }
  __device__ __forceinline__ void merge(const KAcc& o) {
    sum += o.sum;
    mn = o.mn < mn ? o.mn : mn;
    mx = o.mx > mx ? o.mx : mx;
  }
};

// One tile.  INTERIOR: x window fully inside the array and ey == BY, so all
// lanes hold VPL in-bounds columns of full-width blocks.  K = padding kind
// for the statistics (compile time; ignored for MODE_ZERO).
template <int ND, int B, int VPL, int MODE, int K, bool INTERIOR>
__device__ __forceinline__ void fast_tile(const FastArgs& fa, uint32_t tile, const TileXY& tc,
                                          int lane, float* ring, uint64_t* bars,
                                          Producer<ND, B, VPL>& prod, Consumer<ND, B, VPL>& cons,
                                          uint32_t nwarps, KAcc<K>& gacc, long long& gcnt,
                                          uint32_t* nfail_s) {
  using S = Shape<ND, B, VPL>;
  using F = FastShape<ND, B, VPL>;
  constexpr int BZ = S::BZ, BY = S::BY, BX = S::BX, W = S::W, LPB = S::LPB;
  constexpr unsigned MAGIC_BITS = 0x4B400000u;  // bit pattern of 1.5 * 2^23
  const CompressArgs& a = fa.c;
  const Geo& g = a.g;
  const QP& q = a.q;
  const int R = q.radius;
  const unsigned span = (unsigned)(2 * R - 2);  // in range iff (delta + R - 1) <= 2R - 2

  const int64_t z0 = (int64_t)tc.bz * BZ, y0 = (int64_t)tc.by * BY;
  const int ez = (int)imin64(BZ, g.D0 - z0);
  const int ey = INTERIOR ? BY : (int)imin64(BY, g.D1 - y0);
  const int64_t xl0 = (int64_t)tc.wx * W + lane * VPL;
  const int xin = (lane * VPL) % BX;
  const int nvalid = INTERIOR ? VPL : (int)imax64(0, imin64(VPL, g.D2 - xl0));
  const bool lane_valid = INTERIOR || nvalid > 0;
  const int64_t bxg = xl0 / BX;
  const int ex = INTERIOR ? BX : (int)imax64(0, imin64(BX, g.D2 - bxg * BX));
  const int64_t bi = ((int64_t)tc.bz * g.P1 + tc.by) * g.P2 + bxg;
  const int64_t bstart = block_start(g, tc.bz, tc.by, bxg, BZ, BY, BX, ez, ey);
  const bool vec_store = INTERIOR || ((nvalid == VPL) && (ex == BX));
  const unsigned vmask = INTERIOR ? ((1u << VPL) - 1u) : ((1u << nvalid) - 1u);
  // the x-difference at a block's first column reads the zero halo: feed the
  // magic-number bias there so that the biased bit patterns cancel exactly
  const bool xhead = (xin == 0);

  int* const pplane = reinterpret_cast<int*>(ring + FAST_STAGES * F::STAGE_FLOATS) + lane * VPL;
  if (ND == 3) {  // previous-plane state starts at zero (Dz zero fill)
#pragma unroll 1
    for (int yl = 0; yl < BY; ++yl) {
      int z[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) z[j] = 0;
      st_vec<VPL>(pplane + yl * W, z);
    }
  }
  int run = 0;
  bool wide = false;
  int d_origin = 0;
  bool bad_origin = false;
  float v_origin = 0.f;
  KAcc<K> tacc;
  KAcc<K> face[ND];
  long long tcnt = 0;
  uint16_t* cptr = a.codes + bstart + xin;  // advances by ex per row
  // interior tiles stage their codes in shared memory (see the copy-out)
  constexpr bool STAGE_CODES = INTERIOR && F::SPLIT == 1 && BX == 8;  // 16-byte block rows
  const int stage_chunk0 = (lane * VPL * 2) >> 4, stage_sub = (lane * VPL * 2) & 15;
  const int64_t bstart0 =
      block_start(g, tc.bz, tc.by, (int64_t)tc.wx * (W / BX), BZ, BY, BX, ez, ey);
  const int64_t bsize = (int64_t)ez * BY * BX;  // codes per block of this layer

  for (int zl = 0; zl < ez; ++zl) {
    int prow[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) prow[j] = 0;  // Dy zero fill at the block's first row
    int psum = 0;  // |sum of a stage| < STAGE_ROWS * VPL * 2^24 < 2^31 (flushed per stage)
    for (int part = 0; part < F::SPLIT; ++part) {
    const float* plane = ring + cons.stage * F::STAGE_FLOATS + lane * VPL;
    unsigned char* const stage_bytes = reinterpret_cast<unsigned char*>(ring + cons.stage * F::STAGE_FLOATS);
    const uint32_t stage_s = smem_u32(stage_bytes);
    mbar_wait(&bars[cons.stage], cons.parity);
    if (zl == 0 && part == 0) {
      // the block origins sit in row 0 of the layer's first stage: take their
      // value and prequantized d here, once per tile, instead of a predicated
      // capture in every row (same quant_fast / quant_exact decision as the row)
      v_origin = plane[0];
      bool fok, ob = false, oo;
      int n0 = quant_fast(v_origin, q, fok);
      if (!fok) n0 = quant_exact(v_origin, q, ob, oo);
      d_origin = n0;
      bad_origin = ob;
    }
    int rstart = 0;  // first row of the stage for the per-row loop
    constexpr bool BATCH = VLZ_BIG_BATCH_C && INTERIOR && F::SPLIT > 1 && ND == 3;
#if VLZ_BIG_BATCH_C
    if constexpr (BATCH) {
#pragma unroll 1
      for (int h = 0; h < F::STAGE_ROWS; h += VLZ_BATCH_ROWS) {
      // b >= 32 interior stage as one batch: few tiles (512^3 b=64 is one
      // warp per block, ~3.5 warps per SM) leave each row's dependent chain
      // exposed; the rows' loads, quotients, x-shuffles and plane accesses
      // are independent and interleave here, only Dy runs in row order.  A
      // stage with an element off the fast quotient takes the per-row loop.
      constexpr int RB = VLZ_BATCH_ROWS;
      float vb[RB][VPL];
      unsigned nbb[RB][VPL];
      bool okb = true;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        ld_vec<VPL>(plane + (h + r) * W, vb[r]);
#pragma unroll
        for (int j = 0; j < VPL; j += 2) {
          const float2 qq = __fmul2_rn(make_float2(vb[r][j], vb[r][j + 1]),
                                       make_float2(q.inv32, q.inv32));
          const float2 rr = __fadd2_rn(qq, make_float2(12582912.0f, 12582912.0f));
          nbb[r][j] = __float_as_uint(rr.x);
          nbb[r][j + 1] = __float_as_uint(rr.y);
          const float2 rn = __fadd2_rn(rr, make_float2(-12582912.0f, -12582912.0f));
          const float2 e = __ffma2_rn(rn, make_float2(-1.0f, -1.0f), qq);
          const float2 lim = __ffma2_rn(make_float2(fabsf(qq.x), fabsf(qq.y)),
                                        make_float2(-q.kq, -q.kq), make_float2(q.lim0, q.lim0));
          okb = okb && (fabsf(e.x) < lim.x) && (fabsf(e.y) < lim.y);
        }
      }
      if (__all_sync(FULL, okb)) {
        int dlb[RB][VPL];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          unsigned left = __shfl_up_sync(FULL, nbb[r][VPL - 1], 1);
          if (xhead) left = MAGIC_BITS;
          dlb[r][0] = (int)(nbb[r][0] - left);
#pragma unroll
          for (int j = 1; j < VPL; ++j) dlb[r][j] = (int)(nbb[r][j] - nbb[r][j - 1]);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            const int t = dlb[r][j] - prow[j];
            prow[j] = dlb[r][j];
            dlb[r][j] = t;
          }
        }
        if (ND == 3) {
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            int* pp = pplane + (part * F::STAGE_ROWS + h + r) * W;
            int prev[VPL];
            ld_vec<VPL>(pp, prev);
            st_vec<VPL>(pp, dlb[r]);
#pragma unroll
            for (int j = 0; j < VPL; ++j) dlb[r][j] -= prev[j];
          }
        }
        unsigned ub[RB][VPL];
        unsigned umax = 0;
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            ub[r][j] = (unsigned)(dlb[r][j] + (R - 1));
            umax = ub[r][j] > umax ? ub[r][j] : umax;
          }
        unsigned cadd_rows = 0xffu;  // bit r: row r takes the common +1 in its packed store
        if (__any_sync(FULL, umax > span)) {
          // rare: outliers, ranked inside the block in traversal order
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const int yl = part * F::STAGE_ROWS + h + r;
            unsigned rmax = 0;
#pragma unroll
            for (int j = 0; j < VPL; ++j) rmax = ub[r][j] > rmax ? ub[r][j] : rmax;
            if (!__any_sync(FULL, rmax > span)) continue;
            unsigned om = 0;
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
              const bool o = ub[r][j] > span;
              ub[r][j] = o ? 0u : ub[r][j] + 1u;
              om |= o ? (1u << j) : 0u;
            }
            cadd_rows &= ~(1u << r);
            if ((zl == 0) && (yl == 0) && xhead) om &= ~1u;  // the origin is settled at the tile end
            int tot;
            const int excl = group_excl_scan<LPB>(__popc(om), lane, tot);
            int k = run + excl;
            float* slot = a.scratch + scratch_base(a.scratch_dense, bstart, bi) + 1;
            const int slim = scratch_limit(a.scratch_dense);
#pragma unroll
            for (int j = 0; j < VPL; ++j)
              if ((om >> j) & 1u) {
                if (k < slim) slot[k] = vb[r][j];
                ++k;
              }
            run += tot;
          }
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          st_codes<VPL>(cptr, ub[r], ((cadd_rows >> r) & 1u) ? 0x00010001u : 0u);
          cptr += ex;
          const int yl = part * F::STAGE_ROWS + h + r;
          if (MODE == MODE_GLOBAL) {
            if (K == 3) {
              unsigned rs = nbb[r][0];
#pragma unroll
              for (int j = 1; j < VPL; ++j) rs += nbb[r][j];
              psum += (int)(rs - (unsigned)VPL * MAGIC_BITS);
            } else {
#pragma unroll
              for (int j = 0; j < VPL; ++j) tacc.add((int)(nbb[r][j] - MAGIC_BITS));
            }
          } else if (MODE == MODE_BLOCK) {
#pragma unroll
            for (int j = 0; j < VPL; ++j) face[0].add((int)(nbb[r][j] - MAGIC_BITS));
          } else if (MODE == MODE_EDGE) {
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
              const int d = (int)(nbb[r][j] - MAGIC_BITS);
              const bool x0 = (xin + j) == 0;
              if (ND == 3) {
                if (zl == 0) face[0].add(d);
                if (yl == 0) face[1 % ND].add(d);
                if (x0) face[ND - 1].add(d);
              } else {
                if (yl == 0) face[0].add(d);
                if (x0) face[ND - 1].add(d);
              }
            }
          }
        }
        rstart = h + RB;
      } else {
        break;  // rows h.. take the per-row loop
      }
      }
    }
#endif
#pragma unroll 2
    for (int r = BATCH ? rstart : 0; r < F::STAGE_ROWS; ++r) {
      const int yl = part * F::STAGE_ROWS + r;
      if (!INTERIOR && yl >= ey) break;
      float v[VPL];
      ld_vec<VPL>(plane + r * W, v);
      // ---- float32 fast prequantization; nb = biased bit pattern of n
      unsigned nb[VPL];
      bool allok = true;
      // paired FP32 (FMUL2/FADD2/FFMA2, sm_100): the same IEEE RN operations
      // element by element, two per instruction
#pragma unroll
      for (int j = 0; j < VPL; j += 2) {
        const float2 qq = __fmul2_rn(make_float2(v[j], v[j + 1]), make_float2(q.inv32, q.inv32));
        const float2 r = __fadd2_rn(qq, make_float2(12582912.0f, 12582912.0f));
        nb[j] = __float_as_uint(r.x);
        nb[j + 1] = __float_as_uint(r.y);
        const float2 rn = __fadd2_rn(r, make_float2(-12582912.0f, -12582912.0f));  // exact
        const float2 e = __ffma2_rn(rn, make_float2(-1.0f, -1.0f), qq);              // qq - n, exact
        const float2 lim = __ffma2_rn(make_float2(fabsf(qq.x), fabsf(qq.y)),
                                      make_float2(-q.kq, -q.kq), make_float2(q.lim0, q.lim0));
        allok = allok && (fabsf(e.x) < lim.x) && (fabsf(e.y) < lim.y);
      }
      if (!INTERIOR) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (j >= nvalid) nb[j] = MAGIC_BITS;  // out-of-bounds columns act as d = 0
      }
      unsigned badm = 0;  // narrowing-check failures (exact path only)
      if (!__all_sync(FULL, allok)) {
        // rare: exact float64 re-evaluation of the flagged elements, one at a
        // time (one inlined copy of quant_exact; operands picked by select)
        unsigned sm = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          bool ok;
          quant_fast(v[j], q, ok);
          if (!ok && (INTERIOR || j < nvalid)) sm |= 1u << j;
        }
        while (sm) {
          const int j = __ffs(sm) - 1;
          sm &= sm - 1;
          float vj = v[0];
#pragma unroll
          for (int k = 1; k < VPL; ++k) vj = (j == k) ? v[k] : vj;
          bool bj, ovf;
          const int nj = quant_exact(vj, q, bj, ovf);
#pragma unroll
          for (int k = 0; k < VPL; ++k) nb[k] = (j == k) ? (unsigned)nj + MAGIC_BITS : nb[k];
          if (bj) badm |= 1u << j;
          if (ovf) {
            const unsigned long long fi =
                (unsigned long long)(((z0 + zl) * g.D1 + (y0 + yl)) * g.D2 + xl0 + j);
            ws_wait(a.init);
            if (!isfinite(vj)) atomicMin(a.first_nonfinite, fi);
            atomicMin(a.first_overflow, fi);
          }
          wide |= (nj >= (1 << 24)) || (nj <= -(1 << 24));
        }
      }
      // ---- Dx, Dy, Dz in int32 (exact: |d| < 2^24 unless `wide`).  The bias
      // cancels in every difference; the block head subtracts the bias itself.
      unsigned left = __shfl_up_sync(FULL, nb[VPL - 1], 1);
      if (xhead) left = MAGIC_BITS;
      int dl[VPL];
      dl[0] = (int)(nb[0] - left);
#pragma unroll
      for (int j = 1; j < VPL; ++j) dl[j] = (int)(nb[j] - nb[j - 1]);
      if (ND >= 2) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int t = dl[j] - prow[j];
          prow[j] = dl[j];
          dl[j] = t;
        }
      }
      if (ND == 3) {
        int* pp = pplane + yl * W;
        int prev[VPL];
        ld_vec<VPL>(pp, prev);
        st_vec<VPL>(pp, dl);
#pragma unroll
        for (int j = 0; j < VPL; ++j) dl[j] -= prev[j];
      }
      // ---- postquantization: code = delta + R, or 0 for an outlier.
      // u = delta + R - 1 is in range iff u <= 2R - 2 (unsigned): one max per
      // lane tells whether the warp needs the per-element outlier path; in
      // the common path the +1 is added to the packed code pairs
      unsigned u[VPL];
      unsigned umax = 0;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        u[j] = (unsigned)(dl[j] + (R - 1));
        umax = u[j] > umax ? u[j] : umax;
      }
      unsigned cadd = 0x00010001u;  // per 16-bit half: code = u + 1
      if (__any_sync(FULL, umax > span || badm != 0u)) {
        // rare: outliers (code 0; narrowing failures included), ranked inside
        // the block in traversal order
        unsigned om = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const bool o = u[j] > span || ((badm >> j) & 1u);
          u[j] = o ? 0u : u[j] + 1u;
          om |= o ? (1u << j) : 0u;
        }
        cadd = 0u;
        om &= vmask;
        if ((zl == 0) && (yl == 0) && xhead) om &= ~1u;  // the origin is settled at the tile end
        int tot;
        const int excl = group_excl_scan<LPB>(__popc(om), lane, tot);
        int k = run + excl;
        float* slot = a.scratch + scratch_base(a.scratch_dense, bstart, bi) + 1;
        const int slim = scratch_limit(a.scratch_dense);
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if ((om >> j) & 1u) {
            if (k < slim) slot[k] = v[j];
            ++k;
          }
        run += tot;
      }
      if (STAGE_CODES) {
        // this row's codes go into the consumed input row (16-byte chunks
        // rotated by row: conflict-free here and in the copy-out below)
        constexpr int CPR = W / 8;
        const int pos = (stage_chunk0 + r * (BX / 8)) & (CPR - 1);
        // 32-bit shared address (st.shared): no generic-to-shared window
        // arithmetic per row
        const uint32_t sa = stage_s + (uint32_t)(r * W * 4 + pos * 16 + stage_sub);
        if constexpr (VPL == 4) {
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(sa),
                       "r"(__byte_perm(u[0], u[1], 0x5410) + cadd),
                       "r"(__byte_perm(u[2], u[3], 0x5410) + cadd)
                       : "memory");
        } else {
          st_codes<VPL>(reinterpret_cast<uint16_t*>(stage_bytes + r * W * 4 + pos * 16 +
                                                    stage_sub), u, cadd);
        }
      } else if (vec_store) {
        st_codes<VPL>(cptr, u, cadd);
      } else if (lane_valid) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (j < nvalid) cptr[j] = (uint16_t)(u[j] + (cadd & 1u));
      }
      cptr += ex;
      // ---- padding statistics on d = nb - bias (in-bounds columns only)
      if (MODE == MODE_GLOBAL) {
        if (K == 3) {
          unsigned rs = nb[0];
#pragma unroll
          for (int j = 1; j < VPL; ++j) rs += nb[j];
          psum += (int)(rs - (unsigned)VPL * MAGIC_BITS);  // out-of-bounds columns hold the bias
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (INTERIOR || j < nvalid) tacc.add((int)(nb[j] - MAGIC_BITS));
        }
      } else if (MODE == MODE_BLOCK) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (INTERIOR || j < nvalid) face[0].add((int)(nb[j] - MAGIC_BITS));
      } else if (MODE == MODE_EDGE) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          if (!INTERIOR && j >= nvalid) continue;
          const int d = (int)(nb[j] - MAGIC_BITS);
          const bool x0 = (xin + j) == 0;
          if (ND == 3) {
            if (zl == 0) face[0].add(d);
            if (yl == 0) face[1 % ND].add(d);
            if (x0) face[ND - 1].add(d);
          } else {
            if (yl == 0) face[0].add(d);
            if (x0) face[ND - 1].add(d);
          }
        }
      }
    }
    if (STAGE_CODES) {
      // copy the plane's codes out: each block's plane is BY*BX contiguous
      // codes, so every 8 lanes store 128 contiguous bytes (full L2 lines
      // instead of one 8-byte piece per block row)
      __syncwarp();
      constexpr int CPR = W / 8, KB = BY * BX / 8, NCH = BY * CPR;
      uint16_t* const cbase = a.codes + bstart0 + (int64_t)zl * (BY * BX);
#pragma unroll
      for (int i = 0; i < NCH / 32; ++i) {
        const int t = i * 32 + lane;
        const int j = t / KB, k = t % KB;
        const int r = k / (BX / 8), cx = k % (BX / 8);
        const int pos = (j * (BX / 8) + cx + r * (BX / 8)) % CPR;
        const uint4 val = *reinterpret_cast<const uint4*>(stage_bytes + r * W * 4 + pos * 16);
        *reinterpret_cast<uint4*>(cbase + j * bsize + k * 8) = val;
      }
    }
    // release the stage and refill it FAST_STAGES half planes ahead
    __syncwarp();
    fence_proxy_async_smem();
    prod.issue(g, &fa.tmap, ring, bars, lane, nwarps);
    cons.advance();
    if (MODE == MODE_GLOBAL && K == 3) {  // per stage: |psum| < STAGE_ROWS * VPL * 2^24
      tacc.sum += psum;
      psum = 0;
    }
    }
    if (MODE == MODE_GLOBAL) tcnt += (long long)nvalid * ey;
  }

  // int32 stencil may have wrapped: the warp redoes the whole tile in int64
  // after its loop (slot k of this warp; the kernel's tail)
  if (__any_sync(FULL, wide)) {
    if (lane == 0) {
      const uint32_t k = *nfail_s;
      a.redo_list[(size_t)k * nwarps + tile % nwarps] = tile;
      *nfail_s = k + 1;
    }
    return;
  }

  // ---- tile end: padding scalars, block origins, counts (as dq_compress.cuh)
  const bool group_lead = lane_valid && xhead;
  int64_t s0 = 0;
  if (MODE == MODE_BLOCK || MODE == MODE_EDGE) {
    constexpr int NF = (MODE == MODE_BLOCK) ? 1 : ND;
    const int64_t ext[3] = {ND == 3 ? (int64_t)ez : (int64_t)ey,
                            ND == 3 ? (int64_t)ey : (int64_t)ex, (int64_t)ex};
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int64_t sum = K == 3 ? group_sum<LPB>(face[f].sum) : 0;
      const int mn = K == 1 ? group_min<LPB>(face[f].mn) : 0;
      const int mx = K == 2 ? group_max<LPB>(face[f].mx) : 0;
      int64_t cnt;
      if (MODE == MODE_BLOCK) {
        cnt = ext[0] * ext[1] * (ND == 3 ? ext[2] : 1);
      } else {
        cnt = 1;
#pragma unroll
        for (int d = 0; d < ND; ++d)
          if (d != f) cnt *= ext[d];
      }
      const int64_t sv = stat_value(K, sum, cnt, mn, mx);
      if (f == 0) s0 = sv;
      if (group_lead) a.scalars[MODE == MODE_BLOCK ? bi : bi * ND + f] = sv;
    }
  }
  if (MODE == MODE_GLOBAL) {
    gacc.merge(tacc);
    gcnt += tcnt;
  }
  if (group_lead) {
    int64_t total = run;
    if (MODE != MODE_GLOBAL) {
      const int64_t d = (int64_t)d_origin - s0;
      const bool o = bad_origin || d > (int64_t)(R - 1) || d < -(int64_t)(R - 1);
      a.codes[bstart] = o ? (uint16_t)0 : (uint16_t)(d + R);
      if (o) {
        a.scratch[scratch_base(a.scratch_dense, bstart, bi)] = v_origin;
        total += 1;
      }
    }
    // *:global: the origin is still pending -- hand the scan kernel its
    // prequantized value and narrowing verdict packed beside the count
    a.counts[bi] = (MODE == MODE_GLOBAL) ? pack_origin(total, d_origin, bad_origin) : total;
    if (MODE == MODE_GLOBAL) a.origin_vals[bi] = v_origin;
  }
}

template <int ND, int B, int VPL, int MODE, int K>
__global__ void __launch_bounds__(FAST_WARPS * 32, (FastShape<ND, B, VPL>::MINB))
    dq_compress_fast_kernel(const __grid_constant__ FastArgs fa) {
  pdl_enter();
  using S = Shape<ND, B, VPL>;
  using F = FastShape<ND, B, VPL>;
  extern __shared__ __align__(128) unsigned char smem_fast[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* ring = reinterpret_cast<float*>(smem_fast + (size_t)wib * F::WARP_SMEM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_fast + (size_t)wib * F::WARP_SMEM +
                                               FAST_STAGES * F::STAGE_BYTES + F::PREV_BYTES);
  const Geo& g = fa.c.g;

  uint32_t* const nfail_s = reinterpret_cast<uint32_t*>(bars + FAST_STAGES);  // tiles left for the tail
  if (lane == 0) {
    for (int s = 0; s < FAST_STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    *nfail_s = 0u;
  }
  __syncwarp();

  const uint32_t nwarps = gridDim.x * FAST_WARPS;
  const uint32_t first = blockIdx.x * FAST_WARPS + wib;
  if (threadIdx.x == 0) prefetch_tmap(&fa.tmap);
  Producer<ND, B, VPL> prod;
  prod.start(g, first);
  for (int s = 0; s < FAST_STAGES; ++s) prod.issue(g, &fa.tmap, ring, bars, lane, nwarps);
  if (blockIdx.x == 0 && wib == 0) ws_reset_warp(fa.c.init, lane);  // (behind the first loads)
  Consumer<ND, B, VPL> cons{0, 0u};
  KAcc<K> gacc;
  long long gcnt = 0;

  for (uint32_t tile = first; tile < (uint32_t)g.ntiles; tile += nwarps) {
    const TileXY tc = decode_tile(g, tile);
    const bool interior = ((int64_t)(tc.wx + 1) * S::W <= g.D2) &&
                          ((int64_t)(tc.by + 1) * S::BY <= g.D1);
    if (interior)
      fast_tile<ND, B, VPL, MODE, K, true>(fa, tile, tc, lane, ring, bars, prod, cons, nwarps,
                                           gacc, gcnt, nfail_s);
    else
      fast_tile<ND, B, VPL, MODE, K, false>(fa, tile, tc, lane, ring, bars, prod, cons, nwarps,
                                            gacc, gcnt, nfail_s);
  }

  if (MODE == MODE_GLOBAL) commit_global_stats(fa.c, gacc.sum, gcnt, gacc.mn, gacc.mx, lane);

  // tail: tiles whose |d| reached 2^24 (usually none), redone in int64 by the
  // warp that met them.  Shapes whose int64 plane lives in shared memory take
  // turns on the CTA's whole allocation (all rings are idle by then).
  __syncwarp();
#if VLZ_TAIL_MODE == 0
  const uint32_t nfail = 0u;
#else
  const uint32_t nfail = *nfail_s;
#endif
  if constexpr (S::PLANE_SMEM) {
    static_assert(fast_smem_bytes<ND, B, VPL>() >= plane_smem_bytes<ND, B, VPL>(), "tail plane");
    if (__syncthreads_or(nfail != 0u)) {
      for (int w = 0; w < FAST_WARPS; ++w) {
        if (w == wib && nfail)
          compress_redo_tail<ND, B, VPL, MODE>(fa.c, first, nwarps, nfail, lane,
                                               reinterpret_cast<long long*>(smem_fast));
        __syncthreads();
      }
    }
  } else if (nfail) {
    compress_redo_tail<ND, B, VPL, MODE>(fa.c, first, nwarps, nfail, lane, nullptr);
  }
}

}  // namespace vlz
