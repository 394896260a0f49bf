// dq_compress.cuh -- fused dual-quantization compress kernel (K1) for sm_100a.
//
// One warp owns a "tile": one block layer along dim 0 (BZ planes), one block
// row along dim 1 (BY rows) and a window of W = 32*VPL columns along the
// fastest dim (W/BX whole blocks).  Lane l holds VPL consecutive columns.
// The tile streams plane by plane, row by row; per element it
//   1. prequantizes v -> d (exact float64 rules of quantize.py:50-79),
//   2. forms the Lorenzo delta with the separable difference operator
//        delta = Dz Dy Dx (d)   with zero fill at the block's low faces,
//      Dx across lanes by one shuffle, Dy against the previous row held in
//      registers, Dz against the previous plane (registers for B <= 16,
//      shared memory for B >= 32).  For every padding policy this equals the
//      reference's halo-padded 7-point stencil (kernel.py:58-101) everywhere
//      except the block origin, whose delta is d(origin) - s0 (DESIGN.md,
//      "finding 1"); the origin is therefore resolved separately once the
//      padding scalar s0 is known,
//   3. postquantizes: code = delta + R unless |delta| > R-1 or the float32
//      narrowed reconstruction misses the bound (vector.py:72-78),
//   4. writes uint16 codes in canonical block-major order and places outlier
//      values in a per-block scratch slot (slot 0 = origin, 1.. = the others
//      in traversal order); the scan/gather kernel (dq_scan.cuh) compacts them.
// Padding statistics (padding.py:62-110) are accumulated on the fly: per warp
// for *:global (reduced once per CTA at the end), per block / per face in the
// lane group for *:block / *:edge.
//
// The stencil runs in wrapping uint32 when every |d| of the tile is < 2^28 (then no
// intermediate can wrap: |delta| < 8 * 2^28); otherwise the tile is redone in
// int64 (the redo is idempotent: codes and scratch slots are overwritten,
// counts / scalars / statistics are committed only by the final pass).
#pragma once

#include "vlz_common.cuh"

namespace vlz {

enum Mode { MODE_ZERO = 0, MODE_GLOBAL = 1, MODE_BLOCK = 2, MODE_EDGE = 3 };

struct CompressArgs {
  Geo g;
  QP q;
  const float* in;
  uint16_t* codes;
  float* scratch;  // outlier slots (vlz_common.cuh)
  int scratch_dense;  // 1: one slot per element (dense layout)
  int64_t* counts;
  int64_t* scalars;
  float* origin_vals;  // *:global: verbatim origin value per block (workspace, coalesced)
  unsigned long long* first_nonfinite;  // device result fields (atomicMin)
  unsigned long long* first_overflow;
  unsigned long long* gsum;  // global statistics accumulators
  unsigned long long* gcount;
  long long* gmin;
  long long* gnegmax;
  // failed-tile slots of the fused kernels (tile ids redone in int64 by the
  // same warp at the end of its loop: slot k of warp w is redo_list[k * nwarps + w])
  long long* redo_list;
  InitArgs init;  // per-call reset done by CTA 0 (vlz_common.cuh)
};

// the warp's global statistics -> the call's accumulators (after the reset)
__device__ __forceinline__ void commit_global_stats(const CompressArgs& a, long long s, long long c,
                                                    int mn, int mx, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(FULL, s, o);
    c += __shfl_xor_sync(FULL, c, o);
    const int m1 = __shfl_xor_sync(FULL, mn, o);
    const int m2 = __shfl_xor_sync(FULL, mx, o);
    mn = m1 < mn ? m1 : mn;
    mx = m2 > mx ? m2 : mx;
  }
  if (lane == 0 && c > 0) {
    ws_wait(a.init);
    atomicAdd(a.gsum, (unsigned long long)s);
    atomicAdd(a.gcount, (unsigned long long)c);
    atomicMin(a.gmin, (long long)mn);
    atomicMin(a.gnegmax, -(long long)mx);
  }
}

// per-warp statistics for MODE_GLOBAL (lane partials)
struct GlobalAcc {
  int64_t sum = 0, cnt = 0;
  int mn = 0x7fffffff, mx = (int)0x80000000;
};

struct FaceAcc {
  int64_t sum = 0;
  int mn = 0x7fffffff, mx = (int)0x80000000;
  __device__ __forceinline__ void add(int v) {
    sum += v;
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
};

template <int ND, int B, int VPL>
struct Shape {
  static constexpr int BZ = ND == 3 ? B : 1;
  static constexpr int BY = ND >= 2 ? B : 1;
  static constexpr int BX = B;
  static constexpr int W = 32 * VPL;
  static constexpr int LPB = BX / VPL;  // lanes per block
  static constexpr bool PLANE_SMEM = (ND == 3) && (B >= 32);
  static_assert(BX % VPL == 0 && W % BX == 0, "window must hold whole blocks");
};

// shared-memory bytes per warp for the previous-plane store (B >= 32, 3D)
template <int ND, int B, int VPL>
__host__ __device__ constexpr int plane_smem_bytes() {
  return Shape<ND, B, VPL>::PLANE_SMEM ? Shape<ND, B, VPL>::BY * Shape<ND, B, VPL>::W * 8 : 0;
}

template <int ND, int B, int VPL, int MODE, typename IT>
__device__ __forceinline__ bool compress_tile(const CompressArgs& a, int64_t tile, int lane,
                                              IT* plane_smem, GlobalAcc& gacc) {
  using S = Shape<ND, B, VPL>;
  constexpr int BZ = S::BZ, BY = S::BY, BX = S::BX, W = S::W, LPB = S::LPB;
  const Geo& g = a.g;
  const int R = a.q.radius;

  const int64_t wx = tile % g.NW;
  const int64_t t2 = tile / g.NW;
  const int64_t by = t2 % g.P1;
  const int64_t bz = t2 / g.P1;
  const int64_t z0 = bz * BZ, y0 = by * BY;
  const int ez = (int)imin64(BZ, g.D0 - z0);
  const int ey = (int)imin64(BY, g.D1 - y0);
  const int64_t xl0 = wx * W + (int64_t)lane * VPL;
  const int xin = (lane * VPL) % BX;  // column of element 0 inside its block
  const int nvalid = (int)imax64(0, imin64(VPL, g.D2 - xl0));
  const bool lane_valid = nvalid > 0;
  const int64_t bxg = xl0 / BX;
  const int ex = (int)imax64(0, imin64(BX, g.D2 - bxg * BX));
  const int64_t bi = (bz * g.P1 + by) * g.P2 + bxg;
  const int64_t bstart = block_start(g, bz, by, bxg, BZ, BY, BX, ez, ey);
  const bool vec_ok = (VPL % 4 == 0) && (g.D2 % 4 == 0) && (nvalid == VPL);
  const bool vec_store = (nvalid == VPL) && (ex == BX);

  IT prow[VPL];
  IT pplane_r[(ND == 3 && !S::PLANE_SMEM) ? BY : 1][VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) prow[j] = 0;

  int run = 0;  // non-origin outliers of this lane's block so far
  bool wide = false;
  // origin bookkeeping (lane with xin == 0)
  int d_origin = 0;
  bool bad_origin = false;
  float v_origin = 0.f;
  // statistics
  GlobalAcc tacc;
  FaceAcc face[ND];

  constexpr int UNR = (ND == 3 && !S::PLANE_SMEM) ? BY : 1;
  for (int zl = 0; zl < ez; ++zl) {
#pragma unroll UNR
    for (int yl = 0; yl < BY; ++yl) {
      if (yl >= ey) break;
      const int64_t row = ((z0 + zl) * g.D1 + (y0 + yl)) * g.D2;
      float v[VPL];
      if (vec_ok) {
#pragma unroll
        for (int j = 0; j < VPL; j += 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(a.in + row + xl0 + j));
          v[j] = f.x; v[j + 1] = f.y; v[j + 2] = f.z; v[j + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < VPL; ++j) v[j] = j < nvalid ? __ldg(a.in + row + xl0 + j) : 0.f;
      }
      int n[VPL];
      unsigned badm = 0;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        // exact-fast float32 quotient first (DESIGN.md proof: when it reports
        // ok the rounding and the narrowing check are already decided), fp64
        // only for the undecided elements
        bool bad = false, ovf = false, fok;
        n[j] = quant_fast(v[j], a.q, fok);
        if (!fok) n[j] = quant_exact(v[j], a.q, bad, ovf);
        if (j < nvalid) {
          if (bad) badm |= 1u << j;
          if (ovf) {
            const unsigned long long fi = (unsigned long long)(row + xl0 + j);
            ws_wait(a.init);
            if (!isfinite(v[j])) atomicMin(a.first_nonfinite, fi);
            atomicMin(a.first_overflow, fi);
          }
          if (sizeof(IT) == 4) wide |= (n[j] >= (1 << 28)) || (n[j] <= -(1 << 28));
        } else {
          n[j] = 0;
        }
      }
      // ---- Dx: within the lane, then one shuffle across the lane boundary
      IT left = (IT)__shfl_up_sync(FULL, n[VPL - 1], 1);
      if (xin == 0) left = 0;
      IT dl[VPL];
      dl[0] = (IT)n[0] - left;
#pragma unroll
      for (int j = 1; j < VPL; ++j) dl[j] = (IT)n[j] - (IT)n[j - 1];
      // ---- Dy against the previous row of the block
      if (ND >= 2) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const IT t = dl[j] - (yl ? prow[j] : (IT)0);
          prow[j] = dl[j];
          dl[j] = t;
        }
      }
      // ---- Dz against the previous plane of the block
      if (ND == 3) {
        if (S::PLANE_SMEM) {
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            IT* slot = plane_smem + (yl * W + lane * VPL + j);
            const IT prev = zl ? *slot : (IT)0;
            *slot = dl[j];
            dl[j] -= prev;
          }
        } else {
#pragma unroll
          for (int yy = 0; yy < BY; ++yy) {
            if (yy == yl) {
#pragma unroll
              for (int j = 0; j < VPL; ++j) {
                const IT prev = zl ? pplane_r[yy][j] : (IT)0;
                pplane_r[yy][j] = dl[j];
                dl[j] -= prev;
              }
            }
          }
        }
      }
      // ---- postquantization + outliers
      const bool origin_row = (zl == 0) && (yl == 0) && (xin == 0);
      unsigned om = 0;
      uint16_t c[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const IT d = dl[j];
        const bool out = ((unsigned)(d + (IT)(R - 1)) > (unsigned)(2 * R - 2)) ||
                         (sizeof(IT) == 8 && (d > (IT)(R - 1) || d < -(IT)(R - 1))) ||
                         ((badm >> j) & 1u);
        c[j] = out ? (uint16_t)0 : (uint16_t)(d + (IT)R);
        if (out && j < nvalid && !(j == 0 && origin_row)) om |= 1u << j;
      }
      if (origin_row && lane_valid) {
        d_origin = n[0];
        bad_origin = badm & 1u;
        v_origin = v[0];
      }
      // ---- store codes (canonical block-major position)
      if (lane_valid) {
        uint16_t* dst = a.codes + bstart + ((int64_t)zl * ey + yl) * ex + xin;
        if (vec_store && VPL == 4) {
          uint2 pk;
          pk.x = (unsigned)c[0] | ((unsigned)c[1] << 16);
          pk.y = (unsigned)c[2 % VPL] | ((unsigned)c[3 % VPL] << 16);
          *reinterpret_cast<uint2*>(dst) = pk;
        } else if (vec_store && VPL == 8) {
          uint4 pk;
          pk.x = (unsigned)c[0] | ((unsigned)c[1] << 16);
          pk.y = (unsigned)c[2] | ((unsigned)c[3] << 16);
          pk.z = (unsigned)c[4 % VPL] | ((unsigned)c[5 % VPL] << 16);
          pk.w = (unsigned)c[6 % VPL] | ((unsigned)c[7 % VPL] << 16);
          *reinterpret_cast<uint4*>(dst) = pk;
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (j < nvalid) dst[j] = c[j];
        }
      }
      // ---- outlier placement: rank inside the block in traversal order
      if (__any_sync(FULL, om != 0)) {
        int tot;
        const int cnt = __popc(om);
        const int excl = group_excl_scan<LPB>(cnt, lane, tot);
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
      // ---- statistics over in-bounds prequantized values (padding.py:62-110)
      if (MODE == MODE_GLOBAL) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (j < nvalid) {
            tacc.sum += n[j];
            tacc.mn = n[j] < tacc.mn ? n[j] : tacc.mn;
            tacc.mx = n[j] > tacc.mx ? n[j] : tacc.mx;
          }
        tacc.cnt += nvalid;
      } else if (MODE == MODE_BLOCK) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (j < nvalid) face[0].add(n[j]);
      } else if (MODE == MODE_EDGE) {
        // face d = elements whose block-local coordinate along real dim d is 0
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          if (j >= nvalid) continue;
          const bool x0 = (xin + j) == 0;
          if (ND == 3) {
            if (zl == 0) face[0].add(n[j]);
            if (yl == 0) face[ND >= 2 ? 1 : 0].add(n[j]);
            if (x0) face[ND - 1].add(n[j]);
          } else if (ND == 2) {
            if (yl == 0) face[0].add(n[j]);
            if (x0) face[ND - 1].add(n[j]);
          } else {
            if (x0) face[0].add(n[j]);
          }
        }
      }
    }
  }

  // int32 stencil could have wrapped: redo this tile in int64
  if (sizeof(IT) == 4 && __any_sync(FULL, wide)) return true;

  // ---- tile end: padding scalars, block origins, counts
  const bool group_lead = lane_valid && (xin == 0);
  int64_t s0 = 0;
  if (MODE == MODE_BLOCK || MODE == MODE_EDGE) {
    constexpr int NF = (MODE == MODE_BLOCK) ? 1 : ND;
    const int64_t ext[3] = {ND == 3 ? (int64_t)ez : (ND == 2 ? (int64_t)ey : (int64_t)ex),
                            ND == 3 ? (int64_t)ey : (int64_t)ex, (int64_t)ex};
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int64_t sum = group_sum<LPB>(face[f].sum);
      const int mn = group_min<LPB>(face[f].mn);
      const int mx = group_max<LPB>(face[f].mx);
      int64_t cnt;
      if (MODE == MODE_BLOCK) {
        cnt = ext[0] * (ND >= 2 ? ext[1] : 1) * (ND == 3 ? ext[2] : 1);
      } else {
        cnt = 1;
#pragma unroll
        for (int d = 0; d < ND; ++d)
          if (d != f) cnt *= ext[d];
      }
      const int64_t sv = stat_value(a.q.kind, sum, cnt, mn, mx);
      if (f == 0) s0 = sv;
      if (group_lead) a.scalars[MODE == MODE_BLOCK ? bi : bi * ND + f] = sv;
    }
  }
  if (MODE == MODE_GLOBAL) {
    gacc.sum += tacc.sum;
    gacc.cnt += tacc.cnt;
    gacc.mn = tacc.mn < gacc.mn ? tacc.mn : gacc.mn;
    gacc.mx = tacc.mx > gacc.mx ? tacc.mx : gacc.mx;
  }
  if (group_lead) {
    int64_t total = run;
    if (MODE != MODE_GLOBAL) {
      // origin: delta = d(origin) - s0  (finding 1; s0 = 0 for zero padding)
      const int64_t d = (int64_t)d_origin - s0;
      const bool out = bad_origin || d > (int64_t)(R - 1) || d < -(int64_t)(R - 1);
      a.codes[bstart] = out ? (uint16_t)0 : (uint16_t)(d + R);
      if (out) {
        a.scratch[scratch_base(a.scratch_dense, bstart, bi)] = v_origin;
        total += 1;
      }
    }
    // *:global: the origin is still pending -- hand the scan kernel its
    // prequantized value and narrowing verdict packed beside the count
    a.counts[bi] = (MODE == MODE_GLOBAL) ? pack_origin(total, d_origin, bad_origin) : total;
    if (MODE == MODE_GLOBAL) a.origin_vals[bi] = v_origin;
  }
  return false;
}

// Every tile in the uint32 stencil, redone in int64 on demand.
template <int ND, int B, int VPL, int MODE>
__global__ void __launch_bounds__(128) dq_compress_kernel(CompressArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PB = plane_smem_bytes<ND, B, VPL>();
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  if (blockIdx.x == 0 && wib == 0) ws_reset_warp(a.init, lane);
  unsigned char* wsm = smem_raw + (size_t)wib * PB;
  GlobalAcc gacc;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; i < a.g.ntiles; i += nwarps) {
    if (compress_tile<ND, B, VPL, MODE, unsigned>(a, i, lane, reinterpret_cast<unsigned*>(wsm),
                                                  gacc)) {
      compress_tile<ND, B, VPL, MODE, long long>(a, i, lane,
                                                 reinterpret_cast<long long*>(wsm), gacc);
    }
  }
  if (MODE == MODE_GLOBAL) commit_global_stats(a, gacc.sum, gacc.cnt, gacc.mn, gacc.mx, lane);
}

// int64 redo of the tiles a fused kernel's warp could not finish in int32
// (slot k of warp `first` is redo_list[k * nwarps + first]); kept out of line
// so that the fused kernels' register allocation is that of their hot loops
#ifndef VLZ_TAIL_MODE
#define VLZ_TAIL_MODE 2  // 2: inlined (C5 fused compress: neutral; 1, out of line: +1.7 %);
                         // 0: absent (timing experiments only)
#endif
#if VLZ_TAIL_MODE == 2
#define VLZ_TAIL_ATTR __forceinline__
#else
#define VLZ_TAIL_ATTR __noinline__
#endif
template <int ND, int B, int VPL, int MODE>
__device__ VLZ_TAIL_ATTR void compress_redo_tail(const CompressArgs& a, uint32_t first,
                                                uint32_t nwarps, uint32_t nfail, int lane,
                                                long long* plane_smem) {
  GlobalAcc gacc;
  for (uint32_t k = 0; k < nfail; ++k)
    compress_tile<ND, B, VPL, MODE, long long>(a, a.redo_list[(size_t)k * nwarps + first], lane,
                                               plane_smem, gacc);
  if (MODE == MODE_GLOBAL) commit_global_stats(a, gacc.sum, gacc.cnt, gacc.mn, gacc.mx, lane);
}

}  // namespace vlz
