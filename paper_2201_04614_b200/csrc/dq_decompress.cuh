// dq_decompress.cuh -- fused reconstruction kernel (K4) for sm_100a.
//
// Inverse of dq_compress.cuh with the same warp tiling.  With E = d - s0 the
// compressor emitted delta = Dz Dy Dx E (zero fill at the block's low faces),
// so reconstruction is three nested prefix sums, streamed plane by plane:
//     H(z,y,x) = H(z,y,x-1) + delta      (segmented scan along x: in-lane,
//                                          then across the block's lane group)
//     G(z,y,x) = G(z,y-1,x) + H          (previous row, registers)
//     E(z,y,x) = E(z-1,y,x) + G          (previous plane, registers / smem)
//     d = E + s0;  out = float32((2.0 * d) * eb)
// A sentinel (code 0) carries its verbatim value v; its d is re-derived with
// the compressor's float64 rule (reconstruct.py:55-60) and the scan is RESET
// there: H := (d - s0) - E(z-1,y,x) - G(z,y-1,x).  This reproduces the
// reference's strictly sequential per-element decoder (reconstruct.py:30-71)
// exactly, for any number of outliers per block.  Outliers are written back
// verbatim (reconstruct.py:68-71).
//
// Stream validation mirrors reconstruct.py:43-66 / 87-91: codes >= 2R, more
// sentinels than the block's stored outliers (exhausted) or fewer (leftover)
// are recorded per block as (block << 4 | status) with an atomicMin, so the
// host reports the first failing block like the sequential reference does.
#pragma once

#include "dq_compress.cuh"

namespace vlz {

struct DecompressArgs {
  Geo g;
  QP q;
  int mode;  // padding granularity as Mode (for s0 lookup)
  int nd;
  const void* codes;
  const float* outliers;
  long long n_outliers;
  const long long* n_out_dev;  // non-null: the stored outlier count lives in device memory
  const int64_t* counts;
  const int64_t* offsets;  // exclusive prefix of counts
  const int64_t* scalars;
  float* out;
  unsigned long long* first_bad;  // (block << 4) | status
  unsigned long long* sentinels;  // total sentinel count
  unsigned int* done;             // finished-CTA counter (last CTA finalises)
  int* status;
  long long* index;
  long long* n_sent_out;
  // failed-tile slots of the fused kernels (redone in int64 by the same warp
  // after its loop: slot k of warp w is redo_list[k * nwarps + w])
  long long* redo_list;
  unsigned long long* flag;  // the call's reset flag, cleared by the last CTA
};

// the stream's outlier count: a host value, or a device word written by an
// earlier kernel (vlz_dq_decompress_dn: no host round trip between calls)
__device__ __forceinline__ long long n_outliers_of(const DecompressArgs& a) {
  return a.n_out_dev ? *a.n_out_dev : a.n_outliers;
}

template <typename CT, int VPL>
__device__ __forceinline__ void load_codes(const CT* p, bool vec, int nvalid, unsigned (&c)[VPL]) {
  if (sizeof(CT) == 2 && vec && VPL == 4) {
    const uint2 pk = *reinterpret_cast<const uint2*>(p);
    c[0] = pk.x & 0xffffu; c[1 % VPL] = pk.x >> 16;
    c[2 % VPL] = pk.y & 0xffffu; c[3 % VPL] = pk.y >> 16;
  } else if (sizeof(CT) == 2 && vec && VPL == 8) {
    const uint4 pk = *reinterpret_cast<const uint4*>(p);
    const unsigned w[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
    for (int j = 0; j < VPL; ++j) c[j] = (w[(j / 2) % 4] >> (16 * (j & 1))) & 0xffffu;
  } else {
#pragma unroll
    for (int j = 0; j < VPL; ++j) c[j] = j < nvalid ? (unsigned)p[j] : (unsigned)0;
  }
}

template <int ND, int B, int VPL, typename CT>
__device__ __forceinline__ void decompress_tile(const DecompressArgs& a, int64_t tile, int lane,
                                                long long* plane_smem, long long& sent_acc) {
  using S = Shape<ND, B, VPL>;
  constexpr int BZ = S::BZ, BY = S::BY, BX = S::BX, W = S::W, LPB = S::LPB;
  const Geo& g = a.g;
  const int R = a.q.radius;
  const CT* codes = reinterpret_cast<const CT*>(a.codes);

  const int64_t wx = tile % g.NW;
  const int64_t t2 = tile / g.NW;
  const int64_t by = t2 % g.P1;
  const int64_t bz = t2 / g.P1;
  const int64_t z0 = bz * BZ, y0 = by * BY;
  const int ez = (int)imin64(BZ, g.D0 - z0);
  const int ey = (int)imin64(BY, g.D1 - y0);
  const int64_t xl0 = wx * W + (int64_t)lane * VPL;
  const int xin = (lane * VPL) % BX;
  const int nvalid = (int)imax64(0, imin64(VPL, g.D2 - xl0));
  const bool lane_valid = nvalid > 0;
  const int64_t bxg = xl0 / BX;
  const int ex = (int)imax64(0, imin64(BX, g.D2 - bxg * BX));
  const int64_t bi = (bz * g.P1 + by) * g.P2 + bxg;
  const int64_t bstart = block_start(g, bz, by, bxg, BZ, BY, BX, ez, ey);
  const bool vec_ld = (nvalid == VPL) && (ex == BX);
  const bool vec_st = (VPL % 4 == 0) && (g.D2 % 4 == 0) && (nvalid == VPL);

  // block's padding scalar s0 (apply_padding, padding.py:113-129: only the
  // dim-0 halo scalar reaches the codes) and its outlier slice
  long long s0 = 0, off = 0, avail = 0;
  if (lane_valid) {
    if (a.mode == MODE_GLOBAL) s0 = a.scalars[0];
    else if (a.mode == MODE_BLOCK) s0 = a.scalars[bi];
    else if (a.mode == MODE_EDGE) s0 = a.scalars[bi * a.nd];
    off = a.offsets[bi];
    const long long cnt = a.counts[bi];
    avail = imax64(0, imin64(cnt, n_outliers_of(a) - off));
  }

  long long grow[VPL];
  long long pplane_r[(ND == 3 && !S::PLANE_SMEM) ? BY : 1][VPL];
  int run = 0;
  bool badcode = false;

  constexpr int UNR = (ND == 3 && !S::PLANE_SMEM) ? BY : 1;
  for (int zl = 0; zl < ez; ++zl) {
#pragma unroll UNR
    for (int yl = 0; yl < BY; ++yl) {
      if (yl >= ey) break;
      unsigned c[VPL];
      const CT* src = codes + bstart + ((int64_t)zl * ey + yl) * ex + xin;
      if (lane_valid) load_codes<CT, VPL>(src, vec_ld, nvalid, c);
      else {
#pragma unroll
        for (int j = 0; j < VPL; ++j) c[j] = 1;
      }
      unsigned sm = 0;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        if (j < nvalid) {
          if (c[j] == 0) sm |= 1u << j;
          if (c[j] >= (unsigned)(2 * R)) badcode = true;
        }
      }
      // previous-row G and previous-plane E at this row
      long long gp[VPL], ep[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) gp[j] = yl ? grow[j] : 0;
      if (ND == 3) {
        if (S::PLANE_SMEM) {
#pragma unroll
          for (int j = 0; j < VPL; ++j) ep[j] = zl ? plane_smem[yl * W + lane * VPL + j] : 0;
        } else {
#pragma unroll
          for (int yy = 0; yy < BY; ++yy)
            if (yy == yl) {
#pragma unroll
              for (int j = 0; j < VPL; ++j) ep[j] = zl ? pplane_r[yy][j] : 0;
            }
        }
      } else {
#pragma unroll
        for (int j = 0; j < VPL; ++j) ep[j] = 0;
      }
      // sentinel values (rank inside the block, traversal order)
      float vs[VPL];
      long long hs[VPL];
      if (__any_sync(FULL, sm != 0)) {
        int tot;
        const int excl = group_excl_scan<LPB>(__popc(sm), lane, tot);
        int k = run + excl;
        // loads first (in flight together), then the exact-fast quotient
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          vs[j] = 0.f;
          if ((sm >> j) & 1u) {
            if (k < avail) vs[j] = __ldg(a.outliers + off + k);
            ++k;
          }
        }
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          hs[j] = 0;
          if ((sm >> j) & 1u) {
            bool qok;
            const int nq = quant_fast(vs[j], a.q, qok);
            const long long ds = qok ? (long long)nq : quant_value(vs[j], a.q.twoeb);
            hs[j] = (ds - s0) - ep[j] - gp[j];
          }
        }
        run += tot;
      }
      // segmented inclusive scan of delta along x with resets at sentinels
      long long h[VPL];
      long long acc = 0;
      bool reset = false;
      unsigned before = 0;  // elements not yet covered by an in-lane reset
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        if ((sm >> j) & 1u) {
          acc = hs[j];
          reset = true;
        } else {
          acc += (long long)c[j] - R;
        }
        if (!reset) before |= 1u << j;
        h[j] = acc;
      }
      // exclusive carry from earlier lanes of the block: (flag, value)
      long long cv = acc;
      bool cf = reset;
      const int gl = lane & (LPB - 1);
#pragma unroll
      for (int o = 1; o < LPB; o <<= 1) {
        const long long uv = __shfl_up_sync(FULL, cv, o);
        const bool uf = __shfl_up_sync(FULL, cf, o);
        if (gl >= o && !cf) {
          cv += uv;
          cf = uf;
        }
      }
      // cv/cf now inclusive over lanes [group start .. lane]; make exclusive
      long long pv = __shfl_up_sync(FULL, cv, 1);
      if (gl == 0) pv = 0;
#pragma unroll
      for (int j = 0; j < VPL; ++j)
        if ((before >> j) & 1u) h[j] += pv;
      // G, E, output
      float o[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const long long gv = h[j] + gp[j];
        grow[j] = gv;
        const long long ev = gv + ep[j];
        ep[j] = ev;
        o[j] = ((sm >> j) & 1u) ? vs[j] : dequant(ev + s0, a.q.eb);
      }
      if (ND == 3) {
        if (S::PLANE_SMEM) {
#pragma unroll
          for (int j = 0; j < VPL; ++j) plane_smem[yl * W + lane * VPL + j] = ep[j];
        } else {
#pragma unroll
          for (int yy = 0; yy < BY; ++yy)
            if (yy == yl) {
#pragma unroll
              for (int j = 0; j < VPL; ++j) pplane_r[yy][j] = ep[j];
            }
        }
      }
      if (lane_valid) {
        float* dst = a.out + ((z0 + zl) * g.D1 + (y0 + yl)) * g.D2 + xl0;
        if (vec_st) {
#pragma unroll
          for (int j = 0; j < VPL; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (j < nvalid) dst[j] = o[j];
        }
      }
    }
  }
  // per-block validation
  const bool bad_any = group_any<LPB>(badcode, lane);
  if (lane_valid && xin == 0) {
    sent_acc += run;
    int st = 0;
    if (bad_any) st = 4;               // VLZ_ST_CORRUPT_CODE
    else if (run > avail) st = 5;      // VLZ_ST_EXHAUSTED
    else if (run < avail) st = 6;      // VLZ_ST_LEFTOVER
    if (st) atomicMin(a.first_bad, ((unsigned long long)bi << 4) | (unsigned long long)st);
  }
}

// End of every decompress kernel (all threads of the CTA): the warp's sentinel
// count joins the total, and the last CTA to finish turns the per-block
// findings into the reference's error order: sentinel total vs stored outliers
// first (reconstruct.py:87-91), then the first failing block
// (reconstruct.py:43-66, sequential block order).
__device__ __forceinline__ void decompress_finish(const DecompressArgs& a, long long sent,
                                                  int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sent += __shfl_xor_sync(FULL, sent, o);
  if (lane == 0 && sent) atomicAdd(a.sentinels, (unsigned long long)sent);
#ifdef VLZ_NO_DFINISH  // (timing experiments only)
  return;
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long ns = atomicAdd(a.sentinels, 0ull);
      const unsigned long long fb = atomicAdd(a.first_bad, 0ull);
      *a.flag = 0ull;  // a graph replay of this call starts from a cleared flag
      *a.n_sent_out = (long long)ns;
      if ((long long)ns != n_outliers_of(a)) {
        *a.status = 7;  // VLZ_ST_SENTINEL_TOTAL
        *a.index = -1;
      } else if (fb != 0x7fffffffffffffffull) {
        *a.status = (int)(fb & 15ull);
        *a.index = (long long)(fb >> 4);
      }
    }
  }
}

// int64 redo of the tiles a fused kernel's warp could not finish in int32
// (slot k of warp `first` is redo_list[k * nwarps + first]); out of line so
// that the fused kernels keep the register allocation of their hot loops
#ifndef VLZ_DTAIL_MODE
#define VLZ_DTAIL_MODE 1  // 1: out of line; 2: inlined
#endif
#if VLZ_DTAIL_MODE == 2
#define VLZ_DTAIL_ATTR __forceinline__
#else
#define VLZ_DTAIL_ATTR __noinline__
#endif
template <int ND, int B, int VPL>
__device__ VLZ_DTAIL_ATTR void decompress_redo_tail(const DecompressArgs& a, uint32_t first,
                                                  uint32_t nwarps, uint32_t nfail, int lane,
                                                  long long* plane_smem, long long& sent) {
  for (uint32_t k = 0; k < nfail; ++k)
    decompress_tile<ND, B, VPL, uint16_t>(a, a.redo_list[(size_t)k * nwarps + first], lane,
                                          plane_smem, sent);
}

// every tile in int64 (shapes and code widths without a fused kernel)
template <int ND, int B, int VPL, typename CT>
__global__ void __launch_bounds__(128) dq_decompress_kernel(DecompressArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PB = plane_smem_bytes<ND, B, VPL>();
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  long long* wsm = reinterpret_cast<long long*>(smem_raw + (size_t)wib * PB);
  long long sent = 0;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; i < a.g.ntiles; i += nwarps)
    decompress_tile<ND, B, VPL, CT>(a, i, lane, wsm, sent);
  decompress_finish(a, sent, lane);
}

}  // namespace vlz
