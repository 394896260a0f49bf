// dq_decompress_fast.cuh -- production fused reconstruction kernel (sm_100a).
//
// Same warp tiling and recurrences as dq_decompress.cuh (H: segmented scan of
// delta along x with resets at sentinels, G = H + G(prev row),
// E = G + E(prev plane), d = E + s0, out = float32(fl64(2 d eb))), specialised
// for the throughput shapes (3-D b=8/16, 2-D b=8/16) and interior tiles:
//
//  * each plane of a tile is W/BX contiguous block slices of BY*BX uint16
//    codes; they stream into a per-warp shared ring with TMA bulk copies
//    (one cp.async.bulk per block slice, slices padded so that the lanes'
//    vector LDS hit distinct banks), FAST_STAGES planes ahead;
//  * arithmetic is wrapping int32.  It is exact whenever every reconstructed
//    |E| and every sentinel |d - s0| stays below 2^28 and |s0| < 2^28: by
//    induction over the traversal order each true value is then a sum of
//    7 earlier values (< 7 * 2^28) plus a code (< 2^15), i.e. it lies in
//    (-2^31, 2^31) where congruence mod 2^32 is equality.  The kernel checks
//    exactly that and hands any tile that fails it -- and every edge tile --
//    to the int64 kernel (dq_decompress_kernel<..., LIST=true>);
//  * output rows leave with 16-byte stores straight from registers.
#pragma once

#include "dq_compress_fast.cuh"
#include "dq_decompress.cuh"

namespace vlz {

template <int ND, int B, int VPL>
struct DFastShape {
  using S = Shape<ND, B, VPL>;
  static constexpr int NBLK = S::W / S::BX;                 // blocks per window
  static constexpr int SLICE_CODES = S::BY * S::BX;          // codes per block plane
  static constexpr int SLICE_BYTES = SLICE_CODES * 2;
  // pad each slice so consecutive blocks start 4 (B=8) / 8 (B>=16) banks apart
  static constexpr int PAD_BYTES = (S::BX == 8) ? 16 : 32;
  static constexpr int SLOT_BYTES = SLICE_BYTES + PAD_BYTES;
  static constexpr int STAGE_BYTES = NBLK * SLOT_BYTES;
  static constexpr int PREV_BYTES = (ND == 3) ? S::BY * S::W * 4 : 0;
  static constexpr int WARP_SMEM = FAST_STAGES * STAGE_BYTES + PREV_BYTES + 64;
};

template <int ND, int B, int VPL>
__host__ __device__ constexpr int dfast_smem_bytes() {
  return FAST_WARPS * DFastShape<ND, B, VPL>::WARP_SMEM;
}

struct DFastArgs {
  DecompressArgs d;
  unsigned int* redo_count;
  long long* redo_list;
};

template <int ND, int B, int VPL>
__device__ __forceinline__ bool tile_interior(const Geo& g, const TileXY& c) {
  using S = Shape<ND, B, VPL>;
  return ((int64_t)(c.wx + 1) * S::W <= g.D2) && ((int64_t)(c.by + 1) * S::BY <= g.D1);
}

// producer of code planes (interior tiles only; others are skipped)
template <int ND, int B, int VPL>
struct DProducer {
  using S = Shape<ND, B, VPL>;
  using F = DFastShape<ND, B, VPL>;
  uint32_t tile;
  int zl, ez;
  const uint16_t* src;  // block 0's slice of the current plane
  int64_t plane_stride; // codes between consecutive planes of one block
  int stage;

  __device__ __forceinline__ void seek(const Geo& g, const uint16_t* codes, uint32_t nwarps) {
    while (tile < (uint32_t)g.ntiles) {
      const TileXY c = decode_tile(g, tile);
      if (tile_interior<ND, B, VPL>(g, c)) {
        const int64_t z0 = (int64_t)c.bz * S::BZ;
        ez = (int)imin64(S::BZ, g.D0 - z0);
        const int64_t bx0 = (int64_t)c.wx * F::NBLK;
        src = codes + block_start(g, c.bz, c.by, bx0, S::BZ, S::BY, S::BX, ez, S::BY);
        plane_stride = F::SLICE_CODES;
        zl = 0;
        return;
      }
      tile += nwarps;
    }
  }
  __device__ __forceinline__ void start(const Geo& g, const uint16_t* codes, uint32_t t,
                                        uint32_t nwarps) {
    tile = t;
    stage = 0;
    seek(g, codes, nwarps);
  }
  __device__ __forceinline__ void issue(const Geo& g, const uint16_t* codes,
                                        unsigned char* ring, uint64_t* bars, int lane,
                                        uint32_t nwarps) {
    if (tile >= (uint32_t)g.ntiles) return;
    unsigned char* buf = ring + stage * F::STAGE_BYTES;
    uint64_t* bar = &bars[stage];
    if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(F::NBLK * F::SLICE_BYTES));
    __syncwarp();
    // block k of the window: its whole (full) block holds ez*BY*BX codes
    if (lane < F::NBLK)
      bulk_g2s(buf + lane * F::SLOT_BYTES,
               src + (int64_t)lane * ez * F::SLICE_CODES + (int64_t)zl * plane_stride,
               (uint32_t)F::SLICE_BYTES, bar);
    if (++stage == FAST_STAGES) stage = 0;
    if (++zl >= ez) {
      tile += nwarps;
      seek(g, codes, nwarps);
    }
  }
};

template <int ND, int B, int VPL>
__device__ __forceinline__ void dfast_tile(const DFastArgs& fa, uint32_t tile, const TileXY& tc,
                                           int lane, unsigned char* ring, uint64_t* bars,
                                           DProducer<ND, B, VPL>& prod,
                                           Consumer<ND, B, VPL>& cons, uint32_t nwarps,
                                           long long& sent_acc) {
  using S = Shape<ND, B, VPL>;
  using F = DFastShape<ND, B, VPL>;
  constexpr int BZ = S::BZ, BY = S::BY, BX = S::BX, W = S::W, LPB = S::LPB;
  const DecompressArgs& a = fa.d;
  const Geo& g = a.g;
  const int R = a.q.radius;
  const uint16_t* codes = reinterpret_cast<const uint16_t*>(a.codes);

  const int64_t z0 = (int64_t)tc.bz * BZ, y0 = (int64_t)tc.by * BY;
  const int ez = (int)imin64(BZ, g.D0 - z0);
  const int xin = (lane * VPL) % BX;
  const int blk = (lane * VPL) / BX;
  const int64_t xl0 = (int64_t)tc.wx * W + lane * VPL;
  const int64_t bxg = (int64_t)tc.wx * F::NBLK + blk;
  const int64_t bi = ((int64_t)tc.bz * g.P1 + tc.by) * g.P2 + bxg;
  const int gl = lane & (LPB - 1);

  int s0 = 0;
  bool wide = false;
  long long s064 = 0;
  if (a.mode == MODE_GLOBAL) s064 = a.scalars[0];
  else if (a.mode == MODE_BLOCK) s064 = a.scalars[bi];
  else if (a.mode == MODE_EDGE) s064 = a.scalars[bi * a.nd];
  wide |= (s064 >= (1ll << 28)) || (s064 <= -(1ll << 28));
  s0 = (int)s064;
  const long long off = a.offsets[bi];
  const long long avail = imax64(0, imin64(a.counts[bi], a.n_outliers - off));

  int* const pplane = reinterpret_cast<int*>(ring + FAST_STAGES * F::STAGE_BYTES) + lane * VPL;
  if (ND == 3) {
#pragma unroll 1
    for (int yl = 0; yl < BY; ++yl) {
      if (VPL == 4) *reinterpret_cast<int4*>(pplane + yl * W) = make_int4(0, 0, 0, 0);
      else *reinterpret_cast<int2*>(pplane + yl * W) = make_int2(0, 0);
    }
  }
  int run = 0;
  bool badcode = false;
  unsigned emag = 0;  // OR of (E + 2^28): stays < 2^29 iff every |E| < 2^28
  float* orow = a.out + (z0 * g.D1 + y0) * g.D2 + xl0;

  for (int zl = 0; zl < ez; ++zl) {
    const unsigned char* slot = ring + cons.stage * F::STAGE_BYTES + blk * F::SLOT_BYTES + xin * 2;
    mbar_wait(&bars[cons.stage], cons.parity);
    int grow[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) grow[j] = 0;
#pragma unroll 1
    for (int yl = 0; yl < BY; ++yl) {
      unsigned c[VPL];
      if (VPL == 4) {
        const uint2 pk = *reinterpret_cast<const uint2*>(slot + yl * BX * 2);
        c[0] = pk.x & 0xffffu; c[1 % VPL] = pk.x >> 16;
        c[2 % VPL] = pk.y & 0xffffu; c[3 % VPL] = pk.y >> 16;
      } else {
        const unsigned pk = *reinterpret_cast<const unsigned*>(slot + yl * BX * 2);
        c[0] = pk & 0xffffu; c[1 % VPL] = pk >> 16;
      }
      int ep[VPL];
      int* pp = pplane + yl * W;
      if (ND == 3) {
        if (VPL == 4) {
          const int4 p4 = *reinterpret_cast<const int4*>(pp);
          ep[0] = p4.x; ep[1 % VPL] = p4.y; ep[2 % VPL] = p4.z; ep[3 % VPL] = p4.w;
        } else {
          const int2 p2 = *reinterpret_cast<const int2*>(pp);
          ep[0] = p2.x; ep[1 % VPL] = p2.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < VPL; ++j) ep[j] = 0;
      }
      bool anysent = false, anybig = false;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        anysent = anysent || (c[j] == 0u);
        anybig = anybig || (c[j] >= (unsigned)(2 * R));
      }
      badcode |= anybig;
      // in-lane inclusive scan of delta (no resets on the fast path)
      int h[VPL];
      h[0] = (int)c[0] - R;
#pragma unroll
      for (int j = 1; j < VPL; ++j) h[j] = h[j - 1] + ((int)c[j] - R);
      bool reset_any = false;
      unsigned before = (1u << VPL) - 1u;
      unsigned smask = 0;
      float vs[VPL];
      if (__any_sync(FULL, anysent)) {
        // rare: sentinels reset the scan to (d - s0) - E(prev plane) - G(prev row)
#pragma unroll
        for (int j = 0; j < VPL; ++j) smask |= (c[j] == 0u) ? (1u << j) : 0u;
        int tot;
        const int excl = group_excl_scan<LPB>(__popc(smask), lane, tot);
        int k = run + excl;
        int acc = 0;
        before = 0;
        bool reset = false;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          vs[j] = 0.f;
          if ((smask >> j) & 1u) {
            if (k < avail) vs[j] = a.outliers[off + k];
            ++k;
            const long long ds = quant_value(vs[j], a.q.twoeb) - s064;
            wide |= (ds >= (1ll << 28)) || (ds <= -(1ll << 28));
            acc = (int)ds - ep[j] - grow[j];
            reset = true;
          } else {
            acc += (int)c[j] - R;
          }
          if (!reset) before |= 1u << j;
          h[j] = acc;
        }
        reset_any = reset;
        run += tot;
      }
      // carry across the block's lanes: segmented (flag, value) scan
      int cv = h[VPL - 1];
      bool cf = reset_any;
#pragma unroll
      for (int o = 1; o < LPB; o <<= 1) {
        const int uv = __shfl_up_sync(FULL, cv, o);
        const bool uf = __shfl_up_sync(FULL, cf, o);
        if (gl >= o && !cf) {
          cv += uv;
          cf = uf;
        }
      }
      int pv = __shfl_up_sync(FULL, cv, 1);
      if (gl == 0) pv = 0;
      float o[VPL];
      int ev[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int hv = ((before >> j) & 1u) ? h[j] + pv : h[j];
        const int gv = hv + grow[j];
        grow[j] = gv;
        ev[j] = gv + ep[j];
        emag |= (unsigned)(ev[j] + (1 << 28));
        o[j] = __double2float_rn(__dmul_rn((double)(ev[j] + s0), a.q.twoeb));
      }
      if (smask) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if ((smask >> j) & 1u) o[j] = vs[j];
      }
      if (ND == 3) {
        if (VPL == 4) *reinterpret_cast<int4*>(pp) = make_int4(ev[0], ev[1 % VPL], ev[2 % VPL], ev[3 % VPL]);
        else *reinterpret_cast<int2*>(pp) = make_int2(ev[0], ev[1 % VPL]);
      }
      float* dst = orow + yl * g.D2;
      if (VPL == 4) *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1 % VPL], o[2 % VPL], o[3 % VPL]);
      else *reinterpret_cast<float2*>(dst) = make_float2(o[0], o[1 % VPL]);
    }
    orow += g.D1 * g.D2;
    __syncwarp();
    fence_proxy_async_smem();
    prod.issue(g, codes, ring, bars, lane, nwarps);
    cons.advance();
  }
  wide |= emag >= (1u << 29);
  if (__any_sync(FULL, wide)) {
    if (lane == 0) fa.redo_list[atomicAdd(fa.redo_count, 1u)] = tile;
    return;
  }
  const bool bad_any = group_any<LPB>(badcode, lane);
  if (xin == 0) {
    sent_acc += run;
    int st = 0;
    if (bad_any) st = 4;
    else if (run > avail) st = 5;
    else if (run < avail) st = 6;
    if (st) atomicMin(a.first_bad, ((unsigned long long)bi << 4) | (unsigned long long)st);
  }
}

template <int ND, int B, int VPL>
__global__ void __launch_bounds__(FAST_WARPS * 32, 4) dq_decompress_fast_kernel(DFastArgs fa) {
  using F = DFastShape<ND, B, VPL>;
  extern __shared__ __align__(128) unsigned char smem_dfast[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* ring = smem_dfast + (size_t)wib * F::WARP_SMEM;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + FAST_STAGES * F::STAGE_BYTES + F::PREV_BYTES);
  const Geo& g = fa.d.g;
  const uint16_t* codes = reinterpret_cast<const uint16_t*>(fa.d.codes);

  if (lane == 0) {
    for (int s = 0; s < FAST_STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint32_t nwarps = gridDim.x * FAST_WARPS;
  const uint32_t first = blockIdx.x * FAST_WARPS + wib;
  DProducer<ND, B, VPL> prod;
  prod.start(g, codes, first, nwarps);
  for (int s = 0; s < FAST_STAGES; ++s) prod.issue(g, codes, ring, bars, lane, nwarps);
  Consumer<ND, B, VPL> cons{0, 0u};
  long long sent = 0;
  for (uint32_t tile = first; tile < (uint32_t)g.ntiles; tile += nwarps) {
    const TileXY tc = decode_tile(g, tile);
    if (!tile_interior<ND, B, VPL>(g, tc)) {
      if (lane == 0) fa.redo_list[atomicAdd(fa.redo_count, 1u)] = tile;
      continue;
    }
    dfast_tile<ND, B, VPL>(fa, tile, tc, lane, ring, bars, prod, cons, nwarps, sent);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sent += __shfl_xor_sync(FULL, sent, o);
  if (lane == 0 && sent) atomicAdd(fa.d.sentinels, (unsigned long long)sent);
}

}  // namespace vlz
