// dq_decompress_fast.cuh -- production fused reconstruction kernel (sm_100a).
//
// Same warp tiling and recurrences as dq_decompress.cuh (H: segmented scan of
// delta along x with resets at sentinels, G = H + G(prev row),
// E = G + E(prev plane), d = E + s0, out = float32(fl64(2 d eb))), specialised
// for the throughput shapes (3-D b=8/16, 2-D b=8/16) and interior tiles:
//
//  * each lane streams its own VPL codes of every row of a plane into a
//    per-warp shared ring with cp.async (LDGSTS), DSTAGES planes ahead
//    and across tile boundaries; the [row][lane] layout makes the later
//    vector LDS conflict-free and needs no cross-lane barrier;
//  * arithmetic is wrapping int32.  It is exact whenever |s0| < 2^27 and every
//    computed |d| < 2^27: by induction over the traversal order, the true
//    E = d - s0 of each element is a signed sum of 7 earlier exact values
//    (each < 2^28) plus a code (< 2^15), so it lies in (-2^31, 2^31) where
//    congruence mod 2^32 is equality.  The kernel checks exactly that and
//    hands any tile that fails it to the int64 kernel
//    (dq_decompress_kernel<..., LIST=true>);
//  * edge tiles (partial last block row / window) run inline in grids that
//    have them (EDGES variants), the same recurrence instantiated with EDGE:
//    codes are fetched synchronously into a slot of their own (partial blocks
//    are not 4-byte aligned) and positions beyond the array read as "delta 0"
//    -- they trail every valid position of their block in x and y, so they
//    never feed one;
//  * output rows leave with 16-byte stores straight from registers; rows are
//    unrolled by two so that the dequantisation of one row overlaps the
//    scans of the next;
//  * grids of full 8x8x8 blocks take the TMA variant (dq_decompress_tma_kernel):
//    one tensor load per plane brings 16 block planes, 128-byte swizzled.
#pragma once

#ifndef VLZ_BIG_BATCH
#define VLZ_BIG_BATCH 1  // b >= 32 decompress: sentinel-free 8-row stages as one batch
                         // (512^3 b=64 799 -> 318 us, b=32 260 -> 180 us; 2-D unchanged)
#endif
#ifndef VLZ_SENT_PAIRED
#define VLZ_SENT_PAIRED 1  // sentinel quotients in paired FP32 (0: scalar quant_fast; A/B on B200: C5 equal, stress 78.1 vs 78.2 us)
#endif

#include "dq_compress_fast.cuh"
#include "dq_decompress.cuh"

namespace vlz {

#ifndef VLZ_DQ_I2F
#define VLZ_DQ_I2F 0  // 1: int->double by I2F.F64 instead of the magic-number DADD
#endif

// ring depth of the decompress producers (planes in flight per warp)
#ifndef VLZ_DSTAGES
#define VLZ_DSTAGES 2
#endif
constexpr int DSTAGES = VLZ_DSTAGES;

template <int ND, int B, int VPL>
struct DFastShape {
  using S = Shape<ND, B, VPL>;
  static constexpr int NBLK = S::W / S::BX;         // blocks per window
  static constexpr int SLICE_CODES = S::BY * S::BX;  // codes per block plane
  // stage layout [row][lane] x VPL codes: every lane copies (cp.async) and
  // later reads its own VPL codes of each row -- conflict-free, no barrier
  static constexpr int LANE_BYTES = VPL * 2;
  // a plane streams in SPLIT stages of STAGE_ROWS rows (b >= 32: 8-row
  // stages, so the ring stays small enough for several CTAs per SM)
  static constexpr int SPLIT = S::BY >= 32 ? S::BY / 8 : 1;
  static constexpr int STAGE_ROWS = S::BY / SPLIT;
  static constexpr int STAGE_BYTES = STAGE_ROWS * 32 * LANE_BYTES;
  static constexpr int PLANE_BYTES = S::BY * 32 * LANE_BYTES;
  static constexpr int PREV_BYTES = (ND == 3) ? S::BY * S::W * 4 : 0;
  // edge tiles fill a whole plane of codes synchronously into a slot of their
  // own, so the ring of interior planes keeps streaming underneath
  static constexpr int EDGE_OFF = DSTAGES * STAGE_BYTES + PREV_BYTES;
  static constexpr int WARP_SMEM = EDGE_OFF + PLANE_BYTES;
  // per-warp footprint of a kernel variant (the edge slot only when it has edge tiles)
  __host__ __device__ static constexpr int warp_smem(bool edges) { return edges ? WARP_SMEM : EDGE_OFF; }
};

template <int ND, int B, int VPL, bool EDGES = true>
__host__ __device__ constexpr int dfast_smem_bytes() {
  return FAST_WARPS * DFastShape<ND, B, VPL>::warp_smem(EDGES);
}

struct DFastArgs {
  CUtensorMap tmap;  // TMA path: codes as (64, BZ, nblocks) uint16, box (64, 1, NBLK)
  DecompressArgs d;
};

template <int ND, int B, int VPL>
__device__ __forceinline__ bool tile_interior(const Geo& g, const TileXY& c) {
  using S = Shape<ND, B, VPL>;
  return ((int64_t)(c.wx + 1) * S::W <= g.D2) && ((int64_t)(c.by + 1) * S::BY <= g.D1);
}

// per-lane producer of code planes (interior tiles only; others are skipped).
// Every issue() commits exactly one cp.async group (possibly empty), so
// cp.async.wait_group<DSTAGES-1> always retires the plane being consumed.
template <int ND, int B, int VPL>
struct DProducer {
  using S = Shape<ND, B, VPL>;
  using F = DFastShape<ND, B, VPL>;
  static constexpr bool TMAP = false;
  uint32_t tile;
  int zl, ez, part;
  const uint16_t* src;  // this lane's codes in plane 0, row 0 of the current tile
  int stage;

  __device__ __forceinline__ void seek(const Geo& g, const uint16_t* codes, uint32_t nwarps,
                                       int lane) {
    while (tile < (uint32_t)g.ntiles) {
      const TileXY c = decode_tile(g, tile);
      if (tile_interior<ND, B, VPL>(g, c)) {
        const int64_t z0 = (int64_t)c.bz * S::BZ;
        ez = (int)imin64(S::BZ, g.D0 - z0);
        const int blk = (lane * VPL) / S::BX;
        const int64_t bx0 = (int64_t)c.wx * F::NBLK;
        // consecutive full blocks of the window: ez * BY * BX codes each
        src = codes + block_start(g, c.bz, c.by, bx0, S::BZ, S::BY, S::BX, ez, S::BY) +
              (int64_t)blk * ez * F::SLICE_CODES + (lane * VPL) % S::BX;
        zl = 0;
        part = 0;
        return;
      }
      tile += nwarps;
    }
  }
  __device__ __forceinline__ void start(const Geo& g, const uint16_t* codes, uint32_t t,
                                        uint32_t nwarps, int lane) {
    tile = t;
    stage = 0;
    seek(g, codes, nwarps, lane);
  }
  __device__ __forceinline__ void issue(const Geo& g, const uint16_t* codes,
                                        unsigned char* ring, uint32_t nwarps, int lane) {
    if (tile < (uint32_t)g.ntiles) {
      unsigned char* dst = ring + stage * F::STAGE_BYTES + lane * F::LANE_BYTES;
      const uint16_t* s = src + (int64_t)zl * F::SLICE_CODES + part * F::STAGE_ROWS * S::BX;
#pragma unroll
      for (int yl = 0; yl < F::STAGE_ROWS; ++yl)
        cp_async<F::LANE_BYTES>(dst + yl * 32 * F::LANE_BYTES, s + yl * S::BX);
      if (++part == F::SPLIT) {
        part = 0;
        if (++zl >= ez) {
          tile += nwarps;
          seek(g, codes, nwarps, lane);
        }
      }
    }
    cp_async_commit();
    if (++stage == DSTAGES) stage = 0;
  }
};

// TMA producer (3-D b=8 grids whose blocks are all full, so block b's codes
// start at b * 512): one tensor load per plane brings plane zl of the
// window's NBLK consecutive blocks, [block][64 codes], 128-byte swizzled so
// that the consumer's row reads (all lanes on the same row of different
// blocks) are conflict-free.  mbarrier ring as in the compress kernel.
template <int ND, int B, int VPL>
struct DTProducer {
  using S = Shape<ND, B, VPL>;
  using F = DFastShape<ND, B, VPL>;
  static constexpr bool TMAP = true;
  uint32_t tile;
  int zl, ez;
  int b0;  // first block of the window
  int stage;
  __device__ __forceinline__ void seek(const Geo& g, uint32_t nwarps) {
    while (tile < (uint32_t)g.ntiles) {
      const TileXY c = decode_tile(g, tile);
      if (tile_interior<ND, B, VPL>(g, c)) {
        ez = (int)imin64(S::BZ, g.D0 - (int64_t)c.bz * S::BZ);
        b0 = (int)(((int64_t)c.bz * g.P1 + c.by) * g.P2 + (int64_t)c.wx * F::NBLK);
        zl = 0;
        return;
      }
      tile += nwarps;
    }
  }
  __device__ __forceinline__ void start(const Geo& g, uint32_t t, uint32_t nwarps) {
    tile = t;
    stage = 0;
    seek(g, nwarps);
  }
  __device__ __forceinline__ void issue(const Geo& g, const CUtensorMap* tmap,
                                        unsigned char* ring, uint64_t* bars, int lane,
                                        uint32_t nwarps) {
    if (tile >= (uint32_t)g.ntiles) return;
    if (lane == 0) {
      uint64_t* bar = &bars[stage];
      mbar_arrive_expect_tx(bar, (uint32_t)F::STAGE_BYTES);
      tma_load_3d(ring + stage * F::STAGE_BYTES, tmap, 0, zl, b0, bar);
    }
    if (++stage == DSTAGES) stage = 0;
    if (++zl >= ez) {
      tile += nwarps;
      seek(g, nwarps);
    }
  }
};

template <int ND, int B, int VPL, bool EDGE, class Prod>
__device__ __forceinline__ void dfast_tile(const DFastArgs& fa, uint32_t tile, const TileXY& tc,
                                           int lane, unsigned char* ring, uint64_t* bars,
                                           Prod& prod, Consumer<ND, B, VPL, DSTAGES>& cons,
                                           uint32_t nwarps, long long& sent_acc,
                                           uint32_t* nfail_s) {
  constexpr bool TMAP = Prod::TMAP;
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
  // edge tiles: valid rows, valid columns of this lane's block (<= 0: the
  // block lies beyond the array and the lane only carries zeros)
  const int ey = EDGE ? (int)imin64(BY, g.D1 - y0) : BY;
  const int ex = EDGE ? (int)imax64(0, imin64(BX, g.D2 - bxg * BX)) : BX;
  const bool bvalid = !EDGE || ex > 0;

  int s0 = 0;
  bool wide = false;
  long long s064 = 0;
  long long off = 0, avail = 0;
  if (bvalid) {
    if (a.mode == MODE_GLOBAL) s064 = a.scalars[0];
    else if (a.mode == MODE_BLOCK) s064 = a.scalars[bi];
    else if (a.mode == MODE_EDGE) s064 = a.scalars[bi * a.nd];
    off = a.offsets[bi];
    avail = imax64(0, imin64(a.counts[bi], n_outliers_of(a) - off));
  }
  wide |= (s064 >= (1ll << 27)) || (s064 <= -(1ll << 27));
  s0 = (int)s064;

  // The outermost prefix state is primed with s0 (3-D: the previous-plane
  // state starts at s0; 1-D/2-D: the previous-row state does), so d = E + s0
  // comes out of the recurrence directly and a sentinel resets the x-scan to
  // d_s - E'(prev plane) - G(prev row) with no s0 term.
  int* const pplane = reinterpret_cast<int*>(ring + DSTAGES * F::STAGE_BYTES) + lane * VPL;
  if (ND == 3) {
#pragma unroll 1
    for (int yl = 0; yl < BY; ++yl) {
      if (VPL == 4) *reinterpret_cast<int4*>(pplane + yl * W) = make_int4(s0, s0, s0, s0);
      else *reinterpret_cast<int2*>(pplane + yl * W) = make_int2(s0, s0);
    }
  }
  int run = 0;
  unsigned cmax_run = 0u;  // running max of the tile's codes (>= 2R: corrupt stream)
  int dmax = 0, dmin = 0;  // range of every d of the tile (exact iff within +-2^27)
  float* orow = a.out + (z0 * g.D1 + y0) * g.D2 + xl0;
  const unsigned char* const slot0 = ring + (EDGE ? F::EDGE_OFF : 0) + lane * F::LANE_BYTES;

  const uint16_t* esrc = nullptr;
  if (EDGE) esrc = codes + block_start(g, tc.bz, tc.by, bxg, BZ, BY, BX, ez, ey) + xin;
  for (int zl = 0; zl < ez; ++zl) {
    const unsigned char* slot;
    if (EDGE) {
      // synchronous fill of stage 0: invalid positions read as code R
      unsigned char* fill = ring + F::EDGE_OFF + lane * F::LANE_BYTES;
      const uint16_t* zs = esrc + (int64_t)zl * ey * ex;
#pragma unroll
      for (int yl = 0; yl < BY; ++yl) {
        unsigned v[VPL];
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          v[j] = (yl < ey && xin + j < ex) ? (unsigned)zs[yl * ex + j] : (unsigned)R;
        if (VPL == 4)
          *reinterpret_cast<uint2*>(fill + yl * 32 * F::LANE_BYTES) =
              make_uint2(v[0] | (v[1 % VPL] << 16), v[2 % VPL] | (v[3 % VPL] << 16));
        else
          *reinterpret_cast<unsigned*>(fill + yl * 32 * F::LANE_BYTES) = v[0] | (v[1 % VPL] << 16);
      }
      slot = slot0;
    } else if (TMAP) {
      slot = ring + cons.stage * F::STAGE_BYTES;  // swizzled [block][64 codes]
      mbar_wait(&bars[cons.stage], cons.parity);
    } else {
      slot = slot0 + cons.stage * F::STAGE_BYTES;
      cp_async_wait<DSTAGES - 1>();
    }
    int grow[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) grow[j] = (ND == 3) ? 0 : s0;
    int* pp = pplane;
    float* dst = orow;
#pragma unroll 2
    for (int yl = 0; yl < ey; ++yl) {
      if constexpr (!EDGE && !TMAP && F::SPLIT > 1) {
        if (yl > 0 && yl % F::STAGE_ROWS == 0) {  // next stage of this plane
          prod.issue(g, codes, ring, nwarps, lane);
          cons.advance();
          slot = slot0 + cons.stage * F::STAGE_BYTES;
          cp_async_wait<DSTAGES - 1>();
        }
#if VLZ_BIG_BATCH
        // b >= 32: few tiles (512^3 b=64 is one warp per block, ~3.5 warps
        // per SM), so a row's dependent chain -- the x-scan's shuffles, the
        // plane load, the dequantisation -- is exposed.  A stage without
        // sentinels runs its STAGE_ROWS rows as one batch: the x-scans are
        // independent and interleave; only the y/z accumulation is sequential.
        if (yl % F::STAGE_ROWS == 0 && yl + F::STAGE_ROWS <= ey) {
          constexpr int RB = F::STAGE_ROWS;
          unsigned cb[RB][VPL];
          unsigned cmn = 0xffffffffu;
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const unsigned char* rp = slot + r * 32 * F::LANE_BYTES;
            if (VPL == 4) {
              const uint2 pk = *reinterpret_cast<const uint2*>(rp);
              cb[r][0] = pk.x & 0xffffu; cb[r][1 % VPL] = pk.x >> 16;
              cb[r][2 % VPL] = pk.y & 0xffffu; cb[r][3 % VPL] = pk.y >> 16;
            } else {
              const unsigned pk = *reinterpret_cast<const unsigned*>(rp);
              cb[r][0] = pk & 0xffffu; cb[r][1 % VPL] = pk >> 16;
            }
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
              cmn = cb[r][j] < cmn ? cb[r][j] : cmn;
              cmax_run = cb[r][j] > cmax_run ? cb[r][j] : cmax_run;
            }
          }
          if (!__any_sync(FULL, cmn == 0u)) {
            int hb[RB][VPL], inc[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              hb[r][0] = (int)cb[r][0] - R;
#pragma unroll
              for (int j = 1; j < VPL; ++j) hb[r][j] = hb[r][j - 1] + ((int)cb[r][j] - R);
              inc[r] = hb[r][VPL - 1];
            }
#pragma unroll
            for (int o = 1; o < LPB; o <<= 1) {
#pragma unroll
              for (int r = 0; r < RB; ++r) {
                const int u = __shfl_up_sync(FULL, inc[r], o);
                if (gl >= o) inc[r] += u;
              }
            }
#pragma unroll
            for (int r = 0; r < RB; ++r) {
              const int pvc = inc[r] - hb[r][VPL - 1];  // exclusive lane carry
              int ep[VPL];
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
              float o[VPL];
              int dv[VPL];
#pragma unroll
              for (int j = 0; j < VPL; ++j) {
                const int gv = hb[r][j] + grow[j] + pvc;
                grow[j] = gv;
                dv[j] = gv + ep[j];
                const double dd = __dadd_rn(__hiloint2double(0x43300000, dv[j] ^ (int)0x80000000),
                                            -4503601774854144.0);
                o[j] = __double2float_rn(__dmul_rn(dd, a.q.twoeb));
                dmax = max(dmax, dv[j]);
                dmin = min(dmin, dv[j]);
              }
              if (ND == 3) {
                if (VPL == 4) *reinterpret_cast<int4*>(pp) = make_int4(dv[0], dv[1 % VPL], dv[2 % VPL], dv[3 % VPL]);
                else *reinterpret_cast<int2*>(pp) = make_int2(dv[0], dv[1 % VPL]);
              }
              pp += W;
              if (VPL == 4) *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1 % VPL], o[2 % VPL], o[3 % VPL]);
              else *reinterpret_cast<float2*>(dst) = make_float2(o[0], o[1 % VPL]);
              dst += g.D2;
            }
            slot += RB * 32 * F::LANE_BYTES;
            yl += RB - 1;
            continue;
          }
        }
#endif
      }
      unsigned c[VPL];
      const unsigned char* rowp = slot;
      if (TMAP && !EDGE)  // block blk, row yl: 16-byte chunk yl of line blk, XOR-swizzled
        rowp = slot + blk * 128 + (((yl ^ blk) & 7) << 4) + (xin * 2);
      if (VPL == 4) {
        const uint2 pk = *reinterpret_cast<const uint2*>(rowp);
        c[0] = pk.x & 0xffffu; c[1 % VPL] = pk.x >> 16;
        c[2 % VPL] = pk.y & 0xffffu; c[3 % VPL] = pk.y >> 16;
      } else {
        const unsigned pk = *reinterpret_cast<const unsigned*>(rowp);
        c[0] = pk & 0xffffu; c[1 % VPL] = pk >> 16;
      }
      if (!TMAP || EDGE) slot += 32 * F::LANE_BYTES;
      int ep[VPL];
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
      // sentinel test by a min over the row's codes; the code-range check
      // only keeps a running max, tested once per tile
      unsigned cmin = c[0];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        cmin = c[j] < cmin ? c[j] : cmin;
        cmax_run = c[j] > cmax_run ? c[j] : cmax_run;
      }
      const bool anysent = cmin == 0u;
      int h[VPL];
      int pvc = 0;  // carry from earlier lanes not yet in h (common path)
      unsigned smask = 0;
      float vs[VPL];
      if (!__any_sync(FULL, anysent)) {
        // common path: plain prefix of delta within the block's lanes
        h[0] = (int)c[0] - R;
#pragma unroll
        for (int j = 1; j < VPL; ++j) h[j] = h[j - 1] + ((int)c[j] - R);
        int inc = h[VPL - 1];
#pragma unroll
        for (int o = 1; o < LPB; o <<= 1) {
          const int u = __shfl_up_sync(FULL, inc, o);
          if (gl >= o) inc += u;
        }
        pvc = inc - h[VPL - 1];  // exclusive carry, added with grow below (one IADD3)
      } else {
        // rare: sentinels reset the scan to d_s - E'(prev plane) - G(prev row)
#pragma unroll
        for (int j = 0; j < VPL; ++j) smask |= (c[j] == 0u) ? (1u << j) : 0u;
        int tot;
        const int excl = group_excl_scan<LPB>(__popc(smask), lane, tot);
        // all of the row's outlier loads first (independent, predicated
        // addresses: the j-th sentinel of the lane is outlier run + excl +
        // popc(smask below j)), so they are in flight together
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const long long kj = run + excl + __popc(smask & ((1u << j) - 1u));
          vs[j] = (((smask >> j) & 1u) && kj < avail) ? __ldg(a.outliers + off + kj) : 0.f;
        }
        // d of every sentinel value, branch free: the compress side's
        // exact-fast quotient in paired FP32 (equal to round_half_away(fl64(v
        // / 2eb)) whenever it reports ok) ...
        int dsv[VPL];
        unsigned okm = 0;
#if VLZ_SENT_PAIRED
#pragma unroll
        for (int j = 0; j < VPL; j += 2) {
          const float2 qq = __fmul2_rn(make_float2(vs[j], vs[j + 1]),
                                       make_float2(a.q.inv32, a.q.inv32));
          const float2 r = __fadd2_rn(qq, make_float2(12582912.0f, 12582912.0f));
          const float2 rn = __fadd2_rn(r, make_float2(-12582912.0f, -12582912.0f));
          const float2 e = __ffma2_rn(rn, make_float2(-1.0f, -1.0f), qq);
          const float2 lim = __ffma2_rn(make_float2(fabsf(qq.x), fabsf(qq.y)),
                                        make_float2(-a.q.kq, -a.q.kq),
                                        make_float2(a.q.lim0, a.q.lim0));
          dsv[j] = __float_as_int(r.x) - 0x4B400000;
          dsv[j + 1] = __float_as_int(r.y) - 0x4B400000;
          okm |= (fabsf(e.x) < lim.x ? 1u : 0u) << j;
          okm |= (fabsf(e.y) < lim.y ? 2u : 0u) << j;
        }
#else
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          bool qok;
          dsv[j] = quant_fast(vs[j], a.q, qok);
          okm |= qok ? (1u << j) : 0u;
        }
#endif
        // ... and the fp64 division for the sentinels it rejects (rare)
        const unsigned need = smask & ~okm;
        if (__any_sync(FULL, need != 0u)) {
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            if ((need >> j) & 1u) {
              const long long ds = quant_value(vs[j], a.q.twoeb);
              wide |= (ds >= (1ll << 27)) || (ds <= -(1ll << 27));
              dsv[j] = (int)ds;
            }
          }
        }
        int acc = 0;
        unsigned before = 0;
        bool reset = false;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const bool sj = (smask >> j) & 1u;
          acc = sj ? dsv[j] - ep[j] - grow[j] : acc + ((int)c[j] - R);
          reset = reset || sj;
          before |= reset ? 0u : (1u << j);
          h[j] = acc;
        }
        run += tot;
        int cv = h[VPL - 1];
        bool cf = reset;
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
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if ((before >> j) & 1u) h[j] += pv;
      }
      float o[VPL];
      int dv[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int gv = h[j] + grow[j] + pvc;
        grow[j] = gv;
        dv[j] = gv + ep[j];  // = d (primed state)
#if VLZ_DQ_I2F
        const double dd = (double)dv[j];
#else
        // float64(d) without the quarter-rate I2F: 2^52 + 2^31 + d has d in
        // its low word exactly, one DADD removes the offset (exact)
        const double dd = __dadd_rn(__hiloint2double(0x43300000, dv[j] ^ (int)0x80000000),
                                    -4503601774854144.0);
#endif
        o[j] = __double2float_rn(__dmul_rn(dd, a.q.twoeb));
      }
#pragma unroll
      for (int j = 0; j < VPL; j += 2) {
        dmax = max(dmax, max(dv[j], dv[j + 1 < VPL ? j + 1 : j]));
        dmin = min(dmin, min(dv[j], dv[j + 1 < VPL ? j + 1 : j]));
      }
      if (smask) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if ((smask >> j) & 1u) o[j] = vs[j];
      }
      if (ND == 3) {
        if (VPL == 4) *reinterpret_cast<int4*>(pp) = make_int4(dv[0], dv[1 % VPL], dv[2 % VPL], dv[3 % VPL]);
        else *reinterpret_cast<int2*>(pp) = make_int2(dv[0], dv[1 % VPL]);
      }
      pp += W;
      // (D2 % 4 == 0: a lane's VPL columns are all inside or all outside)
      if (!EDGE || xl0 < g.D2) {
        if (VPL == 4) *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1 % VPL], o[2 % VPL], o[3 % VPL]);
        else *reinterpret_cast<float2*>(dst) = make_float2(o[0], o[1 % VPL]);
      }
      dst += g.D2;
    }
    orow += g.D1 * g.D2;
    if constexpr (TMAP && !EDGE) {
      __syncwarp();
      fence_proxy_async_smem();
      prod.issue(g, &fa.tmap, ring, bars, lane, nwarps);
      cons.advance();
    } else if constexpr (!EDGE && !TMAP) {
      prod.issue(g, codes, ring, nwarps, lane);
      cons.advance();
    }
  }
  wide |= dmax >= (1 << 27) || dmin < -(1 << 27);
  if (__any_sync(FULL, wide)) {
    if (lane == 0) {  // slot k of this warp: redone in int64 after the loop
      const uint32_t k = *nfail_s;
      a.redo_list[(size_t)k * nwarps + tile % nwarps] = tile;
      *nfail_s = k + 1;
    }
    return;
  }
  const bool bad_any = group_any<LPB>(cmax_run >= (unsigned)(2 * R), lane);
  if (xin == 0 && bvalid) {
    sent_acc += run;
    int st = 0;
    if (bad_any) st = 4;
    else if (run > avail) st = 5;
    else if (run < avail) st = 6;
    if (st) atomicMin(a.first_bad, ((unsigned long long)bi << 4) | (unsigned long long)st);
  }
}

// EDGES: the grid has edge tiles (processed inline, at the cost of the
// registers of a second instantiation of the tile body); grids without them
// take the lean variant
template <int ND, int B, int VPL, bool EDGES>
__global__ void __launch_bounds__(FAST_WARPS * 32,
                                  ((EDGES && B == 8) || (ND == 3 && (B == 16 || B == 64))) ? 3 : 4)
    dq_decompress_fast_kernel(const __grid_constant__ DFastArgs fa) {
  pdl_enter();
  using F = DFastShape<ND, B, VPL>;
  extern __shared__ __align__(128) unsigned char smem_dfast[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* ring = smem_dfast + (size_t)wib * F::warp_smem(EDGES);
  // tiles left for the int64 tail of this warp: a register (a static shared
  // array would push 3 CTAs of the b = 16 shape past the 196 KB carve-out step
  // and halve their L1: C4 b=16 decompress 178 -> 199 us)
  uint32_t nfail_reg = 0u;
  uint32_t* const s_nfail = &nfail_reg - wib;
  static_assert(!Shape<ND, B, VPL>::PLANE_SMEM ||
                    dfast_smem_bytes<ND, B, VPL, false>() >= plane_smem_bytes<ND, B, VPL>(),
                "tail plane");
  const Geo& g = fa.d.g;
  const uint16_t* codes = reinterpret_cast<const uint16_t*>(fa.d.codes);

  const uint32_t nwarps = gridDim.x * FAST_WARPS;
  const uint32_t first = blockIdx.x * FAST_WARPS + wib;
  DProducer<ND, B, VPL> prod;
  prod.start(g, codes, first, nwarps, lane);
  for (int s = 0; s < DSTAGES; ++s) prod.issue(g, codes, ring, nwarps, lane);
  Consumer<ND, B, VPL, DSTAGES> cons{0, 0u};
  long long sent = 0;
  for (uint32_t tile = first; tile < (uint32_t)g.ntiles; tile += nwarps) {
    const TileXY tc = decode_tile(g, tile);
    if (tile_interior<ND, B, VPL>(g, tc))
      dfast_tile<ND, B, VPL, false>(fa, tile, tc, lane, ring, nullptr, prod, cons, nwarps, sent, &s_nfail[wib]);
    else if constexpr (EDGES)  // same recurrence, synchronous fill (the ring keeps streaming)
      dfast_tile<ND, B, VPL, true>(fa, tile, tc, lane, ring, nullptr, prod, cons, nwarps, sent, &s_nfail[wib]);
  }
  // tail: tiles outside the int32-exact range (usually none), redone in int64
  // by the warp that met them; shapes whose int64 plane lives in shared memory
  // take turns on the CTA's whole allocation (every ring is idle by then)
  __syncwarp();
#if VLZ_DTAIL_MODE == 0
  const uint32_t nfail = 0u;
#else
  const uint32_t nfail = __shfl_sync(FULL, s_nfail[wib], 0);  // (lane 0 keeps the count)
#endif
  if constexpr (Shape<ND, B, VPL>::PLANE_SMEM) {
    if (__syncthreads_or(nfail != 0u)) {
      for (int w = 0; w < FAST_WARPS; ++w) {
        if (w == wib && nfail)
          decompress_redo_tail<ND, B, VPL>(fa.d, first, nwarps, nfail, lane,
                                           reinterpret_cast<long long*>(smem_dfast), sent);
        __syncthreads();
      }
    }
  } else if (nfail) {
    decompress_redo_tail<ND, B, VPL>(fa.d, first, nwarps, nfail, lane, nullptr, sent);
  }
  decompress_finish(fa.d, sent, lane);
}

// TMA variant (DTProducer): per-warp [stages | previous plane | barriers],
// 1024-byte aligned for the 128-byte swizzle
template <int ND, int B, int VPL, bool EDGES>
struct DTmaShape {
  using F = DFastShape<ND, B, VPL>;
  static constexpr int BAR_OFF = F::warp_smem(EDGES);  // stages | previous plane [| edge slot]
  static constexpr int WARP_SMEM = (BAR_OFF + 64 + 1023) / 1024 * 1024;
};
template <int ND, int B, int VPL, bool EDGES>
__host__ __device__ constexpr int dtma_smem_bytes() {
  return FAST_WARPS * DTmaShape<ND, B, VPL, EDGES>::WARP_SMEM + 1024;
}

#ifndef VLZ_DTMA_MINB
#define VLZ_DTMA_MINB 4  // CTAs per SM of the lean TMA decompress kernel (102 regs; 5 CTAs at 95 regs measured
                         // -1.7 % on one box and +3 % on two others, 6 spills)
#endif
template <int ND, int B, int VPL, bool EDGES>
__global__ void __launch_bounds__(FAST_WARPS * 32, EDGES ? 3 : VLZ_DTMA_MINB)
    dq_decompress_tma_kernel(const __grid_constant__ DFastArgs fa) {
  pdl_enter();
  using T = DTmaShape<ND, B, VPL, EDGES>;
  extern __shared__ __align__(1024) unsigned char smem_dtma[];
  // align by an offset from the shared array itself (keeps the accesses LDS/STS)
  unsigned char* base = smem_dtma + ((1024u - (smem_u32(smem_dtma) & 1023u)) & 1023u);
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* ring = base + (size_t)wib * T::WARP_SMEM;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + T::BAR_OFF);
  // tiles left for the int64 tail, per warp (a word of the barrier area: a
  // static array would pad the 1024-byte aligned dynamic allocation by 1 KB)
  uint32_t* const s_nfail = reinterpret_cast<uint32_t*>(bars + DSTAGES) - wib;
  if (lane == 0) s_nfail[wib] = 0u;
  const Geo& g = fa.d.g;
  if (lane == 0) {
    for (int s = 0; s < DSTAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0) prefetch_tmap(&fa.tmap);

  const uint32_t nwarps = gridDim.x * FAST_WARPS;
  const uint32_t first = blockIdx.x * FAST_WARPS + wib;
  DTProducer<ND, B, VPL> prod;
  prod.start(g, first, nwarps);
  for (int s = 0; s < DSTAGES; ++s) prod.issue(g, &fa.tmap, ring, bars, lane, nwarps);
  Consumer<ND, B, VPL, DSTAGES> cons{0, 0u};
  long long sent = 0;
  for (uint32_t tile = first; tile < (uint32_t)g.ntiles; tile += nwarps) {
    const TileXY tc = decode_tile(g, tile);
    if (tile_interior<ND, B, VPL>(g, tc))
      dfast_tile<ND, B, VPL, false>(fa, tile, tc, lane, ring, bars, prod, cons, nwarps, sent, &s_nfail[wib]);
    else if constexpr (EDGES)
      dfast_tile<ND, B, VPL, true>(fa, tile, tc, lane, ring, bars, prod, cons, nwarps, sent, &s_nfail[wib]);
  }
  // tail: tiles outside the int32-exact range (usually none), redone in int64
  // by the warp that met them; shapes whose int64 plane lives in shared memory
  // take turns on the CTA's whole allocation (every ring is idle by then)
  __syncwarp();
#if VLZ_DTAIL_MODE == 0
  const uint32_t nfail = 0u;
#else
  const uint32_t nfail = __shfl_sync(FULL, s_nfail[wib], 0);  // (lane 0 keeps the count)
#endif
  if constexpr (Shape<ND, B, VPL>::PLANE_SMEM) {
    if (__syncthreads_or(nfail != 0u)) {
      for (int w = 0; w < FAST_WARPS; ++w) {
        if (w == wib && nfail)
          decompress_redo_tail<ND, B, VPL>(fa.d, first, nwarps, nfail, lane,
                                           reinterpret_cast<long long*>(base), sent);
        __syncthreads();
      }
    }
  } else if (nfail) {
    decompress_redo_tail<ND, B, VPL>(fa.d, first, nwarps, nfail, lane, nullptr, sent);
  }
  decompress_finish(fa.d, sent, lane);
}

// edge tiles: the last window of every block row when W does not divide D2,
// and every window of the last block row when BY does not divide D1
template <int ND, int B, int VPL>
__host__ __device__ inline int64_t edge_tile_count(const Geo& g) {
  using S = Shape<ND, B, VPL>;
  const bool xp = (g.D2 % S::W) != 0, yp = (g.D1 % S::BY) != 0;
  return (xp ? g.P0 * g.P1 : 0) + (yp ? g.P0 * (g.NW - (xp ? 1 : 0)) : 0);
}

}  // namespace vlz
