// dq_1d.cuh -- fused 1-D dual-quant kernels (sm_100a).
//
// 1-D blocks are runs of b consecutive elements (b = 8 ... 256), and the
// canonical code order is the element order itself (vector.py:193-202 with one
// axis), so a warp can stream the array in rows of 256 elements -- lane l owns
// 8 consecutive elements, 1 ... 32 lanes form a block -- and every block lies
// inside one row.  Tiles of 4 rows (4 KB of float32, 2 KB of codes) reach a
// per-warp shared-memory ring through the bulk-copy engine (one
// cp.async.bulk per tile, mbarrier completion); the partial tail tile reads
// global memory directly.
//
//   compress  : exact-fast float32 prequantization (quant_fast, fp64 exact
//               path for the flagged elements), Dx by one shuffle, postquant
//               by one max per lane, outliers ranked inside the block into the
//               block's scratch slots, per-block origin/padding work at the
//               end of the row (kernel.py:124-193, vector.py:41-79 with nd=1);
//   decompress: segmented prefix sum of (code - R) across the block's lanes,
//               sentinels reset it to the verbatim value's prequantized d
//               (reconstruct.py:30-71), exact fp64 dequantization.
//
// Rows whose values leave the int32-exact range (|d| >= 2^30) are redone in
// int64 by the same warp after its loop, as the generic tiles that cover the
// row (W = 32 * vpl_for(1, b) elements each).
#pragma once

#include <type_traits>

#include "dq_compress_fast.cuh"
#include "dq_decompress.cuh"

namespace vlz {

constexpr int D1_VPL = 8;                  // elements per lane per row
constexpr int D1_ROW = 32 * D1_VPL;        // 256 elements per warp row
#ifndef VLZ_D1_ROWS
#define VLZ_D1_ROWS 4
#endif
constexpr int D1_ROWS = VLZ_D1_ROWS;       // rows per tile
constexpr int D1_TILE = D1_ROW * D1_ROWS;  // elements per tile
constexpr int D1_STAGES = 2;               // tiles in flight per warp
constexpr int D1_WARPS = 4;                // warps per CTA

// generic-kernel window of a 1-D block edge (launch.cuh vpl_for)
template <int B>
__host__ __device__ constexpr int d1_generic_w() {
  return 32 * (B == 256 ? 8 : 4);
}

struct D1Args {
  CompressArgs c;
  DecompressArgs d;
  int meta_smem;  // decompress: per-block counts/offsets/scalars also streamed by the ring
};

// decompress ring stage: codes | counts | offsets | scalars of the tile's blocks
template <int B>
struct D1DStage {
  static constexpr int MB = D1_TILE / B;  // blocks per tile
  static constexpr int CODES = 0, COUNTS = D1_TILE * 2, OFFS = COUNTS + MB * 8,
                       SCAL = OFFS + MB * 8;
  static constexpr int BYTES = (SCAL + MB * 8 + 127) / 128 * 128;
};
template <int B>
__host__ __device__ constexpr int d1d_warp_smem() {
  return D1_STAGES * D1DStage<B>::BYTES + 128;
}

template <int ELEM_BYTES>
__host__ __device__ constexpr int d1_warp_smem() {
  return (D1_STAGES * D1_TILE * ELEM_BYTES + 64 + 127) / 128 * 128;
}

// per-warp ring of whole tiles: issue / wait helpers
struct D1Ring {
  unsigned char* ring;
  uint64_t* bars;
  int stage;
  uint32_t parity;
  template <int ELEM_BYTES>
  __device__ __forceinline__ void issue(const void* base, uint32_t tile, int64_t nfull, int slot,
                                        int lane) {
    if ((int64_t)tile < nfull && lane == 0) {
      constexpr uint32_t BYTES = D1_TILE * ELEM_BYTES;
      mbar_arrive_expect_tx(&bars[slot], BYTES);
      bulk_g2s(ring + slot * BYTES,
               static_cast<const unsigned char*>(base) + (int64_t)tile * BYTES, BYTES, &bars[slot]);
    }
  }
};

// queue the generic tiles that cover row [e0, e0 + 256) for the warp's int64
// redo after its loop (slot k of warp `first` is list[k * nwarps + first])
template <int B>
__device__ __forceinline__ void d1_redo_row(uint32_t* nfail_s, long long* list, uint32_t first,
                                            uint32_t nwarps, int64_t e0, int64_t ntiles_generic,
                                            int lane) {
  constexpr int WG = d1_generic_w<B>();
  constexpr int PER = D1_ROW / WG;  // 1 or 2
  if (lane == 0) {
    uint32_t k = *nfail_s;
    for (int i = 0; i < PER; ++i) {
      const int64_t t = e0 / WG + i;
      if (t < ntiles_generic) list[(size_t)(k++) * nwarps + first] = t;
    }
    *nfail_s = k;
  }
}

// ---------------------------------------------------------------- compress
template <int B, int MODE, int K>
__global__ void __launch_bounds__(D1_WARPS * 32, 4)
    dq_compress_1d_kernel(const __grid_constant__ D1Args fa) {
  pdl_enter();
  constexpr int VPL = D1_VPL;
  constexpr int LPB = B / VPL;  // lanes per block: 1 ... 32
  constexpr unsigned MAGIC_BITS = 0x4B400000u;
  constexpr int WS = d1_warp_smem<4>();
  extern __shared__ __align__(128) unsigned char smem_d1c[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const CompressArgs& a = fa.c;
  const QP& q = a.q;
  const int R = q.radius;
  const unsigned span = (unsigned)(2 * R - 2);
  const int64_t N = a.g.D2;
  const int64_t ntiles = (N + D1_TILE - 1) / D1_TILE;
  const int64_t nfull = N / D1_TILE;
  D1Ring rg{smem_d1c + (size_t)wib * WS,
            reinterpret_cast<uint64_t*>(smem_d1c + (size_t)wib * WS + D1_STAGES * D1_TILE * 4), 0,
            0u};
  uint32_t* const nfail_s = reinterpret_cast<uint32_t*>(rg.bars + D1_STAGES);  // tiles left for the tail
  if (lane == 0) {
    for (int s = 0; s < D1_STAGES; ++s) mbar_init(&rg.bars[s], 1);
    fence_mbar_init();
    *nfail_s = 0u;
  }
  __syncwarp();
  const uint32_t nwarps = gridDim.x * D1_WARPS;
  const uint32_t first = blockIdx.x * D1_WARPS + wib;
  for (int s = 0; s < D1_STAGES; ++s) rg.issue<4>(a.in, first + s * nwarps, nfull, s, lane);
  if (blockIdx.x == 0 && wib == 0) ws_reset_warp(a.init, lane);  // (behind the first loads)

  const int xin = (lane * VPL) % B;  // position of element 0 inside its block
  const int gl = lane & (LPB - 1);
  const bool lead = xin == 0;
  KAcc<K> gacc;
  long long gcnt = 0;

  for (uint32_t tile = first; (int64_t)tile < ntiles; tile += nwarps) {
    const bool full = (int64_t)tile < nfull;
    const float* sm = reinterpret_cast<const float*>(rg.ring + rg.stage * D1_TILE * 4);
    if (full) mbar_wait(&rg.bars[rg.stage], rg.parity);
    // one row of 256 elements; FULL rows (whole tiles) carry no bounds checks
    auto row = [&](auto full_tag, int r, int64_t e0) {
        constexpr bool WHOLE = decltype(full_tag)::value;  // (FULL is the warp mask)
        const int64_t el = e0 + lane * VPL;
        const int nvalid = WHOLE ? VPL : (int)imax64(0, imin64(VPL, N - el));
        float v[VPL];
        if (WHOLE) {
          const float4 p0 = *reinterpret_cast<const float4*>(sm + r * D1_ROW + lane * VPL);
          const float4 p1 = *reinterpret_cast<const float4*>(sm + r * D1_ROW + lane * VPL + 4);
          v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
          v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j) v[j] = j < nvalid ? __ldg(a.in + el + j) : 0.f;
        }
        // ---- float32 fast prequantization; nb = biased bits of n
        unsigned nb[VPL];
        bool allok = true;
#pragma unroll
        for (int j = 0; j < VPL; j += 2) {
          const float2 qq = __fmul2_rn(make_float2(v[j], v[j + 1]), make_float2(q.inv32, q.inv32));
          const float2 rr = __fadd2_rn(qq, make_float2(12582912.0f, 12582912.0f));
          nb[j] = __float_as_uint(rr.x);
          nb[j + 1] = __float_as_uint(rr.y);
          const float2 rn = __fadd2_rn(rr, make_float2(-12582912.0f, -12582912.0f));
          const float2 e = __ffma2_rn(rn, make_float2(-1.0f, -1.0f), qq);
          const float2 lim = __ffma2_rn(make_float2(fabsf(qq.x), fabsf(qq.y)),
                                        make_float2(-q.kq, -q.kq), make_float2(q.lim0, q.lim0));
          allok = allok && (fabsf(e.x) < lim.x) && (fabsf(e.y) < lim.y);
        }
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (j >= nvalid) nb[j] = MAGIC_BITS;  // beyond the array: d = 0
        unsigned badm = 0;
        bool wide = false;
        if (!__all_sync(FULL, allok)) {
          // rare: exact float64 re-evaluation of the flagged elements
          unsigned smk = 0;
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            bool ok;
            quant_fast(v[j], q, ok);
            if (!ok && j < nvalid) smk |= 1u << j;
          }
          while (smk) {
            const int j = __ffs(smk) - 1;
            smk &= smk - 1;
            float vj = v[0];
#pragma unroll
            for (int k = 1; k < VPL; ++k) vj = (j == k) ? v[k] : vj;
            bool bj, ovf;
            const int nj = quant_exact(vj, q, bj, ovf);
#pragma unroll
            for (int k = 0; k < VPL; ++k) nb[k] = (j == k) ? (unsigned)nj + MAGIC_BITS : nb[k];
            if (bj) badm |= 1u << j;
            if (ovf) {
              const unsigned long long fi = (unsigned long long)(el + j);
              ws_wait(a.init);
              if (!isfinite(vj)) atomicMin(a.first_nonfinite, fi);
              atomicMin(a.first_overflow, fi);
            }
            wide |= (nj >= (1 << 30)) || (nj <= -(1 << 30));
          }
        }
        if (__any_sync(FULL, wide)) {  // int32 differences could wrap: int64 redo
          d1_redo_row<B>(nfail_s, a.redo_list, first, nwarps, e0, a.g.ntiles, lane);
          return;
        }
        // ---- Dx inside the block (the block head reads the zero halo)
        unsigned left = __shfl_up_sync(FULL, nb[VPL - 1], 1);
        if (lead) left = MAGIC_BITS;
        unsigned u[VPL];
        unsigned umax = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int dl = (int)(nb[j] - (j ? nb[j - 1] : left));
          u[j] = (unsigned)(dl + (R - 1));
          umax = (j == 0 && lead) ? umax : (u[j] > umax ? u[j] : umax);
        }
        const int d_origin = (int)(nb[0] - MAGIC_BITS);  // meaningful on block leads
        const bool bad_origin = badm & 1u;
        // ---- padding statistic of the block (block / edge) and the origin code
        int64_t s0 = 0;
        if (MODE == MODE_BLOCK) {
          long long ls = 0;
          int mn = 0x7fffffff, mx = (int)0x80000000;
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            if (j < nvalid) {
              const int d = (int)(nb[j] - MAGIC_BITS);
              if (K == 3) ls += d;
              mn = d < mn ? d : mn;
              mx = d > mx ? d : mx;
            }
          }
          const int64_t sum = K == 3 ? group_sum<LPB>(ls) : 0;
          const int gmn = K == 1 ? group_min<LPB>(mn) : 0;
          const int gmx = K == 2 ? group_max<LPB>(mx) : 0;
          const int64_t cnt = imax64(0, imin64(B, N - (e0 + (lane - gl) * VPL)));
          s0 = stat_value(K, sum, cnt, gmn, gmx);
        } else if (MODE == MODE_EDGE) {
          s0 = d_origin;  // the block's dim-0 face is its origin alone
        }
        // origin code: delta d - s0 (finding 1); under *:global the provisional
        // code of s0 = 0, which the scan kernel rewrites once s0 is known
        bool o_out = false;  // origin outlier (non-global policies)
        unsigned ocode = 0;
        if (lead) {
          const int64_t dd = (int64_t)d_origin - s0;
          o_out = bad_origin || dd > (int64_t)(R - 1) || dd < -(int64_t)(R - 1);
          ocode = o_out ? 0u : (unsigned)(dd + R);
        }
        // ---- outliers: code 0, ranked inside the block (origin handled apart)
        unsigned cadd = 0x00010001u;  // common path: code = u + 1 per packed half
        int tot = 0;
        const unsigned orig_mask = lead ? 1u : 0u;
        if (__any_sync(FULL, umax > span || (badm & ~orig_mask) != 0u)) {
          unsigned om = 0;
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            const bool isorig = (j == 0) && lead;
            const bool o = !isorig && j < nvalid && (u[j] > span || ((badm >> j) & 1u));
            om |= o ? (1u << j) : 0u;
          }
#pragma unroll
          for (int j = 0; j < VPL; ++j) u[j] = ((om >> j) & 1u) ? 0u : u[j] + 1u;
          if (lead) u[0] = ocode;
          cadd = 0u;
          const int excl = group_excl_scan<LPB>(__popc(om), lane, tot);
          const int64_t bstart = (e0 + (lane - gl) * VPL);  // block start = its first element
          float* slot = a.scratch + scratch_base(a.scratch_dense, bstart, bstart / B) + 1;
          const int slim = scratch_limit(a.scratch_dense);
          int k = excl;  // rank among the block's non-origin outliers
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if ((om >> j) & 1u) {
              if (k < slim) slot[k] = v[j];
              ++k;
            }
        } else if (lead) {
          u[0] = 0u;  // packed below without a carry; the origin code is patched in
        }
        // ---- codes (element order is the canonical order in 1-D); the
        // origin code (0 for an outlier origin) replaces the lead's low half
        if (nvalid == VPL) {
          uint32_t w[VPL / 2];
#pragma unroll
          for (int k = 0; k < VPL / 2; ++k) w[k] = __byte_perm(u[2 * k], u[2 * k + 1], 0x5410) + cadd;
          if (lead) w[0] = (w[0] & 0xffff0000u) | ocode;
          *reinterpret_cast<uint4*>(a.codes + el) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (j < nvalid)
              a.codes[el + j] = (j == 0 && lead) ? (uint16_t)ocode : (uint16_t)(u[j] + (cadd & 1u));
        }
        // ---- block end (the block lies inside this row)
        if (lead && nvalid > 0) {
          const int64_t bi = el / B;
          int64_t total = tot;
          if (MODE != MODE_GLOBAL) {
            if (o_out) {
              a.scratch[scratch_base(a.scratch_dense, el, bi)] = v[0];
              total += 1;
            }
            if (MODE == MODE_BLOCK || MODE == MODE_EDGE) a.scalars[bi] = s0;
            a.counts[bi] = total;
          } else {
            a.counts[bi] = pack_origin(total, d_origin, bad_origin);
            a.origin_vals[bi] = v[0];
          }
        }
        // ---- global statistics (in-bounds elements)
        if (MODE == MODE_GLOBAL) {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (j < nvalid) gacc.add((int)(nb[j] - MAGIC_BITS));
          gcnt += nvalid;
        }
        };
    if (full) {
#pragma unroll 1
      for (int r = 0; r < D1_ROWS; ++r)
        row(std::true_type{}, r, (int64_t)tile * D1_TILE + r * D1_ROW);
    } else {
#pragma unroll 1
      for (int r = 0; r < D1_ROWS; ++r) {
        const int64_t e0 = (int64_t)tile * D1_TILE + r * D1_ROW;
        if (e0 >= N) break;  // tail tile: warp-uniform
        row(std::false_type{}, r, e0);
      }
    }
    // release the stage, refill it D1_STAGES tiles ahead
    __syncwarp();
    fence_proxy_async_smem();
    rg.issue<4>(a.in, tile + D1_STAGES * nwarps, nfull, rg.stage, lane);
    if (++rg.stage == D1_STAGES) {
      rg.stage = 0;
      rg.parity ^= 1u;
    }
  }

  if (MODE == MODE_GLOBAL) commit_global_stats(a, gacc.sum, gcnt, gacc.mn, gacc.mx, lane);
  // tail: rows whose |d| reached 2^30 (usually none) as generic int64 tiles
  __syncwarp();
  const uint32_t nfail = *nfail_s;
  if (nfail)
    compress_redo_tail<1, B, (B == 256 ? 8 : 4), MODE>(a, first, nwarps, nfail, lane, nullptr);
}

// -------------------------------------------------------------- decompress
#ifndef VLZ_D1D_MINB
#define VLZ_D1D_MINB 5  // CTAs per SM the 1-D decompress register budget targets
                        // (4: 116 regs, 0.44 ms at 1-D 256M b=256; 5: 0.41 ms; 6: 0.51 ms)
#endif
template <int B>
__global__ void __launch_bounds__(D1_WARPS * 32, VLZ_D1D_MINB)
    dq_decompress_1d_kernel(const __grid_constant__ D1Args fa) {
  pdl_enter();
  constexpr int VPL = D1_VPL;
  constexpr int LPB = B / VPL;
  using DS = D1DStage<B>;
  constexpr int WS = d1d_warp_smem<B>();
  extern __shared__ __align__(128) unsigned char smem_d1d[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const DecompressArgs& a = fa.d;
  const int R = a.q.radius;
  const uint16_t* codes = reinterpret_cast<const uint16_t*>(a.codes);
  const int64_t N = a.g.D2;
  const int64_t ntiles = (N + D1_TILE - 1) / D1_TILE;
  const int64_t nfull = N / D1_TILE;
  D1Ring rg{smem_d1d + (size_t)wib * WS,
            reinterpret_cast<uint64_t*>(smem_d1d + (size_t)wib * WS + D1_STAGES * DS::BYTES), 0,
            0u};
  // generic tiles left for the int64 tail, per warp (a word of the barrier area)
  uint32_t* const s_nfail = reinterpret_cast<uint32_t*>(rg.bars + D1_STAGES) - wib;
  if (lane == 0) s_nfail[wib] = 0u;
  const bool meta = fa.meta_smem != 0;
  const bool scal_blocks = a.mode == MODE_BLOCK || a.mode == MODE_EDGE;
  // one stage: the tile's codes and, with `meta`, its blocks' counts /
  // offsets (/ scalars) -- one mbarrier transaction
  auto issue = [&](uint32_t t, int slot) {
    if ((int64_t)t < nfull && lane == 0) {
      unsigned char* dst = rg.ring + slot * DS::BYTES;
      const uint32_t bytes = D1_TILE * 2 + (meta ? DS::MB * 8 * (scal_blocks ? 3 : 2) : 0);
      mbar_arrive_expect_tx(&rg.bars[slot], bytes);
      bulk_g2s(dst + DS::CODES, codes + (int64_t)t * D1_TILE, D1_TILE * 2, &rg.bars[slot]);
      if (meta) {
        const int64_t b0 = (int64_t)t * DS::MB;
        bulk_g2s(dst + DS::COUNTS, a.counts + b0, DS::MB * 8, &rg.bars[slot]);
        bulk_g2s(dst + DS::OFFS, a.offsets + b0, DS::MB * 8, &rg.bars[slot]);
        if (scal_blocks) bulk_g2s(dst + DS::SCAL, a.scalars + b0, DS::MB * 8, &rg.bars[slot]);
      }
    }
  };
  if (lane == 0) {
    for (int s = 0; s < D1_STAGES; ++s) mbar_init(&rg.bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint32_t nwarps = gridDim.x * D1_WARPS;
  const uint32_t first = blockIdx.x * D1_WARPS + wib;
  for (int s = 0; s < D1_STAGES; ++s) issue(first + s * nwarps, s);

  const int xin = (lane * VPL) % B;
  const int gl = lane & (LPB - 1);
  const bool lead = xin == 0;
  long long sent_acc = 0;
  const long long s0g = a.mode == MODE_GLOBAL ? a.scalars[0] : 0;

  for (uint32_t tile = first; (int64_t)tile < ntiles; tile += nwarps) {
    const bool full = (int64_t)tile < nfull;
    const unsigned char* stg = rg.ring + rg.stage * DS::BYTES;
    const uint16_t* sm = reinterpret_cast<const uint16_t*>(stg + DS::CODES);
    const long long* smc = reinterpret_cast<const long long*>(stg + DS::COUNTS);
    const long long* smo = reinterpret_cast<const long long*>(stg + DS::OFFS);
    const long long* sms = reinterpret_cast<const long long*>(stg + DS::SCAL);
    if (full) mbar_wait(&rg.bars[rg.stage], rg.parity);
    auto row = [&](auto full_tag, int r, int64_t e0) {
        constexpr bool WHOLE = decltype(full_tag)::value;  // (FULL is the warp mask)
        const int64_t el = e0 + lane * VPL;
        const int nvalid = WHOLE ? VPL : (int)imax64(0, imin64(VPL, N - el));
        const int64_t bi = el / B;
        const bool bvalid = nvalid > 0;
        // block metadata (every lane of a block reads the same words): from
        // the stage when the ring streams it, else from global memory
        const int lb = (r * D1_ROW + lane * VPL) / B;  // block within the tile
        const bool msm = WHOLE && meta;
        long long s064 = s0g, cnt = 0;
        if (bvalid) {
          if (scal_blocks) s064 = msm ? sms[lb] : a.scalars[bi];
          cnt = msm ? smc[lb] : a.counts[bi];
        }
        auto offset_of = [&]() -> long long { return msm ? smo[lb] : a.offsets[bi]; };
        unsigned c[VPL];
        if (WHOLE) {
          const uint4 pk = *reinterpret_cast<const uint4*>(sm + r * D1_ROW + lane * VPL);
          c[0] = pk.x & 0xffffu; c[1] = pk.x >> 16; c[2] = pk.y & 0xffffu; c[3] = pk.y >> 16;
          c[4] = pk.z & 0xffffu; c[5] = pk.z >> 16; c[6] = pk.w & 0xffffu; c[7] = pk.w >> 16;
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j) c[j] = j < nvalid ? (unsigned)codes[el + j] : (unsigned)R;
        }
        // sentinels other than the block origins decide the path: an origin
        // sentinel only re-bases its block (d = d_s + prefix of later deltas)
        unsigned cmin = lead ? c[1] : c[0], cmax = c[0];
#pragma unroll
        for (int j = 1; j < VPL; ++j) {
          cmin = c[j] < cmin ? c[j] : cmin;
          cmax = c[j] > cmax ? c[j] : cmax;
        }
        if (!lead) cmin = c[0] < cmin ? c[0] : cmin;
        bool wide = (s064 >= (1ll << 30)) || (s064 <= -(1ll << 30));
        const int s0 = (int)s064;
        int sb = s0;  // base of the block's prefix
        int h[VPL];
        int pvc = 0;
        unsigned smask = 0;
        int run = 0;  // sentinels of this lane's block in this row (block total on the lead)
        float vs[VPL];
        if (!__any_sync(FULL, cmin == 0u)) {
          // common path: prefix of delta across the block's lanes
          if (lead && c[0] == 0u && bvalid) {  // origin sentinel
            const long long off = offset_of();
            const long long avail = imax64(0, imin64(cnt, n_outliers_of(a) - off));
            vs[0] = avail > 0 ? a.outliers[off] : 0.f;
            bool qok;
            const int nq = quant_fast(vs[0], a.q, qok);
            const long long ds = qok ? (long long)nq : quant_value(vs[0], a.q.twoeb);
            wide |= (ds >= (1ll << 30)) || (ds <= -(1ll << 30));
            sb = (int)ds;
            c[0] = (unsigned)R;  // delta 0: the base carries the origin
            smask = 1u;
            run = 1;
          }
          if (LPB > 1) sb = __shfl_sync(FULL, sb, lane & ~(LPB - 1));
          h[0] = (int)c[0] - R;
#pragma unroll
          for (int j = 1; j < VPL; ++j) h[j] = h[j - 1] + ((int)c[j] - R);
          int inc = h[VPL - 1];
#pragma unroll
          for (int o = 1; o < LPB; o <<= 1) {
            const int uu = __shfl_up_sync(FULL, inc, o);
            if (gl >= o) inc += uu;
          }
          pvc = inc - h[VPL - 1];
        } else {
          // rare: sentinels reset the prefix to d_s - s0 (d = s0 + prefix)
#pragma unroll
          for (int j = 0; j < VPL; ++j) smask |= (c[j] == 0u && j < nvalid) ? (1u << j) : 0u;
          const int excl = group_excl_scan<LPB>(__popc(smask), lane, run);
          long long off = 0, avail = 0;
          if (smask) {
            off = offset_of();
            avail = imax64(0, imin64(cnt, n_outliers_of(a) - off));
          }
          int k = excl;
          int acc = 0;
          unsigned before = 0;
          bool reset = false;
          // the row's outlier loads first (in flight together), then the resets
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            vs[j] = 0.f;
            if ((smask >> j) & 1u) {
              if (k < avail) vs[j] = __ldg(a.outliers + off + k);
              ++k;
            }
          }
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            if ((smask >> j) & 1u) {
              bool qok;
              const int nq = quant_fast(vs[j], a.q, qok);
              const long long ds = qok ? (long long)nq : quant_value(vs[j], a.q.twoeb);
              wide |= (ds >= (1ll << 30)) || (ds <= -(1ll << 30));
              acc = (int)ds - s0;
              reset = true;
            } else {
              acc += (int)c[j] - R;
            }
            if (!reset) before |= 1u << j;
            h[j] = acc;
          }
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
        int dmax = 0, dmin = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int dv = sb + h[j] + pvc;
          dmax = max(dmax, dv);
          dmin = min(dmin, dv);
          const double dd = __dadd_rn(__hiloint2double(0x43300000, dv ^ (int)0x80000000),
                                      -4503601774854144.0);
          o[j] = __double2float_rn(__dmul_rn(dd, a.q.twoeb));
        }
        wide |= dmax >= (1 << 30) || dmin < -(1 << 30);
        if (__any_sync(FULL, wide)) {  // leave the row to the int64 kernel
          d1_redo_row<B>(&s_nfail[wib], a.redo_list, first, nwarps, e0, a.g.ntiles, lane);
          return;
        }
        if (smask) {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if ((smask >> j) & 1u) o[j] = vs[j];
        }
        if (nvalid == VPL) {
          float4* dst = reinterpret_cast<float4*>(a.out + el);
          dst[0] = make_float4(o[0], o[1], o[2], o[3]);
          dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
          for (int j = 0; j < VPL; ++j)
            if (j < nvalid) a.out[el + j] = o[j];
        }
        // block end: sentinel count against the stored outliers, code range
        const bool bad_any = group_any<LPB>(cmax >= (unsigned)(2 * R), lane);
        if (lead && bvalid) {
          sent_acc += run;
          // (a block with no stored and no found outliers needs no offset)
          const long long off = (cnt != 0 || run != 0) ? offset_of() : 0;
          const long long avail = imax64(0, imin64(cnt, n_outliers_of(a) - off));
          int st = 0;
          if (bad_any) st = 4;
          else if (run > avail) st = 5;
          else if (run < avail) st = 6;
          if (st) atomicMin(a.first_bad, ((unsigned long long)bi << 4) | (unsigned long long)st);
        }
        };
    if (full) {
#pragma unroll 1
      for (int r = 0; r < D1_ROWS; ++r)
        row(std::true_type{}, r, (int64_t)tile * D1_TILE + r * D1_ROW);
    } else {
#pragma unroll 1
      for (int r = 0; r < D1_ROWS; ++r) {
        const int64_t e0 = (int64_t)tile * D1_TILE + r * D1_ROW;
        if (e0 >= N) break;
        row(std::false_type{}, r, e0);
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
    issue(tile + D1_STAGES * nwarps, rg.stage);
    if (++rg.stage == D1_STAGES) {
      rg.stage = 0;
      rg.parity ^= 1u;
    }
  }
  // tail: rows outside the int32-exact range (usually none) as generic int64 tiles
  __syncwarp();
  const uint32_t nfail = s_nfail[wib];
  if (nfail)
    decompress_redo_tail<1, B, (B == 256 ? 8 : 4)>(a, first, nwarps, nfail, lane, nullptr, sent_acc);
  decompress_finish(a, sent_acc, lane);
}

}  // namespace vlz
