#include <cstdlib>
// k_decompress.cu -- reconstruction kernel instantiations and dispatch.
//   fast shapes (3-D b=8/16, 2-D b=8/16), uint16 codes, aligned buffers:
//       dq_decompress_fast_kernel (int32 with exactness check; its warps redo
//       flagged tiles in int64 themselves and the last CTA settles the status)
//   everything else: dq_decompress_kernel (int64)
#include "dq_decompress_fast.cuh"
#include "launch.cuh"
#include "launch_compress.cuh"  // encode_tiled

namespace vlz {

// codes of a grid of full 8x8x8 blocks as a (64, 8, nblocks) uint16 tensor:
// box (64, 1, 16) = plane zl of 16 consecutive blocks, 128-byte swizzle
static bool make_code_map(CUtensorMap* m, const void* codes, int64_t nblocks) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[3] = {64, 8, (cuuint64_t)nblocks};
  const cuuint64_t strides[2] = {128, 1024};
  const cuuint32_t box[3] = {64, 1, 16};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(codes), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ND, int B>
constexpr bool has_dfast() {
  return (ND == 3 || ND == 2) && (B == 8 || B == 16 || B == 32 || B == 64);
}

template <int ND, int B, int VPL>
static cudaError_t run_d(bool u32, const DecompressArgs& a, cudaStream_t st) {
  constexpr int smem = 4 * plane_smem_bytes<ND, B, VPL>();
  if constexpr (has_dfast<ND, B>()) {
    const bool aligned = !u32 && (a.g.D2 % 4 == 0) &&
                         ((reinterpret_cast<uintptr_t>(a.codes) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0) &&
                         a.redo_list != nullptr && a.g.ntiles < (1ll << 30) &&
                         (a.q.twoeb < 1e300);
    if (aligned) {
      DFastArgs fa{};
      fa.d = a;
      const bool edges = edge_tile_count<ND, B, VPL>(a.g) > 0;
      auto kern = edges ? dq_decompress_fast_kernel<ND, B, VPL, true>
                        : dq_decompress_fast_kernel<ND, B, VPL, false>;
      int fsmem = edges ? dfast_smem_bytes<ND, B, VPL, true>() : dfast_smem_bytes<ND, B, VPL, false>();
      if constexpr (ND == 3 && B == 8 && VPL == 4) {
        // every block full (block b starts at b * 512): TMA tensor loads
        if (a.g.D0 % 8 == 0 && a.g.D1 % 8 == 0 && a.g.D2 % 8 == 0 &&
            a.g.nblocks < (1ll << 31) && make_code_map(&fa.tmap, a.codes, a.g.nblocks)) {
          kern = edges ? dq_decompress_tma_kernel<ND, B, VPL, true>
                       : dq_decompress_tma_kernel<ND, B, VPL, false>;
          fsmem = edges ? dtma_smem_bytes<ND, B, VPL, true>() : dtma_smem_bytes<ND, B, VPL, false>();
        }
      }
      int per_sm = 0;
      cudaError_t e = occupancy(kern, FAST_WARPS * 32, fsmem, per_sm);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) per_sm = 1;
      {  // (experiments: fewer resident CTAs per SM than the occupancy allows)
        static const int cap = [] { const char* e = std::getenv("VLZ_DGRID_PER_SM"); return e ? std::atoi(e) : 0; }();
        if (cap > 0 && cap < per_sm) per_sm = cap;
      }
      int64_t grid = (int64_t)per_sm * num_sms();
      const int64_t need = (a.g.ntiles + FAST_WARPS - 1) / FAST_WARPS;
      if (grid > need) grid = need;
      if (grid < 1) grid = 1;
      const bool t = g_timing.load(std::memory_order_relaxed);
      if (t) timing_mark(TK_DECOMPRESS, true, st);
      e = launch_k(kern, (unsigned)grid, FAST_WARPS * 32, fsmem, st, fa);
      if (e != cudaSuccess) return e;
      if (t) timing_mark(TK_DECOMPRESS, false, st);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return cudaGetLastError();
    }
  }
  if (u32) return launch_tiles(dq_decompress_kernel<ND, B, VPL, uint32_t>, a.g.ntiles, smem, st, a);
  return launch_tiles(dq_decompress_kernel<ND, B, VPL, uint16_t>, a.g.ntiles, smem, st, a);
}

cudaError_t launch_decompress(int nd, int B, bool u32, const DecompressArgs& a, cudaStream_t st) {
  if (nd == 1 && d1_fast_decompress_ok(u32, a)) return launch_decompress_1d(B, a, st);
  if (nd == 1) {
    switch (B) {
      case 8: return run_d<1, 8, 4>(u32, a, st);
      case 16: return run_d<1, 16, 4>(u32, a, st);
      case 32: return run_d<1, 32, 4>(u32, a, st);
      case 64: return run_d<1, 64, 4>(u32, a, st);
      case 256: return run_d<1, 256, 8>(u32, a, st);
    }
  } else if (nd == 2) {
    switch (B) {
      case 8: return run_d<2, 8, 4>(u32, a, st);
      case 16: return run_d<2, 16, 4>(u32, a, st);
      case 32: return run_d<2, 32, 4>(u32, a, st);
      case 64: return run_d<2, 64, 4>(u32, a, st);
    }
  } else if (nd == 3) {
    switch (B) {
      case 8: return run_d<3, 8, VLZ_VPL_3D8>(u32, a, st);
      case 16: return run_d<3, 16, VLZ_DVPL_3D16>(u32, a, st);
      case 32: return run_d<3, 32, 2>(u32, a, st);
      case 64: return run_d<3, 64, 2>(u32, a, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace vlz
