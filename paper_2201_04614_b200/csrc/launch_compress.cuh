// launch_compress.cuh -- per-shape launch of the compress kernels.
//   fast shapes (2-D / 3-D, b = 8 ... 64) with 16-byte aligned rows:
//       dq_compress_fast_kernel (its warps redo int32-unsafe tiles in int64 themselves)
//   everything else: dq_compress_kernel (generic, uint32/int64 per tile)
#pragma once

#include <cstdint>
#include <cstdlib>

#include "dq_compress_fast.cuh"
#include "launch.cuh"

namespace vlz {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return EncodeTiledFn(nullptr);
  }();
  return fn;
}

// input float32 array as a (D2, D1, D0) uint32 tensor (bit-exact copies), box
// (W, rows, 1): part of one plane of one tile; out-of-bounds elements read as zero
inline bool make_plane_map(CUtensorMap* m, const float* in, const Geo& g, int W, int BY) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  if (g.D0 > 0xffffffffll || g.D1 > 0xffffffffll || g.D2 > 0xffffffffll) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.D2, (cuuint64_t)g.D1, (cuuint64_t)g.D0};
  const cuuint64_t strides[2] = {(cuuint64_t)g.D2 * 4, (cuuint64_t)(g.D1 * g.D2) * 4};
  const cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)BY, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<float*>(in), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ND, int B>
constexpr bool has_fast() {
  return (ND == 3 || ND == 2) && (B == 8 || B == 16 || B == 32 || B == 64);
}

template <int ND, int B, int VPL, int MODE, int K>
cudaError_t run_compress_shape(const CompressArgs& a, cudaStream_t st) {
  constexpr int smem = 4 * plane_smem_bytes<ND, B, VPL>();
  if constexpr (has_fast<ND, B>()) {
    const bool aligned = (a.g.D2 % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.in) & 15) == 0);
    FastArgs fa{};
    if (aligned && a.redo_list != nullptr && a.g.ntiles < (1ll << 30) &&
        make_plane_map(&fa.tmap, a.in, a.g, Shape<ND, B, VPL>::W,
                       FastShape<ND, B, VPL>::STAGE_ROWS)) {
      auto kern = dq_compress_fast_kernel<ND, B, VPL, MODE, K>;
      constexpr int fsmem = fast_smem_bytes<ND, B, VPL>();
      int per_sm = 0;
      cudaError_t e = occupancy(kern, FAST_WARPS * 32, fsmem, per_sm);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) per_sm = 1;
      {  // (experiments: fewer resident CTAs per SM than the occupancy allows)
        static const int cap = [] { const char* e = std::getenv("VLZ_CGRID_PER_SM"); return e ? std::atoi(e) : 0; }();
        if (cap > 0 && cap < per_sm) per_sm = cap;
      }
      int64_t grid = (int64_t)per_sm * num_sms();
      const int64_t need = (a.g.ntiles + FAST_WARPS - 1) / FAST_WARPS;
      if (grid > need) grid = need;
      if (grid < 1) grid = 1;
      fa.c = a;
      const bool t = g_timing.load(std::memory_order_relaxed);
      if (t) timing_mark(TK_COMPRESS, true, st);
      e = launch_k(kern, (unsigned)grid, FAST_WARPS * 32, fsmem, st, fa);
      if (e != cudaSuccess) return e;
      if (t) timing_mark(TK_COMPRESS, false, st);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return cudaGetLastError();
    }
  }
  return launch_tiles(dq_compress_kernel<ND, B, VPL, MODE>, a.g.ntiles, smem, st, a);
}

template <int ND, int B, int VPL, int MODE>
cudaError_t run_compress_k(int kind, const CompressArgs& a, cudaStream_t st) {
  if constexpr (has_fast<ND, B>()) {
    if (kind == 1) return run_compress_shape<ND, B, VPL, MODE, 1>(a, st);
    if (kind == 2) return run_compress_shape<ND, B, VPL, MODE, 2>(a, st);
    return run_compress_shape<ND, B, VPL, MODE, 3>(a, st);
  } else {
    return run_compress_shape<ND, B, VPL, MODE, 3>(a, st);
  }
}

template <int ND, int B, int VPL>
cudaError_t run_compress_b(int mode, const CompressArgs& a, cudaStream_t st) {
  switch (mode) {
    case MODE_ZERO: return run_compress_shape<ND, B, VPL, MODE_ZERO, 0>(a, st);
    case MODE_GLOBAL: return run_compress_k<ND, B, VPL, MODE_GLOBAL>(a.q.kind, a, st);
    case MODE_BLOCK: return run_compress_k<ND, B, VPL, MODE_BLOCK>(a.q.kind, a, st);
    default: return run_compress_k<ND, B, VPL, MODE_EDGE>(a.q.kind, a, st);
  }
}

}  // namespace vlz
