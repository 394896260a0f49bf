// k_1d.cu -- launch of the fused 1-D kernels (dq_1d.cuh).
#include "dq_1d.cuh"
#include "launch.cuh"

#include <cstdlib>

namespace vlz {

template <typename Kern>
static cudaError_t d1_grid(Kern kern, int smem, int64_t ntiles1, int64_t& grid) {
  int per_sm = 0;
  cudaError_t e = occupancy(kern, D1_WARPS * 32, smem, per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  grid = (int64_t)per_sm * num_sms();
  const int64_t need = (ntiles1 + D1_WARPS - 1) / D1_WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  return cudaSuccess;
}

template <int B, int MODE, int K>
static cudaError_t run_c1d(const CompressArgs& a, cudaStream_t st) {
  D1Args fa{};
  fa.c = a;
  auto kern = dq_compress_1d_kernel<B, MODE, K>;
  constexpr int smem = D1_WARPS * d1_warp_smem<4>();
  int64_t grid = 0;
  cudaError_t e = d1_grid(kern, smem, (a.g.D2 + D1_TILE - 1) / D1_TILE, grid);
  if (e != cudaSuccess) return e;
  const bool t = g_timing.load(std::memory_order_relaxed);
  if (t) timing_mark(TK_COMPRESS, true, st);
  e = launch_k(kern, (unsigned)grid, D1_WARPS * 32, smem, st, fa);
  if (e != cudaSuccess) return e;
  if (t) timing_mark(TK_COMPRESS, false, st);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int B, int MODE>
static cudaError_t run_c1d_k(const CompressArgs& a, cudaStream_t st) {
  if (MODE == MODE_ZERO) return run_c1d<B, MODE, 0>(a, st);
  if (a.q.kind == 1) return run_c1d<B, MODE, 1>(a, st);
  if (a.q.kind == 2) return run_c1d<B, MODE, 2>(a, st);
  return run_c1d<B, MODE, 3>(a, st);
}

template <int B>
static cudaError_t run_c1d_b(int mode, const CompressArgs& a, cudaStream_t st) {
  switch (mode) {
    case MODE_ZERO: return run_c1d_k<B, MODE_ZERO>(a, st);
    case MODE_GLOBAL: return run_c1d_k<B, MODE_GLOBAL>(a, st);
    case MODE_BLOCK: return run_c1d_k<B, MODE_BLOCK>(a, st);
    default: return run_c1d_k<B, MODE_EDGE>(a, st);
  }
}

// arrays below this many elements take the generic kernel (VLZ_D1_MIN_N
// overrides it for A/B runs).  At C1 (2^20 elements) the fused kernels run
// 12.5 / 12.8 us against 13.9 / 14.8 us for the generic ones (with the redo
// launch, round 1, the fused path lost there and the threshold was 2^22).
static int64_t d1_min_n() {
  static const int64_t v = [] {
    const char* e = std::getenv("VLZ_D1_MIN_N");  // A/B runs of the threshold
    return e ? (int64_t)std::atoll(e) : (1ll << 19);
  }();
  return v;
}

bool d1_fast_compress_ok(const CompressArgs& a) {
  return a.g.D2 >= d1_min_n() && a.redo_list != nullptr && (reinterpret_cast<uintptr_t>(a.in) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.codes) & 15) == 0 && a.g.D2 < (1ll << 40) &&
         (a.g.D2 + D1_TILE - 1) / D1_TILE < (1ll << 31);
}

cudaError_t launch_compress_1d(int B, int mode, const CompressArgs& a, cudaStream_t st) {
  switch (B) {
    case 8: return run_c1d_b<8>(mode, a, st);
    case 16: return run_c1d_b<16>(mode, a, st);
    case 32: return run_c1d_b<32>(mode, a, st);
    case 64: return run_c1d_b<64>(mode, a, st);
    case 256: return run_c1d_b<256>(mode, a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int B>
static cudaError_t run_d1d(const DecompressArgs& a, cudaStream_t st) {
  D1Args fa{};
  fa.d = a;
  // the ring also streams counts / offsets / block scalars when aligned
  const bool scal = a.mode == MODE_BLOCK || a.mode == MODE_EDGE;
  fa.meta_smem = ((reinterpret_cast<uintptr_t>(a.counts) & 15) == 0) &&
                 ((reinterpret_cast<uintptr_t>(a.offsets) & 15) == 0) &&
                 (!scal || (reinterpret_cast<uintptr_t>(a.scalars) & 15) == 0);
  auto kern = dq_decompress_1d_kernel<B>;
  constexpr int smem = D1_WARPS * d1d_warp_smem<B>();
  int64_t grid = 0;
  cudaError_t e = d1_grid(kern, smem, (a.g.D2 + D1_TILE - 1) / D1_TILE, grid);
  if (e != cudaSuccess) return e;
  const bool t = g_timing.load(std::memory_order_relaxed);
  if (t) timing_mark(TK_DECOMPRESS, true, st);
  e = launch_k(kern, (unsigned)grid, D1_WARPS * 32, smem, st, fa);
  if (e != cudaSuccess) return e;
  if (t) timing_mark(TK_DECOMPRESS, false, st);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

bool d1_fast_decompress_ok(bool u32, const DecompressArgs& a) {
  return a.g.D2 >= d1_min_n() && !u32 && a.redo_list != nullptr && (reinterpret_cast<uintptr_t>(a.codes) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 && a.g.D2 < (1ll << 40) &&
         (a.g.D2 + D1_TILE - 1) / D1_TILE < (1ll << 31) && a.q.twoeb < 1e300;
}

cudaError_t launch_decompress_1d(int B, const DecompressArgs& a, cudaStream_t st) {
  switch (B) {
    case 8: return run_d1d<8>(a, st);
    case 16: return run_d1d<16>(a, st);
    case 32: return run_d1d<32>(a, st);
    case 64: return run_d1d<64>(a, st);
    case 256: return run_d1d<256>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlz
