// launch.cuh -- host-side launch helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <type_traits>

#include "dq_decompress.cuh"

#ifndef VLZ_VPL_3D8
#define VLZ_VPL_3D8 4  // columns per lane for 3-D b=8 tiles (window 32*VPL)
#endif
#ifndef VLZ_DVPL_3D16
#define VLZ_DVPL_3D16 4  // columns per lane of the 3-D b=16 decompress tiles
                         // (C4 b=16: 4 -> 0.183 ms, 2 -> 0.206 ms)
#endif
#ifndef VLZ_CVPL_3D16
#define VLZ_CVPL_3D16 2  // ... of the 3-D b=16 compress tiles
#endif
#ifndef VLZ_VPL_C3D8
#define VLZ_VPL_C3D8 4  // ... for the 3-D b=8 compress tiles (one block row per lane)
#endif

namespace vlz {

// total kernel launches issued by the library (evidence for bench.py)
extern std::atomic<long long> g_launches;

int num_sms();

extern std::atomic<int> g_timing;  // per-kernel CUDA-event timing on (vlz_timing)
// Resident CTAs per SM of a kernel at (block, dynamic smem), with the
// dynamic-smem opt-in done first -- both once per (kernel, device, config):
// the driver queries cost microseconds per call, which launch-bound small
// arrays would pay on every compress/decompress.
cudaError_t occupancy_cached(const void* kern, int block, int smem, int& per_sm);
template <typename... KArgs>
inline cudaError_t occupancy(void (*kern)(KArgs...), int block, int smem, int& per_sm) {
  return occupancy_cached(reinterpret_cast<const void*>(kern), block, smem, per_sm);
}

// launch with the programmatic-stream-serialization attribute (PDL; the
// kernels call pdl_enter() first).  VLZ_PDL=0 in the environment disables it.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                            cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // per-kernel event timing (vlz_timing) brackets exactly one kernel: no PDL then
  cfg.numAttrs = (pdl_enabled() && !g_timing.load(std::memory_order_relaxed)) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// optional per-kernel CUDA-event timing (vlz_timing / vlz_timing_collect)
enum TimedKind { TK_INIT = 0, TK_COMPRESS = 1, TK_SCAN_C = 2, TK_SCAN_D = 3, TK_DECOMPRESS = 4,
                 TK_MINMAX = 5, TK_REDO = 6, TK_EDGE = 7, TK_COUNT = 8 };
extern std::atomic<int> g_timing;
void timing_mark(int kind, bool start, cudaStream_t st);

// grid = min(resident CTAs, tiles/4) for a 128-thread warp-per-tile kernel
template <typename Kern, typename Arg>
inline cudaError_t launch_tiles(Kern kernel, int64_t ntiles, int smem, cudaStream_t st,
                                const Arg& arg) {
  int per_sm = 0;
  cudaError_t e = occupancy(kernel, 128, smem, per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * num_sms();
  const int64_t need = (ntiles + 3) / 4;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  const int kind = std::is_same<Arg, CompressArgs>::value ? TK_COMPRESS : TK_DECOMPRESS;
  if (g_timing.load(std::memory_order_relaxed)) timing_mark(kind, true, st);
  cudaError_t le = launch_k(kernel, (unsigned)grid, 128, smem, st, arg);
  if (g_timing.load(std::memory_order_relaxed)) timing_mark(kind, false, st);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return le != cudaSuccess ? le : cudaGetLastError();
}

// per-(nd) dispatch entry points, one translation unit each
cudaError_t launch_compress_nd1(int B, int mode, const CompressArgs& a, cudaStream_t st);
cudaError_t launch_compress_nd2(int B, int mode, const CompressArgs& a, cudaStream_t st);
cudaError_t launch_compress_nd3(int B, int mode, const CompressArgs& a, cudaStream_t st);
cudaError_t launch_decompress(int nd, int B, bool u32, const DecompressArgs& a, cudaStream_t st);
// fused 1-D kernels (k_1d.cu) and when they apply
bool d1_fast_compress_ok(const CompressArgs& a);
bool d1_fast_decompress_ok(bool u32, const DecompressArgs& a);
cudaError_t launch_compress_1d(int B, int mode, const CompressArgs& a, cudaStream_t st);
cudaError_t launch_decompress_1d(int B, const DecompressArgs& a, cudaStream_t st);

// window width (columns per warp tile) used for (nd, B)
inline int vpl_for(int nd, int B, bool compress = false) {
  if (compress && nd == 3 && B == 8) return VLZ_VPL_C3D8;
  if (nd == 1 && B == 256) return 8;
  if (nd == 3 && B == 64) return 2;
  if (nd == 3 && B == 32) return 2;
  if (nd == 3 && B == 16) return compress ? VLZ_CVPL_3D16 : VLZ_DVPL_3D16;
  if (nd == 3 && B == 8) return VLZ_VPL_3D8;
  return 4;
}

}  // namespace vlz
