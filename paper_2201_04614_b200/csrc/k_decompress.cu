// k_decompress.cu -- instantiations of the fused reconstruction kernel.
#include "launch.cuh"

namespace vlz {

template <int ND, int B, int VPL>
static cudaError_t run_d(bool u32, const DecompressArgs& a, cudaStream_t st) {
  constexpr int smem = 4 * plane_smem_bytes<ND, B, VPL>();
  if (u32) return launch_tiles(dq_decompress_kernel<ND, B, VPL, uint32_t>, a.g.ntiles, smem, st, a);
  return launch_tiles(dq_decompress_kernel<ND, B, VPL, uint16_t>, a.g.ntiles, smem, st, a);
}

cudaError_t launch_decompress(int nd, int B, bool u32, const DecompressArgs& a, cudaStream_t st) {
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
      case 8: return run_d<3, 8, 4>(u32, a, st);
      case 16: return run_d<3, 16, 4>(u32, a, st);
      case 32: return run_d<3, 32, 4>(u32, a, st);
      case 64: return run_d<3, 64, 2>(u32, a, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace vlz
