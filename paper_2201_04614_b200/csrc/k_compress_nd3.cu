// k_compress_nd3.cu -- instantiations of the fused compress kernel for 3-D arrays.
#include "launch.cuh"

namespace vlz {

template <int B, int VPL>
static cudaError_t run_b(int mode, const CompressArgs& a, cudaStream_t st) {
  constexpr int smem = 4 * plane_smem_bytes<3, B, VPL>();
  switch (mode) {
    case MODE_ZERO: return launch_tiles(dq_compress_kernel<3, B, VPL, MODE_ZERO>, a.g.ntiles, smem, st, a);
    case MODE_GLOBAL: return launch_tiles(dq_compress_kernel<3, B, VPL, MODE_GLOBAL>, a.g.ntiles, smem, st, a);
    case MODE_BLOCK: return launch_tiles(dq_compress_kernel<3, B, VPL, MODE_BLOCK>, a.g.ntiles, smem, st, a);
    default: return launch_tiles(dq_compress_kernel<3, B, VPL, MODE_EDGE>, a.g.ntiles, smem, st, a);
  }
}

cudaError_t launch_compress_nd3(int B, int mode, const CompressArgs& a, cudaStream_t st) {
  switch (B) {
    case 8: return run_b<8, 4>(mode, a, st);
    case 16: return run_b<16, 4>(mode, a, st);
    case 32: return run_b<32, 4>(mode, a, st);
    case 64: return run_b<64, 2>(mode, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlz
