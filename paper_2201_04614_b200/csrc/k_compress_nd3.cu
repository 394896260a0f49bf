// k_compress_nd3.cu -- compress kernel instantiations for 3-D arrays.
#include "launch_compress.cuh"

namespace vlz {

cudaError_t launch_compress_nd3(int B, int mode, const CompressArgs& a, cudaStream_t st) {
  switch (B) {
    case 8: return run_compress_b<3, 8, VLZ_VPL_C3D8>(mode, a, st);
    case 16: return run_compress_b<3, 16, VLZ_CVPL_3D16>(mode, a, st);
    case 32: return run_compress_b<3, 32, 2>(mode, a, st);
    case 64: return run_compress_b<3, 64, 2>(mode, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlz
