// k_compress_nd2.cu -- compress kernel instantiations for 2-D arrays.
#include "launch_compress.cuh"

namespace vlz {

cudaError_t launch_compress_nd2(int B, int mode, const CompressArgs& a, cudaStream_t st) {
  switch (B) {
    case 8: return run_compress_b<2, 8, 4>(mode, a, st);
    case 16: return run_compress_b<2, 16, 4>(mode, a, st);
    case 32: return run_compress_b<2, 32, 4>(mode, a, st);
    case 64: return run_compress_b<2, 64, 4>(mode, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlz
