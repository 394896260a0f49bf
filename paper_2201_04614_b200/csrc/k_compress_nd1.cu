// k_compress_nd1.cu -- compress kernel instantiations for 1-D arrays.
#include "launch_compress.cuh"

namespace vlz {

cudaError_t launch_compress_nd1(int B, int mode, const CompressArgs& a, cudaStream_t st) {
  if (d1_fast_compress_ok(a)) return launch_compress_1d(B, mode, a, st);
  switch (B) {
    case 8: return run_compress_b<1, 8, 4>(mode, a, st);
    case 16: return run_compress_b<1, 16, 4>(mode, a, st);
    case 32: return run_compress_b<1, 32, 4>(mode, a, st);
    case 64: return run_compress_b<1, 64, 4>(mode, a, st);
    case 256: return run_compress_b<1, 256, 8>(mode, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlz
