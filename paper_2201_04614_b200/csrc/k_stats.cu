// k_stats.cu -- border-outlier census on the device (vector.py:82-87 and the
// collect_border result of dualquant_vector, vector.py:257-259; consumed by
// padding.outlier_report, padding.py:162-205).
//
// An element is a border element when any of its block-local coordinates is
// 0 (its Lorenzo prediction reads the halo); the census counts the outliers
// (code 0) among them.  One thread per block walks the block's low faces in
// the canonical in-block order; partial blocks use their own extents.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"

namespace vlz {
namespace {

__global__ void border_kernel(const uint16_t* __restrict__ codes, Geo g, int nd, int BZ, int BY,
                              int BX, unsigned long long* total) {
  unsigned long long cnt = 0;
  for (int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bi < g.nblocks;
       bi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bx = bi % g.P2, t = bi / g.P2;
    const int64_t by = t % g.P1, bz = t / g.P1;
    const int ez = (int)imin64(BZ, g.D0 - bz * BZ);
    const int ey = (int)imin64(BY, g.D1 - by * BY);
    const int ex = (int)imin64(BX, g.D2 - bx * BX);
    const uint16_t* blk = codes + block_start(g, bz, by, bx, BZ, BY, BX, ez, ey);
    for (int z = 0; z < ez; ++z) {
      for (int y = 0; y < ey; ++y) {
        const uint16_t* row = blk + (z * ey + y) * ex;
        const bool face = (nd == 3 && z == 0) || (nd >= 2 && y == 0);
        if (face) {
          for (int x = 0; x < ex; ++x) cnt += row[x] == 0;
        } else {
          cnt += row[0] == 0;  // x == 0 column
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(total, cnt);
}

}  // namespace
}  // namespace vlz

extern "C" {

// border outliers of a canonical uint16 code stream; *d_total (device int64)
// is overwritten; stream-ordered
int vlz_border_outliers(const uint16_t* d_codes, const vlz_geom* gg, int64_t* d_total,
                        void* stream) {
  if (!gg || !d_total || !d_codes || vlz_block_count(gg) < 0) return VLZ_E_ARG;
  const int b = gg->block_edge;
  vlz::Geo g{};
  int64_t D[3] = {1, 1, 1};
  for (int d = 0; d < gg->nd; ++d) D[3 - gg->nd + d] = gg->dims[d];
  g.D0 = D[0];
  g.D1 = D[1];
  g.D2 = D[2];
  g.P0 = gg->nd == 3 ? (D[0] + b - 1) / b : D[0];
  g.P1 = gg->nd >= 2 ? (D[1] + b - 1) / b : D[1];
  g.P2 = (D[2] + b - 1) / b;
  g.nblocks = g.P0 * g.P1 * g.P2;
  g.N = D[0] * D[1] * D[2];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(d_total, 0, 8, st) != cudaSuccess) return VLZ_E_CUDA;
  int64_t grid = (g.nblocks + 255) / 256;
  const int64_t cap = (int64_t)vlz::num_sms() * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  vlz::border_kernel<<<(unsigned)grid, 256, 0, st>>>(
      d_codes, g, gg->nd, gg->nd == 3 ? b : 1, gg->nd >= 2 ? b : 1, b,
      reinterpret_cast<unsigned long long*>(d_total));
  vlz::g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

}  // extern "C"
