// k_census.cu -- one-pass padding-policy census for outlier_report
// (reference padding.py:162-205, which compresses the array once per policy).
//
// By finding 1 every padding policy gives the same Lorenzo deltas
// except at block origins, where the prediction is the block's dim-0 halo
// scalar s0 (kernel.py:72-101).  The narrowing check (vector.py:73-76) does
// not depend on the policy either.  So a policy's outliers are the zero-
// padding outliers away from the origins plus the origins with
// |d_o - s0| > R-1 or a failed narrowing check -- and an origin is always a
// border element (vector.py:82-87).  This file counts, per policy, the block
// origins that are outliers:
//   census_block_kernel   one warp per block: d of every element (the
//                         kernels' exact-fast prequantizer), the block's
//                         min / max / wrapping sum (padding.py:62-69, block
//                         granularity) and the same over its dim-0 low face
//                         (edge granularity; s0 is the dim-0 edge scalar),
//                         the origin's d and narrowing verdict; origin
//                         verdicts of zero, *:block and *:edge padding;
//                         global min / max / sum.
//   census_global_kernel  origin verdicts of the three *:global policies
//                         from the global statistics.
// Output (device int64[12]): [0] zero padding, [3*kind + gran] for kind
// 1 min / 2 max / 3 mean and gran 0 global / 1 block / 2 edge.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"

namespace vlz {

QP make_qp(const vlz_params* p);

namespace {

constexpr int CENSUS_WARPS = 8;

struct CensusArgs {
  const float* in;
  Geo g;
  QP q;
  int nd, BZ, BY, BX;
  long long* origin;             // per block: d_o * 2 | bad_o
  unsigned long long* counts;    // [12]
  long long* gstats;             // sum (wrapping), min, max
};

__device__ __forceinline__ bool origin_out(long long d, bool bad, long long s0, int R) {
  const long long dl = d - s0;
  return bad || dl > R - 1 || dl < -(R - 1);
}

__global__ void __launch_bounds__(CENSUS_WARPS * 32) census_block_kernel(CensusArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * CENSUS_WARPS + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * CENSUS_WARPS;
  const Geo& g = a.g;
  const int R = a.q.radius;
  unsigned long long cnt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // zero, then (kind, gran) block/edge
  long long gsum = 0, gmin = 0x7fffffffffffffffll, gmax = -0x7fffffffffffffffll - 1;
  for (int64_t bi = warp; bi < g.nblocks; bi += nwarps) {
    const int64_t bx = bi % g.P2, t = bi / g.P2;
    const int64_t by = t % g.P1, bz = t / g.P1;
    const int ez = (int)imin64(a.BZ, g.D0 - bz * a.BZ);
    const int ey = (int)imin64(a.BY, g.D1 - by * a.BY);
    const int ex = (int)imin64(a.BX, g.D2 - bx * a.BX);
    const int size = ez * ey * ex;
    const int fsize = a.nd == 3 ? ey * ex : (a.nd == 2 ? ex : 1);
    const float* base = a.in + ((bz * a.BZ) * g.D1 + by * a.BY) * g.D2 + bx * a.BX;
    long long bmin = 0x7fffffffffffffffll, bmax = -0x7fffffffffffffffll - 1, bsum = 0;
    long long fmin = bmin, fmax = bmax, fsum = 0;
    long long d_o = 0;
    bool bad_o = false;
    for (int e = lane; e < size; e += 32) {
      const int x = e % ex, r = e / ex;
      const int y = r % ey, z = r / ey;
      const float v = base[((int64_t)z * g.D1 + y) * g.D2 + x];
      bool ok;
      int d = quant_fast(v, a.q, ok);
      bool bad = false;
      if (!ok) {
        bool ovf;
        d = quant_exact(v, a.q, bad, ovf);
      }
      const long long dl = d;
      bmin = dl < bmin ? dl : bmin;
      bmax = dl > bmax ? dl : bmax;
      bsum = (long long)((unsigned long long)bsum + (unsigned long long)dl);
      const bool face = a.nd == 3 ? z == 0 : (a.nd == 2 ? y == 0 : x == 0);
      if (face) {
        fmin = dl < fmin ? dl : fmin;
        fmax = dl > fmax ? dl : fmax;
        fsum = (long long)((unsigned long long)fsum + (unsigned long long)dl);
      }
      if (e == 0) {
        d_o = dl;
        bad_o = bad;
      }
    }
    bmin = group_min<32>(bmin);
    bmax = group_max<32>(bmax);
    bsum = (long long)group_sum<32>((unsigned long long)bsum);
    fmin = group_min<32>(fmin);
    fmax = group_max<32>(fmax);
    fsum = (long long)group_sum<32>((unsigned long long)fsum);
    if (lane == 0) {
      a.origin[bi] = d_o * 2 + (bad_o ? 1 : 0);
      cnt[0] += origin_out(d_o, bad_o, 0, R);
#pragma unroll
      for (int k = 1; k <= 3; ++k) {
        cnt[k] += origin_out(d_o, bad_o, stat_value(k, bsum, size, bmin, bmax), R);       // block
        cnt[3 + k] += origin_out(d_o, bad_o, stat_value(k, fsum, fsize, fmin, fmax), R);  // edge
      }
      gsum = (long long)((unsigned long long)gsum + (unsigned long long)bsum);
      gmin = bmin < gmin ? bmin : gmin;
      gmax = bmax > gmax ? bmax : gmax;
    }
  }
  if (lane == 0) {
    atomicAdd(&a.counts[0], cnt[0]);
#pragma unroll
    for (int k = 1; k <= 3; ++k) {
      atomicAdd(&a.counts[3 * k + 1], cnt[k]);
      atomicAdd(&a.counts[3 * k + 2], cnt[3 + k]);
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.gstats[0]), (unsigned long long)gsum);
    atomicMin(&a.gstats[1], gmin);
    atomicMax(&a.gstats[2], gmax);
  }
}

__global__ void census_global_kernel(CensusArgs a) {
  const int R = a.q.radius;
  const long long sum = a.gstats[0], mn = a.gstats[1], mx = a.gstats[2];
  long long s0[3];
#pragma unroll
  for (int k = 1; k <= 3; ++k) s0[k - 1] = stat_value(k, sum, a.g.N, mn, mx);
  unsigned long long c[3] = {0, 0, 0};
  for (int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bi < a.g.nblocks;
       bi += (int64_t)gridDim.x * blockDim.x) {
    const long long w = a.origin[bi];
    const long long d = w >> 1;  // arithmetic: d_o * 2 + bad, bad in the low bit
    const bool bad = w & 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] += origin_out(d, bad, s0[k], R);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = group_sum<32>(c[k]);
    if ((threadIdx.x & 31) == 0 && c[k]) atomicAdd(&a.counts[3 * (k + 1)], c[k]);
  }
}

__global__ void census_init(unsigned long long* counts, long long* gstats) {
  if (threadIdx.x < 12) counts[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    gstats[0] = 0;
    gstats[1] = 0x7fffffffffffffffll;
    gstats[2] = -0x7fffffffffffffffll - 1;
  }
}

bool census_geo(const vlz_geom* gg, Geo& g, int& BZ, int& BY, int& BX) {
  if (!gg || gg->nd < 1 || gg->nd > 3 || vlz_block_count(gg) < 0) return false;
  const int b = gg->block_edge;
  int64_t D[3] = {1, 1, 1};
  for (int d = 0; d < gg->nd; ++d) D[3 - gg->nd + d] = gg->dims[d];
  BZ = gg->nd == 3 ? b : 1;
  BY = gg->nd >= 2 ? b : 1;
  BX = b;
  g = Geo{};
  g.D0 = D[0];
  g.D1 = D[1];
  g.D2 = D[2];
  g.P0 = (D[0] + BZ - 1) / BZ;
  g.P1 = (D[1] + BY - 1) / BY;
  g.P2 = (D[2] + BX - 1) / BX;
  g.nblocks = g.P0 * g.P1 * g.P2;
  g.N = D[0] * D[1] * D[2];
  return true;
}

}  // namespace
}  // namespace vlz

extern "C" {

size_t vlz_padding_census_ws_size(const vlz_geom* gg) {
  const int64_t nb = vlz_block_count(gg);
  return nb < 0 ? 0 : 256 + (size_t)nb * 8;
}

int vlz_padding_census(const float* d_in, const vlz_geom* gg, double eb, int32_t radius,
                       int64_t* d_counts, void* d_ws, size_t ws_bytes, void* stream) {
  vlz::CensusArgs a{};
  if (!d_in || !d_counts || !d_ws || !(eb > 0.0) || radius < 2 || radius > 32768 ||
      !vlz::census_geo(gg, a.g, a.BZ, a.BY, a.BX) || ws_bytes < vlz_padding_census_ws_size(gg))
    return VLZ_E_ARG;
  vlz_params p{};
  p.eb = eb;
  p.radius = radius;
  a.in = d_in;
  a.q = vlz::make_qp(&p);
  a.nd = gg->nd;
  a.counts = reinterpret_cast<unsigned long long*>(d_counts);
  a.gstats = static_cast<long long*>(d_ws);
  a.origin = reinterpret_cast<long long*>(static_cast<char*>(d_ws) + 256);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  vlz::census_init<<<1, 32, 0, st>>>(a.counts, a.gstats);
  const int64_t sms = vlz::num_sms();
  int64_t grid = (a.g.nblocks + vlz::CENSUS_WARPS - 1) / vlz::CENSUS_WARPS;
  if (grid > sms * 8) grid = sms * 8;
  vlz::census_block_kernel<<<(unsigned)grid, vlz::CENSUS_WARPS * 32, 0, st>>>(a);
  int64_t g2 = (a.g.nblocks + 255) / 256;
  if (g2 > sms * 4) g2 = sms * 4;
  vlz::census_global_kernel<<<(unsigned)(g2 < 1 ? 1 : g2), 256, 0, st>>>(a);
  vlz::g_launches.fetch_add(3, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

}  // extern "C"
