// vlz_capi.cu -- the C ABI declared in include/vlz_gpu.h.
//
// Host orchestration only: argument validation (model.py:48-231 rules),
// workspace carving, and the launch sequence
//   compress   : init -> fused K1 (dq_compress) -> scan/origin-fix/gather
//   decompress : init -> scan (offsets) -> fused K4 (dq_decompress)
// Every kernel is stream-ordered on the caller's stream; nothing synchronises
// except the *_host entry points, which stage through cached device buffers.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <tuple>
#include <map>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/vlz_gpu.h"
#include "dq_scan.cuh"
#include "launch.cuh"

namespace vlz {

std::atomic<long long> g_launches{0};
std::atomic<int> g_timing{0};

namespace {
struct TimedRec {
  int kind;
  cudaEvent_t a, b;
};
std::mutex g_tmu;
std::vector<TimedRec> g_trecs;
std::vector<cudaEvent_t> g_epool;
cudaEvent_t g_open[TK_COUNT];

cudaEvent_t take_event() {
  if (!g_epool.empty()) {
    cudaEvent_t e = g_epool.back();
    g_epool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void timing_mark(int kind, bool start, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_tmu);
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  if (start) {
    g_open[kind] = e;
  } else {
    g_trecs.push_back({kind, g_open[kind], e});
  }
}

cudaError_t occupancy_cached(const void* kern, int block, int smem, int& per_sm) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(kern, dev, block, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      per_sm = it->second;
      return cudaSuccess;
    }
  }
  if (smem > 40 * 1024) {  // (with margin for a kernel's small static arrays)
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
  if (e != cudaSuccess) return e;
  static const bool dbg = std::getenv("VLZ_DEBUG_OCC") != nullptr;
  if (dbg) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    std::fprintf(stderr, "vlz_gpu: kernel %p block %d dyn smem %d static %zu regs %d local %zu -> %d CTAs/SM\n",
                 kern, block, smem, fa.sharedSizeBytes, fa.numRegs, fa.localSizeBytes, per_sm);
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = per_sm;
  return cudaSuccess;
}

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("VLZ_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

int num_sms() {
  static const int n = [] {  // thread-safe one-time query (same GPU model per node)
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

namespace {


size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool valid_geom(const vlz_geom* g) {
  if (!g || g->nd < 1 || g->nd > 3) return false;
  const int b = g->block_edge;
  const bool b_ok = b == 8 || b == 16 || b == 32 || b == 64 || (b == 256 && g->nd == 1);
  if (!b_ok) return false;
  for (int d = 0; d < g->nd; ++d)
    if (g->dims[d] < 1) return false;
  return true;
}

// compress = true: the tile window of the compress kernels (vpl_for)
bool make_geo(const vlz_geom* gg, Geo& g, bool compress = false) {
  if (!valid_geom(gg)) return false;
  const int b = gg->block_edge;
  int64_t D[3] = {1, 1, 1};
  for (int d = 0; d < gg->nd; ++d) D[3 - gg->nd + d] = gg->dims[d];
  const int BZ = gg->nd == 3 ? b : 1, BY = gg->nd >= 2 ? b : 1, BX = b;
  g.D0 = D[0];
  g.D1 = D[1];
  g.D2 = D[2];
  g.P0 = (D[0] + BZ - 1) / BZ;
  g.P1 = (D[1] + BY - 1) / BY;
  g.P2 = (D[2] + BX - 1) / BX;
  const int W = 32 * vpl_for(gg->nd, b, compress);
  g.NW = (D[2] + W - 1) / W;
  g.ntiles = g.P0 * g.P1 * g.NW;
  g.nblocks = g.P0 * g.P1 * g.P2;
  g.N = D[0] * D[1] * D[2];
  g.divNW.init((uint32_t)(g.NW < 0xffffffffll ? g.NW : 1));
  g.divP1.init((uint32_t)(g.P1 < 0xffffffffll ? g.P1 : 1));
  g.divP2.init((uint32_t)(g.P2 < 0xffffffffll ? g.P2 : 1));
  return true;
}

int mode_of(int kind, int gran) {
  if (kind == VLZ_PAD_ZERO) return MODE_ZERO;
  if (gran == VLZ_GRAN_GLOBAL) return MODE_GLOBAL;
  if (gran == VLZ_GRAN_BLOCK) return MODE_BLOCK;
  return MODE_EDGE;
}

bool valid_params(const vlz_params* p) {
  if (!p) return false;
  if (p->radius < 2 || p->radius > 32768) return false;
  if (p->pad_kind < 0 || p->pad_kind > 3 || p->pad_gran < 0 || p->pad_gran > 2) return false;
  return true;
}

constexpr size_t REDO_SLACK = 65536;  // >= 8 * (warps of the largest persistent grid)

// workspace layout
struct WS {
  unsigned int* ticket;      // scan chunk ticket
  unsigned int* done;        // finished-CTA counter
  unsigned long long* flag;  // per-call reset flag (InitArgs)
  long long* stats;          // sum, count, min, neg_max (single-GPU compress)
  long long* aux;            // 8 spare words
  unsigned long long* lb;    // look-back words, one per scan chunk
  long long* redo_list;      // ntiles + slack: per-warp slots of the int64 tails
  int64_t* offsets;          // nblocks
  float* scratch;            // SCRATCH_SLOTS per block
  size_t bytes;
};

WS carve(const Geo& g, void* base, bool dense = false) {
  WS w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  w.ticket = reinterpret_cast<unsigned int*>(p + off);
  w.done = reinterpret_cast<unsigned int*>(p + off + 8);
  w.flag = reinterpret_cast<unsigned long long*>(p + off + 32);
  w.stats = reinterpret_cast<long long*>(p + off + 64);
  w.aux = reinterpret_cast<long long*>(p + off + 128);
  off += 256;
  const int64_t nchunks = (g.nblocks + SCAN_MIN_CH - 1) / SCAN_MIN_CH;
  w.lb = reinterpret_cast<unsigned long long*>(p + off);
  off += align256((size_t)nchunks * 8);
  w.redo_list = reinterpret_cast<long long*>(p + off);
  // slot k of warp w is entry k * nwarps + w: below ntiles + 8 * nwarps
  off += align256(((size_t)g.ntiles + REDO_SLACK) * 8);
  w.offsets = reinterpret_cast<int64_t*>(p + off);
  off += align256((size_t)g.nblocks * 8);
  w.scratch = reinterpret_cast<float*>(p + off);
  off += align256(dense ? (size_t)g.N * 4 : (size_t)g.nblocks * SCRATCH_SLOTS * 4);
  w.bytes = off;
  return w;
}

// Per-call reset record for the first kernel of a call (vlz_common.cuh
// InitArgs): there is no init launch.  The nonce is unique per call in this
// process and never 0 (the value the call's last kernel leaves in the flag, so
// that a CUDA-graph replay of the same launches starts from a cleared flag).
unsigned long long next_nonce() {
  static std::atomic<unsigned long long> ctr{[] {
    unsigned long long s =
        (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count();
    s ^= (unsigned long long)reinterpret_cast<uintptr_t>(&s) << 17;
    return s * 0x9E3779B97F4A7C15ull;
  }()};
  unsigned long long v = ctr.fetch_add(1, std::memory_order_relaxed) + 1;
  while (v == 0) v = ctr.fetch_add(1, std::memory_order_relaxed) + 1;
  return v;
}

InitArgs make_init(vlz_result* res, const WS& w, long long* stats, int64_t nchunks) {
  InitArgs ia{};
  ia.res = reinterpret_cast<unsigned long long*>(res);
  ia.hdr = w.ticket;
  ia.stats = stats;
  ia.lb = w.lb;
  ia.nchunks = nchunks;
  ia.flag = w.flag;
  ia.nonce = next_nonce();
  return ia;
}

// resident CTAs of the offsets kernel on this device (its grid never exceeds it)
int64_t offsets_ranges() {
  int per_sm = 0;
  if (occupancy(dq_offsets_kernel, SCAN_THREADS, 0, per_sm) != cudaSuccess || per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  return (int64_t)per_sm * num_sms();
}

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t st) {
  const bool t = g_timing.load(std::memory_order_relaxed);
  const int kind = a.gather ? TK_SCAN_C : TK_SCAN_D;
  cudaError_t le = cudaSuccess;
  if (t) timing_mark(kind, true, st);
  if (a.gather) {
    const unsigned nchunks = (unsigned)scan_chunks(a.g.nblocks);
    switch (scan_ipt(a.g.nblocks)) {
      case 1: le = launch_k(dq_scan_kernel<1>, nchunks, SCAN_THREADS, 0, st, a); break;
      case 2: le = launch_k(dq_scan_kernel<2>, nchunks, SCAN_THREADS, 0, st, a); break;
      case 4: le = launch_k(dq_scan_kernel<4>, nchunks, SCAN_THREADS, 0, st, a); break;
      default: le = launch_k(dq_scan_kernel<8>, nchunks, SCAN_THREADS, 0, st, a); break;
    }
  } else {
    const int64_t ranges = offsets_ranges();
    const unsigned nchunks = (unsigned)offsets_chunks(a.g.nblocks, ranges);
    le = launch_k(dq_offsets_kernel, nchunks, SCAN_THREADS, 0, st, a,
                  offsets_span(a.g.nblocks, ranges));
  }
  if (t) timing_mark(kind, false, st);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return le != cudaSuccess ? le : cudaGetLastError();
}

int to_rc(cudaError_t e) {
  if (e == cudaSuccess) return VLZ_OK;
  std::fprintf(stderr, "vlz_gpu: CUDA error %s\n", cudaGetErrorString(e));
  return VLZ_E_CUDA;
}


// ---- value range (ErrorBound.relative) -------------------------------
__device__ __forceinline__ unsigned fkey(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void minmax_kernel(const float* in, int64_t n, unsigned int* kmin, unsigned int* kmax,
                              unsigned int* nan, unsigned int* done, double* out) {
  unsigned lo = 0xffffffffu, hi = 0u, isnan = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    if (v != v) {
      isnan = 1u;
    } else {
      const unsigned k = fkey(v);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned a = __shfl_xor_sync(FULL, lo, o), b = __shfl_xor_sync(FULL, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
    isnan |= __shfl_xor_sync(FULL, isnan, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(kmin, lo);
    atomicMax(kmax, hi);
    if (isnan) atomicOr(nan, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      __threadfence();
      const unsigned a = atomicAdd(kmin, 0u), b = atomicAdd(kmax, 0u), c = atomicAdd(nan, 0u);
      if (c) {
        out[0] = __longlong_as_double(0x7ff8000000000000ll);
        out[1] = out[0];
      } else {
        out[0] = (double)fkey_inv(a);
        out[1] = (double)fkey_inv(b);
      }
    }
  }
}

__global__ void minmax_init(unsigned int* w) {
  w[0] = 0xffffffffu;
  w[1] = 0u;
  w[2] = 0u;
  w[3] = 0u;
}

}  // namespace

// shared with the test-support sweep (k_sweep.cu)
QP make_qp(const vlz_params* p) {
  QP q;
  q.eb = p->eb;
  q.twoeb = 2.0 * p->eb;
  q.radius = p->radius;
  q.kind = p->pad_kind;
  // float32 fast path only where 1/(2eb) is a normal float with margin
  const double inv = 1.0 / q.twoeb;
  const bool fast_ok = q.twoeb > 0.0 && inv > 0x1p-100 && inv < 0x1p100;
  q.inv32 = fast_ok ? (float)inv : 0.0f;
  q.lim0 = fast_ok ? (float)(0.5 - 0x1p-22) : -1.0f;
#ifndef VLZ_KQ_LOG2
#define VLZ_KQ_LOG2 22  // margin per unit of |q|: 2^-22 (2^-21 until late round 2)
#endif
  q.kq = (float)(1.0 / (double)(1u << VLZ_KQ_LOG2));
  return q;
}

}  // namespace vlz

using namespace vlz;

extern "C" {

int64_t vlz_block_count(const vlz_geom* gg) {
  Geo g;
  if (!make_geo(gg, g)) return -1;
  return g.nblocks;
}

int64_t vlz_scalar_count(const vlz_geom* gg, int32_t kind, int32_t gran) {
  Geo g;
  if (!make_geo(gg, g)) return -1;
  if (kind == VLZ_PAD_ZERO) return 0;
  if (gran == VLZ_GRAN_GLOBAL) return 1;
  if (gran == VLZ_GRAN_BLOCK) return g.nblocks;
  return g.nblocks * gg->nd;
}

// the dense scratch layout is used when the caller's workspace has room for it
static bool ws_is_dense(const Geo& gc, size_t ws_bytes) {
  char* null_base = nullptr;
  return ws_bytes >= carve(gc, null_base, true).bytes;
}

size_t vlz_workspace_size_dense(const vlz_geom* gg) {
  Geo gd, gc;
  if (!make_geo(gg, gd) || !make_geo(gg, gc, true)) return 0;
  char* null_base = nullptr;
  const size_t d = carve(gd, null_base).bytes, c = carve(gc, null_base, true).bytes;
  return d > c ? d : c;
}

size_t vlz_workspace_size(const vlz_geom* gg) {
  // large enough for both directions (their tile windows may differ)
  Geo gd, gc;
  if (!make_geo(gg, gd) || !make_geo(gg, gc, true)) return 0;
  char* null_base = nullptr;
  const size_t d = carve(gd, null_base).bytes, c = carve(gc, null_base).bytes;
  return d > c ? d : c;
}

__attribute__((visibility("hidden"))) int vlz_internal_compress_begin(const float* d_in, const vlz_geom* gg, const vlz_params* p,
                               uint16_t* d_codes, int64_t* d_counts, int64_t* d_scalars,
                               vlz_result* d_result, long long* stats, void* d_ws,
                               size_t ws_bytes, cudaStream_t st) {
  Geo g;
  if (!make_geo(gg, g, true) || !valid_params(p) || !(p->eb > 0.0) || !d_in || !d_codes ||
      !d_counts || !d_result || !d_ws)
    return VLZ_E_ARG;
  WS w = carve(g, d_ws);
  if (ws_bytes < w.bytes) return VLZ_E_ARG;
  const int mode = mode_of(p->pad_kind, p->pad_gran);
  if (mode != MODE_ZERO && !d_scalars) return VLZ_E_ARG;
  if (mode == MODE_GLOBAL && !stats) return VLZ_E_ARG;
  const int64_t nchunks = scan_chunks(g.nblocks);
  cudaError_t e = cudaSuccess;
  CompressArgs a{};
  a.init = make_init(d_result, w, stats, nchunks);
  a.g = g;
  a.q = make_qp(p);
  a.in = d_in;
  a.codes = d_codes;
  a.scratch = w.scratch;
  a.scratch_dense = ws_is_dense(g, ws_bytes) ? 1 : 0;
  a.counts = d_counts;
  a.scalars = d_scalars;
  a.origin_vals = reinterpret_cast<float*>(w.offsets);  // offsets are unused by compress
  a.first_nonfinite = reinterpret_cast<unsigned long long*>(&d_result->first_nonfinite);
  a.first_overflow = reinterpret_cast<unsigned long long*>(&d_result->first_overflow);
  a.gsum = reinterpret_cast<unsigned long long*>(stats);
  a.gcount = reinterpret_cast<unsigned long long*>(stats ? stats + 1 : nullptr);
  a.gmin = stats ? stats + 2 : nullptr;
  a.gnegmax = stats ? stats + 3 : nullptr;
  a.redo_list = w.redo_list;
  const int b = gg->block_edge;
  if (gg->nd == 1) e = launch_compress_nd1(b, mode, a, st);
  else if (gg->nd == 2) e = launch_compress_nd2(b, mode, a, st);
  else e = launch_compress_nd3(b, mode, a, st);
  return to_rc(e);
}

static int finish_impl(const float* d_in, const vlz_geom* gg, const vlz_params* p,
                       const long long* gstats, int nstats, uint16_t* d_codes,
                       float* d_outliers, int64_t* d_counts, int64_t* d_scalars,
                       vlz_result* d_result, void* d_ws, size_t ws_bytes, cudaStream_t st,
                       unsigned long long* patch_list, unsigned int* patch_count,
                       long long out_cap = 0x7fffffffffffffffll);

__attribute__((visibility("hidden"))) int vlz_internal_compress_finish(const float* d_in, const vlz_geom* gg, const vlz_params* p,
                                const long long* gstats, uint16_t* d_codes, float* d_outliers,
                                int64_t* d_counts, int64_t* d_scalars, vlz_result* d_result,
                                void* d_ws, size_t ws_bytes, cudaStream_t st,
                                unsigned long long* patch_list, unsigned int* patch_count) {
  return finish_impl(d_in, gg, p, gstats, 1, d_codes, d_outliers, d_counts, d_scalars, d_result,
                     d_ws, ws_bytes, st, patch_list, patch_count);
}

static int finish_impl(const float* d_in, const vlz_geom* gg, const vlz_params* p,
                       const long long* gstats, int nstats, uint16_t* d_codes,
                       float* d_outliers, int64_t* d_counts, int64_t* d_scalars,
                       vlz_result* d_result, void* d_ws, size_t ws_bytes, cudaStream_t st,
                       unsigned long long* patch_list, unsigned int* patch_count,
                       long long out_cap) {
  Geo g;
  if (!make_geo(gg, g, true) || !valid_params(p) || !d_outliers || !d_result || !d_ws)
    return VLZ_E_ARG;
  WS w = carve(g, d_ws);
  if (ws_bytes < w.bytes) return VLZ_E_ARG;
  const int mode = mode_of(p->pad_kind, p->pad_gran);
  const int b = gg->block_edge;
  ScanArgs s{};
  s.g = g;
  s.q = make_qp(p);
  s.BZ = gg->nd == 3 ? b : 1;
  s.BY = gg->nd >= 2 ? b : 1;
  s.BX = b;
  s.fix_origin = mode == MODE_GLOBAL;
  s.gather = 1;
  s.in = d_in;
  s.origin_vals = reinterpret_cast<const float*>(w.offsets);
  s.codes = d_codes;
  s.counts = d_counts;
  s.scratch = w.scratch;
  s.scratch_dense = ws_is_dense(g, ws_bytes) ? 1 : 0;
  s.out = d_outliers;
  s.scalars = d_scalars;
  s.lb = w.lb;
  s.ticket = w.ticket;
  s.flag = w.flag;
  s.n_out = reinterpret_cast<long long*>(&d_result->n_outliers);
  s.gstats = gstats;
  s.nstats = nstats;
  if (nstats < 1) return VLZ_E_ARG;
  s.status = &d_result->status;
  s.index = reinterpret_cast<long long*>(&d_result->index);
  s.first_nonfinite = reinterpret_cast<const unsigned long long*>(&d_result->first_nonfinite);
  s.first_overflow = reinterpret_cast<const unsigned long long*>(&d_result->first_overflow);
  s.patch_list = patch_list;
  s.patch_count = patch_count;
  s.out_cap = out_cap;
  if (mode == MODE_GLOBAL && !gstats) return VLZ_E_ARG;
  return to_rc(launch_scan(s, st));
}

int vlz_dq_compress(const float* d_in, const vlz_geom* g, const vlz_params* p, uint16_t* d_codes,
                    float* d_outliers, int64_t* d_counts, int64_t* d_scalars,
                    vlz_result* d_result, void* d_ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Geo gg;
  if (!make_geo(g, gg, true)) return VLZ_E_ARG;
  WS w = carve(gg, d_ws);
  int rc = vlz_internal_compress_begin(d_in, g, p, d_codes, d_counts, d_scalars, d_result, w.stats,
                               d_ws, ws_bytes, st);
  if (rc != VLZ_OK) return rc;
  return vlz_internal_compress_finish(d_in, g, p, w.stats, d_codes, d_outliers, d_counts, d_scalars,
                              d_result, d_ws, ws_bytes, st, nullptr, nullptr);
}

int vlz_dq_compress_capped(const float* d_in, const vlz_geom* g, const vlz_params* p,
                           uint16_t* d_codes, float* d_outliers, int64_t outlier_capacity,
                           int64_t* d_counts, int64_t* d_scalars, vlz_result* d_result, void* d_ws,
                           size_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Geo gg;
  if (!make_geo(g, gg, true) || outlier_capacity < 0 || (outlier_capacity > 0 && !d_outliers))
    return VLZ_E_ARG;
  WS w = carve(gg, d_ws);
  int rc = vlz_internal_compress_begin(d_in, g, p, d_codes, d_counts, d_scalars, d_result, w.stats,
                                       d_ws, ws_bytes, st);
  if (rc != VLZ_OK) return rc;
  // (a zero-capacity call still needs a non-null pointer for the kernel's base address)
  float* out = d_outliers ? d_outliers : reinterpret_cast<float*>(w.scratch);
  return finish_impl(d_in, g, p, w.stats, 1, d_codes, out, d_counts, d_scalars, d_result, d_ws,
                     ws_bytes, st, nullptr, nullptr, (long long)outlier_capacity);
}

int vlz_dq_compress_begin(const float* d_in, const vlz_geom* g, const vlz_params* p,
                          uint16_t* d_codes, int64_t* d_counts, int64_t* d_scalars,
                          vlz_result* d_result, vlz_stats* d_stats, void* d_ws, size_t ws_bytes,
                          void* stream) {
  return vlz_internal_compress_begin(d_in, g, p, d_codes, d_counts, d_scalars, d_result,
                             reinterpret_cast<long long*>(d_stats), d_ws, ws_bytes,
                             static_cast<cudaStream_t>(stream));
}

int vlz_dq_compress_finish_gathered(const float* d_in, const vlz_geom* g, const vlz_params* p,
                                    const vlz_stats* d_rank_stats, int32_t nranks,
                                    uint16_t* d_codes, float* d_outliers, int64_t* d_counts,
                                    int64_t* d_scalars, vlz_result* d_result, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  return finish_impl(d_in, g, p, reinterpret_cast<const long long*>(d_rank_stats), nranks,
                     d_codes, d_outliers, d_counts, d_scalars, d_result, d_ws, ws_bytes,
                     static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

int vlz_dq_compress_finish(const float* d_in, const vlz_geom* g, const vlz_params* p,
                           const vlz_stats* d_global_stats, uint16_t* d_codes, float* d_outliers,
                           int64_t* d_counts, int64_t* d_scalars, vlz_result* d_result,
                           void* d_ws, size_t ws_bytes, void* stream) {
  return vlz_internal_compress_finish(d_in, g, p, reinterpret_cast<const long long*>(d_global_stats),
                              d_codes, d_outliers, d_counts, d_scalars, d_result, d_ws,
                              ws_bytes, static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

static int decompress_impl(const void* d_codes, bool u32, const float* d_outliers,
                           int64_t n_outliers, const int64_t* d_n_outliers, const int64_t* d_counts,
                           const int64_t* d_scalars, const vlz_geom* gg, const vlz_params* p,
                           float* d_out, vlz_result* d_result, void* d_ws, size_t ws_bytes,
                           cudaStream_t st);

__attribute__((visibility("hidden"))) int vlz_internal_decompress(const void* d_codes, bool u32, const float* d_outliers,
                           int64_t n_outliers, const int64_t* d_counts, const int64_t* d_scalars,
                           const vlz_geom* gg, const vlz_params* p, float* d_out,
                           vlz_result* d_result, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  return decompress_impl(d_codes, u32, d_outliers, n_outliers, nullptr, d_counts, d_scalars, gg, p,
                         d_out, d_result, d_ws, ws_bytes, st);
}

static int decompress_impl(const void* d_codes, bool u32, const float* d_outliers,
                           int64_t n_outliers, const int64_t* d_n_outliers, const int64_t* d_counts,
                           const int64_t* d_scalars, const vlz_geom* gg, const vlz_params* p,
                           float* d_out, vlz_result* d_result, void* d_ws, size_t ws_bytes,
                           cudaStream_t st) {
  Geo g;
  if (!make_geo(gg, g) || !valid_params(p) || !d_codes || !d_counts || !d_out || !d_result ||
      !d_ws || n_outliers < 0)
    return VLZ_E_ARG;
  WS w = carve(g, d_ws);
  if (ws_bytes < w.bytes) return VLZ_E_ARG;
  const int mode = mode_of(p->pad_kind, p->pad_gran);
  if (mode != MODE_ZERO && !d_scalars) return VLZ_E_ARG;
  const int64_t nchunks = offsets_chunks(g.nblocks, offsets_ranges());
  cudaError_t e = cudaSuccess;
  const int b = gg->block_edge;
  ScanArgs s{};
  s.init = make_init(d_result, w, nullptr, nchunks);
  s.g = g;
  s.q = make_qp(p);
  s.BZ = gg->nd == 3 ? b : 1;
  s.BY = gg->nd >= 2 ? b : 1;
  s.BX = b;
  s.fix_origin = 0;
  s.gather = 0;
  s.counts = const_cast<int64_t*>(d_counts);
  s.offsets = w.offsets;
  s.lb = w.lb;
  s.ticket = w.ticket;
  s.n_out = w.aux;  // sum of counts (unused by the checks; kept for debugging)
  e = launch_scan(s, st);
  if (e != cudaSuccess) return to_rc(e);
  DecompressArgs a{};
  a.g = g;
  a.q = make_qp(p);
  a.mode = mode;
  a.nd = gg->nd;
  a.codes = d_codes;
  a.outliers = d_outliers;
  a.n_outliers = n_outliers;
  a.n_out_dev = reinterpret_cast<const long long*>(d_n_outliers);
  a.counts = d_counts;
  a.offsets = w.offsets;
  a.scalars = d_scalars;
  a.out = d_out;
  a.first_bad = reinterpret_cast<unsigned long long*>(&d_result->first_bad_block);
  a.sentinels = reinterpret_cast<unsigned long long*>(&d_result->sentinels);
  a.done = w.done;
  a.status = &d_result->status;
  a.index = reinterpret_cast<long long*>(&d_result->index);
  a.n_sent_out = reinterpret_cast<long long*>(&d_result->n_outliers);
  a.redo_list = w.redo_list;
  a.flag = w.flag;
  return to_rc(launch_decompress(gg->nd, b, u32, a, st));
}

int vlz_dq_decompress(const uint16_t* d_codes, const float* d_outliers, int64_t n_outliers,
                      const int64_t* d_counts, const int64_t* d_scalars, const vlz_geom* g,
                      const vlz_params* p, float* d_out, vlz_result* d_result, void* d_ws,
                      size_t ws_bytes, void* stream) {
  return vlz_internal_decompress(d_codes, false, d_outliers, n_outliers, d_counts, d_scalars, g, p, d_out,
                         d_result, d_ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int vlz_dq_decompress_dn(const uint16_t* d_codes, const float* d_outliers,
                         const int64_t* d_n_outliers, const int64_t* d_counts,
                         const int64_t* d_scalars, const vlz_geom* g, const vlz_params* p,
                         float* d_out, vlz_result* d_result, void* d_ws, size_t ws_bytes,
                         void* stream) {
  if (!d_n_outliers) return VLZ_E_ARG;
  return decompress_impl(d_codes, false, d_outliers, 0, d_n_outliers, d_counts, d_scalars, g, p,
                         d_out, d_result, d_ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int vlz_dq_decompress_u32(const uint32_t* d_codes, const float* d_outliers, int64_t n_outliers,
                          const int64_t* d_counts, const int64_t* d_scalars, const vlz_geom* g,
                          const vlz_params* p, float* d_out, vlz_result* d_result, void* d_ws,
                          size_t ws_bytes, void* stream) {
  return vlz_internal_decompress(d_codes, true, d_outliers, n_outliers, d_counts, d_scalars, g, p, d_out,
                         d_result, d_ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int vlz_minmax(const float* d_in, int64_t n, double* d_minmax, void* stream) {
  if (!d_in || n < 1 || !d_minmax) return VLZ_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // 4 scratch words live in a lazily allocated device buffer per device
  static unsigned int* scratch[64] = {nullptr};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!scratch[dev]) {
      cudaError_t e = cudaMalloc(&scratch[dev], 64);
      if (e != cudaSuccess) return to_rc(e);
    }
  }
  unsigned int* w = scratch[dev];
  minmax_init<<<1, 1, 0, st>>>(w);
  int64_t blocks = (n + 1023) / 1024;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  minmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_in, n, w, w + 1, w + 2, w + 3, d_minmax);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return to_rc(cudaGetLastError());
}

int64_t vlz_launch_count(void) { return g_launches.load(); }

void vlz_timing(int enable) { g_timing.store(enable ? 1 : 0); }

int vlz_timing_collect(double* ms, int64_t* launches, int n) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (int k = 0; k < n; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
  }
  for (const TimedRec& r : g_trecs) {
    float t = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.kind < n) {
      ms[r.kind] += t;
      launches[r.kind] += 1;
    }
    g_epool.push_back(r.a);
    g_epool.push_back(r.b);
  }
  g_trecs.clear();
  return VLZ_OK;
}

const char* vlz_version(void) { return "vlz_gpu 0.1 sm_100a"; }

}  // extern "C"
