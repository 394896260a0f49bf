// k_huffenc.cu -- canonical Huffman encoding of the code stream on the GPU
// (the reference's encode, huffman.py:91-122: MSB-first codewords packed back
// to back, np.packbits zero-pads the last byte).
//
// One pass, no memset of the output:
//  * a chunk of HE_CH symbols per CTA (dynamic ticket order); every thread
//    looks up the lengths of its 32 symbols (u8 table) for the scan and the
//    (codeword, length) entries again when packing (L1-resident tables);
//  * block scan of the lengths + decoupled look-back (lookback.cuh) give the
//    chunk's global bit offset;
//  * the chunk assembles its bits in shared memory, aligned to the global
//    32-bit word grid: each thread shifts its codewords into a 64-bit
//    accumulator and emits whole words (atomicOr only for the words it
//    shares with its neighbours);
//  * a chunk OWNS the output words whose first bit lies inside its bit range;
//    the one word it shares with the next chunk is completed by reading that
//    chunk's leading symbols (<= 31 bits, every codeword has >= 1 bit), so
//    each word is written exactly once, with a plain coalesced store
//    (byte-swapped: bit 0 of the stream is the MSB of byte 0).
// Codewords up to 58 bits are supported (table entry = codeword << 6 | len);
// a stream needs > 10^12 symbols before a Huffman code can be that deep.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/vlz_gpu.h"
#include "launch.cuh"
#include "lookback.cuh"

namespace vlz {
namespace {

constexpr int HE_THREADS = 256;
constexpr int HE_SPT = 32;                  // symbols per thread
constexpr int HE_CH = HE_THREADS * HE_SPT;  // symbols per chunk
constexpr int HE_MAXLEN = 58;
constexpr long long HE_NONE = 0x7fffffffffffffffll;
constexpr size_t HE_TAB = 65536 * 8;        // entries
constexpr size_t HE_LEN = 65536;            // lengths (u8)

struct HEArgs {
  const uint16_t* codes;
  int64_t n;
  const unsigned long long* tab;  // [65536] codeword << 6 | length, 0 = absent
  const uint8_t* len;             // [65536] length, 0 = absent
  int32_t nsym_span;              // max codebook symbol + 1 (huffman.py:96)
  uint32_t* out;
  int64_t out_words;
  unsigned long long* lb;
  unsigned int* ticket;
  long long* info;  // [0] bits, [1] first symbol >= span, [2] overflow, [3] first absent symbol
};

__global__ void he_init_kernel(unsigned long long* lb, int64_t nchunks, unsigned int* ticket,
                               long long* info) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    *ticket = 0;
    info[0] = 0;
    info[1] = HE_NONE;
    info[2] = 0;
    info[3] = HE_NONE;
  }
  for (int64_t k = i; k < nchunks; k += (int64_t)gridDim.x * blockDim.x) lb[k] = 0;
}

__global__ void he_table_kernel(const unsigned long long* staged, int32_t nsym,
                                unsigned long long* tab, uint8_t* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsym) {
    const unsigned long long e = staged[2 * i + 1];
    tab[staged[2 * i]] = e;
    len[staged[2 * i]] = (uint8_t)(e & 63);
  }
}

__device__ __forceinline__ unsigned sym_at(const uint4* pk, int k) {
  const uint4 v = pk[k >> 3];
  const int w = (k >> 1) & 3;
  const unsigned x = w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
  return (k & 1) ? (x >> 16) : (x & 0xffffu);
}

__global__ void __launch_bounds__(HE_THREADS, 4) huff_encode_kernel(HEArgs a) {
  extern __shared__ uint32_t s_words[];  // sized for HE_CH * max_len bits
  __shared__ int s_warp[HE_THREADS / 32];
  __shared__ long long s_start;
  __shared__ unsigned int s_tile;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * HE_CH;
  const int64_t i0 = base + (int64_t)tid * HE_SPT;
  const bool full = i0 + HE_SPT <= a.n;

  // ---- symbols (packed, 16 B vectors) and the next chunk's leading symbols
  uint4 pk[HE_SPT / 8];
  if (full) {
    const uint4* v = reinterpret_cast<const uint4*>(a.codes + i0);
#pragma unroll
    for (int q = 0; q < HE_SPT / 8; ++q) pk[q] = v[q];
  } else {
#pragma unroll
    for (int q = 0; q < HE_SPT / 8; ++q) pk[q] = make_uint4(0, 0, 0, 0);
  }
  unsigned long long tail_e = 0;
  const bool need_tail_sym = (wid == 1) && (base + HE_CH < a.n);
  if (need_tail_sym) {
    const int64_t i = base + HE_CH + lane;
    if (i < a.n) tail_e = __ldg(a.tab + a.codes[i]);
  }
  auto sym_of = [&](int k) -> int {  // -1 past the end
    if (full) return (int)sym_at(pk, k);
    return (i0 + k < a.n) ? (int)a.codes[i0 + k] : -1;
  };

  // ---- lengths -> bits of this thread
  int tbits = 0;
  int lmin = 64, lmax = 0;
#pragma unroll
  for (int k = 0; k < HE_SPT; ++k) {
    const int s = sym_of(k);
    if (s < 0) continue;
    const int L = __ldg(a.len + s);
    lmin = min(lmin, L);
    lmax = max(lmax, L);
    tbits += L;
  }
  if (lmin == 0) {  // symbols not in the codebook (reported, contribute no bits)
#pragma unroll 1
    for (int k = 0; k < HE_SPT; ++k) {
      const int s = sym_of(k);
      if (s >= 0 && __ldg(a.len + s) == 0)
        atomicMin(&a.info[s >= a.nsym_span ? 1 : 3], ((i0 + k) << 16) | (long long)s);
    }
  }
  // common case: every symbol present, every codeword <= 32 bits
  const bool simple = full && lmin > 0 && lmax <= 32;

  // ---- chunk scan of bit lengths
  int inc = tbits;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  int wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < HE_THREADS / 32; ++w) {
    if (w < wid) wbase += s_warp[w];
    agg += s_warp[w];
  }
  const int texcl = wbase + inc - tbits;
  // the chunk's bits are assembled at LOCAL offsets (bit 0 = the chunk's
  // first bit), so only the final store waits for the look-back; the next
  // chunk's leading <= 32 bits are appended after them
  const int nwords = (agg + 32 + 31) / 32 + 1;
  for (int w = tid; w < nwords; w += HE_THREADS) s_words[w] = 0;
  __syncthreads();

  auto compose = [&]() {
    if (simple) {  // branch-light path: every codeword 1..32 bits
      const int p0 = texcl;
      int w = p0 >> 5;
      int nacc = p0 & 31;
      unsigned long long acc = 0;
      int emitted = 0;
#pragma unroll
      for (int k = 0; k < HE_SPT; ++k) {
        const unsigned long long e = __ldg(a.tab + sym_at(pk, k));
        const int L = (int)(e & 63);
        acc = (acc << L) | (e >> 6);
        nacc += L;
        if (nacc >= 32) {
          const uint32_t word = (uint32_t)(acc >> (nacc - 32));
          nacc -= 32;
          if (emitted == 0) atomicOr(&s_words[w], word);
          else s_words[w] = word;
          ++emitted;
          ++w;
        }
      }
      if (nacc > (emitted ? 0 : (p0 & 31))) atomicOr(&s_words[w], (uint32_t)(acc << (32 - nacc)));
      return;
    }
    // 64-bit accumulator per thread; words wholly inside the thread's bit
    // range are plain shared stores, the (at most two) words shared with the
    // neighbouring threads are atomicOr
    const int p0 = texcl;
    int w = p0 >> 5;
    int nacc = p0 & 31;  // leading zero bits of the first word
    unsigned long long acc = 0;
    bool first = true;
    auto push = [&](unsigned long long bits, int L) {  // nacc < 32, L <= 32
      acc = (acc << L) | bits;
      nacc += L;
      if (nacc >= 32) {
        const uint32_t word = (uint32_t)(acc >> (nacc - 32));
        nacc -= 32;
        if (first) atomicOr(&s_words[w], word);
        else s_words[w] = word;
        first = false;
        ++w;
      }
    };
#pragma unroll
    for (int k = 0; k < HE_SPT; ++k) {
      const int s = sym_of(k);
      if (s < 0) continue;
      const unsigned long long e = __ldg(a.tab + s);
      const int L = (int)(e & 63);
      const unsigned long long cw = e >> 6;
      if (L <= 32) {
        push(cw, L);
      } else {  // deep codeword: high part, then the low 32 bits
        push(cw >> 32, L - 32);
        push(cw & 0xffffffffull, 32);
      }
    }
    if (nacc > (first ? (p0 & 31) : 0)) atomicOr(&s_words[w], (uint32_t)(acc << (32 - nacc)));
  };

  if (wid == 0) {  // look-back first, then this warp's share of the bits
    const long long excl = lookback_exclusive(a.lb, tile, agg, lane);
    if (lane == 0) {
      s_start = excl;
      if (base + HE_CH >= a.n) a.info[0] = excl + agg;
    }
    compose();
  } else {
    compose();
    if (wid == 1 && base + HE_CH < a.n) {
      // the next chunk's leading bits, 32 of them, at local [agg, agg + 32)
      // (every codeword has >= 1 bit, so 32 symbols always suffice)
      const int L = (int)(tail_e & 63);
      int x = L;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      const int excl = x - L;
      if (L > 0 && excl < 32) {
        const int take = L < 32 - excl ? L : 32 - excl;
        const unsigned long long bits =
            (((tail_e >> 6) << (64 - L)) >> (64 - take)) << (64 - take);  // left-aligned
        const int p = agg + excl;
        const unsigned long long y = bits >> (p & 31);
        atomicOr(&s_words[p >> 5], (uint32_t)(y >> 32));
        if ((uint32_t)y) atomicOr(&s_words[(p >> 5) + 1], (uint32_t)y);
      }
    }
  }
  __syncthreads();

  // ---- store the owned words (first bit inside [start, start + agg)): output
  // word gw holds local bits [32 gw - start, +32), a funnel of two local words
  const long long start = s_start;
  const int sh = (int)(start & 31);
  const int64_t gw0 = start >> 5;
  const int nout = (sh + agg + 31) / 32;
  for (int m = (sh ? 1 : 0) + tid; m < nout; m += HE_THREADS) {
    const uint32_t word = sh ? __funnelshift_r(s_words[m], s_words[m - 1], sh) : s_words[m];
    const int64_t gw = gw0 + m;
    if (gw < a.out_words) a.out[gw] = __byte_perm(word, 0, 0x0123);
    else a.info[2] = 1;
  }
}

}  // namespace
}  // namespace vlz

extern "C" {

size_t vlz_huff_table_bytes(void) { return vlz::HE_TAB + vlz::HE_LEN + 65536 * 16; }

int vlz_huff_table(const uint16_t* h_syms, const uint8_t* h_lens, int32_t nsym, void* d_table,
                   void* stream) {
  if (!d_table || nsym < 1 || nsym > 65536 || !h_syms || !h_lens) return VLZ_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // canonical codewords of the (length, symbol)-sorted book (huffman.py:33-45)
  std::vector<unsigned long long> staged(2 * (size_t)nsym);
  unsigned long long code = 0;
  for (int i = 0; i < nsym; ++i) {
    const int L = h_lens[i];
    if (L < 1 || L > vlz::HE_MAXLEN || (i && L < h_lens[i - 1])) return VLZ_E_ARG;
    staged[2 * i] = h_syms[i];
    staged[2 * i + 1] = (code << 6) | (unsigned long long)L;
    code += 1;
    if (i + 1 < nsym) code <<= (int)h_lens[i + 1] - L;
  }
  auto* tab = static_cast<unsigned long long*>(d_table);
  auto* len = static_cast<uint8_t*>(d_table) + vlz::HE_TAB;
  auto* dst = reinterpret_cast<unsigned long long*>(len + vlz::HE_LEN);
  if (cudaMemsetAsync(tab, 0, vlz::HE_TAB + vlz::HE_LEN, st) != cudaSuccess) return VLZ_E_CUDA;
  // pageable source: returns once the bytes are staged, `staged` may go
  if (cudaMemcpyAsync(dst, staged.data(), staged.size() * 8, cudaMemcpyHostToDevice, st) !=
      cudaSuccess)
    return VLZ_E_CUDA;
  vlz::he_table_kernel<<<(nsym + 255) / 256, 256, 0, st>>>(dst, nsym, tab, len);
  vlz::g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

size_t vlz_huff_encode_ws_size(int64_t n) {
  const int64_t nchunks = n > 0 ? (n + vlz::HE_CH - 1) / vlz::HE_CH : 1;
  return 256 + (size_t)nchunks * 8;
}

int vlz_huff_encode_device(const uint16_t* d_codes, int64_t n, const void* d_table,
                           int32_t nsym_span, int32_t max_len, uint8_t* d_out, int64_t out_cap, int64_t* d_info,
                           void* d_ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !d_table || !d_info || !d_ws || (n > 0 && (!d_codes || !d_out))) return VLZ_E_ARG;
  if ((reinterpret_cast<uintptr_t>(d_codes) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 3))
    return VLZ_E_ARG;
  if (ws_bytes < vlz_huff_encode_ws_size(n) || max_len < 1 || max_len > vlz::HE_MAXLEN)
    return VLZ_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nchunks = n > 0 ? (n + vlz::HE_CH - 1) / vlz::HE_CH : 1;
  auto* ticket = static_cast<unsigned int*>(d_ws);
  auto* lb = reinterpret_cast<unsigned long long*>(static_cast<char*>(d_ws) + 256);
  int64_t ig = (nchunks + 255) / 256;
  if (ig > 1024) ig = 1024;
  vlz::he_init_kernel<<<(unsigned)ig, 256, 0, st>>>(lb, nchunks, ticket,
                                                     reinterpret_cast<long long*>(d_info));
  vlz::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (n == 0) return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
  vlz::HEArgs a{};
  a.codes = d_codes;
  a.n = n;
  a.tab = static_cast<const unsigned long long*>(d_table);
  a.len = static_cast<const uint8_t*>(d_table) + vlz::HE_TAB;
  a.nsym_span = nsym_span;
  a.out = reinterpret_cast<uint32_t*>(d_out);
  a.out_words = out_cap / 4;
  a.lb = lb;
  a.ticket = ticket;
  a.info = reinterpret_cast<long long*>(d_info);
  // shared words: the chunk's bits at max_len per symbol, plus alignment
  const size_t smem = ((size_t)vlz::HE_CH * max_len / 32 + 4) * 4;
  // opt in to > 48 KB (books up to 58 bits); per device, so set every call
  if (cudaFuncSetAttribute(vlz::huff_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           ((size_t)vlz::HE_CH * vlz::HE_MAXLEN / 32 + 4) * 4) != cudaSuccess)
    return VLZ_E_CUDA;
  vlz::huff_encode_kernel<<<(unsigned)nchunks, vlz::HE_THREADS, smem, st>>>(a);
  vlz::g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? VLZ_OK : VLZ_E_CUDA;
}

}  // extern "C"
