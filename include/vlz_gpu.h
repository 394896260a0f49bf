/*
 * vlz_gpu.h -- C ABI of the B200-native dual-quantization path.
 *
 * Drop-in boundary for the reference package `vlz` (Python, numpy).  The
 * reference has no FFI of its own; its seams are Python functions, so each
 * entry point below names the reference function it replaces (paths relative
 * to /root/reference/pkg/src/vlz/).  INTEGRATION.md shows the ctypes binding a
 * maintainer adds on the reference side.
 *
 * Conventions
 *  - plain pointers + sizes, no torch types; every `d_*` pointer is device
 *    memory, every `h_*` pointer is host memory (pinned for full speed).
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *  - all device entry points are asynchronous and stream-ordered; errors found
 *    on the device (non-finite input, quantizer overflow, corrupt streams) are
 *    reported in a caller-allocated device `vlz_result` the caller reads back.
 *  - return value: VLZ_OK or a launch/argument error (VLZ_E_ARG, VLZ_E_CUDA).
 *  - the library allocates nothing on the device paths (workspace is caller
 *    owned); the *_host paths keep a per-device pool of staging buffers.
 */
#ifndef VLZ_GPU_H_
#define VLZ_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes of the entry points */
#define VLZ_OK 0
#define VLZ_E_ARG 1  /* invalid geometry / parameters (host-side check) */
#define VLZ_E_CUDA 2 /* CUDA launch / memory error                      */

/* device-side status codes (vlz_result.status).  Mapped by the Python layer
 * onto the reference's exception classes (errors.py:8-62):               */
#define VLZ_ST_OK 0
#define VLZ_ST_NONFINITE 1       /* ConfigError: non-finite value at flat index   */
#define VLZ_ST_OVERFLOW 2        /* BoundTooSmallError(index, value, eb)          */
#define VLZ_ST_CORRUPT_CODE 4    /* CorruptStreamError: code >= 2R (first block)  */
#define VLZ_ST_EXHAUSTED 5       /* CorruptStreamError: outliers exhausted        */
#define VLZ_ST_LEFTOVER 6        /* CorruptStreamError: leftover outliers         */
#define VLZ_ST_SENTINEL_TOTAL 7  /* CorruptStreamError: sentinels != outliers     */
#define VLZ_ST_OUTLIER_CAPACITY 8 /* vlz_dq_compress_capped: more outliers than the caller's array holds */

/* padding policy codes: container.py:57-58 ordering */
#define VLZ_PAD_ZERO 0
#define VLZ_PAD_MIN 1
#define VLZ_PAD_MAX 2
#define VLZ_PAD_MEAN 3
#define VLZ_GRAN_GLOBAL 0
#define VLZ_GRAN_BLOCK 1
#define VLZ_GRAN_EDGE 2

/* Array geometry + block tiling (model.py:48-159).  dims are the reference's
 * row-major extents, dims[0] slowest; only the first nd entries are read. */
typedef struct vlz_geom {
  int32_t nd;         /* 1, 2 or 3                                         */
  int32_t block_edge; /* 8, 16, 32, 64 (256 accepted for nd == 1)          */
  int64_t dims[3];
} vlz_geom;

/* Quantizer parameters (model.py:200-231, padding policy model.py:162-197) */
typedef struct vlz_params {
  double eb;          /* resolved absolute error bound (model.py:94-110)  */
  int32_t radius;     /* 2 .. 32768                                        */
  int32_t pad_kind;   /* VLZ_PAD_*                                         */
  int32_t pad_gran;   /* VLZ_GRAN_*                                        */
  int32_t reserved;
} vlz_params;

/* Device-written result block (64 bytes). */
typedef struct vlz_result {
  int32_t status;        /* VLZ_ST_*                                          */
  int32_t reserved;
  int64_t index;         /* flat element index (compress) / block index      */
  int64_t n_outliers;    /* compress: outliers written; decompress: sentinels */
  int64_t first_nonfinite; /* raw minima, INT64_MAX when none                */
  int64_t first_overflow;
  int64_t first_bad_block; /* (block << 4) | status, INT64_MAX when none     */
  int64_t sentinels;
  int64_t pad0;
} vlz_result;

/* Global padding statistics over the prequantized field (padding.py:62-69),
 * accumulated by compress_begin; all-reduced across ranks for sharded runs
 * (sum: wrapping int64 add; count: add; min: min; neg_max: min of -max). */
typedef struct vlz_stats {
  int64_t sum;
  int64_t count;
  int64_t min;
  int64_t neg_max;
} vlz_stats;

/* ---- geometry helpers (host) --------------------------------------- */
int64_t vlz_block_count(const vlz_geom* g);
/* PaddingPolicy.scalar_count (model.py:167-175) */
int64_t vlz_scalar_count(const vlz_geom* g, int32_t pad_kind, int32_t pad_gran);
/* Device workspace bytes needed by compress/decompress for this geometry.
 * The workspace needs no initialisation and may be reused across calls and
 * geometries: the first kernel of every call resets the state the call uses
 * (there is no separate init launch).  One workspace serves one call at a
 * time (calls ordered on one stream, or otherwise not overlapping). */
size_t vlz_workspace_size(const vlz_geom* g);
/* Optional larger workspace (4 bytes per element more): with at least this many
 * bytes the compress path keeps one outlier scratch slot per element instead
 * of 8 per block, and its scan kernel copies the outliers of outlier-dense
 * blocks (> 8 per block) instead of regenerating them from the codes and the
 * input.  Same results; worth it only for outlier-dense data (a 17.8 %-outlier
 * 256^3 field: compress call 72 us instead of 148 us).  The library picks the
 * layout from the ws_bytes it is given, so begin / finish / capped calls of
 * one compression must be given the same ws_bytes. */
size_t vlz_workspace_size_dense(const vlz_geom* g);

/* ---- compress: replaces vector.dualquant_vector (vector.py:205-260) ---- *
 * d_in         float32[N] row-major input
 * d_codes      uint16[N] quantization codes, canonical block-major order
 *              (0 = outlier sentinel; CodeStream.codes, model.py:254)
 * d_outliers   float32[N] capacity; the first n_outliers hold the verbatim
 *              outlier values in canonical order (CodeStream.outlier_values)
 * d_counts     int64[nblocks] outliers per block (CodeStream.outlier_counts)
 * d_scalars    int64[scalar_count] padding scalars (PaddingScalars.values)
 * d_result     status, first error indices and n_outliers                    */
int vlz_dq_compress(const float* d_in, const vlz_geom* g, const vlz_params* p,
                    uint16_t* d_codes, float* d_outliers, int64_t* d_counts,
                    int64_t* d_scalars, vlz_result* d_result, void* d_ws,
                    size_t ws_bytes, void* stream);

/* The same compression with an outlier array of `outlier_capacity` floats
 * (any size from 0 to N; vlz_dq_compress needs the worst case, N).  Codes,
 * counts, scalars and n_outliers are always complete.  When the stream has
 * more outliers than fit, d_outliers holds the first outlier_capacity of them
 * and the status is VLZ_ST_OUTLIER_CAPACITY: call again with at least
 * n_outliers floats.  With the 8-slots-per-block scratch of the workspace this
 * bounds the device memory of a compression by the stream it produces
 * (C5: 17.2 GB in + 8.6 GB codes + 0.3 GB workspace + the outliers kept). */
int vlz_dq_compress_capped(const float* d_in, const vlz_geom* g, const vlz_params* p,
                           uint16_t* d_codes, float* d_outliers, int64_t outlier_capacity,
                           int64_t* d_counts, int64_t* d_scalars, vlz_result* d_result,
                           void* d_ws, size_t ws_bytes, void* stream);

/* Two-phase form for slab-sharded multi-GPU runs (each rank compresses a
 * block-aligned slab along dims[0]).  begin = fused prequant + Lorenzo +
 * postquant + block/edge padding; for *:global policies it also writes this
 * shard's partial statistics to d_stats and leaves block origins pending.
 * The caller all-reduces d_stats (NCCL) and then calls finish, which resolves
 * the global scalar, the origin codes and compacts the outliers.  d_in, the
 * codes and the workspace must stay untouched between begin and finish:
 * finish reads the values of outlier-dense blocks (more than 8 outliers) back
 * from d_in at the positions the codes mark. */
int vlz_dq_compress_begin(const float* d_in, const vlz_geom* g, const vlz_params* p,
                          uint16_t* d_codes, int64_t* d_counts, int64_t* d_scalars,
                          vlz_result* d_result, vlz_stats* d_stats, void* d_ws,
                          size_t ws_bytes, void* stream);
int vlz_dq_compress_finish(const float* d_in, const vlz_geom* g, const vlz_params* p,
                           const vlz_stats* d_global_stats, uint16_t* d_codes,
                           float* d_outliers, int64_t* d_counts, int64_t* d_scalars,
                           vlz_result* d_result, void* d_ws, size_t ws_bytes, void* stream);
/* As finish, with the statistics of every rank as gathered (one all-gather
 * of nranks vlz_stats records, rank order) instead of pre-reduced: the
 * reduction (wrapping sum, count, min, min of -max) runs inside the scan
 * kernel, so a sharded step needs no reduction kernels of its own. */
int vlz_dq_compress_finish_gathered(const float* d_in, const vlz_geom* g, const vlz_params* p,
                                    const vlz_stats* d_rank_stats, int32_t nranks,
                                    uint16_t* d_codes, float* d_outliers, int64_t* d_counts,
                                    int64_t* d_scalars, vlz_result* d_result, void* d_ws,
                                    size_t ws_bytes, void* stream);

/* ---- decompress: replaces reconstruct.decompress_parsed minus the Huffman
 * decode (reconstruct.py:30-124).  Codes uint16 (container symbol width) or
 * uint32 (CodeStream width).  d_out float32[N] row-major.  Stream corruption
 * is reported in d_result (status, index = first failing block). ---------- */
int vlz_dq_decompress(const uint16_t* d_codes, const float* d_outliers,
                      int64_t n_outliers, const int64_t* d_counts, const int64_t* d_scalars,
                      const vlz_geom* g, const vlz_params* p, float* d_out,
                      vlz_result* d_result, void* d_ws, size_t ws_bytes, void* stream);
/* As vlz_dq_decompress, with the stored outlier count read from device
 * memory (e.g. &d_result->n_outliers of the vlz_dq_compress that produced the
 * stream): a compress -> decompress round trip on one stream then needs no
 * host synchronisation in between.  Replaces the host-side
 * len(CodeStream.outlier_values) of reconstruct.py:87-91.  d_n_outliers must not
 * alias d_result (the decompressor resets its own result block first). */
int vlz_dq_decompress_dn(const uint16_t* d_codes, const float* d_outliers,
                         const int64_t* d_n_outliers, const int64_t* d_counts,
                         const int64_t* d_scalars, const vlz_geom* g, const vlz_params* p,
                         float* d_out, vlz_result* d_result, void* d_ws, size_t ws_bytes,
                         void* stream);
int vlz_dq_decompress_u32(const uint32_t* d_codes, const float* d_outliers,
                          int64_t n_outliers, const int64_t* d_counts,
                          const int64_t* d_scalars, const vlz_geom* g, const vlz_params* p,
                          float* d_out, vlz_result* d_result, void* d_ws, size_t ws_bytes,
                          void* stream);

/* ---- value range for ErrorBound.relative (model.py:104-110) ------------ *
 * d_minmax[0] = float(min), d_minmax[1] = float(max), NaN-propagating like
 * numpy's min/max. */
int vlz_minmax(const float* d_in, int64_t n, double* d_minmax, void* stream);

/* ---- host-buffer entry points (end-to-end: H2D + kernels + D2H) -------- *
 * Same semantics as the device versions; buffers are host memory (pinned for
 * full PCIe speed).  Synchronous: returns after the results are in host
 * memory.  *h_result receives the status block.  Thread-safe: concurrent
 * calls (up to 4 per device) run on their own streams and staging buffers,
 * so a compress (mostly H2D) and a decompress (mostly D2H) issued from two
 * host threads overlap on the full-duplex link. */
int vlz_dq_compress_host(const float* h_in, const vlz_geom* g, const vlz_params* p,
                         uint16_t* h_codes, float* h_outliers, int64_t* h_counts,
                         int64_t* h_scalars, vlz_result* h_result, int device);
int vlz_dq_decompress_host(const uint16_t* h_codes, const float* h_outliers,
                           int64_t n_outliers, const int64_t* h_counts,
                           const int64_t* h_scalars, const vlz_geom* g, const vlz_params* p,
                           float* h_out, vlz_result* h_result, int device);
/* release the cached staging buffers of the host entry points */
void vlz_host_release(void);

/* ---- entropy stage after the path (huffman.py, container.py) ------------ *
 * canonical Huffman coding of the uint16 code stream with the reference's
 * codebook, bit order and error verdicts (see csrc/huffman.cpp). */
/* symbol frequencies (np.bincount, huffman.py:62) on the device; d_freqs is
 * uint64[65536]; radius centres the shared-memory window */
int vlz_histogram(const uint16_t* d_codes, int64_t n, int32_t radius, uint64_t* d_freqs,
                  void* stream);
void vlz_histogram_host(const uint16_t* h_codes, int64_t n, uint64_t* h_freqs);
/* build_codebook (huffman.py:56-88): canonical (length, symbol) order; returns
 * 0, -1 for an empty stream, -2 if a code length exceeds 64 bits */
int vlz_huff_build(const uint64_t* h_freqs, uint16_t* h_syms, uint8_t* h_lens, int32_t* h_nsym);
/* encode (huffman.py:91-122): MSB-first; returns 0 or -1 (*bad_symbol set) */
int vlz_huff_encode(const uint16_t* h_codes, int64_t n, const uint16_t* h_syms,
                    const uint8_t* h_lens, int32_t nsym, uint8_t* h_out, int64_t out_cap,
                    int64_t* h_nbits, int64_t* h_bad_symbol);
/* device encode (huffman.py:91-122 on the GPU, csrc/k_huffenc.cu).
 * vlz_huff_table uploads a canonical book (symbols/lengths in (length,
 * symbol) order, lengths <= 58) into d_table (vlz_huff_table_bytes()).
 * vlz_huff_encode_device packs n uint16 codes (16-byte aligned) into d_out
 * (4-byte aligned, out_cap bytes; whole 32-bit words are written, bits past
 * the end are zero) and fills d_info (int64[4], device): [0] bit length,
 * [1] (index << 16 | symbol) of the first symbol >= nsym_span (= largest book
 * symbol + 1) or INT64_MAX, [2] 1 if out_cap was too small, [3] first symbol
 * absent from the book or INT64_MAX.  max_len = longest book codeword (sizes
 * shared memory).  Stream-ordered, no host sync. */
size_t vlz_huff_table_bytes(void);
int vlz_huff_table(const uint16_t* h_syms, const uint8_t* h_lens, int32_t nsym, void* d_table,
                   void* stream);
size_t vlz_huff_encode_ws_size(int64_t n);
int vlz_huff_encode_device(const uint16_t* d_codes, int64_t n, const void* d_table,
                           int32_t nsym_span, int32_t max_len, uint8_t* d_out, int64_t out_cap, int64_t* d_info,
                           void* d_ws, size_t ws_bytes, void* stream);
/* device decode (huffman.py:125-207 on the GPU, csrc/k_huffdec.cu):
 * self-synchronising parallel decode of the single MSB-first stream.
 * d_payload: 4-byte aligned device copy of the payload (nbytes) followed by
 * >= 16 zero bytes past nbytes rounded up to 4; d_out 16-byte aligned.  Returns the
 * same verdict codes as vlz_huff_decode (0 ok, 1..5) with *h_consumed, or a
 * negative VLZ_E_*; synchronises `stream`.  Code lengths <= 58. */
size_t vlz_huff_decode_ws_size(int64_t nbytes);
int vlz_huff_decode_device(const uint8_t* d_payload, int64_t nbytes, int64_t bit_length,
                           const uint16_t* h_syms, const uint8_t* h_lens, int32_t nsym,
                           int64_t count, uint16_t* d_out, int64_t* h_consumed, void* d_ws,
                           size_t ws_bytes, void* stream);
/* decode (huffman.py:125-207): exactly `count` symbols; returns 0 or the
 * reference's verdict 1..5 (empty/short payload/underrun/invalid prefix/
 * consumed != declared bits) */
int vlz_huff_decode(const uint8_t* h_payload, int64_t nbytes, int64_t bit_length,
                    const uint16_t* h_syms, const uint8_t* h_lens, int32_t nsym, int64_t count,
                    uint16_t* h_out, int64_t* h_consumed);

/* border-outlier census (vector.py:82-87, collect_border): outliers (code 0)
 * whose block-local coordinates include a 0, over a canonical uint16 code
 * stream; *d_total (device int64) receives the count, stream-ordered */
int vlz_border_outliers(const uint16_t* d_codes, const vlz_geom* g, int64_t* d_total,
                        void* stream);

/* padding-policy census for outlier_report (padding.py:162-205): for every
 * policy, the block origins that are outliers (|d_o - s0| > R-1 or a failed
 * narrowing check; by finding 1 the only elements whose verdict depends on
 * the policy).  One pass over d_in (float32, row-major).  d_counts (device
 * int64[12]) is overwritten: [0] zero padding, [3*kind + gran] for
 * VLZ_PAD_MIN/MAX/MEAN x VLZ_GRAN_GLOBAL/BLOCK/EDGE.  Stream-ordered. */
size_t vlz_padding_census_ws_size(const vlz_geom* g);
int vlz_padding_census(const float* d_in, const vlz_geom* g, double eb, int32_t radius,
                       int64_t* d_counts, void* d_ws, size_t ws_bytes, void* stream);

/* CRC-32 (zlib: polynomial 0xEDB88320 reflected, init/xorout 0xFFFFFFFF) of
 * n device bytes -- the VLZ1 payload CRC (container.py:160-163, 214-217).
 * *d_crc (device uint32) receives zlib.crc32(bytes); any alignment; workspace
 * of vlz_crc32_ws_size(n) device bytes.  Stream-ordered. */
size_t vlz_crc32_ws_size(int64_t n);
int vlz_crc32_device(const uint8_t* d_data, int64_t n, uint32_t* d_crc, void* d_ws,
                     size_t ws_bytes, void* stream);

/* number of kernel launches the library issued since load (bench evidence) */
int64_t vlz_launch_count(void);
/* per-kernel CUDA-event timing: when enabled every launch is bracketed by
 * events on its stream; collect() synchronises and returns, per kind
 * (0 unused since the reset moved into the first kernel, 1 fused compress,
 * 2 compress scan/gather, 3 decompress scan, 4 fused decompress, 5 minmax,
 * 6 unused since the fused kernels redo int32-unsafe tiles themselves), the
 * summed milliseconds and launch counts
 * since the last collect. */
void vlz_timing(int enable);
int vlz_timing_collect(double* ms, int64_t* launches, int n);
/* library build string (arch, commit) */
const char* vlz_version(void);

/* ---- test support (not on any product path; tests/test_gpu_sweep.py) ---- *
 * Exhaustive check of the float32 exact-fast prequantizer against the exact
 * float64 one (quantize.py:31-42,66-78; vector.py:72-77) over all 2^32 float
 * bit patterns at bound eb.  d_counts (device uint64[6]) receives: accepted
 * by the fast path, finite but sent to the exact path, non-finite, accepted
 * but wrong (n differs, overflow or narrowing failure -- must be 0), scalar
 * vs paired-FP32 form disagreements (must be 0), first offending pattern
 * (UINT64_MAX when none).  Stream-ordered. */
int vlz_test_prequant_sweep(double eb, unsigned long long* d_counts, void* stream);
/* 1 when the fast path is enabled for this eb (1/(2eb) in (2^-100, 2^100)) */
int vlz_test_fast_enabled(double eb);

/* ---- measurement support (not a product path; bench.py) -------------- *
 * One arithmetic-free streaming kernel over n_elems elements (a multiple of
 * 8, 16-byte aligned buffers) with the read : write mix of a fused kernel:
 * kind 0 copy f32 -> f32 (4 B read + 4 B written per element), 1 narrow
 * f32 -> u16 (4 + 2: the compress mix), 2 widen u16 -> f32 (2 + 4: the
 * decompress mix); ctas_per_sm (1..8) CTAs of 256 threads per SM.  The caller
 * times it with events on `stream`. */
int vlz_bench_stream(int32_t kind, const void* d_src, void* d_dst, int64_t n_elems,
                     int32_t ctas_per_sm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VLZ_GPU_H_ */
