/*
 * vlz_oracle.c -- CPU restatement of the reference dual-quantization path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2201_04614_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It is never
 * the thing measured as the GPU result and never a fallback for the product.
 *
 * It restates, element by element, the algorithm of the reference Python
 * package `vlz` (paths relative to /root/reference/pkg/src/vlz/):
 *
 *   prequantize          quantize.py:31-42 (round_half_away, quantize_value),
 *                        quantize.py:50-79 (prequantize: non-finite check over
 *                        the whole array first, then the 2^31-1 overflow guard)
 *   padding statistics   padding.py:53-59 (_round_half_away_ratio),
 *                        padding.py:62-69 (_statistic), padding.py:72-110
 *                        (compute_padding: global/block/edge, in-bounds only)
 *   halo + prediction    padding.py:113-129 (apply_padding),
 *                        kernel.py:72-79 (PaddedBlock.value_at: a neighbour
 *                        below several faces takes the highest such dim's
 *                        scalar), kernel.py:82-101 (lorenzo_predict)
 *   postquant + outliers kernel.py:162-185 / vector.py:72-78 (delta range test
 *                        plus the float32-narrowed reconstruction bound test;
 *                        outliers keep the verbatim float32)
 *   canonical order      model.py:113-159 (BlockGrid: row-major blocks, partial
 *                        edge blocks), vector.py:193-202 (codes[inb], per-block
 *                        int64 outlier counts)
 *   reconstruction       reconstruct.py:30-71 (reconstruct_block: sequential,
 *                        sentinel -> quantize_value(verbatim)), reconstruct.py:
 *                        74-124 (decompress_parsed minus the Huffman decode)
 *
 * Unlike the CUDA kernels it deliberately does NOT use the separable
 * difference / prefix-sum reformulation: it evaluates
 * the reference's own 7-point stencil with the reference's halo rule, so that
 * agreement between the two is evidence for the reformulation.
 *
 * Floating point: compiled with -O2 -fno-fast-math -ffp-contract=off so every
 * double expression is a single IEEE round-to-nearest op, as in numpy.
 *
 * Parity pin: tests/test_oracle_golden.py checks this oracle against vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* status codes shared with oracle/oracle.py */
enum {
  VLZO_OK = 0,
  VLZO_NONFINITE = 1,      /* ConfigError("...non-finite value at flat index i") */
  VLZO_OVERFLOW = 2,       /* BoundTooSmallError(i, v, eb)                      */
  VLZO_BAD_CONFIG = 3,     /* ConfigError (eb <= 0, bad geometry)               */
  VLZO_CORRUPT_CODE = 4,   /* CorruptStreamError: code >= 2R in block           */
  VLZO_EXHAUSTED = 5,      /* CorruptStreamError: outliers exhausted            */
  VLZO_LEFTOVER = 6,       /* CorruptStreamError: leftover outliers             */
  VLZO_SENTINEL_TOTAL = 7, /* CorruptStreamError: sentinel total != outliers    */
  VLZO_NOMEM = 8
};

/* padding kinds / granularities: container.py:57-58 ordering */
enum { PAD_ZERO = 0, PAD_MIN = 1, PAD_MAX = 2, PAD_MEAN = 3 };
enum { GRAN_GLOBAL = 0, GRAN_BLOCK = 1, GRAN_EDGE = 2 };

#define OVERFLOW_LIMIT 2147483647.0 /* quantize.py:28 */

/* quantize.py:31-37 */
static inline int64_t round_half_away(double q) {
  if (q > 0.0) return (int64_t)floor(q + 0.5);
  if (q < 0.0) return -(int64_t)floor(-q + 0.5);
  return 0;
}

/* quantize.py:40-42 (v / (2.0 * eb) evaluated in float64) */
static inline int64_t quantize_value(double v, double eb) {
  return round_half_away(v / (2.0 * eb));
}

/* quantize.py:45-47 / 82-84: float32((2.0 * d) * eb) */
static inline float reconstruct_value(int64_t d, double eb) {
  return (float)((2.0 * (double)d) * eb);
}

typedef struct {
  int nd;
  int64_t dims[3];
  int b;
  int64_t per[3];   /* blocks per dim, model.py:154 */
  int64_t nblocks;
} grid_t;

static void grid_init(grid_t* g, int nd, const int64_t* dims, int b) {
  g->nd = nd;
  g->b = b;
  g->nblocks = 1;
  for (int d = 0; d < nd; ++d) {
    g->dims[d] = dims[d];
    g->per[d] = (dims[d] + b - 1) / b;
    g->nblocks *= g->per[d];
  }
}

/* model.py:126-145: block coords (row-major), origin and extents */
static void block_geom(const grid_t* g, int64_t bi, int64_t* origin, int64_t* ext) {
  int64_t rem = bi;
  int64_t c[3];
  for (int d = g->nd - 1; d >= 0; --d) {
    c[d] = rem % g->per[d];
    rem /= g->per[d];
  }
  for (int d = 0; d < g->nd; ++d) {
    origin[d] = c[d] * g->b;
    int64_t e = g->dims[d] - origin[d];
    ext[d] = e < g->b ? e : g->b;
  }
}

static inline int64_t flat_index(const grid_t* g, const int64_t* idx) {
  int64_t f = 0;
  for (int d = 0; d < g->nd; ++d) f = f * g->dims[d] + idx[d];
  return f;
}

/* quantize.py:50-79.  Non-finite check over the whole array first, then the
 * overflow guard in row-major order; returns the first offending index. */
int vlzo_prequantize(const float* data, int64_t n, double eb, int64_t* dq,
                     int64_t* err_index) {
  if (eb <= 0.0) return VLZO_BAD_CONFIG; /* quantize.py:58-59 (NaN falls through) */
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for reduction(min : first_bad) schedule(static)
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(data[i]) && i < first_bad) first_bad = i;
  if (first_bad != INT64_MAX) {
    *err_index = first_bad;
    return VLZO_NONFINITE;
  }
  const double twoeb = 2.0 * eb;
  int64_t first_ovf = INT64_MAX;
#pragma omp parallel for reduction(min : first_ovf) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double q = (double)data[i] / twoeb;
    if (fabs(q) >= OVERFLOW_LIMIT || q != q) {
      if (i < first_ovf) first_ovf = i;
      dq[i] = 0;
    } else {
      dq[i] = round_half_away(q);
    }
  }
  if (first_ovf != INT64_MAX) {
    *err_index = first_ovf;
    return VLZO_OVERFLOW;
  }
  return VLZO_OK;
}

/* padding.py:53-59: exact round-half-away of total/count (total is the int64,
 * wrapping numpy sum converted to a Python int). */
static int64_t round_half_away_ratio(int64_t total, int64_t count) {
  uint64_t mag = total < 0 ? (uint64_t)0 - (uint64_t)total : (uint64_t)total;
  uint64_t q = mag / (uint64_t)count, r = mag % (uint64_t)count;
  uint64_t res = q + ((2 * r >= (uint64_t)count) ? 1 : 0);
  return total < 0 ? -(int64_t)res : (int64_t)res;
}

typedef struct {
  int64_t mn, mx;
  uint64_t sum; /* wraps like np.sum(dtype=int64) */
  int64_t cnt;
} stat_t;

static inline void stat_reset(stat_t* s) {
  s->mn = INT64_MAX;
  s->mx = INT64_MIN;
  s->sum = 0;
  s->cnt = 0;
}
static inline void stat_add(stat_t* s, int64_t v) {
  if (v < s->mn) s->mn = v;
  if (v > s->mx) s->mx = v;
  s->sum += (uint64_t)v;
  s->cnt++;
}
/* padding.py:62-69 */
static inline int64_t stat_value(const stat_t* s, int kind) {
  if (kind == PAD_MIN) return s->mn;
  if (kind == PAD_MAX) return s->mx;
  return round_half_away_ratio((int64_t)s->sum, s->cnt);
}

/* element-of-block iteration helpers */
static inline int64_t block_elems(const grid_t* g, const int64_t* ext) {
  int64_t n = 1;
  for (int d = 0; d < g->nd; ++d) n *= ext[d];
  return n;
}

/* padding.py:72-110 */
static int64_t padding_scalar_count(const grid_t* g, int kind, int gran) {
  if (kind == PAD_ZERO) return 0;
  if (gran == GRAN_GLOBAL) return 1;
  if (gran == GRAN_BLOCK) return g->nblocks;
  return g->nblocks * g->nd;
}

static void compute_padding(const grid_t* g, const int64_t* dq, int kind, int gran,
                            int64_t* scalars) {
  if (kind == PAD_ZERO) return;
  int64_t n = 1;
  for (int d = 0; d < g->nd; ++d) n *= g->dims[d];
  if (gran == GRAN_GLOBAL) {
    /* the int64 sum wraps like numpy's; unsigned addition is associative */
    uint64_t sum = 0;
    int64_t mn = INT64_MAX, mx = INT64_MIN;
#pragma omp parallel for reduction(+ : sum) reduction(min : mn) reduction(max : mx) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      sum += (uint64_t)dq[i];
      if (dq[i] < mn) mn = dq[i];
      if (dq[i] > mx) mx = dq[i];
    }
    stat_t s = {mn, mx, sum, n};
    scalars[0] = stat_value(&s, kind);
    return;
  }
  const int nd = g->nd;
#pragma omp parallel for schedule(static)
  for (int64_t bi = 0; bi < g->nblocks; ++bi) {
    int64_t org[3], ext[3] = {1, 1, 1};
    block_geom(g, bi, org, ext);
    int64_t e0 = ext[0], e1 = nd > 1 ? ext[1] : 1, e2 = nd > 2 ? ext[2] : 1;
    if (gran == GRAN_BLOCK) {
      stat_t s;
      stat_reset(&s);
      for (int64_t i = 0; i < e0; ++i)
        for (int64_t j = 0; j < e1; ++j)
          for (int64_t k = 0; k < e2; ++k) {
            int64_t idx[3] = {org[0] + i, nd > 1 ? org[1] + j : 0, nd > 2 ? org[2] + k : 0};
            stat_add(&s, dq[flat_index(g, idx)]);
          }
      scalars[bi] = stat_value(&s, kind);
    } else {
      /* edge: face of dim d is the block's coord_d == 0 slice */
      for (int fd = 0; fd < nd; ++fd) {
        stat_t s;
        stat_reset(&s);
        for (int64_t i = 0; i < e0; ++i)
          for (int64_t j = 0; j < e1; ++j)
            for (int64_t k = 0; k < e2; ++k) {
              int64_t loc[3] = {i, j, k};
              if (loc[fd] != 0) continue;
              int64_t idx[3] = {org[0] + i, nd > 1 ? org[1] + j : 0, nd > 2 ? org[2] + k : 0};
              stat_add(&s, dq[flat_index(g, idx)]);
            }
        scalars[bi * nd + fd] = stat_value(&s, kind);
      }
    }
  }
}

/* padding.py:113-129 */
static void apply_padding(const grid_t* g, const int64_t* scalars, int kind, int gran,
                          int64_t bi, int64_t* halo) {
  for (int d = 0; d < g->nd; ++d) {
    if (kind == PAD_ZERO) halo[d] = 0;
    else if (gran == GRAN_GLOBAL) halo[d] = scalars[0];
    else if (gran == GRAN_BLOCK) halo[d] = scalars[bi];
    else halo[d] = scalars[bi * g->nd + d];
  }
}

/* kernel.py:72-79: PaddedBlock.value_at over a block-local int64 tile */
typedef struct {
  int nd;
  int64_t ext[3];
  const int64_t* halo;
  const int64_t* vals; /* block-local row-major, shape ext */
} padded_t;

static inline int64_t value_at(const padded_t* p, int64_t i, int64_t j, int64_t k) {
  int64_t c[3] = {i, j, k};
  int pad_dim = -1;
  for (int d = 0; d < p->nd; ++d)
    if (c[d] < 0) pad_dim = d;
  if (pad_dim >= 0) return p->halo[pad_dim];
  if (p->nd == 1) return p->vals[i];
  if (p->nd == 2) return p->vals[i * p->ext[1] + j];
  return p->vals[(i * p->ext[1] + j) * p->ext[2] + k];
}

/* kernel.py:82-101 */
static inline int64_t lorenzo_predict(const padded_t* p, int64_t i, int64_t j, int64_t k) {
  if (p->nd == 1) return value_at(p, i - 1, 0, 0);
  if (p->nd == 2) return value_at(p, i, j - 1, 0) + value_at(p, i - 1, j, 0) - value_at(p, i - 1, j - 1, 0);
  return value_at(p, i, j, k - 1) + value_at(p, i, j - 1, k) + value_at(p, i - 1, j, k) -
         value_at(p, i, j - 1, k - 1) - value_at(p, i - 1, j, k - 1) -
         value_at(p, i - 1, j - 1, k) + value_at(p, i - 1, j - 1, k - 1);
}

/* grow-only scratch arena (not re-entrant: the oracle is called serially) */
static void* g_arena = NULL;
static size_t g_arena_cap = 0;

static void* arena_get(size_t bytes) {
  if (bytes > g_arena_cap) {
    free(g_arena);
    g_arena = malloc(bytes);
    g_arena_cap = g_arena ? bytes : 0;
  }
  return g_arena;
}

/* closed-form canonical start of a block's codes (sum of sizes of all
 * earlier blocks in row-major block order) */
static int64_t block_code_start(const grid_t* g, int64_t bi) {
  int64_t org[3], ext[3];
  block_geom(g, bi, org, ext);
  if (g->nd == 1) return org[0];
  if (g->nd == 2) return org[0] * g->dims[1] + ext[0] * org[1];
  return org[0] * g->dims[1] * g->dims[2] + ext[0] * org[1] * g->dims[2] +
         ext[0] * ext[1] * org[2];
}

int64_t vlzo_scalar_count(int nd, const int64_t* dims, int b, int kind, int gran) {
  grid_t g;
  grid_init(&g, nd, dims, b);
  return padding_scalar_count(&g, kind, gran);
}

int64_t vlzo_block_count(int nd, const int64_t* dims, int b) {
  grid_t g;
  grid_init(&g, nd, dims, b);
  return g.nblocks;
}

/* Slab-sharded runs (SURVEY 8c "full-size parity strategy"): a shard of a
 * block-aligned slab must use the scalar of the WHOLE array for *:global
 * policies, as if compute_padding had been handed the full field.  The test
 * harness computes per-shard partial statistics with vlzo_global_stats,
 * all-reduces them and injects the result here. */
static int g_override_on = 0;
static int64_t g_override_value = 0;

void vlzo_set_global_scalar_override(int enable, int64_t value) {
  g_override_on = enable;
  g_override_value = value;
}

/* partial statistics of a slab's prequantized field: out = {wrapping sum,
 * count, min, max}; returns a VLZO_* status (prequantize errors) */
int vlzo_global_stats(const float* data, int64_t n, double eb, int64_t* out,
                      int64_t* err_index) {
  const size_t nn = (size_t)(n > 0 ? n : 1);
  int64_t* dq = (int64_t*)malloc(nn * sizeof(int64_t));
  if (!dq) return VLZO_NOMEM;
  int rc = vlzo_prequantize(data, n, eb, dq, err_index);
  if (rc == VLZO_OK) {
    uint64_t sum = 0;
    int64_t mn = INT64_MAX, mx = INT64_MIN;
    for (int64_t i = 0; i < n; ++i) {
      sum += (uint64_t)dq[i];
      if (dq[i] < mn) mn = dq[i];
      if (dq[i] > mx) mx = dq[i];
    }
    out[0] = (int64_t)sum;
    out[1] = n;
    out[2] = mn;
    out[3] = mx;
  }
  free(dq);
  return rc;
}

/* exact rounding of the global mean from reduced statistics (padding.py:53-69) */
int64_t vlzo_stat_value(int kind, int64_t sum, int64_t count, int64_t mn, int64_t mx) {
  stat_t s = {mn, mx, (uint64_t)sum, count};
  return stat_value(&s, kind);
}

/*
 * Full dual-quant compress (vector.py:205-260 semantics, scalar evaluation).
 * codes: N uint32 (canonical order); outlier_vals: capacity N; counts: nblocks;
 * scalars: vlzo_scalar_count(); *n_out = number of outliers written.
 * threads <= 0 uses the OpenMP default.
 */
int vlzo_dualquant(const float* data, int nd, const int64_t* dims, int b, double eb,
                   int radius, int pad_kind, int pad_gran, int threads, uint32_t* codes,
                   float* outlier_vals, int64_t* counts, int64_t* scalars, int64_t* n_out,
                   int64_t* err_index) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  grid_t g;
  grid_init(&g, nd, dims, b);
  int64_t n = 1;
  for (int d = 0; d < nd; ++d) n *= dims[d];
  /* dq + scratch come from a grow-only arena: re-faulting hundreds of MB of
   * fresh pages per call serialises on the kernel's mm lock and would make
   * the CPU baseline measure page faults instead of the algorithm */
  const size_t nn = (size_t)(n > 0 ? n : 1);
  char* arena = (char*)arena_get(nn * (sizeof(int64_t) + sizeof(float)));
  if (!arena) return VLZO_NOMEM;
  int64_t* dq = (int64_t*)arena;
  float* scratch = (float*)(arena + nn * sizeof(int64_t));
  int rc = vlzo_prequantize(data, n, eb, dq, err_index);
  if (rc != VLZO_OK) return rc;
  compute_padding(&g, dq, pad_kind, pad_gran, scalars);
  if (g_override_on && pad_kind != PAD_ZERO && pad_gran == GRAN_GLOBAL) scalars[0] = g_override_value;
  const int64_t keep_max = radius - 1;
  const int64_t bmax = (int64_t)b * (nd > 1 ? b : 1) * (nd > 2 ? b : 1);

#pragma omp parallel
  {
    int64_t* tile = (int64_t*)malloc(sizeof(int64_t) * (size_t)bmax);
#pragma omp for schedule(dynamic, 64)
    for (int64_t bi = 0; bi < g.nblocks; ++bi) {
      int64_t org[3], ext[3] = {1, 1, 1}, halo[3];
      block_geom(&g, bi, org, ext);
      apply_padding(&g, scalars, pad_kind, pad_gran, bi, halo);
      int64_t e0 = ext[0], e1 = nd > 1 ? ext[1] : 1, e2 = nd > 2 ? ext[2] : 1;
      /* gather the block's d values (row-major within block) */
      int64_t t = 0;
      for (int64_t i = 0; i < e0; ++i)
        for (int64_t j = 0; j < e1; ++j)
          for (int64_t k = 0; k < e2; ++k) {
            int64_t idx[3] = {org[0] + i, nd > 1 ? org[1] + j : 0, nd > 2 ? org[2] + k : 0};
            tile[t++] = dq[flat_index(&g, idx)];
          }
      padded_t p = {nd, {e0, e1, e2}, halo, tile};
      int64_t pos = block_code_start(&g, bi);
      int64_t nout = 0;
      t = 0;
      for (int64_t i = 0; i < e0; ++i)
        for (int64_t j = 0; j < e1; ++j)
          for (int64_t k = 0; k < e2; ++k, ++t) {
            int64_t idx[3] = {org[0] + i, nd > 1 ? org[1] + j : 0, nd > 2 ? org[2] + k : 0};
            float v = data[flat_index(&g, idx)];
            int64_t d = tile[t];
            int64_t pred = nd == 1 ? lorenzo_predict(&p, i, 0, 0)
                         : nd == 2 ? lorenzo_predict(&p, i, j, 0)
                                   : lorenzo_predict(&p, i, j, k);
            int64_t delta = d - pred;
            float w = reconstruct_value(d, eb);
            int in_range = (delta <= keep_max) && (delta >= -keep_max);
            int in_bound = fabs((double)w - (double)v) <= eb;
            if (in_range && in_bound) {
              codes[pos + t] = (uint32_t)(delta + radius);
            } else {
              codes[pos + t] = 0;
              scratch[pos + nout] = v;
              ++nout;
            }
          }
      counts[bi] = nout;
    }
    free(tile);
  }
  /* canonical outlier order: block-major, within-block traversal order */
  int64_t off = 0;
  for (int64_t bi = 0; bi < g.nblocks; ++bi) {
    if (counts[bi]) {
      memcpy(outlier_vals + off, scratch + block_code_start(&g, bi),
             sizeof(float) * (size_t)counts[bi]);
      off += counts[bi];
    }
  }
  *n_out = off;
  return VLZO_OK;
}

/*
 * Decompress (reconstruct.py:74-124 minus Huffman decode; per block
 * reconstruct.py:30-71).  Returns VLZO_OK or a CorruptStreamError flavour with
 * *err_index = failing block (lowest index; sequential semantics) and
 * *err_value = the offending code (VLZO_CORRUPT_CODE) or the consumed count
 * (VLZO_LEFTOVER).
 */
int vlzo_reconstruct(const uint32_t* codes, const float* outlier_vals, int64_t n_out,
                     const int64_t* counts, const int64_t* scalars, int nd,
                     const int64_t* dims, int b, double eb, int radius, int pad_kind,
                     int pad_gran, int threads, float* out, int64_t* err_index,
                     int64_t* err_value) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  grid_t g;
  grid_init(&g, nd, dims, b);
  int64_t n = 1;
  for (int d = 0; d < nd; ++d) n *= dims[d];
  /* reconstruct.py:87-91: sentinel total must equal the outlier count */
  int64_t nsent = 0;
#pragma omp parallel for reduction(+ : nsent) schedule(static)
  for (int64_t i = 0; i < n; ++i) nsent += codes[i] == 0;
  if (nsent != n_out) {
    *err_index = nsent;
    *err_value = n_out;
    return VLZO_SENTINEL_TOTAL;
  }
  int64_t* out_start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g.nblocks + 1));
  if (!out_start) return VLZO_NOMEM;
  out_start[0] = 0;
  for (int64_t bi = 0; bi < g.nblocks; ++bi) out_start[bi + 1] = out_start[bi] + counts[bi];
  const int64_t bmax = (int64_t)b * (nd > 1 ? b : 1) * (nd > 2 ? b : 1);
  int64_t first_bad = INT64_MAX;
  int bad_kind = VLZO_OK;
  int64_t bad_val = 0;

#pragma omp parallel
  {
    int64_t* tile = (int64_t*)malloc(sizeof(int64_t) * (size_t)bmax);
    float* ftile = (float*)malloc(sizeof(float) * (size_t)bmax);
    unsigned char* sent = (unsigned char*)malloc((size_t)bmax);
#pragma omp for schedule(dynamic, 64)
    for (int64_t bi = 0; bi < g.nblocks; ++bi) {
      int64_t org[3], ext[3] = {1, 1, 1}, halo[3];
      block_geom(&g, bi, org, ext);
      apply_padding(&g, scalars, pad_kind, pad_gran, bi, halo);
      int64_t e0 = ext[0], e1 = nd > 1 ? ext[1] : 1, e2 = nd > 2 ? ext[2] : 1;
      int64_t ne = e0 * e1 * e2;
      const uint32_t* bc = codes + block_code_start(&g, bi);
      const float* bo = outlier_vals + out_start[bi];
      int64_t bo_n = counts[bi];
      int kind = VLZO_OK;
      int64_t val = 0;
      /* reconstruct.py:44-48: max code check before traversal */
      uint32_t cmax = 0;
      for (int64_t t = 0; t < ne; ++t)
        if (bc[t] > cmax) cmax = bc[t];
      if (ne && cmax >= (uint32_t)(2 * radius)) {
        kind = VLZO_CORRUPT_CODE;
        val = cmax;
      }
      padded_t p = {nd, {e0, e1, e2}, halo, tile};
      int64_t cursor = 0, t = 0;
      for (int64_t i = 0; i < e0 && kind == VLZO_OK; ++i)
        for (int64_t j = 0; j < e1 && kind == VLZO_OK; ++j)
          for (int64_t k = 0; k < e2; ++k, ++t) {
            uint32_t c = bc[t];
            if (c == 0) {
              if (cursor >= bo_n) {
                kind = VLZO_EXHAUSTED;
                break;
              }
              tile[t] = quantize_value((double)bo[cursor], eb);
              sent[t] = 1;
              ++cursor;
            } else {
              int64_t pred = nd == 1 ? lorenzo_predict(&p, i, 0, 0)
                           : nd == 2 ? lorenzo_predict(&p, i, j, 0)
                                     : lorenzo_predict(&p, i, j, k);
              tile[t] = pred + ((int64_t)c - radius);
              sent[t] = 0;
            }
          }
      if (kind == VLZO_OK && cursor != bo_n) {
        kind = VLZO_LEFTOVER;
        val = cursor;
      }
      if (kind != VLZO_OK) {
#pragma omp critical
        {
          if (bi < first_bad) {
            first_bad = bi;
            bad_kind = kind;
            bad_val = val;
          }
        }
        continue;
      }
      int64_t oc = 0;
      for (t = 0; t < ne; ++t) ftile[t] = sent[t] ? bo[oc++] : reconstruct_value(tile[t], eb);
      t = 0;
      for (int64_t i = 0; i < e0; ++i)
        for (int64_t j = 0; j < e1; ++j)
          for (int64_t k = 0; k < e2; ++k, ++t) {
            int64_t idx[3] = {org[0] + i, nd > 1 ? org[1] + j : 0, nd > 2 ? org[2] + k : 0};
            out[flat_index(&g, idx)] = ftile[t];
          }
    }
    free(tile);
    free(ftile);
    free(sent);
  }
  free(out_start);
  if (bad_kind != VLZO_OK) {
    *err_index = first_bad;
    *err_value = bad_val;
    return bad_kind;
  }
  return VLZO_OK;
}

/* model.py:104-110 helper: float(min), float(max) with numpy NaN propagation */
void vlzo_minmax(const float* data, int64_t n, double* lo, double* hi) {
  float mn = data[0], mx = data[0];
  int nan = 0;
  for (int64_t i = 0; i < n; ++i) {
    float v = data[i];
    if (v != v) nan = 1;
    if (v < mn) mn = v;
    if (v > mx) mx = v;
  }
  *lo = nan ? NAN : (double)mn;
  *hi = nan ? NAN : (double)mx;
}
