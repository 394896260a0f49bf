// huffman.cpp -- canonical Huffman coding of the code stream (host, C++).
//
// Restates the reference's entropy stage (huffman.py) natively so that
// compress()/decompress() produce and accept byte-identical VLZ1 containers:
//   vlz_huff_build   huffman.py:56-88 -- heap of (freq, smallest symbol in
//                    subtree); pop two, merge, push (f1+f2, min(m1, m2));
//                    depths by DFS; a lone symbol gets length 1.  The
//                    (freq, min symbol) key is unique among live subtrees, so
//                    the tree -- and every length -- is fully determined.
//                    Canonical order/codewords: huffman.py:33-45.
//   vlz_huff_encode  huffman.py:91-122 -- MSB-first bit packing, zero-padded
//                    last byte (np.packbits).
//   vlz_huff_decode  huffman.py:125-207 -- exactly `count` symbols from the
//                    payload, same error verdicts in the same order.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>

#include "../../include/vlz_gpu.h"

namespace {

struct Node {
  uint64_t freq;
  uint32_t minsym;
  int32_t id;
};
struct Cmp {
  bool operator()(const Node& a, const Node& b) const {  // min-heap on (freq, minsym, id)
    if (a.freq != b.freq) return a.freq > b.freq;
    if (a.minsym != b.minsym) return a.minsym > b.minsym;
    return a.id > b.id;
  }
};

}  // namespace

extern "C" {

// freqs[0..65535] -> canonical (length, symbol) order; returns 0, or -1 for an
// empty stream (ConfigError), -2 when a length exceeds 64 bits
int vlz_huff_build(const uint64_t* freqs, uint16_t* syms_out, uint8_t* lens_out,
                   int32_t* nsym_out) {
  std::vector<uint32_t> present;
  for (uint32_t s = 0; s < 65536; ++s)
    if (freqs[s]) present.push_back(s);
  const int n = (int)present.size();
  *nsym_out = n;
  if (n == 0) return -1;
  std::vector<uint8_t> depth(n, 0);
  if (n == 1) {
    depth[0] = 1;
  } else {
    std::priority_queue<Node, std::vector<Node>, Cmp> heap;
    std::vector<int32_t> left, right;  // children of internal node id - n
    for (int i = 0; i < n; ++i) heap.push({freqs[present[i]], present[i], i});
    while (heap.size() > 1) {
      const Node a = heap.top();
      heap.pop();
      const Node b = heap.top();
      heap.pop();
      left.push_back(a.id);
      right.push_back(b.id);
      heap.push({a.freq + b.freq, a.minsym < b.minsym ? a.minsym : b.minsym,
                 n + (int32_t)left.size() - 1});
    }
    // depths by an explicit stack (huffman.py:79-87)
    std::vector<std::pair<int32_t, int32_t>> stack{{heap.top().id, 0}};
    while (!stack.empty()) {
      auto [id, d] = stack.back();
      stack.pop_back();
      if (id < n) {
        if (d > 64) return -2;
        depth[id] = (uint8_t)d;
      } else {
        stack.push_back({left[id - n], d + 1});
        stack.push_back({right[id - n], d + 1});
      }
    }
  }
  // canonical order: by length, then symbol (np.lexsort((symbols, lengths)))
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (depth[a] != depth[b]) return depth[a] < depth[b];
    return present[a] < present[b];
  });
  for (int i = 0; i < n; ++i) {
    syms_out[i] = (uint16_t)present[order[i]];
    lens_out[i] = depth[order[i]];
  }
  return 0;
}

// canonical codewords for (length, symbol)-sorted lengths (huffman.py:33-45)
static void codewords(const uint8_t* lens, int n, uint64_t* cw) {
  uint64_t code = 0;
  for (int i = 0; i < n; ++i) {
    cw[i] = code;
    code += 1;
    if (i + 1 < n) code <<= (int)lens[i + 1] - (int)lens[i];
  }
}

// returns 0; -1 with *bad_symbol set when a symbol has no codeword
int vlz_huff_encode(const uint16_t* codes, int64_t n, const uint16_t* syms, const uint8_t* lens,
                    int32_t nsym, uint8_t* out, int64_t out_cap, int64_t* nbits_out,
                    int64_t* bad_symbol) {
  std::vector<uint64_t> cw(nsym);
  codewords(lens, nsym, cw.data());
  std::vector<uint64_t> code_of(65536, 0);
  std::vector<uint8_t> len_of(65536, 0);
  for (int i = 0; i < nsym; ++i) {
    code_of[syms[i]] = cw[i];
    len_of[syms[i]] = lens[i];
  }
  uint64_t acc = 0;  // pending bits, MSB-first
  int nacc = 0;
  int64_t pos = 0, nbits = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint16_t s = codes[i];
    const int L = len_of[s];
    if (L == 0) {
      // huffman.py:102-104: a symbol beyond the largest codebook symbol is
      // reported first (anywhere in the stream), else the first absent one
      int span = 0;
      for (int k = 0; k < nsym; ++k) span = syms[k] + 1 > span ? syms[k] + 1 : span;
      *bad_symbol = s;
      for (int64_t j = 0; j < n; ++j)
        if (codes[j] >= span) {
          *bad_symbol = codes[j];
          break;
        }
      return -1;
    }
    uint64_t c = code_of[s];
    int rem = L;
    while (rem > 0) {  // push in pieces that fit the 64-bit accumulator
      const int take = rem < 56 - nacc ? rem : 56 - nacc;
      acc = (acc << take) | ((c >> (rem - take)) & ((take == 64) ? ~0ull : ((1ull << take) - 1)));
      nacc += take;
      rem -= take;
      while (nacc >= 8) {
        if (pos >= out_cap) return -3;
        out[pos++] = (uint8_t)(acc >> (nacc - 8));
        nacc -= 8;
      }
    }
    nbits += L;
  }
  if (nacc > 0) {
    if (pos >= out_cap) return -3;
    out[pos++] = (uint8_t)(acc << (8 - nacc));
  }
  *nbits_out = nbits;
  return 0;
}

// Decode exactly `count` symbols; status (huffman.py:135-207 order):
//  0 ok, 1 nonzero bit length for an empty stream, 2 payload shorter than
//  bit_length, 3 underrun mid-symbol, 4 invalid prefix, 5 consumed != bit_length
//  (*consumed_out set)
int vlz_huff_decode(const uint8_t* payload, int64_t nbytes, int64_t bit_length,
                    const uint16_t* syms, const uint8_t* lens, int32_t nsym, int64_t count,
                    uint16_t* out, int64_t* consumed_out) {
  *consumed_out = 0;
  if (count == 0) return bit_length != 0 ? 1 : 0;
  if (nbytes * 8 < bit_length) return 2;
  int maxlen = 0;
  for (int i = 0; i < nsym; ++i) maxlen = lens[i] > maxlen ? lens[i] : maxlen;
  // first_code grows without bound for an over-subscribed book (Kraft sum
  // > 1, reachable from a crafted container); the reference computes it in
  // Python ints.  Saturating at 2^70 keeps every comparison with a <= 64-bit
  // prefix exact: a saturated first code is above any prefix, as the true one is.
  using u128 = unsigned __int128;
  const u128 kCap = (u128)1 << 70;
  std::vector<u128> first_code(maxlen + 2, 0);
  std::vector<uint64_t> first_idx(maxlen + 2, 0), cnt(maxlen + 2, 0);
  for (int i = 0; i < nsym; ++i) cnt[lens[i]] += 1;
  {
    u128 code = 0;
    uint64_t idx = 0;
    for (int l = 1; l <= maxlen; ++l) {
      first_code[l] = code;
      first_idx[l] = idx;
      code = (code + cnt[l]) << 1;
      if (code > kCap) code = kCap;
      idx += cnt[l];
    }
  }
  // 12-bit lookup table for short codes (same result as the bit loop)
  const int lut_bits = maxlen < 12 ? maxlen : 12;
  std::vector<uint16_t> lut_sym(1u << lut_bits, 0);
  std::vector<uint8_t> lut_len(1u << lut_bits, 0);
  {
    // canonical codewords in (length, symbol) order; an over-subscribed book
    // runs its codewords past the table, where the reference's slice
    // assignment (huffman.py:166-167) truncates -- so do we
    const uint64_t size = 1ull << lut_bits;
    uint64_t code = 0;
    for (int i = 0; i < nsym && lens[i] <= lut_bits; ++i) {
      if (i && lens[i] < lens[i - 1]) break;  // not canonical order: table stays partial
      if (i) code = (code + 1) << (lens[i] - lens[i - 1]);
      if (code >= (size >> (lut_bits - lens[i]))) break;  // later codewords lie further out
      const uint64_t base = code << (lut_bits - lens[i]);
      const uint64_t span = 1ull << (lut_bits - lens[i]);
      for (uint64_t k = 0; k < span && base + k < size; ++k) {
        lut_sym[base + k] = syms[i];
        lut_len[base + k] = lens[i];
      }
    }
  }
  const int64_t total_bits = nbytes * 8;
  int64_t bp = 0;  // bit position in the payload
  auto bit_at = [&](int64_t b) -> uint64_t { return (payload[b >> 3] >> (7 - (b & 7))) & 1u; };
  for (int64_t i = 0; i < count; ++i) {
    if (bp + lut_bits <= total_bits) {
      uint64_t peek = 0;
      for (int k = 0; k < lut_bits; ++k) peek = (peek << 1) | bit_at(bp + k);
      const int L = lut_len[peek];
      if (L) {
        out[i] = lut_sym[peek];
        bp += L;
        continue;
      }
    }
    // a prefix of more than 64 bits (lengths up to 255 are representable)
    // saturates at 2^64: every first code that can match lies below it
    u128 acc = 0;
    int acclen = 0;
    for (;;) {
      if (bp >= total_bits) {
        *consumed_out = bp;
        return 3;
      }
      acc = (acc << 1) | bit_at(bp++);
      if (acc > ((u128)1 << 64)) acc = (u128)1 << 64;
      ++acclen;
      if (acclen > maxlen) {
        *consumed_out = bp;
        return 4;
      }
      if (acc >= first_code[acclen] && (uint64_t)(acc - first_code[acclen]) < cnt[acclen]) {
        const uint64_t off = (uint64_t)(acc - first_code[acclen]);
        out[i] = syms[first_idx[acclen] + off];
        break;
      }
    }
  }
  *consumed_out = bp;
  return bp != bit_length ? 5 : 0;
}

// bincount of uint16 codes (host side of the codebook, huffman.py:62)
void vlz_histogram_host(const uint16_t* codes, int64_t n, uint64_t* freqs) {
  std::memset(freqs, 0, 65536 * sizeof(uint64_t));
  for (int64_t i = 0; i < n; ++i) freqs[codes[i]] += 1;
}

}  // extern "C"
