// Golomb-Rice seed stream: encode (recsplit.py:126-170 BitWriter.rice) and
// decode (_core.pyx:575-635 c_rice_decode).
//
// Encoding is fully parallel: every node's code length (x >> g) + 1 + g is
// known from its seed, an exclusive scan turns lengths into bit positions
// (the stream is preorder per bucket, buckets in order), and every node ORs
// its unary run and its g remainder bits (LSB-first, little-endian 64-bit
// words) into a zeroed word array.  The reference writes long unary runs in
// 63-bit chunks; the resulting bits are identical.
#include "shk_common.cuh"
#include "shk_kernels.h"
#include "shk_rice.cuh"

namespace shk {

__global__ void rice_len_kernel(const int64_t* seeds, const int32_t* g, int64_t nn, int64_t* len) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)seeds[i];
    int gg = g[i];
    len[i] = (int64_t)((x >> gg) + 1 + gg);
  }
}

SHK_D void or_bits(uint64_t* w, uint64_t pos, uint64_t value, int nbits) {
  // value < 2^nbits, nbits <= 64
  if (nbits == 0 || value == 0) return;
  uint64_t i = pos >> 6;
  int sh = (int)(pos & 63);
  atomicOr((unsigned long long*)&w[i], (unsigned long long)(value << sh));
  if (sh && sh + nbits > 64) atomicOr((unsigned long long*)&w[i + 1], (unsigned long long)(value >> (64 - sh)));
}

__global__ void rice_scatter_kernel(const int64_t* seeds, const int32_t* g, const int64_t* pos, int64_t nn,
                                    uint64_t* words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)seeds[i];
    int gg = g[i];
    uint64_t q = x >> gg;
    uint64_t p = (uint64_t)pos[i];
    // unary: q ones at [p, p + q)
    uint64_t a = p, e = p + q;
    while (a < e) {
      int sh = (int)(a & 63);
      uint64_t take = 64 - sh;
      if (take > e - a) take = e - a;
      uint64_t m = (take == 64) ? ~0ull : (((1ull << take) - 1) << sh);
      atomicOr((unsigned long long*)&words[a >> 6], (unsigned long long)m);
      a += take;
    }
    if (gg) or_bits(words, p + q + 1, x & ((1ull << gg) - 1), gg);
  }
}

__global__ void rice_decode_seq_kernel(const uint64_t* words, int64_t bit_len, int64_t pos, const int32_t* g,
                                       int64_t count, int64_t* values, int64_t* positions, int* err) {
  if (blockIdx.x || threadIdx.x) return;
  for (int64_t k = 0; k < count; ++k) {
    int64_t v = 0;
    if (rice_decode(words, bit_len, &pos, g[k], &v)) {
      *err = 1;
      return;
    }
    values[k] = v;
    positions[k] = pos;
  }
}

}  // namespace shk

using namespace shk;

int shk_rice_lengths(const int64_t* seeds, const int32_t* g, int64_t nn, int64_t* len, cudaStream_t st) {
  if (nn <= 0) return 0;
  int64_t b = (nn + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  rice_len_kernel<<<(unsigned)b, 256, 0, st>>>(seeds, g, nn, len);
  SHK_LAUNCHED();
  return 0;
}

int shk_rice_scatter(const int64_t* seeds, const int32_t* g, const int64_t* pos, int64_t nn, uint64_t* words,
                     cudaStream_t st) {
  if (nn <= 0) return 0;
  int64_t b = (nn + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  rice_scatter_kernel<<<(unsigned)b, 256, 0, st>>>(seeds, g, pos, nn, words);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_rice_decode(const uint64_t* words, int64_t bit_len, int64_t pos, const int32_t* g, int64_t count,
                           int64_t* values, int64_t* positions, int* err, cudaStream_t st) {
  rice_decode_seq_kernel<<<1, 1, 0, st>>>(words, bit_len, pos, g, count, values, positions, err);
  SHK_LAUNCHED();
  return 0;
}
