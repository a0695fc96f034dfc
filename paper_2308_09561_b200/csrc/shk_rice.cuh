// Golomb-Rice decode shared by the stream decode, node-index and query kernels.
#pragma once
#include "shk_common.cuh"

namespace shk {

// Sequential decode, bit-exact with _core.pyx:575-623.  Returns 1 on overrun.
SHK_D int rice_decode(const uint64_t* words, int64_t bit_len, int64_t* pos, int g, int64_t* out) {
  int64_t q = 0, p = *pos;
  const int64_t nwords = (bit_len + 63) >> 6;
  for (;;) {
    if (p >= bit_len) return 1;
    int64_t i = p >> 6;
    int sh = (int)(p & 63);
    uint64_t chunk = words[i] >> sh;
    if (sh && i + 1 < nwords) chunk |= words[i + 1] << (64 - sh);
    int64_t avail = bit_len - p;
    if (avail > 64) avail = 64;
    uint64_t inv = ~chunk;
    int t = inv ? __ffsll((long long)inv) - 1 : 64;
    if (t >= avail) {
      q += avail;
      p += avail;
      continue;
    }
    q += t;
    p += t + 1;
    break;
  }
  uint64_t rem = 0;
  if (g) {
    if (p + g > bit_len) return 1;
    int64_t i = p >> 6;
    int sh = (int)(p & 63);
    uint64_t chunk = words[i] >> sh;
    if (sh && i + 1 < nwords) chunk |= words[i + 1] << (64 - sh);
    rem = chunk & ((1ull << g) - 1);
    p += g;
  }
  *out = (int64_t)(((uint64_t)q << g) | rem);
  *pos = p;
  return 0;
}

}  // namespace shk
