// Exclusive prefix sum of int64 values (bucket key counts, Rice code lengths,
// node counts, ribbon chunk counts).  Reduce-then-scan in at most two
// launches (the build runs a dozen small scans back to back, so launches --
// not bytes -- are their cost): tile totals, then each tile adds the totals
// of the tiles before it (a block-wide sum over at most a few thousand
// values) to its own scan; the last tile writes the grand total to out[n].
// A single tile needs only the second launch.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

constexpr int SCAN_T = 256;            // threads per tile
constexpr int SCAN_V = 8;              // values per thread
constexpr int SCAN_B = SCAN_T * SCAN_V;  // values per tile

SHK_D int64_t block_sum(int64_t v, int64_t* red) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_WARP, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int64_t r = 0;
#pragma unroll
  for (int w = 0; w < SCAN_T / 32; ++w) r += red[w];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_T) scan_tile_sum_kernel(const int64_t* in, int64_t n, int64_t* tile_sums) {
  __shared__ int64_t red[SCAN_T / 32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_B;
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < SCAN_V; ++j) {
    const int64_t i = base + j * SCAN_T + threadIdx.x;  // coalesced
    if (i < n) s += in[i];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = s;
}

// tile_off (optional): the tiles' exclusive offsets, scanned already (long
// inputs); otherwise each tile sums tile_sums[0, tile) itself.
__global__ void __launch_bounds__(SCAN_T) scan_tile_kernel(const int64_t* in, int64_t* out, int64_t n,
                                                           const int64_t* tile_sums, const int64_t* tile_off) {
  __shared__ int64_t red[SCAN_T / 32];
  __shared__ int64_t wsum[SCAN_T / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t tile = blockIdx.x;
  // carry-in: the totals of the tiles before this one
  int64_t carry = 0;
  if (tile_off) {
    carry = tile_off[tile];
  } else if (tile) {
    int64_t c = 0;
    for (int64_t k = t; k < tile; k += SCAN_T) c += tile_sums[k];
    carry = block_sum(c, red);
  }
  // this thread's SCAN_V consecutive values
  const int64_t base = tile * SCAN_B + (int64_t)t * SCAN_V;
  int64_t v[SCAN_V];
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < SCAN_V; ++j) {
    const int64_t i = base + j;
    v[j] = (i < n) ? in[i] : 0;
    s += v[j];
  }
  int64_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL_WARP, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int64_t wo = 0;
  for (int w = 0; w < warp; ++w) wo += wsum[w];
  int64_t excl = carry + wo + inc - s;
#pragma unroll
  for (int j = 0; j < SCAN_V; ++j) {
    const int64_t i = base + j;
    if (i < n) out[i] = excl;
    excl += v[j];
  }
  if (tile == gridDim.x - 1 && t == SCAN_T - 1) out[n] = excl;  // grand total
}

}  // namespace shk

using namespace shk;

// Tiles a scan sums in place (carry-in loop per tile); longer inputs scan the
// tile totals recursively first.
constexpr int64_t SCAN_FLAT_TILES = 4096;

size_t shk_scan_scratch(int64_t n) {
  const int64_t tiles = (n + SCAN_B - 1) / SCAN_B;
  size_t b = (size_t)(tiles + 1) * sizeof(int64_t) + 256;
  if (tiles > SCAN_FLAT_TILES) b += (size_t)(tiles + 1) * sizeof(int64_t) + shk_scan_scratch(tiles);
  return b;
}

int shk_exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* scratch, size_t scratch_bytes,
                           cudaStream_t st) {
  if (scratch_bytes < shk_scan_scratch(n)) {
    shk_set_error("scan scratch too small");
    return 3;
  }
  if (n == 0) {
    SHK_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    return 0;
  }
  const int64_t tiles = (n + SCAN_B - 1) / SCAN_B;
  int64_t* sums = (int64_t*)scratch;
  int64_t* offs = nullptr;
  if (tiles > 1) {
    scan_tile_sum_kernel<<<(unsigned)tiles, SCAN_T, 0, st>>>(in, n, sums);
    SHK_LAUNCHED();
  }
  if (tiles > SCAN_FLAT_TILES) {
    offs = sums + tiles + 1;
    void* rest = offs + tiles + 1;
    int rc = shk_exclusive_scan_i64(sums, offs, tiles, rest, shk_scan_scratch(tiles), st);
    if (rc) return rc;
  }
  scan_tile_kernel<<<(unsigned)tiles, SCAN_T, 0, st>>>(in, out, n, sums, offs);
  SHK_LAUNCHED();
  return 0;
}
