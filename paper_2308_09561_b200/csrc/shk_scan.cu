// Exclusive prefix sum of int64 values (bucket key counts, Rice code lengths,
// node counts).  Three-phase: per-block scan with block totals, a recursive
// scan of the totals, then a uniform add.  out[n] receives the grand total.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

constexpr int SCAN_B = 1024;  // elements per block (256 threads x 4)

__global__ void scan_block_kernel(const int64_t* in, int64_t* out, int64_t n, int64_t* block_sums) {
  __shared__ int64_t wsum[8];
  const int64_t base = (int64_t)blockIdx.x * SCAN_B;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t v[4];
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t i = base + t * 4 + j;
    v[j] = (i < n) ? in[i] : 0;
    s += v[j];
  }
  // inclusive warp scan of per-thread sums
  int64_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(FULL_WARP, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < 8) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      int64_t y = __shfl_up_sync(FULL_WARP, w, o);
      if (lane >= o) w += y;
    }
    if (lane < 8) wsum[lane] = w;
  }
  __syncthreads();
  int64_t excl = inc - s + (warp ? wsum[warp - 1] : 0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t i = base + t * 4 + j;
    if (i < n) out[i] = excl;
    excl += v[j];
  }
  if (t == 255) block_sums[blockIdx.x] = excl;  // block total
}

__global__ void scan_add_kernel(int64_t* out, int64_t n, const int64_t* block_off) {
  int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
  int64_t add = block_off[blockIdx.x];
#pragma unroll
  for (int j = 0; j < 4; ++j, i += 256)
    if (i < n) out[i] += add;
}

}  // namespace shk

using namespace shk;

size_t shk_scan_scratch(int64_t n) {
  size_t total = 0;
  int64_t m = n;
  while (true) {
    int64_t nb = (m + SCAN_B - 1) / SCAN_B;
    if (nb < 1) nb = 1;
    total += (size_t)(2 * nb + 2) * sizeof(int64_t);
    if (nb == 1) break;
    m = nb;
  }
  return total + 256;
}

static int scan_rec(const int64_t* in, int64_t* out, int64_t n, int64_t* scratch, cudaStream_t st) {
  int64_t nb = (n + SCAN_B - 1) / SCAN_B;
  if (nb < 1) nb = 1;
  int64_t* sums = scratch;           // [nb]
  int64_t* sums_scan = scratch + nb;  // [nb + 1]
  scan_block_kernel<<<(unsigned)nb, 256, 0, st>>>(in, out, n, sums);
  SHK_LAUNCHED();
  if (nb == 1) {
    // total
    SHK_CUDA(cudaMemcpyAsync(out + n, sums, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  int rc = scan_rec(sums, sums_scan, nb, scratch + 2 * nb + 2, st);
  if (rc) return rc;
  scan_add_kernel<<<(unsigned)nb, 256, 0, st>>>(out, n, sums_scan);
  SHK_LAUNCHED();
  SHK_CUDA(cudaMemcpyAsync(out + n, sums_scan + nb, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  return 0;
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
  return scan_rec(in, out, n, (int64_t*)scratch, st);
}
