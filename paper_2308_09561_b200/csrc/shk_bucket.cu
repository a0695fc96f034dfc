// Bucketing: bucket hash, counting sort by bucket, per-bucket sort by the
// 128-bit code, prefix sums and the duplicate check.
//
// Restates recsplit.py:475-483 (bucket = hash_range(remix(hi, lo, 0,
// TAG_BUCKET), nb); lexsort by (bucket, hi, lo); bincount -> key_prefix) and
// the duplicate check of recsplit.py:433-440 (adjacent equal codes).  Equal
// codes always share a bucket, so one sort serves both.
//
// HBM-bound streaming passes: (1) bucket id + histogram, (2) scan,
// (3) scatter into bucket ranges, (4) one CTA per bucket sorts it in shared
// memory (bitonic on the 64-bit hi word with a 16-bit index, ties on hi
// resolved on lo, which is astronomically rare but exact), gathers, writes
// the interleaved sorted keys and flags adjacent duplicates.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

__global__ void bucket_hist_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N, uint32_t nb, uint32_t* bid,
                                   int64_t* counts) {
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    u2 v = remix_d(split64(hi[i]), split64(lo[i]), x);
    uint32_t b = __umulhi(v.hi, nb);
    bid[i] = b;
    atomicAdd((unsigned long long*)&counts[b], 1ull);
  }
}

__global__ void bucket_scatter_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N, const uint32_t* bid,
                                      int64_t* cursor, ulonglong2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = bid[i];
    int64_t p = (int64_t)atomicAdd((unsigned long long*)&cursor[b], 1ull);
    out[p] = make_ulonglong2(hi[i], lo[i]);
  }
}

SHK_D bool key_less(ulonglong2 a, ulonglong2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// One CTA per bucket, P = power of two >= max bucket size (<= 16384).
__global__ void bucket_sort_kernel(const ulonglong2* in, const int64_t* prefix, int64_t nb, int P, ulonglong2* out,
                                   int* dup_flag) {
  extern __shared__ uint64_t smem[];
  uint64_t* sk = smem;                              // [P] hi words
  uint16_t* si = reinterpret_cast<uint16_t*>(sk + P);  // [P] local index
  __shared__ int ties;
  for (int64_t bu = blockIdx.x; bu < nb; bu += gridDim.x) {
    const int64_t s0 = prefix[bu];
    const int cnt = (int)(prefix[bu + 1] - s0);
    if (cnt == 0) continue;
    int Pb = 1;
    while (Pb < cnt) Pb <<= 1;
    if (threadIdx.x == 0) ties = 0;
    for (int i = threadIdx.x; i < Pb; i += blockDim.x) {
      sk[i] = (i < cnt) ? in[s0 + i].x : ~0ull;
      si[i] = (uint16_t)i;
    }
    __syncthreads();
    // bitonic sort of (hi, idx); padding (~0, idx>=cnt) sorts last because
    // ties compare the index.
    for (int k = 2; k <= Pb; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < (Pb >> 1); t += blockDim.x) {
          int i = 2 * j * (t / j) + (t % j);
          int l = i + j;
          bool up = ((i & k) == 0);
          uint64_t a = sk[i], b = sk[l];
          uint16_t ia = si[i], ib = si[l];
          bool gt = (a > b) || (a == b && ia > ib);
          if (gt == up) {
            sk[i] = b;
            sk[l] = a;
            si[i] = ib;
            si[l] = ia;
          }
        }
        __syncthreads();
      }
    }
    // detect equal hi words (then order by lo, and duplicate check)
    for (int i = threadIdx.x; i + 1 < cnt; i += blockDim.x)
      if (sk[i] == sk[i + 1]) ties = 1;
    __syncthreads();
    if (ties && threadIdx.x == 0) {
      // insertion sort inside runs of equal hi by lo (rare)
      int i = 0;
      while (i < cnt) {
        int j = i + 1;
        while (j < cnt && sk[j] == sk[i]) ++j;
        for (int a2 = i + 1; a2 < j; ++a2) {
          uint16_t v = si[a2];
          uint64_t lv = in[s0 + v].y;
          int b2 = a2 - 1;
          while (b2 >= i && in[s0 + si[b2]].y > lv) {
            si[b2 + 1] = si[b2];
            --b2;
          }
          si[b2 + 1] = v;
        }
        for (int a2 = i + 1; a2 < j; ++a2)
          if (in[s0 + si[a2]].y == in[s0 + si[a2 - 1]].y) atomicOr(dup_flag, 1);
        i = j;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[s0 + i] = in[s0 + si[i]];
    __syncthreads();
  }
}

// Same result by distribution: a bucket's hi words are uniform 64-bit values,
// so one counting pass on their top 12 bits (4096 bins, ~0.5 keys per bin at
// b = 2000) places every key within a few slots of its sorted position; each
// bin (a contiguous output range) is then insertion-sorted by (hi, lo) by one
// thread, which also flags equal codes (they share a bin).  O(cnt) work and
// three block barriers per bucket instead of the bitonic network's 66.
#ifndef SHK_BUCKET_SORT
#define SHK_BUCKET_SORT 2  // 2: distribution sort (bins); 1: bitonic network (+ O(m^2) rank past 16384 keys)
#endif
constexpr int SORT_BINS = 4096;
__global__ void __launch_bounds__(256) bucket_sort_bins_kernel(const ulonglong2* in, const int64_t* prefix, int64_t nb,
                                                               ulonglong2* out, int* dup_flag) {
  __shared__ int cur[SORT_BINS];
  __shared__ int wsum[8];
  for (int64_t bu = blockIdx.x; bu < nb; bu += gridDim.x) {
    const int64_t s0 = prefix[bu];
    const int cnt = (int)(prefix[bu + 1] - s0);
    if (cnt == 0) continue;
    for (int i = threadIdx.x; i < SORT_BINS; i += blockDim.x) cur[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) atomicAdd(&cur[(int)(in[s0 + i].x >> 52)], 1);
    __syncthreads();
    // exclusive scan of the 4096 counts: 16 per thread, then across threads
    {
      const int t = threadIdx.x, base = t * (SORT_BINS / 256);
      int loc[SORT_BINS / 256], run = 0;
#pragma unroll
      for (int k = 0; k < SORT_BINS / 256; ++k) {
        loc[k] = run;
        run += cur[base + k];
      }
      // block scan of the per-thread totals (warp shuffles + 8 warp sums)
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL_WARP, incl, o);
        if ((t & 31) >= o) incl += v;
      }
      if ((t & 31) == 31) wsum[t >> 5] = incl;
      __syncthreads();
      int woff = 0;
      for (int w = 0; w < (t >> 5); ++w) woff += wsum[w];
      const int excl = woff + incl - run;
#pragma unroll
      for (int k = 0; k < SORT_BINS / 256; ++k) cur[base + k] = excl + loc[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const ulonglong2 k = in[s0 + i];
      out[s0 + atomicAdd(&cur[(int)(k.x >> 52)], 1)] = k;
    }
    __syncthreads();
    // cur[bin] is now the end of the bin; its start is the previous bin's end
    for (int bin = threadIdx.x; bin < SORT_BINS; bin += blockDim.x) {
      const int a = bin ? cur[bin - 1] : 0, e = cur[bin];
      for (int x = a + 1; x < e; ++x) {
        const ulonglong2 v = out[s0 + x];
        int y = x - 1;
        while (y >= a && key_less(v, out[s0 + y])) {
          out[s0 + y + 1] = out[s0 + y];
          --y;
        }
        out[s0 + y + 1] = v;
      }
      for (int x = a + 1; x < e; ++x) {
        const ulonglong2 p = out[s0 + x - 1], q = out[s0 + x];
        if (p.x == q.x && p.y == q.y) atomicOr(dup_flag, 1);
      }
    }
    __syncthreads();
  }
}

// Fallback for buckets larger than the shared-memory sort: rank by counting
// (O(cnt^2) per bucket, correct for any size; only reached with huge b).
__global__ void bucket_rank_kernel(const ulonglong2* in, int64_t s0, int cnt, ulonglong2* out, int* dup_flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    ulonglong2 k = in[s0 + i];
    int64_t rank = 0;
    for (int j = 0; j < cnt; ++j) {
      ulonglong2 o = in[s0 + j];
      rank += key_less(o, k) || (o.x == k.x && o.y == k.y && j < i);
      if (j != i && o.x == k.x && o.y == k.y) atomicOr(dup_flag, 1);
    }
    out[s0 + rank] = k;
  }
}

__global__ void max_bucket_kernel(const int64_t* counts, int64_t nb, int64_t* maxv) {
  int64_t m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, counts[i]);
  atomicMax((unsigned long long*)maxv, (unsigned long long)m);
}

// Choice bits of the keys at positions [k0, k1) of the (partitioned) build
// array, written at those keys' positions in the bucket-sorted array: the
// bucket is recomputed from the key, then a binary search by (hi, lo) inside
// it (codes are distinct).
__global__ void choice_sorted_kernel(const ulonglong2* keys, const ulonglong2* sorted, const int64_t* prefix,
                                     uint32_t nb, const uint8_t* choice, int64_t k0, int64_t k1, uint8_t* out) {
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  for (int64_t i = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k1; i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 k = keys[i];
    const uint32_t bu = __umulhi(remix_d(split64(k.x), split64(k.y), x).hi, nb);
    int64_t lo = prefix[bu], hi = prefix[bu + 1] - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key_less(sorted[mid], k))
        lo = mid + 1;
      else
        hi = mid;
    }
    out[lo - k0] = choice[i];
  }
}

}  // namespace shk

using namespace shk;

int shk_launch_choice_sorted(const uint64_t* keys, const uint64_t* sorted, const int64_t* prefix, int64_t nb,
                             const uint8_t* choice, int64_t k0, int64_t k1, uint8_t* out, cudaStream_t st) {
  if (k1 <= k0) return 0;
  int64_t g = (k1 - k0 + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  choice_sorted_kernel<<<(unsigned)g, 256, 0, st>>>((const ulonglong2*)keys, (const ulonglong2*)sorted, prefix,
                                                    (uint32_t)nb, choice, k0, k1, out);
  SHK_LAUNCHED();
  return 0;
}

size_t shk_bucketize_scratch(int64_t N, int64_t nb) {
  size_t s = 0;
  s += ((size_t)N * 4 + 255) & ~(size_t)255;        // bucket ids
  s += ((size_t)N * 16 + 255) & ~(size_t)255;       // unsorted scatter
  s += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;  // counts
  s += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;  // cursor
  s += 256;                                          // max
  s += shk_scan_scratch(nb);
  return s;
}

int shk_bucketize(const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nb, uint64_t* skeys_u64,
                  uint64_t* key_prefix, int* dup_flag, void* scratch, size_t scratch_bytes, int64_t* max_bucket_out,
                  cudaStream_t st, uint64_t* h_prefix) {
  if (scratch_bytes < shk_bucketize_scratch(N, nb)) {
    shk_set_error("bucketize scratch too small");
    return 3;
  }
  if (nb <= 0 || nb > 0xFFFFFFFFll) {
    shk_set_error("bad bucket count");
    return 3;
  }
  char* p = (char*)scratch;
  uint32_t* bid = (uint32_t*)p;
  p += ((size_t)N * 4 + 255) & ~(size_t)255;
  ulonglong2* unsorted = (ulonglong2*)p;
  p += ((size_t)N * 16 + 255) & ~(size_t)255;
  int64_t* counts = (int64_t*)p;
  p += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;
  int64_t* cursor = (int64_t*)p;
  p += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;
  int64_t* maxv = (int64_t*)p;
  p += 256;
  void* scan_scratch = p;
  int64_t* prefix = (int64_t*)key_prefix;
  ulonglong2* out = (ulonglong2*)skeys_u64;

  SHK_CUDA(cudaMemsetAsync(counts, 0, (size_t)(nb + 1) * 8, st));
  SHK_CUDA(cudaMemsetAsync(maxv, 0, 8, st));
  SHK_CUDA(cudaMemsetAsync(dup_flag, 0, sizeof(int), st));
  const int T = 256;
  int64_t g = (N + T - 1) / T;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  if (N > 0) {
    bucket_hist_kernel<<<(unsigned)g, T, 0, st>>>(hi, lo, N, (uint32_t)nb, bid, counts);
    SHK_LAUNCHED();
  }
  int rc = shk_exclusive_scan_i64(counts, prefix, nb, scan_scratch, shk_scan_scratch(nb), st);
  if (rc) return rc;
  SHK_CUDA(cudaMemcpyAsync(cursor, prefix, (size_t)nb * 8, cudaMemcpyDeviceToDevice, st));
  int64_t maxb = 0;
  if (h_prefix) {
    // the caller wants the key prefix early (to prepare the next phase while
    // the scatter and the sort run): wait for the scan only, take the
    // largest bucket from the prefix on the host, and return without waiting
    // for the sort
    SHK_CUDA(cudaMemcpyAsync(h_prefix, prefix, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost, st));
    SHK_CUDA(cudaStreamSynchronize(st));
    for (int64_t bu = 0; bu < nb; ++bu) {
      const int64_t cnt = (int64_t)(h_prefix[bu + 1] - h_prefix[bu]);
      if (cnt > maxb) maxb = cnt;
    }
  }
  if (N > 0) {
    bucket_scatter_kernel<<<(unsigned)g, T, 0, st>>>(hi, lo, N, bid, cursor, unsorted);
    SHK_LAUNCHED();
  }
  if (!h_prefix) {
    max_bucket_kernel<<<64, 256, 0, st>>>(counts, nb, maxv);
    SHK_LAUNCHED();
    SHK_CUDA(cudaMemcpyAsync(&maxb, maxv, 8, cudaMemcpyDeviceToHost, st));
    SHK_CUDA(cudaStreamSynchronize(st));
  }
  if (max_bucket_out) *max_bucket_out = maxb;
  int P = 1;
  while (P < maxb) P <<= 1;
  if (P < 2) P = 2;
  if (SHK_BUCKET_SORT == 2) {
    // distribution sort: any bucket size (bins hold cnt / 4096 keys on average)
    int64_t grid = nb < 148 * 8 ? nb : 148 * 8;
    bucket_sort_bins_kernel<<<(unsigned)grid, 256, 0, st>>>(unsorted, prefix, nb, out, dup_flag);
    SHK_LAUNCHED();
  } else if (maxb <= 16384) {
    size_t sm = (size_t)P * 10;
    if (sm > 48 * 1024)
      SHK_CUDA(cudaFuncSetAttribute(bucket_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int64_t grid = nb < 148 * 8 ? nb : 148 * 8;
    bucket_sort_kernel<<<(unsigned)grid, 256, sm, st>>>(unsorted, prefix, nb, P, out, dup_flag);
    SHK_LAUNCHED();
  } else {
    // Huge buckets: per-bucket counting rank (host loop over buckets).
    int64_t* hp = (int64_t*)malloc((size_t)(nb + 1) * 8);
    SHK_CUDA(cudaMemcpyAsync(hp, prefix, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost, st));
    SHK_CUDA(cudaStreamSynchronize(st));
    for (int64_t bu = 0; bu < nb; ++bu) {
      int cnt = (int)(hp[bu + 1] - hp[bu]);
      if (!cnt) continue;
      bucket_rank_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(unsorted, hp[bu], cnt, out, dup_flag);
    }
    free(hp);
    SHK_LAUNCHED();
  }
  return 0;
}
