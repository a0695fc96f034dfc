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
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

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

// ---------------------------------------------------------------------------
// Shared-memory path (nb <= BK_MAX_NB buckets, buckets <= BK_MAX_SORT keys,
// N < 2^32): three streaming passes and no global atomics.
//   1. bk_hist: CTA c of G histograms its contiguous key chunk in shared
//      memory and writes the counts column-wise, M[b * G + c];
//   2. an exclusive scan of M (bucket-major) gives every (bucket, CTA) its
//      write offset in the bucket-sorted array; key_prefix[b] = M[b * G];
//   3. bk_scatter: CTA c re-reads its chunk, recomputes the bucket hash (no
//      bucket-id array) and places each key at its (bucket, CTA) cursor,
//      advanced with shared-memory atomics;
//   4. bk_sort: one CTA per bucket stages the bucket in shared memory,
//      distributes it over 4096 bins by the top 12 bits of hi, and every
//      key's final position is its bin start + the number of keys of its
//      bin that sort before it by (hi, lo) (~0.5 other keys per bin at
//      b = 2000); equal codes share a bin and raise the duplicate flag.
// Traffic: 16 B read (1) + 32 B (3) + 32 B (4) per key, plus M.
constexpr int BK_G = 296;            // CTAs of the histogram / scatter passes
constexpr int BK_MAX_NB = 40960;     // shared-memory histogram limit (160 KB)
constexpr int BK_MAX_SORT = 11264;   // keys per bucket staged in shared memory

SHK_D uint32_t bucket_of_d(uint64_t hi, uint64_t lo, u2 x, uint32_t nb) {
  return __umulhi(remix_d(split64(hi), split64(lo), x).hi, nb);
}

constexpr int BK_SB = 16;  // buckets per super-bucket (the cluster path below)

// Msb (optional): the CTA's key count per super-bucket of BK_SB buckets,
// Msb[sb * G + c] (the first-level scatter of the cluster path).
__global__ void __launch_bounds__(512) bk_hist_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N, uint32_t nb,
                                                      int64_t* M, int64_t* Msb) {
  extern __shared__ uint32_t h[];
  const int G = gridDim.x, c = blockIdx.x;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  const int64_t c0 = N * c / G, c1 = N * (c + 1) / G;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&h[bucket_of_d(hi[i], lo[i], x, nb)], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) M[(int64_t)b * G + c] = h[b];
  if (Msb) {
    const uint32_t nsb = (nb + BK_SB - 1) / BK_SB;
    for (uint32_t sb = threadIdx.x; sb < nsb; sb += blockDim.x) {
      uint32_t t = 0;
      for (uint32_t b = sb * BK_SB; b < sb * BK_SB + BK_SB && b < nb; ++b) t += h[b];
      Msb[(int64_t)sb * G + c] = t;
    }
  }
}

// key_prefix[b] = offset of (b, CTA 0); key_prefix[nb] = N; and the largest bucket.
__global__ void bk_prefix_kernel(const int64_t* Moff, int G, int64_t nb, int64_t* prefix, int64_t* maxv) {
  int64_t m = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = Moff[b * G];
    prefix[b] = v;
    if (b < nb) m = max(m, Moff[(b + 1) * G] - v);
  }
  atomicMax((unsigned long long*)maxv, (unsigned long long)m);
}

// L2 policies of the scatter: its 16-byte stores land in random bucket
// slots, so a 32-byte sector is completed by a later store of another CTA;
// the destination lines are kept in L2 (evict_last) until they fill, and the
// streamed inputs are dropped first (evict_first), instead of partial
// sectors going to DRAM as read-modify-writes.
SHK_D uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SHK_D uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SHK_D uint64_t ld_hint_u64(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
SHK_D void st_hint_u64x2(ulonglong2* a, ulonglong2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(a), "l"(v.x), "l"(v.y), "l"(pol)
               : "memory");
}
SHK_D ulonglong2 ld_hint_u64x2(const ulonglong2* a, uint64_t pol) {
  ulonglong2 v;
  asm volatile("ld.global.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(a), "l"(pol));
  return v;
}

#ifndef SHK_BUCKET_L2HINT
#define SHK_BUCKET_L2HINT 1
#endif
// Buckets [blo, bhi) only (A/B of a sliced scatter, see the launcher).  One
// pass over the 160 MB destination at C4 reads 374 MB and writes 254 MB of
// DRAM: the random 16-byte stores reach DRAM as partial sectors.
__global__ void __launch_bounds__(512) bk_scatter_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N,
                                                         uint32_t nb, const int64_t* Moff, ulonglong2* out,
                                                         uint32_t blo, uint32_t bhi) {
  extern __shared__ uint32_t cur[];
  const int G = gridDim.x, c = blockIdx.x;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cur[b] = (uint32_t)Moff[(int64_t)b * G + c];
  __syncthreads();
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  const int64_t c0 = N * c / G, c1 = N * (c + 1) / G;
  const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const uint64_t a = SHK_BUCKET_L2HINT ? ld_hint_u64(hi + i, stream) : hi[i];
    const uint64_t z = SHK_BUCKET_L2HINT ? ld_hint_u64(lo + i, stream) : lo[i];
    const uint32_t bu = bucket_of_d(a, z, x, nb);
    if (bu < blo || bu >= bhi) continue;
    const uint32_t p = atomicAdd(&cur[bu], 1u);
    if (SHK_BUCKET_L2HINT)
      st_hint_u64x2(out + p, make_ulonglong2(a, z), keep);
    else
      out[p] = make_ulonglong2(a, z);
  }
}

__global__ void __launch_bounds__(256) bk_sort_kernel(const ulonglong2* in, const int64_t* prefix, int64_t nb,
                                                      ulonglong2* out, int* dup_flag) {
  extern __shared__ __align__(16) unsigned char bk_smem[];
  int* cur = reinterpret_cast<int*>(bk_smem);                                   // [4096]
  ulonglong2* A = reinterpret_cast<ulonglong2*>(bk_smem + SORT_BINS * 4);       // [cnt]
  __shared__ int wsum[8];
  for (int64_t bu = blockIdx.x; bu < nb; bu += gridDim.x) {
    const int64_t s0 = prefix[bu];
    const int cnt = (int)(prefix[bu + 1] - s0);
    if (cnt == 0) continue;
    uint16_t* B = reinterpret_cast<uint16_t*>(A + cnt);  // [cnt] bin-ordered key indices
    for (int i = threadIdx.x; i < SORT_BINS; i += blockDim.x) cur[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const ulonglong2 k = SHK_BUCKET_L2HINT ? ld_hint_u64x2(in + s0 + i, policy_evict_first()) : in[s0 + i];
      A[i] = k;
      atomicAdd(&cur[(int)(k.x >> 52)], 1);
    }
    __syncthreads();
    {  // exclusive scan of the 4096 bin counts (16 per thread)
      const int t = threadIdx.x, base = t * (SORT_BINS / 256);
      int loc[SORT_BINS / 256], run = 0;
#pragma unroll
      for (int k = 0; k < SORT_BINS / 256; ++k) {
        loc[k] = run;
        run += cur[base + k];
      }
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
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) B[atomicAdd(&cur[(int)(A[i].x >> 52)], 1)] = (uint16_t)i;
    __syncthreads();
    // cur[bin] is the end of the bin, its start the previous bin's end
    for (int p = threadIdx.x; p < cnt; p += blockDim.x) {
      const ulonglong2 k = A[B[p]];
      const int bin = (int)(k.x >> 52);
      const int a = bin ? cur[bin - 1] : 0, e = cur[bin];
      int r = a;
      for (int q = a; q < e; ++q) {
        if (q == p) continue;
        const ulonglong2 o = A[B[q]];
        const bool eq = o.x == k.x && o.y == k.y;
        if (eq) atomicOr(dup_flag, 1);
        r += key_less(o, k) || (eq && q < p);
      }
      out[s0 + r] = k;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Cluster path (B200: thread-block clusters + distributed shared memory).
// The scatter above writes 16-byte keys to random slots of 5,000 bucket
// ranges, which reach DRAM as partial sectors (374 MB read + 254 MB written
// for 160 MB of keys at C4).  Here the keys move in two coalesced steps:
//   L1 (bk_l1_scatter): to their SUPER-bucket (BK_SB = 32 consecutive
//      buckets, ~64k keys at C4) -- each CTA sorts a 2,048-key tile by
//      super-bucket in shared memory and writes runs (~13 keys = 208 B);
//   L2 (bk_cluster_sort): one cluster of BK_CL = 8 CTAs per super-bucket,
//      each CTA owning BK_SB / BK_CL = 4 buckets: the CTAs read the
//      super-bucket's range in eighths, count keys per bucket, exchange the
//      counts through distributed shared memory, and store every key straight
//      into the shared memory of the CTA that owns its bucket; after a
//      cluster barrier each CTA sorts its buckets in its own shared memory
//      (rank within 4096 top-bit bins, as bk_sort) and writes them out.
// DRAM traffic: 16 B (hist) + 32 B (L1) + 32 B (L2) per key.
constexpr int BK_CL = 16;              // cluster size (non-portable: set at launch)
constexpr int BK_TILE = 2048;          // keys per L1 tile (512 threads x 4)

// Exclusive scan of n <= 2048 ints in shared memory by 512 threads (4 each);
// out[n] = total.  Both arrays in shared memory; ends synchronized.
SHK_D void block_scan_2048(const uint32_t* in, uint32_t* out, int n, uint32_t* wsum) {
  const int t = threadIdx.x, base = t * 4;
  uint32_t v[4], run = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0u;
    run += v[k];
  }
  uint32_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL_WARP, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    uint32_t w = (t < 16) ? wsum[t] : 0u, wi = w;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL_WARP, wi, o);
      if (t >= o) wi += y;
    }
    if (t < 16) wsum[t] = wi - w;  // exclusive warp offsets
    if (t == 15) wsum[16] = wi;    // total
  }
  __syncthreads();
  uint32_t e = wsum[t >> 5] + incl - run;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (base + k < n) out[base + k] = e;
    e += v[k];
  }
  if (t == 0) out[n] = wsum[16];
  __syncthreads();
}

__global__ void __launch_bounds__(512) bk_l1_scatter_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N,
                                                            uint32_t nb, const int64_t* Msboff, ulonglong2* out) {
  extern __shared__ __align__(16) unsigned char l1sm[];
  const uint32_t nsb = (nb + BK_SB - 1) / BK_SB;
  ulonglong2* stage = reinterpret_cast<ulonglong2*>(l1sm);                 // [BK_TILE]
  uint16_t* ssb = reinterpret_cast<uint16_t*>(stage + BK_TILE);            // [BK_TILE]
  uint32_t* cur = reinterpret_cast<uint32_t*>(ssb + BK_TILE);              // [nsb]
  uint32_t* th = cur + nsb;                                                // [nsb]
  uint32_t* toff = th + nsb;                                               // [nsb + 1]
  __shared__ uint32_t wsum[17];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  for (uint32_t sb = tid; sb < nsb; sb += blockDim.x) cur[sb] = (uint32_t)Msboff[(int64_t)sb * G + c];
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  const uint64_t stream = policy_evict_first();
  const int64_t c0 = N * c / G, c1 = N * (c + 1) / G;
  for (int64_t base = c0; base < c1; base += BK_TILE) {
    const int nt = (int)((c1 - base < BK_TILE) ? (c1 - base) : BK_TILE);
    for (uint32_t sb = tid; sb < nsb; sb += blockDim.x) th[sb] = 0;
    __syncthreads();
    ulonglong2 k[4];
    uint32_t sbk[4], r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = tid + u * 512;
      sbk[u] = 0xFFFFu;
      if (j < nt) {
        const int64_t i = base + j;
        k[u] = make_ulonglong2(ld_hint_u64(hi + i, stream), ld_hint_u64(lo + i, stream));
        sbk[u] = bucket_of_d(k[u].x, k[u].y, x, nb) / BK_SB;
        r[u] = atomicAdd(&th[sbk[u]], 1u);
      }
    }
    __syncthreads();
    block_scan_2048(th, toff, (int)nsb, wsum);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (sbk[u] != 0xFFFFu) {
        const uint32_t p = toff[sbk[u]] + r[u];
        stage[p] = k[u];
        ssb[p] = (uint16_t)sbk[u];
      }
    }
    __syncthreads();
    // write the tile in super-bucket order: consecutive threads, consecutive slots
    for (int t = tid; t < nt; t += blockDim.x) {
      const uint32_t sb = ssb[t];
      out[cur[sb] + (uint32_t)t - toff[sb]] = stage[t];
    }
    __syncthreads();
    for (uint32_t sb = tid; sb < nsb; sb += blockDim.x) cur[sb] += toff[sb + 1] - toff[sb];
    __syncthreads();
  }
}

// One cluster of BK_CL CTAs per super-bucket; CTA k owns bucket BK_SB*sb + k.
constexpr int BK_CBINS = 1024;  // top-10-bit bins of the in-cluster sort (~2 keys per bin at b = 2000)
__global__ void __launch_bounds__(256)
    bk_cluster_sort_kernel(const ulonglong2* in, const int64_t* prefix, int64_t nb, int cap, ulonglong2* out,
                           int* dup_flag) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char csm[];
  ulonglong2* keys = reinterpret_cast<ulonglong2*>(csm);            // [cap] this CTA's bucket
  uint16_t* idx = reinterpret_cast<uint16_t*>(keys + cap);          // [cap]
  int* bins = reinterpret_cast<int*>(idx + ((cap + 7) & ~7));      // [BK_CBINS]
  __shared__ uint32_t cnt[BK_SB];  // keys of my input slice per bucket of the super-bucket (read remotely)
  __shared__ uint32_t dst[BK_SB];  // my write cursor in each owner's key array
  __shared__ int wsum[8];
  const int kr = (int)cluster.block_rank(), tid = threadIdx.x;
  const int64_t sb = blockIdx.x / BK_CL;
  const int64_t b0 = sb * BK_SB, bend = (b0 + BK_SB < nb) ? b0 + BK_SB : nb;
  const int64_t s0 = prefix[b0], s1 = prefix[bend];
  if (tid < BK_SB) cnt[tid] = 0;
  __syncthreads();
  const u2 x = split64(seed_mixer(0, TAG_BUCKET));
  const int64_t na = s1 - s0, a = s0 + na * kr / BK_CL, z = s0 + na * (kr + 1) / BK_CL;
  for (int64_t i = a + tid; i < z; i += blockDim.x) {
    const ulonglong2 k = in[i];
    atomicAdd(&cnt[bucket_of_d(k.x, k.y, x, (uint32_t)nb) - (uint32_t)b0], 1u);
  }
  cluster.sync();  // every CTA's slice counts are final
  if (tid < BK_SB) {
    uint32_t base = 0;
    for (int k2 = 0; k2 < kr; ++k2) base += cluster.map_shared_rank(cnt, k2)[tid];
    dst[tid] = base;
  }
  __syncthreads();
  for (int64_t i = a + tid; i < z; i += blockDim.x) {
    const ulonglong2 k = in[i];
    const uint32_t lb = bucket_of_d(k.x, k.y, x, (uint32_t)nb) - (uint32_t)b0;
    const uint32_t slot = atomicAdd(&dst[lb], 1u);
    cluster.map_shared_rank(keys, (int)lb)[slot] = k;  // DSMEM store into the bucket's CTA
  }
  cluster.sync();  // all keys have arrived; no remote access after this point
  const int64_t b = b0 + kr;
  if (b >= bend) return;
  const int cntb = (int)(prefix[b + 1] - prefix[b]);
  if (cntb == 0) return;
  for (int i = tid; i < BK_CBINS; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  for (int i = tid; i < cntb; i += blockDim.x) atomicAdd(&bins[(int)(keys[i].x >> 54)], 1);
  __syncthreads();
  {  // exclusive scan of the bin counts (4 per thread)
    const int base = tid * (BK_CBINS / 256);
    int loc[BK_CBINS / 256], run = 0;
#pragma unroll
    for (int q = 0; q < BK_CBINS / 256; ++q) {
      loc[q] = run;
      run += bins[base + q];
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL_WARP, incl, o);
      if ((tid & 31) >= o) incl += v;
    }
    if ((tid & 31) == 31) wsum[tid >> 5] = incl;
    __syncthreads();
    int woff = 0;
    for (int w = 0; w < (tid >> 5); ++w) woff += wsum[w];
    const int excl = woff + incl - run;
#pragma unroll
    for (int q = 0; q < BK_CBINS / 256; ++q) bins[base + q] = excl + loc[q];
  }
  __syncthreads();
  for (int i = tid; i < cntb; i += blockDim.x) idx[atomicAdd(&bins[(int)(keys[i].x >> 54)], 1)] = (uint16_t)i;
  __syncthreads();
  const int64_t o0 = prefix[b];
  for (int p = tid; p < cntb; p += blockDim.x) {
    const ulonglong2 k = keys[idx[p]];
    const int bin = (int)(k.x >> 54);
    const int lo_ = bin ? bins[bin - 1] : 0, hi_ = bins[bin];
    int r = lo_;
    for (int q = lo_; q < hi_; ++q) {
      if (q == p) continue;
      const ulonglong2 o = keys[idx[q]];
      const bool eq = o.x == k.x && o.y == k.y;
      if (eq) atomicOr(dup_flag, 1);
      r += key_less(o, k) || (eq && q < p);
    }
    out[o0 + r] = k;
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
  // shared-memory path: M and its scan (nb * BK_G + 1 each) + scan scratch
  const int64_t nm = nb * BK_G + 1;
  const int64_t nms = ((nb + BK_SB - 1) / BK_SB) * BK_G + 1;
  size_t sm_path = ((size_t)nm * 8 + 255) & ~(size_t)255;
  sm_path *= 2;
  sm_path += 2 * (((size_t)nms * 8 + 255) & ~(size_t)255) + shk_scan_scratch(nms) + 256;
  sm_path += ((size_t)N * 16 + 255) & ~(size_t)255;
  sm_path += 256 + shk_scan_scratch(nm);
  s += ((size_t)N * 4 + 255) & ~(size_t)255;        // bucket ids
  s += ((size_t)N * 16 + 255) & ~(size_t)255;       // unsorted scatter
  s += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;  // counts
  s += ((size_t)(nb + 1) * 8 + 255) & ~(size_t)255;  // cursor
  s += 256;                                          // max
  s += shk_scan_scratch(nb);
  return s > sm_path ? s : sm_path;
}

// The shared-memory path; returns 1 when it does not apply (caller falls back).
static int bucketize_smem(const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nb, ulonglong2* out,
                          int64_t* prefix, int* dup_flag, void* scratch, int64_t* max_bucket_out, cudaStream_t st,
                          uint64_t* h_prefix, int* handled) {
  *handled = 0;
  if (nb > BK_MAX_NB || N >= (int64_t(1) << 32) || N < BK_G) return 0;
  const int64_t nm = nb * BK_G + 1;
  char* p = (char*)scratch;
  int64_t* M = (int64_t*)p;
  p += ((size_t)nm * 8 + 255) & ~(size_t)255;
  int64_t* Moff = (int64_t*)p;
  p += ((size_t)nm * 8 + 255) & ~(size_t)255;
  ulonglong2* unsorted = (ulonglong2*)p;
  p += ((size_t)N * 16 + 255) & ~(size_t)255;
  int64_t* maxv = (int64_t*)p;
  p += 256;
  const int64_t nsb = (nb + BK_SB - 1) / BK_SB, nms = nsb * BK_G + 1;
  int64_t* Msb = (int64_t*)p;
  p += ((size_t)nms * 8 + 255) & ~(size_t)255;
  int64_t* Msboff = (int64_t*)p;
  p += ((size_t)nms * 8 + 255) & ~(size_t)255;
  void* scan_scratch2 = p;
  p += shk_scan_scratch(nms) + 256;
  void* scan_scratch = p;
  const size_t hsm = (size_t)nb * 4;
  // (per call: the attribute is per device)
  SHK_CUDA(cudaFuncSetAttribute(bk_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BK_MAX_NB * 4));
  SHK_CUDA(cudaFuncSetAttribute(bk_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BK_MAX_NB * 4));
  SHK_CUDA(cudaFuncSetAttribute(bk_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SORT_BINS * 4 + BK_MAX_SORT * 18 + 16));
  SHK_CUDA(cudaMemsetAsync(maxv, 0, 8, st));
  SHK_CUDA(cudaMemsetAsync(dup_flag, 0, sizeof(int), st));
  SHK_CUDA(cudaMemsetAsync(M + nb * BK_G, 0, 8, st));
  SHK_CUDA(cudaMemsetAsync(Msb + nsb * BK_G, 0, 8, st));
  bk_hist_kernel<<<BK_G, 512, hsm, st>>>(hi, lo, N, (uint32_t)nb, M, Msb);
  SHK_LAUNCHED();
  int rc = shk_exclusive_scan_i64(M, Moff, nb * BK_G, scan_scratch, shk_scan_scratch(nm), st);
  if (rc) return rc;
  rc = shk_exclusive_scan_i64(Msb, Msboff, nsb * BK_G, scan_scratch2, shk_scan_scratch(nms), st);
  if (rc) return rc;
  bk_prefix_kernel<<<(unsigned)((nb + 256) / 256 < 148 ? (nb + 256) / 256 : 148), 256, 0, st>>>(Moff, BK_G, nb,
                                                                                                 prefix, maxv);
  SHK_LAUNCHED();
  // The key prefix and the largest bucket come back through pinned memory
  // behind an event; the super-bucket scatter is queued before the host
  // waits (it does not depend on the largest bucket, which only picks the
  // sort kernel), so the device goes from the scan straight into the scatter.
  static thread_local int64_t* hp = nullptr;
  static thread_local size_t hp_cap = 0;
  static thread_local cudaEvent_t ev = nullptr;
  if (hp_cap < (size_t)(nb + 2)) {
    if (hp) cudaFreeHost(hp);
    hp = nullptr;
    hp_cap = 0;
    SHK_CUDA(cudaMallocHost(&hp, (size_t)(nb + 2) * 8));
    hp_cap = (size_t)(nb + 2);
  }
  if (!ev) SHK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  if (h_prefix) SHK_CUDA(cudaMemcpyAsync(hp, prefix, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaMemcpyAsync(hp + nb + 1, maxv, 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaEventRecord(ev, st));
  static const bool use_cluster = [] {
    const char* e = getenv("SHK_BUCKET_CLUSTER");
    return !(e && e[0] == '0');
  }();
  if (use_cluster) {
    // super-bucket scatter (coalesced runs), then one 16-CTA cluster per super-bucket
    const size_t l1sm = (size_t)BK_TILE * 18 + (size_t)(3 * nsb + 1) * 4;
    SHK_CUDA(cudaFuncSetAttribute(bk_l1_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l1sm));
    bk_l1_scatter_kernel<<<BK_G, 512, l1sm, st>>>(hi, lo, N, (uint32_t)nb, Msboff, unsorted);
    SHK_LAUNCHED();
  }
  // the largest bucket picks the sort kernel; the caller's host work overlaps
  // the scatter and the sort (only the histogram and the scan are waited for)
  SHK_CUDA(cudaEventSynchronize(ev));
  const int64_t maxb = hp[nb + 1];
  if (h_prefix) memcpy(h_prefix, hp, (size_t)(nb + 1) * 8);
  if (max_bucket_out) *max_bucket_out = maxb;
  const int64_t cap = maxb;
  const size_t csm = (size_t)cap * 16 + (size_t)((cap + 7) & ~7) * 2 + BK_CBINS * 4;
  if (use_cluster && csm <= 200 * 1024) {
    SHK_CUDA(cudaFuncSetAttribute(bk_cluster_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
    SHK_CUDA(cudaFuncSetAttribute(bk_cluster_sort_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nsb * BK_CL), 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = csm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = BK_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SHK_CUDA(cudaLaunchKernelEx(&cfg, bk_cluster_sort_kernel, (const ulonglong2*)unsorted, (const int64_t*)prefix, nb,
                                (int)cap, out, dup_flag));
    SHK_LAUNCHED();
    *handled = 1;
    return 0;
  }
  // (A/B: SHK_BUCKET_SLICE_MB=S scatters S-MB destination slices, one pass
  // each; at C4 48 MB slices measured 0.61 ms vs 0.58 ms for one pass)
  static const int64_t slice_bytes = [] {
    const char* e = getenv("SHK_BUCKET_SLICE_MB");
    return e ? (int64_t)atoi(e) << 20 : (int64_t)0;
  }();
  int64_t passes = slice_bytes > 0 ? (N * 16 + slice_bytes - 1) / slice_bytes : 1;
  if (passes < 1) passes = 1;
  if (passes > nb) passes = nb;
  for (int64_t k = 0; k < passes; ++k) {
    const uint32_t blo = (uint32_t)(nb * k / passes), bhi = (uint32_t)(nb * (k + 1) / passes);
    bk_scatter_kernel<<<BK_G, 512, hsm, st>>>(hi, lo, N, (uint32_t)nb, Moff, unsorted, blo, bhi);
    SHK_LAUNCHED();
  }
  if (maxb > BK_MAX_SORT) {
    int64_t grid = nb < 148 * 8 ? nb : 148 * 8;
    bucket_sort_bins_kernel<<<(unsigned)grid, 256, 0, st>>>(unsorted, prefix, nb, out, dup_flag);
    SHK_LAUNCHED();
  } else {
    const size_t ssm = SORT_BINS * 4 + (size_t)maxb * 18 + 16;
    int64_t grid = nb < 148 * 16 ? nb : 148 * 16;
    bk_sort_kernel<<<(unsigned)grid, 256, ssm, st>>>(unsorted, prefix, nb, out, dup_flag);
    SHK_LAUNCHED();
  }
  *handled = 1;
  return 0;
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
#ifndef SHK_BUCKET_SMEM
#define SHK_BUCKET_SMEM 1
#endif
  if (SHK_BUCKET_SMEM) {
    int handled = 0;
    int rc = bucketize_smem(hi, lo, N, nb, (ulonglong2*)skeys_u64, (int64_t*)key_prefix, dup_flag, scratch,
                            max_bucket_out, st, h_prefix, &handled);
    if (rc || handled) return rc;
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
