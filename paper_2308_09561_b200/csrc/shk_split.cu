// RecSplit split-seed brute force + stable partition.
//
// Restates _core.pyx:378-428 (split_parts, split_seed_search) and the
// per-node partition of recsplit.py:553-567 for sm_100a.
//
// Keys are interleaved (premix_hi(hi), lo) pairs (shk_hash.cuh).
// One warp per split node (fetched dynamically).  Lane j tests seed R + j
// over all m keys of the node: key loads are warp-uniform (LDG.128 broadcast
// from L1/L2), part counts live in one 64-bit register as four 16-bit
// remaining-capacity fields biased by 0x8000, so an overflowing part is the
// clearing of that field's sign bit.  The first failing key index of each
// lane is tracked exactly, so the reference's `evals` counter is reproduced.
// The warp votes every 8 keys and leaves the key loop as soon as every lane
// has failed.  The lowest succeeding lane of the first batch with a success
// is the reference's minimum seed.  The warp then stable-partitions the
// node's keys by part with ballots (child order = part order), through a
// scratch buffer, in place.
#include "shk_common.cuh"
#include "shk_kernels.h"
#include "shk_split_dev.cuh"

namespace shk {

__global__ void __launch_bounds__(256) split_kernel(ShkSplitLaunch a) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const ulonglong2* keys = reinterpret_cast<const ulonglong2*>(a.hi);  // interleaved (hi, lo)
  ulonglong2* kw = reinterpret_cast<ulonglong2*>(a.hi);
  ulonglong2* tmp = reinterpret_cast<ulonglong2*>(a.tmp_hi);
  for (;;) {
    int64_t t = 0;
    if (lane == 0) t = atomicAdd(a.counter, 1);
    t = __shfl_sync(FULL_WARP, t, 0);
    if (t >= a.ntasks) break;
    const ShkSplitTask task = a.tasks[t];
    const int m = task.m;
    const ulonglong2* kp = keys + task.start;
    const uint32_t um = (uint32_t)m;
    if (!a.exact_evals && task.fanout >= 2 && task.fanout <= 4) {
      int64_t seed = split_search_build(kp, task, a.max_seed, lane);
      if (lane == 0) {
        a.seeds[task.seed_slot] = seed;
        if (seed < 0 && a.exhausted) atomicOr(a.exhausted, 1);
      }
      if (seed >= 0 && a.partition) split_partition(kp, kw, tmp, task, seed, lane, lt);
      continue;
    }
    // cumulative bounds; unused parts get bound m (never reached by r < m)
    uint32_t b[3];
    uint64_t cap0 = 0;  // biased remaining capacities
    {
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t sz = (j < task.fanout) ? (uint32_t)task.sizes[j] : 0x7FFFu;
        if (j < 3) {
          acc += (j < task.fanout) ? (uint32_t)task.sizes[j] : 0u;
          b[j] = (j < task.fanout - 1) ? acc : um;
        }
        cap0 |= (uint64_t)(0x8000u + sz) << (16 * j);
      }
    }
    const uint32_t b0 = b[0], b1 = b[1], b2 = b[2];
    uint64_t evals = 0;
    int64_t seed = -1;
    for (uint64_t R = 0; R < a.max_seed; R += 32) {
      const uint64_t s = R + lane;
      const bool valid = s < a.max_seed;
      const u2 x = seed_mixer_pre_d(s, TAG_SPLIT);
      uint32_t capl = (uint32_t)cap0, caph = (uint32_t)(cap0 >> 32);
      int fail = valid ? -1 : 0;  // invalid lanes count as failed at key 0
      for (int i0 = 0; i0 < m; i0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          if (i < m) {
            ulonglong2 k = __ldg(kp + i);
            u2 v = remix_pre_d(split64(k.x), split64(k.y), x);
            uint32_t r = __umulhi(v.hi, um);
            uint32_t sh = part_of(r, b0, b1, b2) << 4;
            uint32_t dl = shl_clamp(1u, sh), dh = shl_clamp(1u, sh - 32u);
            // 64-bit subtract of the one-hot decrement
            asm("sub.cc.u32 %0, %0, %2;\n\tsubc.u32 %1, %1, %3;" : "+r"(capl), "+r"(caph) : "r"(dl), "r"(dh));
            bool ovf = ((capl & caph & 0x80008000u) != 0x80008000u);
            if (ovf && fail < 0) fail = i;
          }
        }
        if (__all_sync(FULL_WARP, fail >= 0)) break;
      }
      const bool ok = valid && fail < 0;
      const unsigned ab = __ballot_sync(FULL_WARP, ok);
      const int w = ab ? __ffs(ab) - 1 : 32;
      uint64_t my = 0;
      if (valid) {
        if (lane < w) my = (uint64_t)fail + 1;
        else if (lane == w) my = (uint64_t)m;
      }
      evals += warp_sum(my);
      if (ab) {
        seed = (int64_t)(R + (uint64_t)w);
        break;
      }
    }
    if (lane == 0) {
      a.seeds[task.seed_slot] = seed;
      if (a.evals_out) a.evals_out[t] = (int64_t)evals;
      if (seed < 0 && a.exhausted) atomicOr(a.exhausted, 1);
      if (a.evals_acc) atomicAdd(a.evals_acc, (unsigned long long)evals);
    }
    if (seed >= 0 && a.partition) split_partition(kp, kw, tmp, task, seed, lane, lt);
  }
}

__global__ void split_parts_kernel(const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed,
                                   const int64_t* sizes, int fanout, int64_t* parts) {
  const u2 x = seed_mixer_d(seed, TAG_SPLIT);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    u2 v = remix_d(split64(hi[i]), split64(lo[i]), x);
    uint64_t r = ((uint64_t)v.hi * (uint64_t)m) >> 32;
    // searchsorted(cumsum(sizes), r, side="right")
    int64_t acc = 0, p = 0;
    for (; p < fanout; ++p) {
      acc += sizes[p];
      if ((int64_t)r < acc) break;
    }
    parts[i] = p;
  }
}

__global__ void interleave_kernel(const uint64_t* hi, const uint64_t* lo, int64_t N, ulonglong2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_ulonglong2(hi[i], lo[i]);
}

__global__ void deinterleave_kernel(const ulonglong2* in, int64_t N, uint64_t* hi, uint64_t* lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    ulonglong2 k = in[i];
    hi[i] = k.x;
    lo[i] = k.y;
  }
}

// In-place premix_hi / unpremix_hi of the high words of interleaved pairs.
__global__ void premix_pairs_kernel(ulonglong2* keys, int64_t N, int inverse) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    ulonglong2 k = keys[i];
    k.x = inverse ? unpremix_hi(k.x) : premix_hi(k.x);
    keys[i] = k;
  }
}

}  // namespace shk

using namespace shk;

static unsigned grid256(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

int shk_launch_split_parts(const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed, const int64_t* sizes,
                           int fanout, int64_t* parts, cudaStream_t st) {
  if (m <= 0) return 0;
  split_parts_kernel<<<grid256(m), 256, 0, st>>>(hi, lo, m, seed, sizes, fanout, parts);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_interleave(const uint64_t* hi, const uint64_t* lo, int64_t N, uint64_t* pairs, cudaStream_t st) {
  if (N <= 0) return 0;
  interleave_kernel<<<grid256(N), 256, 0, st>>>(hi, lo, N, (ulonglong2*)pairs);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_deinterleave(const uint64_t* pairs, int64_t N, uint64_t* hi, uint64_t* lo, cudaStream_t st) {
  if (N <= 0) return 0;
  deinterleave_kernel<<<grid256(N), 256, 0, st>>>((const ulonglong2*)pairs, N, hi, lo);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_premix(uint64_t* pairs, int64_t N, int inverse, cudaStream_t st) {
  if (N <= 0) return 0;
  premix_pairs_kernel<<<grid256(N), 256, 0, st>>>((ulonglong2*)pairs, N, inverse);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_split(const ShkSplitLaunch& p, cudaStream_t st) {
  if (p.ntasks <= 0) return 0;
  SHK_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(int), st));
  int occ = 0;
  SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, split_kernel, 256, 0));
  if (occ < 1) occ = 1;
  int sms = p.num_sms > 0 ? p.num_sms : 148;
  int64_t blocks = (int64_t)sms * occ;
  int64_t need = (p.ntasks + 7) / 8;
  if (blocks > need) blocks = need;
  split_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  SHK_LAUNCHED();
  return 0;
}
