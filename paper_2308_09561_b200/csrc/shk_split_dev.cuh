// Split-seed search and stable partition as warp-level device functions,
// shared by the per-level split kernel (shk_split.cu) and the persistent
// construction kernel (shk_tree.cu).  Restates _core.pyx:378-428 and
// recsplit.py:553-567.
#pragma once
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

// Key loads of the split searches: warp-uniform addresses (broadcast).
// Plain coherent loads (L1-cached): inside the persistent tree kernel the
// same key array is partitioned in place by other warps during the launch,
// so the read-only (.nc) path is not allowed; the acquire fence a warp runs
// before it reads a published node orders these loads after the parent's
// partition stores.
SHK_D ulonglong2 load_key(const ulonglong2* p) { return *p; }

// (analysis builds, -DSHK_SPLIT_WORK) lane-key evaluations the fast split
// searches issue: [0] keys x 32 lanes per seed block, [1] seed blocks
#ifdef SHK_SPLIT_WORK
__device__ unsigned long long g_split_work[2];
#define SHK_SPLIT_WORK_ADD(keys)                                     \
  do {                                                               \
    if (lane == 0) {                                                 \
      atomicAdd(&g_split_work[0], 32ull * (unsigned long long)(keys)); \
      atomicAdd(&g_split_work[1], 1ull);                             \
    }                                                                \
  } while (0)
#else
#define SHK_SPLIT_WORK_ADD(keys) \
  do {                           \
  } while (0)
#endif

// Part index of split hash value r against cumulative bounds (up to 4 parts).
SHK_D uint32_t part_of(uint32_t r, uint32_t b0, uint32_t b1, uint32_t b2) {
  return (uint32_t)(r >= b0) + (uint32_t)(r >= b1) + (uint32_t)(r >= b2);
}

// Keys of the split searches are interleaved (premix_hi(hi), lo) pairs.

// Stable partition of a node's keys by part (recsplit.py:558-561): ballots
// rank every key within its part, keys go to tmp and are copied back.
SHK_D void split_partition(const ulonglong2* kp, ulonglong2* kw, ulonglong2* tmp, const ShkSplitTask& task,
                           int64_t seed, int lane, unsigned lt) {
  const int m = task.m;
  const uint32_t um = (uint32_t)m;
  uint32_t b[3], cur[4];
  {
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cur[j] = acc;
      acc += (j < task.fanout) ? (uint32_t)task.sizes[j] : 0u;
      if (j < 3) b[j] = (j < task.fanout - 1) ? acc : um;
    }
  }
  const u2 x = seed_mixer_pre_d((uint64_t)seed, TAG_SPLIT);
  for (int c = 0; c < m; c += 32) {
    const int i = c + lane;
    const bool in = i < m;
    ulonglong2 k = make_ulonglong2(0, 0);
    uint32_t p = 4;
    if (in) {
      k = kp[i];
      u2 v = remix_pre_d(split64(k.x), split64(k.y), x);
      p = part_of(__umulhi(v.hi, um), b[0], b[1], b[2]);
    }
    uint32_t dst = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned bal = __ballot_sync(FULL_WARP, p == (uint32_t)j);
      if (p == (uint32_t)j) dst = cur[j] + __popc(bal & lt);
      cur[j] += __popc(bal);
    }
    if (in) tmp[task.start + dst] = k;
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) kw[task.start + i] = tmp[task.start + i];
  __syncwarp();
}

// High word of remix(hi, lo, seed, tag) (all the split hash needs), from a
// pre-mixed key high word and seed mixer (shk_hash.cuh, premix_hi).
#ifndef SHK_SPLIT_SHIFT_MASK
// bit i: xor-shift i of the split hash takes its high-word shift on the FMA pipe
// (IMAD.HI, two issue slots) instead of the ALU pipe (SHF).  With the
// shared-memory tables the construction kernel is ALU-bound (ncu: ALU 75%,
// FMA-heavy 62%), so two of the four shifts go back to the FMA pipe.  All 16
// masks measured at C4 (10-step A/Bs, two rounds each, tools/ab_bench.sh):
// 0: 91.7 ms, single bits 91.4-91.7, 3: 91.1, 12: 91.1, 5: 90.8 (best),
// three bits 91.3-91.8, 15: 92.0-92.9.
#define SHK_SPLIT_SHIFT_MASK 5
#endif
template <int S, int I>
SHK_D u2 split_xs(u2 z) {
  return ((SHK_SPLIT_SHIFT_MASK >> I) & 1) ? xorshr<S>(z) : xorshr_alu<S>(z);
}
SHK_D uint32_t remix_hi_pre_d(u2 kp, u2 k_lo, u2 xp) {
  u2 z;
  z.lo = kp.lo ^ xp.lo;
  z.hi = kp.hi ^ xp.hi;
  z = mulc<MUL1>(z);
  z = mulc<MUL2>(split_xs<27, 0>(z));
  z = split_xs<31, 1>(z);
  z.lo ^= k_lo.lo;
  z.hi ^= k_lo.hi;
  z = mulc<MUL1>(split_xs<30, 2>(z));
  const uint32_t h = mulc_hi<MUL2>(split_xs<27, 3>(z));
  return h ^ (h >> 31);  // hi word of z ^ (z >> 31)
}

// Fast minimum-seed search for a node with F parts (build path).
// hash_range(v, m) >= b  <=>  v.hi >= ceil(b * 2^32 / m), so parts are
// counted by comparing the remixed high word against F-1 precomputed
// thresholds (thermometer counts g_j = #keys with part >= j).  Overflow is
// checked once per 8 keys (it is monotone, so the seed verdict is exact);
// the exact first-failing key index (the reference's `evals`) is not tracked
// here — the exact path of split_kernel (shk_split.cu) does that for the seam
// API and the instrumented build.
template <int F>
SHK_D int64_t split_search_fast(const ulonglong2* kp, const ShkSplitTask& task, uint64_t max_seed, int lane) {
  const int m = task.m;
  uint32_t T0 = 0, T1 = 0, T2 = 0;
  {
    uint64_t acc = 0;
    acc += (uint64_t)task.sizes[0];
    T0 = (uint32_t)(((acc << 32) + (uint64_t)m - 1) / (uint64_t)m);
    if (F > 2) {
      acc += (uint64_t)task.sizes[1];
      T1 = (uint32_t)(((acc << 32) + (uint64_t)m - 1) / (uint64_t)m);
    }
    if (F > 3) {
      acc += (uint64_t)task.sizes[2];
      T2 = (uint32_t)(((acc << 32) + (uint64_t)m - 1) / (uint64_t)m);
    }
  }
  const int s0 = task.sizes[0], s1 = task.sizes[1], s2 = F > 2 ? task.sizes[2] : 0, s3 = F > 3 ? task.sizes[3] : 0;
  for (uint64_t R = 0; R < max_seed; R += 32) {
    const uint64_t s = R + lane;
    const u2 x = seed_mixer_pre_d(s, TAG_SPLIT);
    int g1 = 0, g2 = 0, g3 = 0;
    bool fail = !(s < max_seed);
    bool all_failed = false;
    int i = 0;
    for (; i + 8 <= m; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const ulonglong2 k = load_key(kp + i + u);
        const uint32_t vh = remix_hi_pre_d(split64(k.x), split64(k.y), x);
        g1 += (vh >= T0);
        if (F > 2) g2 += (vh >= T1);
        if (F > 3) g3 += (vh >= T2);
      }
      const int done = i + 8;
      bool ovf = (done - g1 > s0);
      if (F == 2) ovf |= (g1 > s1);
      if (F == 3) ovf |= (g1 - g2 > s1) | (g2 > s2);
      if (F == 4) ovf |= (g1 - g2 > s1) | (g2 - g3 > s2) | (g3 > s3);
      fail |= ovf;
      if (__all_sync(FULL_WARP, fail)) {
        all_failed = true;
        break;
      }
    }
    if (!all_failed) {
      for (; i < m; ++i) {
        const ulonglong2 k = load_key(kp + i);
        const uint32_t vh = remix_hi_pre_d(split64(k.x), split64(k.y), x);
        g1 += (vh >= T0);
        if (F > 2) g2 += (vh >= T1);
        if (F > 3) g3 += (vh >= T2);
      }
      bool ovf = (m - g1 > s0);
      if (F == 2) ovf |= (g1 > s1);
      if (F == 3) ovf |= (g1 - g2 > s1) | (g2 > s2);
      if (F == 4) ovf |= (g1 - g2 > s1) | (g2 - g3 > s2) | (g3 > s3);
      fail |= ovf;
    }
    SHK_SPLIT_WORK_ADD(all_failed ? i + 8 : m);
    const unsigned ab = __ballot_sync(FULL_WARP, !fail);
    if (ab) return (int64_t)(R + (uint64_t)(__ffs(ab) - 1));
  }
  return -1;
}

// Nodes split into F EQUAL parts (the 4 x 40, 3 x 160 and 2 x 480 nodes of
// C4's plans carry most of the split work).  With s = m / F the part of a key
// is floor(floor(vh m / 2^32) / s) = floor(F vh / 2^32) exactly, so:
//   F = 2: part = vh >> 31, counted with one LEA.HI;
//   F = 3: part = umulhi(vh, 3); a += part, b += part >> 1 give
//          #part2 = b, #part1 = a - 2b;
//   F = 4 (m < 172): part = vh >> 30, one byte counter per part in one
//          register (acc += 1 << 8 part), overflow of any byte past s by one
//          add-and-mask.
// Same seeds as split_search_fast (same exact per-part counts).
#ifndef SHK_SPLIT_EQUAL
// bit F: equal-part counters for fanout F.  Measured at C4 (tools/ab_bench.sh):
// F = 4 saves ~3%; the F = 2 / F = 3 variants are neutral (F = 3's IMAD.HI
// competes for the busy FMA pipe), so only F = 4 is on by default.
#define SHK_SPLIT_EQUAL 0x10
#endif
SHK_D bool equal_split_ok(int F, int m) {
  if (F < 2 || F > 4 || m % F || !((SHK_SPLIT_EQUAL >> F) & 1)) return false;
  return F != 4 || m < 172;
}

#ifndef SHK_SPLIT_EQ_BLOCK
#define SHK_SPLIT_EQ_BLOCK 8  // keys between overflow checks of the equal-part search
#endif
#ifndef SHK_SPLIT_EQ_SEEDS
#define SHK_SPLIT_EQ_SEEDS 1  // seeds per lane (S > 1: lane tests R + lane + 32 j, j < S, per key load)
#endif
// SHK_SPLIT_CNT_LDS: the F = 4 byte counter's increment 1 << 8 part comes from
// a 4-entry shared-memory table (one LDS on the LSU pipe) instead of a mask
// and a variable shift on the ALU pipe, which the construction kernel saturates.
#ifndef SHK_SPLIT_CNT_LDS
#define SHK_SPLIT_CNT_LDS 1
#endif
template <int F>
SHK_D int64_t split_search_equal(const ulonglong2* kp, const ShkSplitTask& task, uint64_t max_seed, int lane) {
  constexpr int U = SHK_SPLIT_EQ_BLOCK, S = SHK_SPLIT_EQ_SEEDS;
  const int m = task.m;
  const int sz = m / F;
  __shared__ uint32_t cnt_tab[4];  // 1 << 8 p (written by every warp before its search: same values)
  if (F == 4 && SHK_SPLIT_CNT_LDS) {
    if (lane < 4) cnt_tab[lane] = 1u << (8 * lane);
    __syncwarp();
  }
  const uint32_t K4 = (uint32_t)(127 - sz) * 0x01010101u;  // byte b > sz <=> bit 7 of (b + 127 - sz)
  for (uint64_t R = 0; R < max_seed; R += 32 * S) {
    u2 x[S];
    uint32_t a[S], b[S];
    bool fail[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const uint64_t s = R + lane + 32 * j;
      x[j] = seed_mixer_pre_d(s, TAG_SPLIT);
      a[j] = 0;
      b[j] = 0;
      fail[j] = !(s < max_seed);
    }
    bool all_failed = false;
    int i = 0;
    auto count = [&](int j, uint32_t vh) {
      if (F == 2) {
        a[j] += vh >> 31;
      } else if (F == 3) {
        const uint32_t p = __umulhi(vh, 3u);
        a[j] += p;
        b[j] += p >> 1;
      } else if (SHK_SPLIT_CNT_LDS) {
        a[j] += cnt_tab[vh >> 30];
      } else {
        a[j] += 1u << ((vh >> 27) & 24u);
      }
    };
    auto over = [&](int j, int done) -> bool {
      if (F == 2) return (done - (int)a[j] > sz) || ((int)a[j] > sz);
      if (F == 3) {
        const int c2 = (int)b[j], c1 = (int)a[j] - 2 * c2;
        return (done - c1 - c2 > sz) || (c1 > sz) || (c2 > sz);
      }
      return ((a[j] + K4) & 0x80808080u) != 0u;
    };
    for (; i + U <= m; i += U) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const ulonglong2 k = load_key(kp + i + u);
#pragma unroll
        for (int j = 0; j < S; ++j) count(j, remix_hi_pre_d(split64(k.x), split64(k.y), x[j]));
      }
      bool af = true;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        fail[j] |= over(j, i + U);
        af &= fail[j];
      }
      if (__all_sync(FULL_WARP, af)) {
        all_failed = true;
        break;
      }
    }
    if (!all_failed) {
      for (; i < m; ++i) {
        const ulonglong2 k = load_key(kp + i);
#pragma unroll
        for (int j = 0; j < S; ++j) count(j, remix_hi_pre_d(split64(k.x), split64(k.y), x[j]));
      }
#pragma unroll
      for (int j = 0; j < S; ++j) fail[j] |= over(j, m);
    }
    SHK_SPLIT_WORK_ADD(S * (all_failed ? i + U : m));
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const unsigned ab = __ballot_sync(FULL_WARP, !fail[j]);
      if (ab) return (int64_t)(R + 32 * j + (uint64_t)(__ffs(ab) - 1));
    }
  }
  return -1;
}

// Dispatch: equal-part nodes take the cheaper counters.
SHK_D int64_t split_search_build(const ulonglong2* kp, const ShkSplitTask& task, uint64_t max_seed, int lane) {
  const int F = task.fanout;
  bool eq = SHK_SPLIT_EQUAL && equal_split_ok(F, task.m);
  for (int j = 1; j < F && eq; ++j) eq = task.sizes[j] == task.sizes[0];
  if (eq) {
    return F == 2 ? split_search_equal<2>(kp, task, max_seed, lane)
           : F == 3 ? split_search_equal<3>(kp, task, max_seed, lane)
                    : split_search_equal<4>(kp, task, max_seed, lane);
  }
  return F == 2 ? split_search_fast<2>(kp, task, max_seed, lane)
         : F == 3 ? split_search_fast<3>(kp, task, max_seed, lane)
                  : split_search_fast<4>(kp, task, max_seed, lane);
}

}  // namespace shk
