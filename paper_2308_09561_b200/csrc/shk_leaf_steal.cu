// Batched PLAIN leaf search with seed-block work stealing (the leaf-only
// configs C1/C3/C5 and the seam's search_plain).  Restates
// _core.pyx:186-229 (minimum seed, counters) and pseudoforest.py:149-201
// (orientation, via orient_edges).
//
// Why: with a fixed team per leaf, a batch ends on its heaviest leaves.  Seed
// counts are geometric, so the worst of 20,000 C5 leaves needs ~10x the mean
// (up to ~5e7 seeds) and runs on one team while the rest of the GPU idles; a
// team also waits at a barrier every round for its slowest warp.
//
// Here every warp works alone (no barriers).  A leaf's seeds are handed out
// in blocks of 32 (one seed per lane) by an atomic block counter in the
// leaf's global state; any number of warps may work on a leaf at once:
//   * main phase: a warp takes the next leaf from the global leaf counter
//     (it is the leaf's owner) and claims its blocks one by one;
//   * tail phase (leaf counter exhausted): the warp joins a leaf some owner
//     is still working on (the `active` board, one slot per warp) and claims
//     blocks of that leaf too, so the last heavy leaves are searched by the
//     whole GPU.
// A lane whose seed passes the coverage filter and the exact pseudoforest
// check proposes it with an atomicMax of its complement (= atomicMin of the
// seed).  A warp stops claiming once the next block starts above the best
// seed found so far (read before the claim; a stale value only costs
// overshoot).  Every claimed block is searched completely, so when the last
// worker leaves (join/leave counter, joins only while it is positive) every
// block below the final best has been searched: the best is the minimum
// seed, exactly the reference's.
//
// Outputs: the minimum seed and its f bits (orientation by the last worker).
// The per-leaf counters (evals, passes, checks) are not produced here: the
// launcher takes this kernel only when no stats are requested (the
// fixed-team kernel of shk_leaf.cu counts them exactly).
#include "shk_kernels.h"
#include "shk_leaf_dev.cuh"

namespace shk {

struct StealLeaf {                 // per-leaf global state, zero-initialised
  unsigned long long next_blk;     // next 32-seed block to hand out
  unsigned long long nbest;        // ~(best seed found), 0 = none yet
  int workers;                     // warps on the leaf; joins only while > 0
  int pad;
};

template <int MAXE>
struct StealSmem {
  uint4 keys[MAXE];
  uint16_t col[MAXE];  // edge column of the candidate being checked
  uint8_t eu[MAXE], ev[MAXE];
  uint64_t inc[MAXE];
  WarpChk chk;
};

SHK_D unsigned long long ldr_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
SHK_D long long ldr_s64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
SHK_D int ldr_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SHK_D void str_s64(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// First lane of `pb` (filter-passing lanes, seeds s0 + lane) whose graph is a
// pseudoforest, or 32.  The warp recomputes each candidate's edge column.
template <class SM>
SHK_D int plain_first_accept(SM& sm, int n, uint64_t s0, unsigned pb, int lane) {
  while (pb) {
    const int L = __ffs(pb) - 1;
    pb &= pb - 1;
    const u2 x = seed_mixer_pre_d(s0 + (uint64_t)L, TAG_LEAF);
    for (int i = lane; i < n; i += 32) {
      const uint4 k = sm.keys[i];
      uint32_t h0, h1;
      leaf_pair_d(remix_pre_d(u2{k.x, k.y}, u2{k.z, k.w}, x), (uint32_t)n, (uint32_t)(n - 1), h0, h1);
      sm.col[i] = (uint16_t)(h0 | (h1 << 8));
    }
    __syncwarp();
    const bool ok = warp_pf_check_col(sm.col, 1, 0, n, lane, sm.chk);
    __syncwarp();
    if (ok) return L;
  }
  return 32;
}

template <bool WIDE, int MAXE>
__global__ void __launch_bounds__(128, 8) leaf_steal_kernel(LeafArgs a, StealLeaf* st, long long* active,
                                                             int* leaf_counter) {
  __shared__ StealSmem<MAXE> sm_all[4];
  __shared__ uint2 onehot_tab[64];  // SHK_PLAIN_ONEHOT_LDS
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  StealSmem<MAXE>& sm = sm_all[w];
  if (SHK_PLAIN_ONEHOT_LDS) fill_onehot_tab(onehot_tab, lane);
  const int gw = blockIdx.x * 4 + w;
  const int nw = gridDim.x * 4;
  bool tail = false;
  for (;;) {
    // ---- take a leaf: own the next one, or join one still being searched
    long long leaf = -1;
    bool owner = false;
    if (!tail) {
      long long l = 0;
      // system scope: the counter may live on another GPU (CUDA IPC, NVLink
      // atomics) and be shared by every rank's launch (cross-GPU leaf queue)
      if (lane == 0) l = atomicAdd_system(leaf_counter, 1);
      l = __shfl_sync(FULL_WARP, l, 0);
      if (l < a.L) {
        leaf = l;
        owner = true;
      } else {
        tail = true;
      }
    }
    if (tail) {
      // active[nw] counts the owners still searching; with none left every
      // leaf is closed and the warp is done
      for (int base = 0; base < nw && leaf < 0; base += 32) {
        if (ldr_s64(active + nw) <= 0) break;
        const int j = base + lane;
        long long cand = -1;
        if (j < nw) {
          int idx = gw + 1 + j;
          if (idx >= nw) idx -= nw;
          cand = ldr_s64(active + idx);
        }
        unsigned m = __ballot_sync(FULL_WARP, cand >= 0);
        while (m && leaf < 0) {
          const int L = __ffs(m) - 1;
          m &= m - 1;
          const long long c = __shfl_sync(FULL_WARP, cand, L);
          int joined = 0;
          if (lane == 0) {
            int* wp = &st[c].workers;
            int cur = ldr_s32(wp);
            while (cur > 0) {
              const int old = atomicCAS(wp, cur, cur + 1);
              if (old == cur) {
                joined = 1;
                break;
              }
              cur = old;
            }
          }
          if (__shfl_sync(FULL_WARP, joined, 0)) leaf = c;
        }
      }
      if (leaf < 0) break;  // nothing left to search
    }
    const int64_t k0 = a.off[leaf];
    const int n = (int)(a.off[leaf + 1] - k0);
    const LeafOut o{a.seed_slot ? a.seed_slot[leaf] : leaf, leaf};
    for (int i = lane; i < n; i += 32) {
      const uint64_t hw = a.hi[(k0 + i) * a.stride];
      const u2 h = split64(a.pre ? hw : premix_hi(hw)), l = split64(a.lo[(k0 + i) * a.stride]);
      sm.keys[i] = make_uint4(h.lo, h.hi, l.lo, l.hi);
    }
    __syncwarp();
    if (n <= 1) {  // _core.pyx: a 1-key leaf is (0, 1, 1, 1, 0); owners only
      leaf_finish<1>(a, sm, k0, n, 0, o, 1, 1, 0, lane);
      continue;
    }
    StealLeaf& L_ = st[leaf];
    if (owner) {
      if (lane == 0) {
        atomicAdd(&L_.workers, 1);
        atomicAdd((unsigned long long*)(active + nw), 1ull);
        str_s64(active + gw, leaf);  // helpers may join from now on
      }
    }
    // ---- claim and search 32-seed blocks.  The loads that decide whether
    // to claim the next block are issued when the current block starts, so
    // their latency hides behind its search (stale values are safe: the
    // best seed only decreases and the block counter only grows).
    unsigned long long nb = 0, nbest = 0;
    if (lane == 0) {
      nb = ldr_u64(&L_.next_blk);
      nbest = ldr_u64(&L_.nbest);
    }
    for (;;) {
      unsigned long long blk = 0;
      int stop = 0;
      if (lane == 0) {
        const unsigned long long s0 = nb * 32ull;
        if (s0 >= a.max_seed || (nbest != 0 && s0 > ~nbest)) {
          stop = 1;
        } else {
          blk = atomicAdd(&L_.next_blk, 1ull);
          nb = ldr_u64(&L_.next_blk);
          nbest = ldr_u64(&L_.nbest);
        }
      }
      if (__shfl_sync(FULL_WARP, stop, 0)) break;
      blk = __shfl_sync(FULL_WARP, blk, 0);
      const uint64_t s0 = (uint64_t)blk * 32ull;
      const uint64_t s = s0 + lane;
      const bool full = s < a.max_seed &&
                        plain_mask_full<WIDE, false>(sm.keys, n, s, nullptr, SHK_PLAIN_ONEHOT_LDS ? onehot_tab : nullptr);
      const unsigned pb = __ballot_sync(FULL_WARP, full);
      if (pb) {
        const int win = plain_first_accept(sm, n, s0, pb, lane);
        if (win < 32 && lane == 0) {
          const unsigned long long c = ~(unsigned long long)(s0 + win);
          atomicMax(&L_.nbest, c);
          if (c > nbest) nbest = c;
        }
      }
    }
    // ---- leave; the last worker finalises the leaf
    int last = 0;
    if (lane == 0) {
      if (owner) {
        str_s64(active + gw, -1);
        atomicAdd((unsigned long long*)(active + nw), ~0ull);
      }
      __threadfence();
      last = atomicSub(&L_.workers, 1) == 1;
      if (last) __threadfence();
    }
    if (!__shfl_sync(FULL_WARP, last, 0)) continue;
    if (lane == 0) nbest = ldr_u64(&L_.nbest);
    nbest = __shfl_sync(FULL_WARP, nbest, 0);
    const int64_t seed = nbest != 0 ? (int64_t)~nbest : -1;
    if (seed >= 0) {
      const u2 x = seed_mixer_pre_d((uint64_t)seed, TAG_LEAF);
      for (int i = lane; i < n; i += 32) {
        const uint4 k = sm.keys[i];
        uint32_t h0, h1;
        leaf_pair_d(remix_pre_d(u2{k.x, k.y}, u2{k.z, k.w}, x), (uint32_t)n, (uint32_t)(n - 1), h0, h1);
        sm.eu[i] = (uint8_t)h0;
        sm.ev[i] = (uint8_t)h1;
      }
    }
    leaf_finish<1>(a, sm, k0, n, seed, o, 0, 0, 0, lane);
    __syncwarp();
  }
}

}  // namespace shk

using namespace shk;

size_t shk_leaf_steal_state_bytes(int64_t L) { return (size_t)L * sizeof(StealLeaf); }

int shk_launch_leaf_steal(const ShkLeafLaunch& p, void* state, long long* active, int max_active, int shared_counter,
                          cudaStream_t st) {
  if (p.L <= 0) return 0;
  LeafArgs a{};
  a.hi = p.hi;
  a.lo = p.lo;
  a.off = p.off;
  a.L = p.L;
  a.max_seed = p.max_seed;
  a.mode = 0;
  a.seed_out = p.seed_out;
  a.fbits_out = p.fbits_out;
  a.choice_out = p.choice_out;
  a.stats_out = nullptr;  // no counters on this path (see top)
  a.error = p.error;
  a.stride = p.stride > 0 ? p.stride : 1;
  a.pre = p.pre;
  a.seed_slot = p.seed_slot;
  a.stats_acc = nullptr;
  a.exhausted = p.exhausted;
  a.place_out = p.place_out;
  const bool wide = p.max_n > 32;
  void (*kfn)(LeafArgs, StealLeaf*, long long*, int*) =
      wide ? leaf_steal_kernel<true, 64> : leaf_steal_kernel<false, 32>;
  int occ = 0;
  SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 128, 0));
  if (occ < 1) occ = 1;
  const int sms = p.num_sms > 0 ? p.num_sms : 148;
  int64_t blocks = (int64_t)sms * occ;
  SHK_CUDA(cudaMemsetAsync(state, 0, shk_leaf_steal_state_bytes(p.L), st));
  if (blocks * 4 + 1 > max_active) blocks = (max_active - 1) / 4;
  SHK_CUDA(cudaMemsetAsync(active, 0xFF, (size_t)blocks * 4 * sizeof(long long), st));
  SHK_CUDA(cudaMemsetAsync(active + blocks * 4, 0, sizeof(long long), st));  // owners searching
  if (!shared_counter) SHK_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(int), st));  // a shared one is reset by its owner
  kfn<<<(unsigned)blocks, 128, 0, st>>>(a, reinterpret_cast<StealLeaf*>(state), active, p.counter);
  SHK_LAUNCHED();
  return 0;
}
