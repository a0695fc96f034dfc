// Batched leaf search kernels (CSR leaves, dynamic fetch) and the standalone
// orientation kernel.  The per-leaf search itself is in shk_leaf_dev.cuh.
#include "shk_kernels.h"
#include "shk_leaf_dev.cuh"

namespace shk {

// CTA = TEAMS independent teams of TW warps; each team fetches leaves with an
// atomic counter, so heavy-tailed leaves do not hold up other teams.
template <int TW, int TEAMS, bool WIDE, int MODE>
__global__ void __launch_bounds__(TW * 32 * TEAMS) leaf_kernel(LeafArgs a) {
  __shared__ LeafSmem<TW> sm_all[TEAMS];
  const int lane = threadIdx.x & 31;
  const int team = (threadIdx.x >> 5) / TW;
  const int warp = (threadIdx.x >> 5) % TW;  // warp within the team
  const int tt = threadIdx.x - team * TW * 32;
  LeafSmem<TW>& sm = sm_all[team];
  for (;;) {
    if (tt == 0) sm.leaf = atomicAdd(a.counter, 1);
    team_sync<TW>(team);
    const int64_t leaf = sm.leaf;
    if (leaf >= a.L) break;
    const int64_t k0 = a.off[leaf];
    const int n = (int)(a.off[leaf + 1] - k0);
    const LeafOut o{a.seed_slot ? a.seed_slot[leaf] : leaf, leaf};
    if (MODE == 0)
      solve_plain<TW, WIDE>(a, sm, k0, n, o, team, warp, lane, tt);
    else
      solve_rotate<TW, WIDE>(a, sm, k0, n, o, team, warp, lane, tt);
  }
}

// Standalone batched orientation (pseudoforest.orient on the GPU): one warp
// per edge list; edges [L][64] as (u, v) bytes.
__global__ void orient_kernel(const uint8_t* eu, const uint8_t* ev, const int64_t* off, int64_t L,
                              uint64_t* fbits, int* ok) {
  __shared__ uint64_t inc[4][64];
  __shared__ uint8_t su[4][64], sv[4][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t leaf = (int64_t)blockIdx.x * 4 + warp;
  if (leaf >= L) return;
  int64_t k0 = off[leaf];
  int n = (int)(off[leaf + 1] - k0);
  for (int i = lane; i < n; i += 32) {
    su[warp][i] = eu[k0 + i];
    sv[warp][i] = ev[k0 + i];
  }
  __syncwarp();
  if (lane == 0) {
    // orient() requires a pseudoforest: check with the union-find first
    uint16_t pk[64];
    for (int i = 0; i < n; ++i) pk[i] = (uint16_t)(su[warp][i] | (sv[warp][i] << 8));
    bool pf = pf_accepts(pk, 1, n, n, 0);
    ok[leaf] = pf ? 1 : 0;
    fbits[leaf] = pf ? orient_edges(su[warp], sv[warp], n, inc[warp]) : 0;
  }
}

}  // namespace shk

using namespace shk;

int shk_launch_leaf_search(const ShkLeafLaunch& p, cudaStream_t st) {
  LeafArgs a{};
  a.hi = p.hi;
  a.lo = p.lo;
  a.off = p.off;
  a.L = p.L;
  a.max_seed = p.max_seed;
  a.mode = p.mode;
  a.cache_k = p.cache_k;
  a.cache_min_leaf = p.cache_min_leaf;
  a.seed_out = p.seed_out;
  a.fbits_out = p.fbits_out;
  a.choice_out = p.choice_out;
  a.stats_out = p.stats_out;
  a.counter = p.counter;
  a.error = p.error;
  a.stride = p.stride > 0 ? p.stride : 1;
  a.pre = p.pre;
  a.seed_slot = p.seed_slot;
  a.stats_acc = p.stats_acc;
  a.exhausted = p.exhausted;
  a.place_out = p.place_out;
  if (p.L <= 0) return 0;
  SHK_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(int), st));
  int sms = p.num_sms > 0 ? p.num_sms : 148;
  const bool wide = p.max_n > 32;
  // Team size: spread heavy plain-mode leaves (large n) over more warps so
  // the heavy-tailed per-leaf seed counts do not leave a lone warp running.
  int tw = p.team_warps;
  if (tw <= 0) tw = (p.mode == 0) ? (p.max_n <= 24 ? 1 : (p.max_n <= 40 ? 4 : 8)) : 1;
  int occ = 0;
  // CTAs of 4 warps (TEAMS = 4 / TW independent teams; TW = 8 -> one team).
#define SHK_LEAF_LAUNCH(TW, TEAMS)                                                                  \
  do {                                                                                              \
    void (*kfn)(LeafArgs);                                                                          \
    if (p.mode == 0)                                                                                \
      kfn = wide ? leaf_kernel<TW, TEAMS, true, 0> : leaf_kernel<TW, TEAMS, false, 0>;              \
    else                                                                                            \
      kfn = wide ? leaf_kernel<TW, TEAMS, true, 1> : leaf_kernel<TW, TEAMS, false, 1>;              \
    SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, TW * 32 * TEAMS, 0));        \
    if (occ < 1) occ = 1;                                                                           \
    int64_t blocks = (int64_t)sms * occ;                                                            \
    int64_t need = (p.L + TEAMS - 1) / TEAMS;                                                       \
    if (blocks > need) blocks = need;                                                               \
    kfn<<<(unsigned)blocks, TW * 32 * TEAMS, 0, st>>>(a);                                           \
  } while (0)
  switch (tw) {
    case 1: SHK_LEAF_LAUNCH(1, 4); break;
    case 2: SHK_LEAF_LAUNCH(2, 2); break;
    case 4: SHK_LEAF_LAUNCH(4, 1); break;
    case 8: SHK_LEAF_LAUNCH(8, 1); break;
    default: shk_set_error("team_warps must be 1, 2, 4 or 8"); return 3;
  }
#undef SHK_LEAF_LAUNCH
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_orient(const uint8_t* eu, const uint8_t* ev, const int64_t* off, int64_t L, uint64_t* fbits, int* ok,
                      cudaStream_t st) {
  if (L <= 0) return 0;
  orient_kernel<<<(unsigned)((L + 3) / 4), 128, 0, st>>>(eu, ev, off, L, fbits, ok);
  SHK_LAUNCHED();
  return 0;
}
