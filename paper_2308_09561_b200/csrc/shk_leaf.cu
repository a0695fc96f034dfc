// ShockHash leaf seed search (plain and rotation fitting) + orientation.
//
// Restates _core.pyx:186-229 (search_plain), :232-334 (search_rotate) and
// pseudoforest.py:149-201 (orient) for sm_100a.
//
// Layout: one TEAM of TW warps owns one leaf at a time (leaves are fetched
// dynamically with an atomic counter, so heavy-tailed leaves do not stall a
// whole CTA).  Every lane tests one candidate (a seed for plain search, a base
// seed for rotation fitting); a team round covers TW*32 consecutive
// candidates.  The leaf's keys sit in shared memory and are read with
// broadcast LDS.128, the coverage mask lives in one (n<=32) or two (n>32)
// registers, and lanes whose mask is full run the exact union-find on edges
// they stored in shared memory while hashing.  After each round the team
// takes the lowest accepting candidate, so the result is the reference's
// minimum seed (lexicographic (base, r) minimum for rotation) and the
// counters (evals, passes, checks, a_evals) are the reference's exactly.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

struct LeafArgs {
  const uint64_t* hi;
  const uint64_t* lo;
  const int64_t* off;  // CSR [L+1]; leaf i = keys [off[i], off[i+1])
  int64_t L;
  uint64_t max_seed;
  int mode;             // 0 plain, 1 rotate
  int cache_k;          // rotate: k-aligned A-set seed when m > cache_min_leaf
  int cache_min_leaf;
  int64_t* seed_out;    // [L]
  uint64_t* fbits_out;  // [L] or null
  uint8_t* choice_out;  // [N] per key (CSR order) or null
  int64_t* stats_out;   // [L][4] or null
  int* counter;         // dynamic leaf fetch
  int* error;           // set on internal inconsistency
  int stride;           // key stride in hi/lo (1 separate arrays, 2 interleaved pairs)
  const int64_t* seed_slot;  // optional: seed_out index per leaf
  unsigned long long* stats_acc;  // optional [4] running totals
  int* exhausted;       // optional: set if a leaf has no seed below max_seed
  int64_t* place_out;   // optional [N]: global slot of each key (leaf start + its cell)
};

template <int TW>
struct LeafSmem {
  uint4 keys[64];                 // (hi.lo, hi.hi, lo.lo, lo.hi)
  uint16_t edges[TW][64 * 32];    // per-lane packed edges, column per lane
  int64_t slot_win[2][TW];        // per-warp lowest accepting candidate (or -1)
  int32_t slot_r[2][TW];          // rotation of that candidate
  uint64_t slot_pass_le[2][TW];   // passes at candidates <= winner in warp
  uint64_t slot_pass[2][TW];      // all passes in warp this round
  uint64_t slot_evals_le[2][TW];
  uint64_t slot_evals[2][TW];
  uint64_t slot_aev_le[2][TW];
  uint64_t slot_aev[2][TW];
  uint8_t eu[64], ev[64];
  uint64_t inc[64];
  int64_t leaf;
};

// A CTA holds TEAMS independent teams of TW warps; a team synchronizes on
// its own named barrier (id team+1), so teams never wait for each other.
template <int TW>
SHK_D void team_sync(int team) {
  if (TW == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TW * 32) : "memory");
}

// -------------------------------------------------------------------------
// Plain search body for one candidate seed per lane.
template <bool WIDE>
SHK_D bool plain_mask_full(const uint4* keys, int n, uint64_t s, uint16_t* e, bool store) {
  u2 x = seed_mixer_d(s, TAG_LEAF);
  const uint32_t un = (uint32_t)n, unm1 = (uint32_t)(n - 1);
  uint32_t m0 = 0, m1 = 0;
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    uint4 k = keys[i];
    u2 v = remix_d(u2{k.x, k.y}, u2{k.z, k.w}, x);
    uint32_t h0, h1;
    leaf_pair_d(v, un, unm1, h0, h1);
    if (!WIDE) {
      m0 |= (1u << h0) | (1u << h1);
    } else {
      m0 |= shl_clamp(1u, h0) | shl_clamp(1u, h1);
      m1 |= shl_clamp(1u, h0 - 32u) | shl_clamp(1u, h1 - 32u);
    }
    if (store) e[i * 32] = (uint16_t)(h0 | (h1 << 8));
  }
  if (!WIDE) {
    uint32_t full = (n == 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    return m0 == full;
  } else {
    // WIDE kernels also serve leaves of <= 32 keys in mixed batches
    const uint32_t fulllo = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    const uint32_t fullhi = (n >= 64) ? 0xFFFFFFFFu : (n > 32 ? ((1u << (n - 32)) - 1u) : 0u);
    return m0 == fulllo && m1 == fullhi;
  }
}

template <int TW, int TEAMS, bool WIDE>
__global__ void __launch_bounds__(TW * 32 * TEAMS) leaf_plain_kernel(LeafArgs a) {
  __shared__ LeafSmem<TW> sm_all[TEAMS];
  const int lane = threadIdx.x & 31;
  const int team = (threadIdx.x >> 5) / TW;
  const int warp = (threadIdx.x >> 5) % TW;  // warp within the team
  const int tt = threadIdx.x - team * TW * 32;
  LeafSmem<TW>& sm = sm_all[team];
  uint16_t* e = &sm.edges[warp][lane];
  const bool store = true;
  for (;;) {
    if (tt == 0) sm.leaf = atomicAdd(a.counter, 1);
    team_sync<TW>(team);
    const int64_t leaf = sm.leaf;
    if (leaf >= a.L) break;
    const int64_t k0 = a.off[leaf];
    const int n = (int)(a.off[leaf + 1] - k0);
    for (int i = tt; i < n; i += TW * 32) {
      u2 h = split64(a.hi[(k0 + i) * a.stride]), l = split64(a.lo[(k0 + i) * a.stride]);
      sm.keys[i] = make_uint4(h.lo, h.hi, l.lo, l.hi);
    }
    team_sync<TW>(team);
    int64_t seed = -1;
    uint64_t passes = 0;
    if (n <= 1) {
      seed = 0;
      passes = 1;
    } else {
      // Rounds of TW*32 consecutive seeds; warp w owns [R + 32w, R + 32w + 32).
      int par = 0;
      for (uint64_t R = 0; R < a.max_seed; R += (uint64_t)TW * 32, par ^= 1) {
        const uint64_t s = R + (uint64_t)warp * 32 + lane;
        const bool valid = s < a.max_seed;
        bool full = valid && plain_mask_full<WIDE>(sm.keys, n, s, e, store);
        unsigned pb = __ballot_sync(FULL_WARP, full);
        bool acc = false;
        if (full) acc = pf_accepts(e, 32, n, n, 0);
        unsigned ab = __ballot_sync(FULL_WARP, acc);
        if (lane == 0) {
          int w = ab ? __ffs(ab) - 1 : 32;
          unsigned le = (w == 32) ? pb : (pb & (0xFFFFFFFFu >> (31 - w)));
          sm.slot_win[par][warp] = ab ? (int64_t)(R + (uint64_t)warp * 32 + w) : -1;
          sm.slot_pass_le[par][warp] = __popc(le);
          sm.slot_pass[par][warp] = __popc(pb);
        }
        team_sync<TW>(team);
        int64_t win = -1;
        uint64_t round_pass = 0;
#pragma unroll
        for (int w = 0; w < TW; ++w) {
          if (win < 0) {
            int64_t sw = sm.slot_win[par][w];
            if (sw >= 0) {
              win = sw;
              round_pass += sm.slot_pass_le[par][w];
            } else {
              round_pass += sm.slot_pass[par][w];
            }
          }
        }
        passes += round_pass;
        if (win >= 0) {
          seed = win;
          break;
        }
      }
    }
    // Orientation of the winning seed (one leaf, tiny): warp 0.
    if (warp == 0) {
      if (seed >= 0 && n >= 2) {
        for (int i = lane; i < n; i += 32) {
          uint4 k = sm.keys[i];
          u2 v = remix_d(u2{k.x, k.y}, u2{k.z, k.w}, seed_mixer_d((uint64_t)seed, TAG_LEAF));
          uint32_t h0, h1;
          leaf_pair_d(v, (uint32_t)n, (uint32_t)(n - 1), h0, h1);
          sm.eu[i] = (uint8_t)h0;
          sm.ev[i] = (uint8_t)h1;
        }
        __syncwarp();
        uint64_t f = 0;
        if (lane == 0) f = orient_edges(sm.eu, sm.ev, n, sm.inc);
        f = __shfl_sync(FULL_WARP, f, 0);
        if (lane == 0) {
          if (a.fbits_out) a.fbits_out[leaf] = f;
        }
        if (a.choice_out)
          for (int i = lane; i < n; i += 32) a.choice_out[k0 + i] = (uint8_t)((f >> i) & 1);
        if (a.place_out)
          for (int i = lane; i < n; i += 32) a.place_out[k0 + i] = k0 + (((f >> i) & 1) ? sm.ev[i] : sm.eu[i]);
      } else if (lane == 0) {
        if (a.fbits_out) a.fbits_out[leaf] = 0;
        if (a.choice_out && n == 1) a.choice_out[k0] = 0;
        if (a.place_out && n == 1) a.place_out[k0] = k0;
      }
      if (lane == 0) {
        a.seed_out[a.seed_slot ? a.seed_slot[leaf] : leaf] = seed;
        uint64_t evals = (n <= 1) ? 1 : (seed >= 0 ? ((uint64_t)seed + 1) * n : a.max_seed * (uint64_t)n);
        if (a.stats_out) {
          int64_t* st = a.stats_out + 4 * leaf;
          st[0] = (int64_t)evals;
          st[1] = (int64_t)passes;
          st[2] = (int64_t)passes;
          st[3] = 0;
        }
        if (a.stats_acc) {
          atomicAdd(&a.stats_acc[0], (unsigned long long)evals);
          atomicAdd(&a.stats_acc[1], (unsigned long long)passes);
          atomicAdd(&a.stats_acc[2], (unsigned long long)passes);
        }
        if (seed < 0 && a.exhausted) atomicOr(a.exhausted, 1);
      }
    }
    team_sync<TW>(team);
  }
}

// -------------------------------------------------------------------------
// Rotation fitting: lane per base seed.
template <int TW, int TEAMS, bool WIDE>
__global__ void __launch_bounds__(TW * 32 * TEAMS) leaf_rotate_kernel(LeafArgs a) {
  __shared__ LeafSmem<TW> sm_all[TEAMS];
  const int lane = threadIdx.x & 31;
  const int team = (threadIdx.x >> 5) / TW;
  const int warp = (threadIdx.x >> 5) % TW;  // warp within the team
  const int tt = threadIdx.x - team * TW * 32;
  LeafSmem<TW>& sm = sm_all[team];
  uint16_t* e = &sm.edges[warp][lane];
  for (;;) {
    if (tt == 0) sm.leaf = atomicAdd(a.counter, 1);
    team_sync<TW>(team);
    const int64_t leaf = sm.leaf;
    if (leaf >= a.L) break;
    const int64_t k0 = a.off[leaf];
    const int n = (int)(a.off[leaf + 1] - k0);
    const int64_t ck = (n > a.cache_min_leaf) ? a.cache_k : 0;
    for (int i = tt; i < n; i += TW * 32) {
      u2 h = split64(a.hi[(k0 + i) * a.stride]), l = split64(a.lo[(k0 + i) * a.stride]);
      sm.keys[i] = make_uint4(h.lo, h.hi, l.lo, l.hi);
    }
    team_sync<TW>(team);
    int64_t q = -1;
    uint64_t passes = 0, evals = 0, aev = 0;
    if (n <= 1) {
      q = 0;
      passes = 1;
      evals = 1;
    } else {
      const uint64_t max_base = a.max_seed / (uint64_t)n + 1;
      const uint32_t un = (uint32_t)n, unm1 = (uint32_t)(n - 1);
      int par = 0;
      for (uint64_t R = 0; R < max_base; R += (uint64_t)TW * 32, par ^= 1) {
        const uint64_t base = R + (uint64_t)warp * 32 + lane;
        const bool valid = base < max_base;
        uint64_t passmask = 0;
        int win_r = -1;
        uint32_t na = 0;
        bool ws = false;
        if (valid) {
          const uint64_t sa = ck ? base - base % (uint64_t)ck : base;
          ws = (base == 0) || (ck == 0) || (base % (uint64_t)ck == 0);
          const u2 xb = seed_mixer_d(sa, TAG_SPLITBIT);
          const u2 xa = seed_mixer_d(sa, TAG_LEAF);
          const u2 xg = seed_mixer_d(base, TAG_LEAF);
          uint32_t ma0 = 0, ma1 = 0, mb0 = 0, mb1 = 0;
#pragma unroll 2
          for (int i = 0; i < n; ++i) {
            uint4 k = sm.keys[i];
            u2 kh{k.x, k.y}, kl{k.z, k.w};
            uint32_t bit = remix_top_d(kh, kl, xb);
            u2 x;
            x.lo = bit ? xg.lo : xa.lo;
            x.hi = bit ? xg.hi : xa.hi;
            u2 v = remix_d(kh, kl, x);
            uint32_t h0, h1;
            leaf_pair_d(v, un, unm1, h0, h1);
            uint32_t c0, c1 = 0;
            if (!WIDE) {
              c0 = (1u << h0) | (1u << h1);
            } else {
              c0 = shl_clamp(1u, h0) | shl_clamp(1u, h1);
              c1 = shl_clamp(1u, h0 - 32u) | shl_clamp(1u, h1 - 32u);
            }
            if (bit) {
              mb0 |= c0;
              mb1 |= c1;
            } else {
              ma0 |= c0;
              ma1 |= c1;
            }
            na += bit ^ 1u;
            e[i * 32] = (uint16_t)(h0 | (h1 << 8) | (bit << 15));
          }
          // Rotation filter: (mask_a | rotl_n(mask_b, r)) == full.
          if (!WIDE) {
            const uint32_t full = (n == 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
            const uint32_t need = ~ma0 & full;
            const uint64_t D = (uint64_t)mb0 | ((uint64_t)mb0 << n);
            for (int r = 0; r < n; ++r) {
              uint32_t rot = (uint32_t)(D >> (n - r));
              if ((need & ~rot) == 0) passmask |= 1ull << r;
            }
          } else {
            const uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
            const uint64_t ma = join64(ma0, ma1), mb = join64(mb0, mb1);
            const uint64_t need = ~ma & full;
            for (int r = 0; r < n; ++r) {
              uint64_t rot = r ? (((mb << r) | (mb >> (n - r))) & full) : mb;
              if ((need & ~rot) == 0) passmask |= 1ull << r;
            }
          }
          uint64_t pm = passmask;
          while (pm) {
            int r = __ffsll((long long)pm) - 1;
            pm &= pm - 1;
            if (pf_accepts(e, 32, n, n, r)) {
              win_r = r;
              break;
            }
          }
        }
        const uint32_t nb = (uint32_t)n - na;
        const uint64_t my_ev = valid ? (uint64_t)nb + (ws ? (uint64_t)n + na : 0) : 0;
        const uint64_t my_aev = (valid && ws) ? na : 0;
        const uint64_t my_pass = __popcll(passmask);
        uint64_t my_pass_le = my_pass;
        if (win_r >= 0) my_pass_le = __popcll(passmask & ((win_r == 63) ? ~0ull : ((2ull << win_r) - 1)));
        unsigned ab = __ballot_sync(FULL_WARP, win_r >= 0);
        int wl = ab ? __ffs(ab) - 1 : 32;
        // Inclusive sums over lanes <= wl (winner) and over all lanes.
        uint64_t c_ev_le = (lane < wl || lane == wl) ? my_ev : 0;
        uint64_t c_aev_le = (lane <= wl) ? my_aev : 0;
        uint64_t c_pass_le = (lane < wl) ? my_pass : (lane == wl ? my_pass_le : 0);
        uint64_t t_ev = warp_sum(my_ev), t_aev = warp_sum(my_aev), t_pass = warp_sum(my_pass);
        c_ev_le = warp_sum(c_ev_le);
        c_aev_le = warp_sum(c_aev_le);
        c_pass_le = warp_sum(c_pass_le);
        int wr = __shfl_sync(FULL_WARP, win_r, wl & 31);
        if (lane == 0) {
          sm.slot_win[par][warp] = ab ? (int64_t)(R + (uint64_t)warp * 32 + wl) : -1;
          sm.slot_r[par][warp] = wr;
          sm.slot_pass_le[par][warp] = c_pass_le;
          sm.slot_pass[par][warp] = t_pass;
          sm.slot_evals_le[par][warp] = c_ev_le;
          sm.slot_evals[par][warp] = t_ev;
          sm.slot_aev_le[par][warp] = c_aev_le;
          sm.slot_aev[par][warp] = t_aev;
        }
        team_sync<TW>(team);
        int64_t winb = -1;
        int winr = 0;
#pragma unroll
        for (int w = 0; w < TW; ++w) {
          if (winb < 0) {
            int64_t sw = sm.slot_win[par][w];
            if (sw >= 0) {
              winb = sw;
              winr = sm.slot_r[par][w];
              passes += sm.slot_pass_le[par][w];
              evals += sm.slot_evals_le[par][w];
              aev += sm.slot_aev_le[par][w];
            } else {
              passes += sm.slot_pass[par][w];
              evals += sm.slot_evals[par][w];
              aev += sm.slot_aev[par][w];
            }
          }
        }
        if (winb >= 0) {
          uint64_t qq = (uint64_t)winb * (uint64_t)n + (uint64_t)winr;
          q = (qq >= a.max_seed) ? -1 : (int64_t)qq;
          break;
        }
      }
    }
    if (warp == 0) {
      if (q >= 0 && n >= 2) {
        const uint64_t base = (uint64_t)q / (uint64_t)n;
        const int r = (int)((uint64_t)q % (uint64_t)n);
        const uint64_t sa = ck ? base - base % (uint64_t)ck : base;
        const u2 xb = seed_mixer_d(sa, TAG_SPLITBIT), xa = seed_mixer_d(sa, TAG_LEAF), xg = seed_mixer_d(base, TAG_LEAF);
        for (int i = lane; i < n; i += 32) {
          uint4 k = sm.keys[i];
          u2 kh{k.x, k.y}, kl{k.z, k.w};
          uint32_t bit = remix_top_d(kh, kl, xb);
          u2 v = remix_d(kh, kl, bit ? xg : xa);
          uint32_t h0, h1;
          leaf_pair_d(v, (uint32_t)n, (uint32_t)(n - 1), h0, h1);
          if (bit) {
            h0 = (h0 + r) % n;
            h1 = (h1 + r) % n;
          }
          sm.eu[i] = (uint8_t)h0;
          sm.ev[i] = (uint8_t)h1;
        }
        __syncwarp();
        uint64_t f = 0;
        if (lane == 0) f = orient_edges(sm.eu, sm.ev, n, sm.inc);
        f = __shfl_sync(FULL_WARP, f, 0);
        if (lane == 0 && a.fbits_out) a.fbits_out[leaf] = f;
        if (a.choice_out)
          for (int i = lane; i < n; i += 32) a.choice_out[k0 + i] = (uint8_t)((f >> i) & 1);
        if (a.place_out)
          for (int i = lane; i < n; i += 32) a.place_out[k0 + i] = k0 + (((f >> i) & 1) ? sm.ev[i] : sm.eu[i]);
      } else if (lane == 0) {
        if (a.fbits_out) a.fbits_out[leaf] = 0;
        if (a.choice_out && n == 1) a.choice_out[k0] = 0;
        if (a.place_out && n == 1) a.place_out[k0] = k0;
      }
      if (lane == 0) {
        a.seed_out[a.seed_slot ? a.seed_slot[leaf] : leaf] = q;
        if (a.stats_out) {
          int64_t* st = a.stats_out + 4 * leaf;
          st[0] = (int64_t)evals;
          st[1] = (int64_t)passes;
          st[2] = (int64_t)passes;
          st[3] = (int64_t)aev;
        }
        if (a.stats_acc) {
          atomicAdd(&a.stats_acc[0], (unsigned long long)evals);
          atomicAdd(&a.stats_acc[1], (unsigned long long)passes);
          atomicAdd(&a.stats_acc[2], (unsigned long long)passes);
          atomicAdd(&a.stats_acc[3], (unsigned long long)aev);
        }
        if (q < 0 && a.exhausted) atomicOr(a.exhausted, 1);
      }
    }
    team_sync<TW>(team);
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
    // Pseudoforest check first (orient requires one): reuse the UF with
    // packed edges in a small local buffer.
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
  LeafArgs a;
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
  a.seed_slot = p.seed_slot;
  a.stats_acc = p.stats_acc;
  a.exhausted = p.exhausted;
  a.place_out = p.place_out;
  if (p.L <= 0) return 0;
  SHK_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(int), st));
  int sms = p.num_sms > 0 ? p.num_sms : 148;
  const bool wide = p.max_n > 32;
  // Team size: spread heavy leaves (large n) over more warps so the
  // heavy-tailed per-leaf seed counts do not leave a lone warp running.
  int tw = p.team_warps;
  if (tw <= 0) {
    if (p.mode == 0)
      tw = p.max_n <= 24 ? 1 : (p.max_n <= 40 ? 4 : 8);
    else
      tw = p.max_n <= 24 ? 1 : 1;
  }
  int occ = 0;
  // CTAs of 4 warps (TEAMS = 4 / TW independent teams; TW = 8 -> one team).
#define SHK_LEAF_LAUNCH(TW, TEAMS)                                                               \
  do {                                                                                           \
    void (*kfn)(LeafArgs);                                                                       \
    if (p.mode == 0)                                                                             \
      kfn = wide ? leaf_plain_kernel<TW, TEAMS, true> : leaf_plain_kernel<TW, TEAMS, false>;     \
    else                                                                                         \
      kfn = wide ? leaf_rotate_kernel<TW, TEAMS, true> : leaf_rotate_kernel<TW, TEAMS, false>;   \
    SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, TW * 32 * TEAMS, 0));     \
    if (occ < 1) occ = 1;                                                                        \
    int64_t blocks = (int64_t)sms * occ;                                                         \
    int64_t need = (p.L + TEAMS - 1) / TEAMS;                                                    \
    if (blocks > need) blocks = need;                                                            \
    kfn<<<(unsigned)blocks, TW * 32 * TEAMS, 0, st>>>(a);                                        \
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
