// ShockHash leaf seed search (plain and rotation fitting) + orientation, as
// team-level device functions shared by the batched leaf kernels
// (shk_leaf.cu) and the persistent construction kernel (shk_tree.cu).
//
// Restates _core.pyx:186-229 (search_plain), :232-334 (search_rotate) and
// pseudoforest.py:149-201 (orient) for sm_100a.
//
// A TEAM of TW warps owns one leaf.  Every lane tests one candidate (a seed
// for plain search, a base seed for rotation fitting); a team round covers
// TW*32 consecutive candidates.  The leaf's keys sit in shared memory and are
// read with broadcast LDS.128, the coverage masks live in registers, and
// every lane stores its candidate's edges in shared memory while hashing.
// Candidates that pass the coverage filter get the exact pseudoforest check
// warp-cooperatively (warp_first_accept, in (lane, r) order).  After each
// round the team takes the lowest accepting candidate, so the result is the
// reference's minimum seed (lexicographic (base, r) minimum for rotation)
// and the counters (evals, passes, checks, a_evals) are the reference's.
#pragma once
#include "shk_common.cuh"

namespace shk {

struct ShkHandoff;

struct LeafArgs {
  const uint64_t* hi;
  const uint64_t* lo;
  const int64_t* off;  // CSR [L+1]; leaf i = keys [off[i], off[i+1])
  int64_t L;
  uint64_t max_seed;
  int mode;             // 0 plain, 1 rotate
  int cache_k;          // rotate: k-aligned A-set seed when m > cache_min_leaf
  int cache_min_leaf;
  int64_t* seed_out;    // [L] (or indexed by seed_slot)
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
  int pre;              // hi words are already premix_hi'ed (build path)
  // Tail hand-off of the persistent construction kernel (shk_tree.cu), rotate
  // search with one-warp teams only: once abort_flag is set, a warp ends its
  // leaf after the current round and records where the search stands; the
  // resume kernel finishes the recorded leaves with multi-warp teams.
  const int* abort_flag;               // optional
  ShkHandoff* handoff;                 // [capacity]
  unsigned long long* handoff_count;
};

// A leaf search stopped at a round boundary: every base below `next_base` is
// searched (no acceptance), the counters cover exactly those bases.
struct ShkHandoff {
  int64_t seed_slot;
  int64_t k0;
  uint64_t next_base;
  uint64_t evals, passes, aev;
  int32_t n;
  int32_t pad;
};

// MAXE: most keys per leaf the team's buffers hold (64, or 40 to fit more
// warps per SM when the build's leaves are small enough).
template <int TW, int MAXE = 64>
struct LeafSmem {
  uint4 keys[MAXE];               // (hp.lo, hp.hi, lo.lo, lo.hi), hp = premix_hi(hi)
  uint16_t edges[TW][MAXE * 32];  // per-lane packed edges, column per lane
  int64_t slot_win[2][TW];        // per-warp lowest accepting candidate (or -1)
  int32_t slot_r[2][TW];          // rotation of that candidate
  uint64_t slot_pass_le[2][TW];   // passes at candidates <= winner in warp
  uint64_t slot_pass[2][TW];      // all passes in warp this round
  uint64_t slot_evals_le[2][TW];
  uint64_t slot_evals[2][TW];
  uint64_t slot_aev_le[2][TW];
  uint64_t slot_aev[2][TW];
  uint8_t eu[MAXE], ev[MAXE];
  uint64_t inc[MAXE];
  WarpChk chk[TW];                // per-warp scratch of the exact check
  int64_t leaf;
};

// A CTA holds independent teams of TW warps; a team synchronizes on its own
// named barrier (id team+1), so teams never wait for each other.
template <int TW>
SHK_D void team_sync(int team) {
  if (TW == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TW * 32) : "memory");
}

// Where a solved leaf writes its results.
struct LeafOut {
  int64_t seed_slot;   // index into a.seed_out
  int64_t leaf_index;  // index into fbits_out / stats_out (or -1)
};

template <int TW, class SM>
SHK_D void load_leaf_keys(const LeafArgs& a, SM& sm, int64_t k0, int n, int tt) {
  for (int i = tt; i < n; i += TW * 32) {
    const uint64_t hw = a.hi[(k0 + i) * a.stride];
    u2 h = split64(a.pre ? hw : premix_hi(hw)), l = split64(a.lo[(k0 + i) * a.stride]);
    sm.keys[i] = make_uint4(h.lo, h.hi, l.lo, l.hi);
  }
}

// Orientation of the final edges in sm.eu/sm.ev (warp 0 of the team) and
// result stores.
template <int TW, class SM>
SHK_D void leaf_finish(const LeafArgs& a, SM& sm, int64_t k0, int n, int64_t q, const LeafOut& o,
                       uint64_t evals, uint64_t passes, uint64_t aev, int lane) {
  if (q >= 0 && n >= 2) {
    __syncwarp();
    uint64_t f = 0;
    if (lane == 0) f = orient_edges(sm.eu, sm.ev, n, sm.inc);
    f = __shfl_sync(FULL_WARP, f, 0);
    if (lane == 0 && a.fbits_out && o.leaf_index >= 0) a.fbits_out[o.leaf_index] = f;
    if (a.choice_out)
      for (int i = lane; i < n; i += 32) a.choice_out[k0 + i] = (uint8_t)((f >> i) & 1);
    if (a.place_out)
      for (int i = lane; i < n; i += 32) a.place_out[k0 + i] = k0 + (((f >> i) & 1) ? sm.ev[i] : sm.eu[i]);
  } else if (lane == 0) {
    if (a.fbits_out && o.leaf_index >= 0) a.fbits_out[o.leaf_index] = 0;
    if (a.choice_out && n == 1) a.choice_out[k0] = 0;
    if (a.place_out && n == 1) a.place_out[k0] = k0;
  }
  if (lane == 0) {
    a.seed_out[o.seed_slot] = q;
    if (a.stats_out && o.leaf_index >= 0) {
      int64_t* st = a.stats_out + 4 * o.leaf_index;
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

// -------------------------------------------------------------------------
// Edge columns of the lanes in `lanes` (their seeds s): the warp recomputes
// them cooperatively (lane i hashes keys i, i+32) instead of every lane
// storing its edges for every seed; only filter-passing seeds need them.
SHK_D void plain_fill_edges(const uint4* keys, int n, uint64_t s, unsigned lanes, uint16_t* ew, int lane) {
  while (lanes) {
    const int L = __ffs(lanes) - 1;
    lanes &= lanes - 1;
    const uint64_t sl = __shfl_sync(FULL_WARP, s, L);
    const u2 x = seed_mixer_pre_d(sl, TAG_LEAF);
    for (int i = lane; i < n; i += 32) {
      const uint4 k = keys[i];
      uint32_t h0, h1;
      leaf_pair_d(remix_pre_d(u2{k.x, k.y}, u2{k.z, k.w}, x), (uint32_t)n, (uint32_t)(n - 1), h0, h1);
      ew[i * 32 + L] = (uint16_t)(h0 | (h1 << 8));
    }
  }
  __syncwarp();
}

// Plain search body for one candidate seed per lane (STORE: also write the
// lane's edge column).
// remix_pre_d's shift placement (AM) in the plain search's filter loop.  The
// loop is FMA-pipe bound with every high-word shift on IMAD.HI (ncu: C3
// fmaheavy 83% / ALU 63%, C5 fmaheavy 85% / ALU 63%), so all five shifts go
// to the ALU pipe (tools/ab_leaf.sh: C3 26.0 -> 25.5 ms; C5 13.03-13.08 ->
// 12.82-12.92 s).  The rotate search in the build was left on the FMA
// placement in round 1 (the tree kernel is ALU-heavier overall); measured
// again once IMAD.HI was known to take two FMA issue slots, it is faster with
// the shifts on the ALU pipe too (SHK_ROT_SHIFT_MASK below).
// Re-swept for the stealing kernel (ncu C3: ALU 76%, fmaheavy 64%): C3 best
// with shift 4 on the FMA pipe (0x0F: 23.62 vs 23.93 ms), C5 with shifts 1
// and 3 there (0x15: 11.20 vs 11.41 s); all-FMA (0x00) is the slowest.
#ifndef SHK_PLAIN_SHIFT_MASK
#define SHK_PLAIN_SHIFT_MASK 0x0F
#endif
#ifndef SHK_PLAIN_SHIFT_MASK_WIDE
#define SHK_PLAIN_SHIFT_MASK_WIDE 0x15
#endif
// SHK_PLAIN_ONEHOT_LDS: the cells' one-hots come from a 64-entry (lo, hi)
// shared-memory table `tab` (LSU) instead of shifts on the ALU pipe (as in the
// rotation search); tab == nullptr keeps the shifts.
#ifndef SHK_PLAIN_ONEHOT_LDS
#define SHK_PLAIN_ONEHOT_LDS 1
#endif
// Fill a 64-entry one-hot table (the calling warp's lanes; same values from
// every warp of the CTA, so concurrent fills are benign).
SHK_D void fill_onehot_tab(uint2* tab, int lane) {
  for (int h = lane; h < 64; h += 32) tab[h] = make_uint2(h < 32 ? 1u << h : 0u, h < 32 ? 0u : 1u << (h - 32));
  __syncwarp();
}
template <bool WIDE, bool STORE = true>
SHK_D bool plain_mask_full(const uint4* keys, int n, uint64_t s, uint16_t* e, const uint2* tab = nullptr) {
  u2 x = seed_mixer_pre_d(s, TAG_LEAF);
  const uint32_t un = (uint32_t)n, unm1 = (uint32_t)(n - 1);
  uint32_t m0 = 0, m1 = 0;
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    uint4 k = keys[i];
    u2 v = remix_pre_d<WIDE ? SHK_PLAIN_SHIFT_MASK_WIDE : SHK_PLAIN_SHIFT_MASK>(u2{k.x, k.y}, u2{k.z, k.w}, x);
    uint32_t h0, h1;
    leaf_pair_d(v, un, unm1, h0, h1);
    if (SHK_PLAIN_ONEHOT_LDS && tab) {
      const uint2 t0 = tab[h0], t1 = tab[h1];
      m0 |= t0.x | t1.x;
      if (WIDE) m1 |= t0.y | t1.y;
    } else if (!WIDE) {
      m0 |= (1u << h0) | (1u << h1);
    } else {
      m0 |= shl_clamp(1u, h0) | shl_clamp(1u, h1);
      m1 |= shl_clamp(1u, h0 - 32u) | shl_clamp(1u, h1 - 32u);
    }
    if (STORE) e[i * 32] = (uint16_t)(h0 | (h1 << 8));
  }
  if (!WIDE) {
    uint32_t full = (n == 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    return m0 == full;
  } else {
    // WIDE code also serves leaves of <= 32 keys in mixed batches
    const uint32_t fulllo = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    const uint32_t fullhi = (n >= 64) ? 0xFFFFFFFFu : (n > 32 ? ((1u << (n - 32)) - 1u) : 0u);
    return m0 == fulllo && m1 == fullhi;
  }
}

// Plain search of one leaf (keys [k0, k0+n)) by a team.  All threads of the
// team call it; it ends team-synchronized.
template <int TW, bool WIDE, class SM>
SHK_D void solve_plain(const LeafArgs& a, SM& sm, int64_t k0, int n, const LeafOut& o, int team, int warp,
                       int lane, int tt) {
  load_leaf_keys<TW>(a, sm, k0, n, tt);
  team_sync<TW>(team);
  uint16_t* e = &sm.edges[warp][lane];
  int64_t seed = -1;
  uint64_t passes = 0;
  if (n <= 1) {
    seed = 0;
    passes = 1;
  } else {
    __shared__ uint2 plain_tab[64];  // SHK_PLAIN_ONEHOT_LDS (one per CTA)
    if (SHK_PLAIN_ONEHOT_LDS) fill_onehot_tab(plain_tab, lane);
    // Rounds of TW*32 consecutive seeds; warp w owns [R + 32w, R + 32w + 32).
    int par = 0;
    for (uint64_t R = 0; R < a.max_seed; R += (uint64_t)TW * 32, par ^= 1) {
      const uint64_t s = R + (uint64_t)warp * 32 + lane;
      const bool valid = s < a.max_seed;
      bool full = valid && plain_mask_full<WIDE, false>(sm.keys, n, s, e, SHK_PLAIN_ONEHOT_LDS ? plain_tab : nullptr);
      unsigned pb = __ballot_sync(FULL_WARP, full);
      if (pb) plain_fill_edges(sm.keys, n, s, pb, sm.edges[warp], lane);
      const bool acc = warp_first_accept(sm.edges[warp], full ? 1ull : 0ull, n, lane, sm.chk[warp]) == 0;
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
  if (warp == 0) {
    if (seed >= 0 && n >= 2) {
      const u2 x = seed_mixer_pre_d((uint64_t)seed, TAG_LEAF);
      for (int i = lane; i < n; i += 32) {
        uint4 k = sm.keys[i];
        u2 v = remix_pre_d(u2{k.x, k.y}, u2{k.z, k.w}, x);
        uint32_t h0, h1;
        leaf_pair_d(v, (uint32_t)n, (uint32_t)(n - 1), h0, h1);
        sm.eu[i] = (uint8_t)h0;
        sm.ev[i] = (uint8_t)h1;
      }
    }
    const uint64_t evals = (n <= 1) ? 1 : (seed >= 0 ? ((uint64_t)seed + 1) * n : a.max_seed * (uint64_t)n);
    leaf_finish<TW>(a, sm, k0, n, seed, o, evals, passes, 0, lane);
  }
  team_sync<TW>(team);
}

// Cells of one key in the rotation search: OR its two cells into the A or B
// coverage mask (bit = split bit, 1 = B) and store its packed edge.
// High-word shift placement of the rotation search's two remixes per key
// (bit i: xor-shift i on the ALU pipe, else IMAD.HI on the FMA pipe; see
// remix_pre_d / remix_top_pre_d).  IMAD.HI takes two FMA issue slots
// (tools/int_peak.py), which made the rotation loop FMA-bound: all nine shifts
// on the ALU pipe measured C4 99.06 -> 98.17 ms (20-step A/Bs; one, two, five
// and four of them in between), and eight of them (the cells remix's first
// shift back on IMAD.HI) 98.31 -> 98.11 ms over 4 pairs; other single or
// double moves back measured equal or slower.
#ifndef SHK_ROT_SHIFT_MASK
#define SHK_ROT_SHIFT_MASK 0x1E
#endif
#ifndef SHK_ROT_TOP_SHIFT_MASK
#define SHK_ROT_TOP_SHIFT_MASK 0xF
#endif
#ifndef SHK_ROT_UNROLL
#define SHK_ROT_UNROLL 3  // keys per iteration of the rotate filter loop (independent hash chains); 3 vs 4: -0.2 ms (C4, 4 A/B pairs)
#endif
constexpr int kRotUnroll = SHK_ROT_UNROLL;
// SHK_ROT_MASK_LDS: the 64-bit one-hots of the two cells come from a
// shared-memory table (LSU pipe) instead of shifts and XORs on the ALU pipe,
// which the rotation loop saturates.  The table is indexed by (split bit,
// cell) and holds the one-hot already placed in the A or the B half of a
// 4-word (ma0, ma1, mb0, mb1) record, so a key's cells OR straight into the
// masks (two LDS.128, four 3-input ORs; no select).  One table per CTA.
// (A (lo, hi) one-hot table with the A/B select kept measured half the gain.)
#ifndef SHK_ROT_MASK_LDS
#define SHK_ROT_MASK_LDS 1
#endif
#ifndef SHK_ROT_FMA_BOOK
#define SHK_ROT_FMA_BOOK 1
#endif
// a * b + c as one IMAD (written in PTX so it stays on the FMA pipe)
SHK_D uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
template <bool WIDE>
SHK_D void rot_key_cells(u2 v, uint32_t un, uint32_t unm1, uint32_t bit, uint32_t& ma0, uint32_t& ma1,
                         uint32_t& mb0, uint32_t& mb1, uint32_t& na, uint16_t* e, const uint2* onehot = nullptr) {
  uint32_t h0, h1;
  leaf_pair_d(v, un, unm1, h0, h1);
  const uint32_t sel = 0u - bit;  // all ones for B
  uint32_t c0, c1 = 0;
  if (!WIDE) {
    c0 = (1u << h0) | (1u << h1);
  } else if (SHK_ROT_MASK_LDS && onehot) {
    const uint4* t4 = reinterpret_cast<const uint4*>(onehot) + (bit << 6);
    const uint4 t0 = t4[h0], t1 = t4[h1];
    ma0 |= t0.x | t1.x;
    ma1 |= t0.y | t1.y;
    mb0 |= t0.z | t1.z;
    mb1 |= t0.w | t1.w;
#if SHK_ROT_FMA_BOOK
    // (table path) na counts the B keys here (the caller turns it into the A
    // count after the loop) and the edge is packed with multiply-adds: the
    // bookkeeping runs on the FMA pipe, the ALU pipe being the bound
    na = imad_u32(bit, 1u, na);
    *e = (uint16_t)imad_u32(bit, 0x8000u, imad_u32(h1, 0x100u, h0));
#else
    na += bit ^ 1u;
    *e = (uint16_t)(h0 | (h1 << 8) | (bit << 15));
#endif
    return;
  } else {
    // 64-bit one-hots: low word clamps to 0 for h >= 32, and the wrapped
    // shift (h mod 32) differs from it exactly when h >= 32
    const uint32_t l0 = shl_clamp(1u, h0), l1 = shl_clamp(1u, h1);
    c0 = l0 | l1;
    c1 = (shl_wrap(1u, h0) ^ l0) | (shl_wrap(1u, h1) ^ l1);
  }
  mb0 |= c0 & sel;
  ma0 |= c0 & ~sel;
  if (WIDE) {
    mb1 |= c1 & sel;
    ma1 |= c1 & ~sel;
  }
  na += bit ^ 1u;
  *e = (uint16_t)(h0 | (h1 << 8) | (bit << 15));
}

// Rotation fitting of one leaf: lane per base seed.
#ifndef SHK_HANDOFF_EVERY
// rounds between abort-flag checks (power of two; 1 and 4 measured equal at C4,
// and the flag load placed at the top of a round or folded into the winner's
// exit measured slower: the hot loop's schedule moves)
#define SHK_HANDOFF_EVERY 1
#endif
// HANDOFF (one-warp teams): check a.abort_flag after every round without an
// acceptance and hand the leaf off if it is set.  Resume: start at base R0
// with the counters of the bases below it.
template <int TW, bool WIDE, bool HANDOFF = false, class SM>
SHK_D void solve_rotate(const LeafArgs& a, SM& sm, int64_t k0, int n, const LeafOut& o, int team,
                        int warp, int lane, int tt, uint64_t R0 = 0, uint64_t ev0 = 0, uint64_t pass0 = 0,
                        uint64_t aev0 = 0) {
  load_leaf_keys<TW>(a, sm, k0, n, tt);
  __shared__ uint4 rot_tab[128];  // SHK_ROT_MASK_LDS: (bit << 6 | h) -> (ma0, ma1, mb0, mb1) one-hot, per CTA
  const uint2* onehot_tab = nullptr;
  if (WIDE && SHK_ROT_MASK_LDS) {
    // every team writes the same values (benign) before its search
    for (int k = tt; k < 128; k += TW * 32) {
      const int h = k & 63;
      const uint32_t lo = h < 32 ? 1u << h : 0u, hi = h < 32 ? 0u : 1u << (h - 32);
      rot_tab[k] = (k >> 6) ? make_uint4(0u, 0u, lo, hi) : make_uint4(lo, hi, 0u, 0u);
    }
    onehot_tab = reinterpret_cast<const uint2*>(rot_tab);
  }
  team_sync<TW>(team);
  uint16_t* e = &sm.edges[warp][lane];
  const int64_t ck = (n > a.cache_min_leaf) ? a.cache_k : 0;
  int64_t q = -1;
  uint64_t passes = pass0, evals = ev0, aev = aev0;
  uint64_t stop_at = 0;  // HANDOFF: next base of a search stopped by the abort flag (0: not stopped)
  if (n <= 1) {
    q = 0;
    passes = 1;
    evals = 1;
  } else {
    const uint64_t max_base = a.max_seed / (uint64_t)n + 1;
    const uint32_t un = (uint32_t)n, unm1 = (uint32_t)(n - 1);
    int par = 0;
    for (uint64_t R = R0; R < max_base; R += (uint64_t)TW * 32, par ^= 1) {
      const uint64_t base = R + (uint64_t)warp * 32 + lane;
      const bool valid = base < max_base;
      uint64_t passmask = 0;
      uint32_t na = 0;
      bool ws = false;
      if (valid) {
        const uint64_t sa = ck ? base - base % (uint64_t)ck : base;
        ws = (base == 0) || (ck == 0) || (base % (uint64_t)ck == 0);
        const u2 xb = seed_mixer_pre_d(sa, TAG_SPLITBIT);
        const u2 xg = seed_mixer_pre_d(base, TAG_LEAF);
        uint32_t ma0 = 0, ma1 = 0, mb0 = 0, mb1 = 0;
        if (ck == 0) {  // A and B keys share the leaf seed (sa == base)
#pragma unroll kRotUnroll
          for (int i = 0; i < n; ++i) {
            const uint4 k = sm.keys[i];
            const u2 kh{k.x, k.y}, kl{k.z, k.w};
            const uint32_t bit = remix_top_pre_d<SHK_ROT_TOP_SHIFT_MASK>(kh, kl, xb);
            rot_key_cells<WIDE>(remix_pre_d<SHK_ROT_SHIFT_MASK>(kh, kl, xg), un, unm1, bit, ma0, ma1, mb0, mb1, na,
                                e + i * 32, onehot_tab);
          }
          if (SHK_ROT_FMA_BOOK && WIDE && SHK_ROT_MASK_LDS) na = (uint32_t)n - na;  // B count -> A count
        } else {
          const u2 xa = seed_mixer_pre_d(sa, TAG_LEAF);
#pragma unroll 2
          for (int i = 0; i < n; ++i) {
            const uint4 k = sm.keys[i];
            const u2 kh{k.x, k.y}, kl{k.z, k.w};
            const uint32_t bit = remix_top_pre_d(kh, kl, xb);
            u2 x;
            x.lo = bit ? xg.lo : xa.lo;
            x.hi = bit ? xg.hi : xa.hi;
            rot_key_cells<WIDE>(remix_pre_d(kh, kl, x), un, unm1, bit, ma0, ma1, mb0, mb1, na, e + i * 32);
          }
        }
        // Rotation filter: the set of r with (mask_a | rotl_n(mask_b, r))
        // == full.  Cell j missing from A needs mask_b[(j - r) mod n], i.e.
        // r in rotl_n(rev, j) with rev[k] = mask_b[(-k) mod n]; intersect
        // over the missing cells (about a third of them), stop when empty.
        const uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
        const uint64_t ma = join64(ma0, ma1), mb = join64(mb0, mb1);
        uint64_t need = ~ma & full;
        // E (128 bits): bit t = mb[(2n - 1 - t) mod n], the B mask written
        // twice and reversed.  Cell j is covered after rotation r iff
        // mb[(j - r) mod n] = E[n - 1 - j + r], so the rotations covering j
        // are the bits of E >> (n - 1 - j): one funnel shift per missing cell.
        const uint64_t dl = (n == 64) ? mb : (mb | (mb << n));   // D = mb | mb << n, low word
        const uint64_t dh = (n == 64) ? mb : (mb >> (64 - n));   // D, high word
        // E = reverse128(D) >> (128 - 2n)
        const uint64_t rl = __brevll(dh), rh = __brevll(dl);     // reverse128(D) = (rh:rl)
        const int sh = 128 - 2 * n;                              // 0 .. 126
        uint64_t el, eh;
        if (sh >= 64) {
          el = rh >> (sh - 64);
          eh = 0;
        } else if (sh > 0) {
          el = (rl >> sh) | (rh << (64 - sh));
          eh = rh >> sh;
        } else {
          el = rl;
          eh = rh;
        }
        // (E >> s) for s in [0, 63] without a select: (eh << 1) << (63 - s)
        const uint64_t eh1 = eh << 1;
        uint64_t Rm = full;
        // missing cells word by word (32-bit lowest-bit extraction is cheap)
        for (int hw = 0; hw < 2; ++hw) {
          uint32_t w = hw ? (uint32_t)(need >> 32) : (uint32_t)need;
          const int nb1 = n - 1 - 32 * hw;
          while (w && Rm) {
            const int s = nb1 - (__ffs(w) - 1);  // n - 1 - j, in [0, n - 1]
            w &= w - 1;
            Rm &= (el >> s) | (eh1 << (63 - s));
          }
        }
        passmask = Rm;
      }
      // exact checks, warp-cooperative, in lexicographic (base, r) order
      const int win_r = warp_first_accept(sm.edges[warp], passmask, n, lane, sm.chk[warp]);
      // per-lane counters (each < 2^8: 32-bit single-instruction warp sums)
      const uint32_t nb = (uint32_t)n - na;
      const uint32_t my_ev = valid ? nb + (ws ? (uint32_t)n + na : 0u) : 0u;
      const uint32_t my_aev = (valid && ws) ? na : 0u;
      const uint32_t my_pass = __popcll(passmask);
      unsigned ab = __ballot_sync(FULL_WARP, win_r >= 0);
      int wl = ab ? __ffs(ab) - 1 : 32;
      // sums over all lanes, and over lanes <= wl (the winner) when there is one
      const uint32_t t_ev = __reduce_add_sync(FULL_WARP, my_ev), t_aev = __reduce_add_sync(FULL_WARP, my_aev),
                     t_pass = __reduce_add_sync(FULL_WARP, my_pass);
      uint32_t c_ev_le = t_ev, c_aev_le = t_aev, c_pass_le = t_pass;
      if (ab) {
        uint32_t my_pass_le = my_pass;
        if (win_r >= 0) my_pass_le = __popcll(passmask & ((win_r == 63) ? ~0ull : ((2ull << win_r) - 1)));
        c_ev_le = __reduce_add_sync(FULL_WARP, lane <= wl ? my_ev : 0u);
        c_aev_le = __reduce_add_sync(FULL_WARP, lane <= wl ? my_aev : 0u);
        c_pass_le = __reduce_add_sync(FULL_WARP, lane < wl ? my_pass : (lane == wl ? my_pass_le : 0u));
      }
      int wr = __shfl_sync(FULL_WARP, win_r, wl & 31);
      if (TW == 1) {  // one-warp team: the round's result stays in registers
        passes += c_pass_le;
        evals += c_ev_le;
        aev += c_aev_le;
        if (ab) {
          const uint64_t qq = (R + (uint64_t)wl) * (uint64_t)n + (uint64_t)wr;
          q = (qq >= a.max_seed) ? -1 : (int64_t)qq;
          break;
        }
        if (HANDOFF && (SHK_HANDOFF_EVERY == 1 || ((R >> 5) & (SHK_HANDOFF_EVERY - 1)) == 0)) {
          int f;  // volatile asm: one relaxed load per round (not hoisted), no memory clobber
          asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(a.abort_flag));
          if (__any_sync(FULL_WARP, f != 0)) {
            stop_at = R + 32;
            break;
          }
        }
        continue;
      }
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
  if (HANDOFF && stop_at) {
    if (lane == 0) {
      ShkHandoff h;
      h.seed_slot = o.seed_slot;
      h.k0 = k0;
      h.next_base = stop_at;
      h.evals = evals;
      h.passes = passes;
      h.aev = aev;
      h.n = n;
      h.pad = 0;
      a.handoff[atomicAdd(a.handoff_count, 1ull)] = h;
    }
    __syncwarp();
    return;
  }
  if (warp == 0) {
    if (q >= 0 && n >= 2) {
      const uint64_t base = (uint64_t)q / (uint64_t)n;
      const int r = (int)((uint64_t)q % (uint64_t)n);
      const uint64_t sa = ck ? base - base % (uint64_t)ck : base;
      const u2 xb = seed_mixer_pre_d(sa, TAG_SPLITBIT), xa = seed_mixer_pre_d(sa, TAG_LEAF),
               xg = seed_mixer_pre_d(base, TAG_LEAF);
      for (int i = lane; i < n; i += 32) {
        uint4 k = sm.keys[i];
        u2 kh{k.x, k.y}, kl{k.z, k.w};
        uint32_t bit = remix_top_pre_d(kh, kl, xb);
        u2 v = remix_pre_d(kh, kl, bit ? xg : xa);
        uint32_t h0, h1;
        leaf_pair_d(v, (uint32_t)n, (uint32_t)(n - 1), h0, h1);
        if (bit) {
          h0 = (h0 + r) % n;
          h1 = (h1 + r) % n;
        }
        sm.eu[i] = (uint8_t)h0;
        sm.ev[i] = (uint8_t)h1;
      }
    }
    leaf_finish<TW>(a, sm, k0, n, q, o, evals, passes, aev, lane);
  }
  team_sync<TW>(team);
}

}  // namespace shk
