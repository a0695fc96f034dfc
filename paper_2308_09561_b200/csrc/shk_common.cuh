// Shared device helpers: error checking, warp utilities, small union-find,
// the canonical 1-orientation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "shk_hash.cuh"

#define SHK_CUDA(call)                                                      \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) {                                                \
      shk_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                    cudaGetErrorString(e_));                                \
      return -(int)e_ - 1000;                                               \
    }                                                                       \
  } while (0)

void shk_set_error(const char* fmt, ...);
void shk_note_launch();

// Every kernel launch goes through this: counts launches (reported as
// gpu_launches by bench.py) and surfaces launch errors.
#define SHK_LAUNCHED()                 \
  do {                                 \
    shk_note_launch();                 \
    SHK_CUDA(cudaGetLastError());      \
  } while (0)

namespace shk {

constexpr unsigned FULL_WARP = 0xFFFFFFFFu;

SHK_D int lane_id() { return threadIdx.x & 31; }

template <typename T>
SHK_D T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_WARP, v, o);
  return v;
}

// Pseudoforest acceptance on <= 64 cells (_core.pyx:125-179).  Acceptance is
// a graph property (every component has exactly as many edges as nodes), so
// any correct union-find gives the reference's answer; this one links by
// index with path halving and keeps the per-root "has a cycle" flags in a
// 64-bit mask.  Edges are packed u16 (h0 | h1 << 8), stride 32 (one column
// per lane of a warp), bit 15 marks a rotation-set-B key whose cells are
// shifted by `rot` mod n.
SHK_D bool pf_accepts(const uint16_t* e, int stride, int nkeys, int n, int rot) {
  uint8_t parent[64];
  for (int i = 0; i < n; ++i) parent[i] = (uint8_t)i;
  uint64_t pseudo = 0;
  for (int i = 0; i < nkeys; ++i) {
    uint32_t w = e[i * stride];
    int u = w & 0x7F, v = (w >> 8) & 0x7F;
    if (w & 0x8000u) {
      u += rot;
      v += rot;
      if (u >= n) u -= n;
      if (v >= n) v -= n;
    }
    while (parent[u] != u) {
      parent[u] = parent[parent[u]];
      u = parent[u];
    }
    while (parent[v] != v) {
      parent[v] = parent[parent[v]];
      v = parent[v];
    }
    uint64_t pu = (pseudo >> u) & 1, pv = (pseudo >> v) & 1;
    if (u == v) {
      if (pu) return false;
      pseudo |= 1ull << u;
    } else {
      if (pu & pv) return false;
      parent[v] = (uint8_t)u;
      pseudo |= pv << u;
    }
  }
  return true;
}

// Warp-cooperative exact pseudoforest check of one candidate (all 32 lanes
// participate; lane t owns edges t and t+32).  Used instead of a per-lane
// union-find so a rare candidate costs ~100 warp instructions, not ~1000
// single-lane ones.
//  1. Degrees (shared atomics).  An isolated edge (both cells of degree 1)
//     is a tree component: reject.  This catches ~84% of the candidates that
//     pass the coverage filter at n=40.
//  2. Components by min-label hooking + pointer jumping (labels only move to
//     smaller indices, so jumping always ends at a root; a round that hooked
//     anything is followed by another, so a lost concurrent hook is redone).
//  3. Pseudoforest iff every component has as many edges as cells.
// ew: edges of the warp, column per lane (ew[i*32 + L] = candidate lane L's
// edge i, packed u | v << 8 | rotation-set-B << 15); rot: B-cell shift.
struct WarpChk {
  int deg[64];
  int par[64];
  int ce[64];
  int cv[64];
};

// col[i * stride] = edge i of the candidate (warp_pf_check: the column of
// lane L in a stride-32 edge table).
SHK_D bool warp_pf_check_col(const uint16_t* col, int stride, int rot, int n, int lane, WarpChk& s) {
  int u0 = -1, v0 = 0, u1 = -1, v1 = 0;
  if (lane < n) {
    uint32_t w = col[lane * stride];
    u0 = w & 0x7F;
    v0 = (w >> 8) & 0x7F;
    if (w & 0x8000u) {
      u0 += rot;
      v0 += rot;
      if (u0 >= n) u0 -= n;
      if (v0 >= n) v0 -= n;
    }
  }
  if (lane + 32 < n) {
    uint32_t w = col[(lane + 32) * stride];
    u1 = w & 0x7F;
    v1 = (w >> 8) & 0x7F;
    if (w & 0x8000u) {
      u1 += rot;
      v1 += rot;
      if (u1 >= n) u1 -= n;
      if (v1 >= n) v1 -= n;
    }
  }
  s.deg[lane] = 0;
  s.deg[lane + 32] = 0;
  s.par[lane] = lane;
  s.par[lane + 32] = lane + 32;
  __syncwarp();
  if (u0 >= 0) {
    atomicAdd(&s.deg[u0], 1);
    atomicAdd(&s.deg[v0], 1);
  }
  if (u1 >= 0) {
    atomicAdd(&s.deg[u1], 1);
    atomicAdd(&s.deg[v1], 1);
  }
  __syncwarp();
  const bool iso = (u0 >= 0 && s.deg[u0] == 1 && s.deg[v0] == 1) || (u1 >= 0 && s.deg[u1] == 1 && s.deg[v1] == 1);
  if (__any_sync(FULL_WARP, iso)) return false;
  for (int it = 0; it < 128; ++it) {
    bool ch = false;
    if (u0 >= 0) {
      int a = s.par[u0], b = s.par[v0];
      if (a != b) {
        atomicMin(&s.par[a > b ? a : b], a < b ? a : b);
        ch = true;
      }
    }
    if (u1 >= 0) {
      int a = s.par[u1], b = s.par[v1];
      if (a != b) {
        atomicMin(&s.par[a > b ? a : b], a < b ? a : b);
        ch = true;
      }
    }
    __syncwarp();
    for (int x = lane; x < n; x += 32) {
      int p = s.par[x];
      while (s.par[p] != p) p = s.par[p];
      s.par[x] = p;
    }
    __syncwarp();
    if (!__any_sync(FULL_WARP, ch)) break;
  }
  s.ce[lane] = 0;
  s.ce[lane + 32] = 0;
  s.cv[lane] = 0;
  s.cv[lane + 32] = 0;
  __syncwarp();
  for (int x = lane; x < n; x += 32) atomicAdd(&s.cv[s.par[x]], 1);
  if (u0 >= 0) atomicAdd(&s.ce[s.par[u0]], 1);
  if (u1 >= 0) atomicAdd(&s.ce[s.par[u1]], 1);
  __syncwarp();
  bool bad = false;
  for (int x = lane; x < n; x += 32)
    if (s.par[x] == x && s.ce[x] != s.cv[x]) bad = true;
  const bool ok = !__any_sync(FULL_WARP, bad);
  __syncwarp();
  return ok;
}

SHK_D bool warp_pf_check(const uint16_t* ew, int L, int rot, int n, int lane, WarpChk& s) {
  return warp_pf_check_col(ew + L, 32, rot, n, lane, s);
}

// First accepted candidate in (lane, r) order among the lanes' candidate
// masks (bit r of cand = the coverage filter passed for rotation r).
// Returns r on the winning lane, -1 elsewhere (all lanes get the same L).
SHK_D int warp_first_accept(const uint16_t* ew, uint64_t cand, int n, int lane, WarpChk& s) {
  unsigned lanes = __ballot_sync(FULL_WARP, cand != 0);
  while (lanes) {
    const int L = __ffs(lanes) - 1;
    lanes &= lanes - 1;
    uint64_t pm = __shfl_sync(FULL_WARP, cand, L);
    while (pm) {
      const int r = __ffsll((long long)pm) - 1;
      pm &= pm - 1;
      if (warp_pf_check(ew, L, r, n, lane, s)) return lane == L ? r : -1;
    }
  }
  return -1;
}

// Canonical 1-orientation of a pseudoforest (pseudoforest.py:149-201):
// peel degree-1 cells (the single remaining edge takes that cell), then walk
// each remaining cycle from its lowest-index key, which takes its first cell.
// The result is independent of peel order, so peeling in
// lowest-cell order is bit-exact with the reference's stack order.
// eu/ev: cells of edge k (edges[k][0], edges[k][1]); inc: scratch[64].
// Returns f bits (bit k = 1 iff key k takes edges[k][1]).
SHK_D uint64_t orient_edges(const uint8_t* eu, const uint8_t* ev, int n, uint64_t* inc) {
  for (int u = 0; u < n; ++u) inc[u] = 0;
  for (int k = 0; k < n; ++k) {
    inc[eu[k]] |= 1ull << k;
    inc[ev[k]] |= 1ull << k;
  }
  uint64_t alive = (n == 64) ? ~0ull : ((1ull << n) - 1);
  uint64_t loops = 0;  // self-loop edges count twice toward a cell's degree
  for (int k = 0; k < n; ++k)
    if (eu[k] == ev[k]) loops |= 1ull << k;
  uint64_t f = 0;
  uint64_t cand = 0;
  for (int u = 0; u < n; ++u)
    if (__popcll(inc[u]) + __popcll(inc[u] & loops) == 1) cand |= 1ull << u;
  while (cand) {
    int u = __ffsll((long long)cand) - 1;
    cand &= cand - 1;
    uint64_t live = inc[u] & alive;
    if (__popcll(live) + __popcll(live & loops) != 1) continue;
    int k = __ffsll((long long)live) - 1;
    int a = eu[k], b = ev[k];
    if (a != u) f |= 1ull << k;
    alive &= ~(1ull << k);
    int other = (a == u) ? b : a;
    uint64_t lo = inc[other] & alive;
    if (__popcll(lo) + __popcll(lo & loops) == 1) cand |= 1ull << other;
  }
  while (alive) {
    int k0 = __ffsll((long long)alive) - 1;
    alive &= ~(1ull << k0);
    int u0 = eu[k0];
    int node = ev[k0];
    int guard = 0;
    while (node != u0 && guard++ <= n) {
      uint64_t live = inc[node] & alive;
      if (!live) break;  // not a pseudoforest; caller guarantees otherwise
      int k = __ffsll((long long)live) - 1;
      int a = eu[k], b = ev[k];
      if (a != node) f |= 1ull << k;
      alive &= ~(1ull << k);
      node = (a == node) ? b : a;
    }
  }
  return f;
}

}  // namespace shk
