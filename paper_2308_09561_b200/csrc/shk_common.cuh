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
