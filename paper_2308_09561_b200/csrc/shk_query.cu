// Batched MPHF evaluation.
//
// Restates _core.pyx:642-742 (query_stream) / _pure.py:489-550 and
// recsplit.py:251-275 (clamp to N-1).  The reference walks the preorder plan
// of the key's bucket and Rice-decodes EVERY node before the key's leaf (the
// seeds of skipped left subtrees included, ~38 decodes per query at n=40,
// b=2000).  Here the whole stream is decoded ONCE per descriptor (one thread
// per bucket decodes the bucket's nodes in order) into a per-node value table
// (split node: its seed's pre-mixed TAG_SPLIT mixer; leaf: its seed, as
// base << 6 | r in the rotate modes), so a
// query decodes nothing: it reads the values on its root-to-leaf path.
// Outputs are identical; so are the FormatError cases: a query fails iff the
// reference's sequential decode would overrun before reaching the key's leaf,
// i.e. iff the first undecodable node of its bucket has preorder index <= the
// leaf's.
#include "shk_common.cuh"
#include "shk_kernels.h"
#include "shk_rice.cuh"
#include "shk_split_dev.cuh"  // remix_hi_pre_d: the routing hashes only need the high word

namespace shk {

__global__ void node_index_kernel(ShkQueryDesc d, uint64_t* node_val, int32_t* bucket_bad) {
  for (int64_t bu = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bu < d.nbuckets;
       bu += (int64_t)gridDim.x * blockDim.x) {
    const int32_t plan = d.bucket_plan[bu];
    int32_t bad = 0x7FFFFFFF;
    if (plan >= 0) {
      const int64_t p0 = d.plan_off[plan], p1 = d.plan_off[plan + 1];
      const int64_t nb = d.node_base[bu];
      int64_t pos = (int64_t)d.bit_offsets[bu];
      for (int64_t j = 0; j < p1 - p0; ++j) {
        int64_t v;
        if (rice_decode(d.stream, d.stream_bit_len, &pos, d.pn_g[p0 + j], &v)) {
          bad = (int32_t)j;
          break;
        }
        uint64_t val;
        if (d.pn_kind[p0 + j] == 0) {
          val = premix_hi(seed_mixer((uint64_t)v, TAG_SPLIT));
        } else if (d.mode != 0 && d.pn_m[p0 + j] > 1) {  // rotate: q = base * m + r stored as base << 6 | r
          const uint64_t m = (uint64_t)d.pn_m[p0 + j], base = (uint64_t)v / m;
          // (a base too large to pack keeps q, flagged by bit 63)
          val = (base >> 57) ? ((uint64_t)v | (1ull << 63)) : ((base << 6) | ((uint64_t)v - base * m));
        } else {
          val = (uint64_t)v;
        }
        node_val[nb + j] = val;
      }
    }
    bucket_bad[bu] = bad;
    uint32_t* bq = reinterpret_cast<uint32_t*>(const_cast<uint4*>(d.bucketq)) + 4 * bu + 1;
    *bq = (*bq & 0xFFFFu) | ((bad < 0xFFFF ? (uint32_t)bad : 0xFFFFu) << 16);
  }
}

// High-word shift placement of the query's full remixes (ribbon patterns,
// leaf cells, split bit): 0 = IMAD.HI on the FMA pipe (two issue slots).
#ifndef SHK_QUERY_SHIFTS_ALU
#define SHK_QUERY_SHIFTS_ALU 1  // all on the ALU pipe: 1e8 queries 3.838 -> 3.826 ms (3 A/B pairs)
#endif
constexpr int QAM = SHK_QUERY_SHIFTS_ALU ? 0x1F : 0, QTM = SHK_QUERY_SHIFTS_ALU ? 0xF : 0;

// Pre-mixed per-descriptor mixers of the query (constant over a launch).
struct QueryMixers {
  u2 bucket, rstart, rpat0, rpat1;
};

SHK_D uint64_t rib_choice(const ShkQueryDesc& d, const QueryMixers& mx, u2 kp, u2 kl) {
  if (!d.rib_m) return 0;
  const uint64_t span = (uint64_t)(d.rib_m - RIBBON_W + 1);
  const int64_t s = (int64_t)(((uint64_t)remix_hi_pre_d(kp, kl, mx.rstart) * span) >> 32);
  const u2 a = remix_pre_d<QAM>(kp, kl, mx.rpat0);
  const u2 b = remix_pre_d<QAM>(kp, kl, mx.rpat1);
  const uint64_t pat0 = join64(a.lo | 1u, a.hi), pat1 = join64(b.lo, b.hi);
  const int64_t wi = s >> 6;
  const int sh = (int)(s & 63);
  // words wi .. wi + 2 in two gathers: the aligned pair holding wi + 1, and
  // the remaining word (the table is padded with a zero word; words past m
  // are zero, as the reference's out-of-range reads)
  const int64_t odd = wi & 1;
  const ulonglong2 pr = __ldg(reinterpret_cast<const ulonglong2*>(d.rib_words + ((wi + 1) & ~1ll)));
  const uint64_t ws = __ldg(d.rib_words + (odd ? wi : wi + 2));
  const uint64_t w0 = odd ? ws : pr.x;
  const uint64_t w1 = odd ? pr.x : pr.y;
  const uint64_t w2 = odd ? pr.y : ws;
  uint64_t v0, v1;
  if (sh) {
    v0 = (w0 >> sh) | (w1 << (64 - sh));
    v1 = (w1 >> sh) | (w2 << (64 - sh));
  } else {
    v0 = w0;
    v1 = w1;
  }
  return (uint64_t)((__popcll(v0 & pat0) + __popcll(v1 & pat1)) & 1);
}

// Cell of a key inside its leaf (leaf_cell, _core.pyx:751-767) from the
// pre-mixed key and the leaf's node value q (plain: the seed; rotate: the
// seed's base << 6 | rotation, split once by node_index_kernel).
SHK_D uint32_t leaf_cell_pre(u2 kp, u2 kl, uint64_t q, uint32_t n, int mode, int64_t cache_k, int choice) {
  if (n <= 1) return 0;  // leaf_pair gives (0, 0)
  uint32_t h0, h1;
  if (mode == 0) {
    leaf_pair_d(remix_pre_d<QAM>(kp, kl, seed_mixer_pre_d(q, TAG_LEAF)), n, n - 1, h0, h1);
    return choice ? h1 : h0;
  }
  uint64_t base = q >> 6, r = q & 63;  // node_index_kernel's packing
  if (q >> 63) {
    q &= ~(1ull << 63);
    base = q / n;
    r = q - base * n;
  }
  const uint64_t sa = (mode == 2 && cache_k && n > 32) ? base - base % (uint64_t)cache_k : base;
  if (remix_top_pre_d<QTM>(kp, kl, seed_mixer_pre_d(sa, TAG_SPLITBIT)) == 0) {
    leaf_pair_d(remix_pre_d<QAM>(kp, kl, seed_mixer_pre_d(sa, TAG_LEAF)), n, n - 1, h0, h1);
    return choice ? h1 : h0;
  }
  leaf_pair_d(remix_pre_d<QAM>(kp, kl, seed_mixer_pre_d(base, TAG_LEAF)), n, n - 1, h0, h1);
  uint32_t h = (choice ? h1 : h0) + (uint32_t)r;  // < 2n
  return h >= n ? h - n : h;
}

// SHK_QUERY_ILP queries per thread (t, t + stride, ...), stepped together
// through their split paths.  The kernel is co-bound by the L1 gather rate
// (one random 8-16 byte gather per level) and integer issue; two interleaved
// queries (58 registers, half the resident warps) measured 3% slower than one
// (profiles/r01_ncu_full_query_v15.csv), so the default is 1.
#ifndef SHK_QUERY_ILP
#define SHK_QUERY_ILP 1
#endif
__global__ void __launch_bounds__(256) query_kernel(ShkQueryDesc d, const uint64_t* hi, const uint64_t* lo, int64_t Q,
                                                    uint64_t* out, int* err, int clamp) {
  constexpr int U = SHK_QUERY_ILP;
  QueryMixers mx;
  mx.bucket = seed_mixer_pre_d(0, TAG_BUCKET);
  mx.rstart = seed_mixer_pre_d(d.rib_seed, TAG_RSTART);
  mx.rpat0 = seed_mixer_pre_d(d.rib_seed, TAG_RPAT0);
  mx.rpat1 = seed_mixer_pre_d(d.rib_seed, TAG_RPAT1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < Q; t0 += U * stride) {
    u2 kp[U], kl[U];
    uint64_t kp0[U], offset[U], x[U];
    uint4 p[U];
    const uint64_t* nv[U];
    const uint4* pq[U];
    int idx[U], bad[U], choice[U];
    bool walk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * stride;
      const bool in = t < Q;
      kp[u] = split64(premix_hi(in ? hi[t] : 0ull));
      kl[u] = split64(in ? lo[t] : 0ull);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t bucket = (int64_t)__umulhi(remix_hi_pre_d(kp[u], kl[u], mx.bucket), (uint32_t)d.nbuckets);
      const uint4 bq = __ldg(d.bucketq + bucket);
      kp0[u] = join64(bq.x, bq.y & 0xFFu);
      bad[u] = (int)(bq.y >> 16);  // 0xFFFF: none (plan-local ids are smaller)
      walk[u] = bq.w != 0xFFFFFFFFu;
      nv[u] = d.node_val + join64(bq.z, (bq.y >> 8) & 0xFFu);
      pq[u] = d.planq + (walk[u] ? bq.w : 0u);
    }
    // the ribbon bit depends on the key alone: its word loads stay in flight
    // across the split-path walk
#pragma unroll
    for (int u = 0; u < U; ++u) choice[u] = (int)rib_choice(d, mx, kp[u], kl[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      offset[u] = 0;
      idx[u] = 0;
      if (walk[u]) {  // a node's plan record and value depend on idx only: loaded together
        p[u] = __ldg(pq[u]);
        x[u] = __ldg(nv[u]);
      }
    }
    bool any = true;
    while (any) {
      any = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (walk[u] && !(p[u].x & 0x8000u) && idx[u] < bad[u]) {  // split node
          const uint32_t r = __umulhi(remix_hi_pre_d(kp[u], kl[u], split64(x[u])), p[u].x & 0x7FFFu);
          const uint32_t part = (uint32_t)(r >= (p[u].x >> 16)) + (uint32_t)(r >= (p[u].y & 0xFFFFu)) +
                                (uint32_t)(r >= (p[u].y >> 16));
          const uint32_t sh = 16 * part;
          offset[u] += (uint32_t)(join64(p[u].x & 0xFFFF0000u, p[u].y) >> sh) & 0xFFFFu;  // lane `part` of (0, b1..b3)
          idx[u] = (int)((uint32_t)(join64(p[u].z, p[u].w) >> sh) & 0xFFFFu);            // lane `part` of (c0..c3)
          p[u] = __ldg(pq[u] + idx[u]);
          x[u] = __ldg(nv[u] + idx[u]);
          any = true;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * stride;
      if (t >= Q) continue;
      if (walk[u]) {
        if (idx[u] >= bad[u]) {
          atomicOr(err, 1);
          out[t] = 0;
          continue;
        }
        offset[u] += leaf_cell_pre(kp[u], kl[u], x[u], p[u].x & 0x7FFFu, d.mode, d.cache_k, choice[u]);
      }
      uint64_t o = kp0[u] + offset[u];
      if (clamp) {
        const uint64_t mxk = d.n_keys > 0 ? (uint64_t)(d.n_keys - 1) : 0;
        if (o > mxk) o = mxk;
      }
      out[t] = o;
    }
  }
}

// Bijection check of query outputs (MphfDescriptor.verify, recsplit.py:383-394):
// first[v] = first input index mapping to v; the offender is the first input
// index whose value is out of range or was produced by an earlier index.
__global__ void first_index_kernel(const uint64_t* v, int64_t Q, int64_t N, unsigned long long* first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = v[i];
    if (x < (uint64_t)N) atomicMin(&first[x], (unsigned long long)i);
  }
}

__global__ void offender_kernel(const uint64_t* v, int64_t Q, int64_t N, const unsigned long long* first,
                                unsigned long long* offender) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Q; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = v[i];
    if (x >= (uint64_t)N || first[x] != (unsigned long long)i) atomicMin(offender, (unsigned long long)i);
  }
}

}  // namespace shk

using namespace shk;

int shk_launch_node_index(const ShkQueryDesc& d, uint64_t* node_val, int32_t* bucket_bad, cudaStream_t st) {
  if (d.nbuckets <= 0) return 0;
  int64_t g = (d.nbuckets + 127) / 128;
  node_index_kernel<<<(unsigned)g, 128, 0, st>>>(d, node_val, bucket_bad);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_query(const ShkQueryDesc& d, const uint64_t* hi, const uint64_t* lo, int64_t Q, uint64_t* out, int* err,
                     int clamp, cudaStream_t st) {
  if (Q <= 0) return 0;
  int64_t g = ((Q + SHK_QUERY_ILP - 1) / SHK_QUERY_ILP + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  query_kernel<<<(unsigned)g, 256, 0, st>>>(d, hi, lo, Q, out, err, clamp);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_bijection(const uint64_t* v, int64_t Q, int64_t N, unsigned long long* first,
                         unsigned long long* offender, cudaStream_t st) {
  SHK_CUDA(cudaMemsetAsync(first, 0xFF, (size_t)N * 8, st));
  SHK_CUDA(cudaMemsetAsync(offender, 0xFF, 8, st));
  if (Q <= 0) return 0;
  int64_t g = (Q + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  first_index_kernel<<<(unsigned)g, 256, 0, st>>>(v, Q, N, first);
  SHK_LAUNCHED();
  offender_kernel<<<(unsigned)g, 256, 0, st>>>(v, Q, N, first, offender);
  SHK_LAUNCHED();
  return 0;
}
