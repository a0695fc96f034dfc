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
    reinterpret_cast<uint32_t*>(const_cast<uint4*>(d.bucketq))[8 * bu + 3] = (uint32_t)bad;
  }
}

// Pre-mixed per-descriptor mixers of the query (constant over a launch).
struct QueryMixers {
  u2 bucket, rstart, rpat0, rpat1;
};

SHK_D uint64_t rib_choice(const ShkQueryDesc& d, const QueryMixers& mx, u2 kp, u2 kl) {
  if (!d.rib_m) return 0;
  const uint64_t span = (uint64_t)(d.rib_m - RIBBON_W + 1);
  const int64_t s = (int64_t)(((uint64_t)remix_hi_pre_d(kp, kl, mx.rstart) * span) >> 32);
  const u2 a = remix_pre_d(kp, kl, mx.rpat0);
  const u2 b = remix_pre_d(kp, kl, mx.rpat1);
  const uint64_t pat0 = join64(a.lo | 1u, a.hi), pat1 = join64(b.lo, b.hi);
  const int64_t wi = s >> 6;
  const int sh = (int)(s & 63);
  const int64_t nw = d.rib_nwords;
  const uint64_t w0 = wi < nw ? d.rib_words[wi] : 0;
  const uint64_t w1 = wi + 1 < nw ? d.rib_words[wi + 1] : 0;
  const uint64_t w2 = wi + 2 < nw ? d.rib_words[wi + 2] : 0;
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
    leaf_pair_d(remix_pre_d(kp, kl, seed_mixer_pre_d(q, TAG_LEAF)), n, n - 1, h0, h1);
    return choice ? h1 : h0;
  }
  uint64_t base = q >> 6, r = q & 63;  // node_index_kernel's packing
  if (q >> 63) {
    q &= ~(1ull << 63);
    base = q / n;
    r = q - base * n;
  }
  const uint64_t sa = (mode == 2 && cache_k && n > 32) ? base - base % (uint64_t)cache_k : base;
  if (remix_top_pre_d(kp, kl, seed_mixer_pre_d(sa, TAG_SPLITBIT)) == 0) {
    leaf_pair_d(remix_pre_d(kp, kl, seed_mixer_pre_d(sa, TAG_LEAF)), n, n - 1, h0, h1);
    return choice ? h1 : h0;
  }
  leaf_pair_d(remix_pre_d(kp, kl, seed_mixer_pre_d(base, TAG_LEAF)), n, n - 1, h0, h1);
  uint32_t h = (choice ? h1 : h0) + (uint32_t)r;  // < 2n
  return h >= n ? h - n : h;
}

__global__ void __launch_bounds__(256) query_kernel(ShkQueryDesc d, const uint64_t* hi, const uint64_t* lo, int64_t Q,
                                                    uint64_t* out, int* err, int clamp) {
  QueryMixers mx;
  mx.bucket = seed_mixer_pre_d(0, TAG_BUCKET);
  mx.rstart = seed_mixer_pre_d(d.rib_seed, TAG_RSTART);
  mx.rpat0 = seed_mixer_pre_d(d.rib_seed, TAG_RPAT0);
  mx.rpat1 = seed_mixer_pre_d(d.rib_seed, TAG_RPAT1);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Q; t += (int64_t)gridDim.x * blockDim.x) {
    const u2 kp = split64(premix_hi(hi[t])), kl = split64(lo[t]);
    const int64_t bucket = (int64_t)__umulhi(remix_hi_pre_d(kp, kl, mx.bucket), (uint32_t)d.nbuckets);
    const uint4 b0 = __ldg(d.bucketq + 2 * bucket), b1 = __ldg(d.bucketq + 2 * bucket + 1);
    // the ribbon bit depends on the key alone: its three word loads are issued
    // here and stay in flight across the split-path walk
    const int choice = (int)rib_choice(d, mx, kp, kl);
    const uint64_t kp0 = join64(b0.x, b0.y);
    uint64_t offset = 0;
    if (b0.z > 0) {  // msize
      const int bad = (int)b0.w;
      const uint64_t* nv = d.node_val + join64(b1.x, b1.y);
      const uint4* pq = d.planq + b1.z;
      int idx = 0;
      // a node's plan record and value are loaded together (both depend on
      // idx only): one dependent load round trip per level
      uint4 p = __ldg(pq);
      uint64_t x = __ldg(nv);
      while (!(p.x & 0x8000u)) {  // split node
        if (idx >= bad) break;
        const uint32_t r = __umulhi(remix_hi_pre_d(kp, kl, split64(x)), p.x & 0x7FFFu);
        const uint32_t part = (uint32_t)(r >= (p.x >> 16)) + (uint32_t)(r >= (p.y & 0xFFFFu)) + (uint32_t)(r >= (p.y >> 16));
        const uint32_t sh = 16 * part;
        offset += (uint32_t)(join64(p.x & 0xFFFF0000u, p.y) >> sh) & 0xFFFFu;  // lane `part` of (0, b1, b2, b3)
        idx = (int)((uint32_t)(join64(p.z, p.w) >> sh) & 0xFFFFu);          // lane `part` of (c0 .. c3)
        p = __ldg(pq + idx);
        x = __ldg(nv + idx);
      }
      if (idx >= bad) {
        atomicOr(err, 1);
        out[t] = 0;
        continue;
      }
      const uint64_t q = x;
      const uint32_t mleaf = p.x & 0x7FFFu;
      offset += leaf_cell_pre(kp, kl, q, mleaf, d.mode, d.cache_k, choice);
    }
    uint64_t o = kp0 + offset;
    if (clamp) {
      const uint64_t mx = d.n_keys > 0 ? (uint64_t)(d.n_keys - 1) : 0;
      if (o > mx) o = mx;
    }
    out[t] = o;
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
  int64_t g = (Q + 255) / 256;
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
