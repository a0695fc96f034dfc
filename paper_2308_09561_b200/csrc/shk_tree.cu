// Persistent construction kernel: every split node and every leaf of a
// bucket range in ONE launch, scheduled through a device task queue.
//
// The per-level schedule (one launch per tree depth, then one leaf launch)
// pays a tail at every level: the slowest node of a level (trial counts are
// geometric, the worst of ~1e4 nodes needs ~10x the mean) runs alone while
// the rest of the GPU idles.  Here each warp pops a ready node from a global
// queue, solves it (split: minimum seed + stable partition; leaf: ShockHash
// search + orientation) and publishes the node's children, so the tail of one
// level overlaps the work of every other level and of the leaves.
//
// Queue protocol: slots are pre-sized to the node count.  The initial slots
// hold the bucket roots; a producer reserves slots with atomicAdd on the tail
// and publishes child ids with release stores after a __threadfence() that
// orders its key partition before them; a consumer takes the next slot with
// atomicAdd on the head and waits (nanosleep) until the id is published, then
// fences (which also drops stale L1 lines of keys partitioned on another SM).
// Every unpublished node is a child of a node that some warp is executing,
// so a waiting warp always gets its task; warps exit once head >= node count.
// Results are exactly those of the per-level schedule: every node sees the
// same keys in the same order and runs the same minimum-seed search.
//
// Warp slots are not equal.  The issue arbiter of a sub-partition serves
// low hardware warp slots (%warpid) first (measured), so in this issue-bound kernel a warp in
// the top CTA slot runs ~16x slower than one in the bottom slot
// (tools/tree_trace.py: mean node time per %warpid at C4, 0.55 ms for slots
// 0-3, 9 ms for slots 28-31).  A split node that lands on a slow slot gates
// its whole subtree: the long nodes of a build were 3 x 160 / 4 x 40 splits
// started in the first milliseconds on slots >= 24 and finished only when
// the queue drained.  So the queue is split in two regions, split nodes
// [0, nsplit) and leaves [nsplit, nnodes), each with its own head and tail:
// warps in the lower half of the slots take split nodes first and leaves
// once every split has been handed out; warps in the upper half take leaves
// only (a leaf gates nothing).  Each region hands out tickets as before
// (atomicAdd on its head, then wait until the slot is published).  A lower
// slot waiting for a split leaves its issue share to the leaf warps, so the
// SM stays busy while the splits run on the fast slots.
#include "shk_kernels.h"
#include "shk_leaf_dev.cuh"
#include "shk_split_dev.cuh"

namespace shk {

struct TreeArgs {
  ulonglong2* keys;
  ulonglong2* tmp;
  const ShkTreeNode* nodes;
  int64_t nnodes;
  int64_t* queue;              // [nnodes]: split region [0, nsplit), leaf region [nsplit, nnodes)
  unsigned long long* head;    // [2]: split head, leaf head (absolute slot indices)
  unsigned long long* tail;    // [2]: split tail, leaf tail
  int64_t nsplit;
  int slow_wid;                // warps with %warpid >= slow_wid take leaves only
  int idle_wid;                // warps with %warpid >= idle_wid take no work (A/B)
  int64_t tail_reserve;        // leaf-only warps take no leaf once fewer than this remain
  uint64_t max_seed;
  int64_t* seeds;
  int* exhausted;
  const int* dup_flag;         // nonzero: equal codes in the input, every warp exits (the host raises)
  int set_abort;               // rotate tail hand-off: raise leaf.abort_flag once the leaf queue is empty
  LeafArgs leaf;
};

#ifdef SHK_TREE_TRACE
// (analysis builds) start / end globaltimer of every node id < 2^20
__device__ unsigned long long g_tree_trace[2 << 20];
// node size m << 8 | fanout (0 for a leaf) | %warpid << 24 of the warp that ran it
__device__ unsigned int g_tree_trace_m[1 << 20];
#endif

SHK_D int64_t load_published(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

SHK_D void publish(int64_t* p, int64_t v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

SHK_D unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// MAXE: leaf buffer capacity; MINB: CTAs per SM requested from ptxas (8 = 64
// registers; see SHK_TREE_MINB).
#ifndef SHK_TREE_MINB
#define SHK_TREE_MINB 8
#endif
template <bool WIDE, int MODE, int MAXE, int MINB>
__global__ void __launch_bounds__(128, MINB) tree_kernel(TreeArgs t) {
  __shared__ LeafSmem<1, MAXE> sm_all[4];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  LeafSmem<1, MAXE>& sm = sm_all[w];
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  // lower slots take split tickets until the split region is used up, then
  // leaf tickets; upper slots take leaf tickets only
  // Progress must not depend on the slot numbering (%warpid is volatile and
  // other kernels / MPS clients may hold the low slots): warp 0 of CTA 0 is
  // always split-capable and never idles, so every split node -- and with it
  // every leaf slot -- is eventually published whatever slots the warps get.
  const bool anchor = blockIdx.x == 0 && w == 0;
  if ((int)wid >= t.idle_wid && !anchor) return;
  // the bucket sort's duplicate flag is checked here rather than by the host
  // before the launch, so the host enqueues the launch while the sort runs
  if (t.dup_flag && *(volatile const int*)t.dup_flag) return;
  const bool slow = (int)wid >= t.slow_wid && !anchor;
  bool splits_done = slow;
  for (;;) {
    unsigned long long h = 0;
    if (!splits_done) {
      if (lane == 0) h = atomicAdd(t.head, 1ull);
      h = __shfl_sync(FULL_WARP, h, 0);
      if (h >= (unsigned long long)t.nsplit) splits_done = true;
    }
    if (splits_done) {
      if (slow && t.tail_reserve > 0) {
        // the last leaves go to the fast slots: a leaf started late on a
        // slow slot would end the launch (a top slot runs ~16x slower)
        unsigned long long hh = 0;
        if (lane == 0) hh = ld_relaxed_u64(t.head + 1);
        hh = __shfl_sync(FULL_WARP, hh, 0);
        if ((int64_t)hh + t.tail_reserve >= t.nnodes) break;
      }
      if (lane == 0) h = atomicAdd(t.head + 1, 1ull);
      h = __shfl_sync(FULL_WARP, h, 0);
      if (h >= (unsigned long long)t.nnodes) {
        // every leaf is handed out: the leaves still searching stop at their
        // next round boundary and tree_resume_kernel finishes them with teams
        if (t.set_abort && lane == 0) *(volatile int*)t.leaf.abort_flag = 1;
        break;
      }
    }
    int64_t id = -1;
    if (lane == 0) {
      while ((id = load_published(t.queue + h)) < 0) __nanosleep(200);
    }
    id = __shfl_sync(FULL_WARP, id, 0);
    __threadfence();  // acquire side for all lanes; invalidates stale L1 lines
#ifdef SHK_TREE_TRACE
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
    const ShkTreeNode nd = t.nodes[id];
    if (nd.kind == 0) {
      ShkSplitTask task;
      task.start = nd.start;
      task.m = nd.m;
      task.fanout = nd.fanout;
      for (int k = 0; k < 4; ++k) task.sizes[k] = nd.sizes[k];
      task.seed_slot = id;
      const ulonglong2* kp = t.keys + nd.start;
      const int64_t seed = split_search_build(kp, task, t.max_seed, lane);
      if (lane == 0) {
        t.seeds[id] = seed;
        if (seed < 0 && t.exhausted) atomicOr(t.exhausted, 1);
      }
      if (seed >= 0) split_partition(kp, t.keys, t.tmp, task, seed, lane, lt);
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        // children are published even after a failed search (the build is
        // flagged exhausted) so that no consumer waits forever
        for (int k = 0; k < nd.fanout; ++k) {
          const int64_t ch = nd.child[k];
          const int r = t.nodes[ch].kind != 0;  // 0: split region, 1: leaf region
          publish(t.queue + atomicAdd(t.tail + r, 1ull), ch);
        }
      }
    } else {
      const LeafOut o{id, -1};
      if (MODE == 0)
        solve_plain<1, WIDE>(t.leaf, sm, nd.start, nd.m, o, 0, 0, lane, lane);
      else
        solve_rotate<1, WIDE, true>(t.leaf, sm, nd.start, nd.m, o, 0, 0, lane, lane);
    }
#ifdef SHK_TREE_TRACE
    if (lane == 0 && id < (1 << 20)) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      g_tree_trace[2 * id] = t0;
      g_tree_trace[2 * id + 1] = now;
      unsigned wid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      g_tree_trace_m[id] = ((unsigned)nd.m << 8) | (nd.kind == 0 ? (unsigned)nd.fanout : 0u) | (wid << 24);
    }
#endif
  }
}

// Tail hand-off, second half: one team of TW warps per CTA takes the leaves
// the construction kernel stopped (ShkHandoff records) and resumes each at its
// recorded base with its recorded counters.  A team round covers TW * 32
// consecutive bases and keeps the lowest accepting (base, r), so the seed,
// the f bits and the counters are those of the uninterrupted one-warp search.
// A leaf's heavy seed tail is thus spread over TW warps instead of ending the
// build on one warp.
static_assert(sizeof(ShkHandoff) == 56, "hand-off record size is part of the host allocation");
template <int TW, bool WIDE, int MAXE>
__global__ void __launch_bounds__(TW * 32) tree_resume_kernel(LeafArgs a, unsigned long long* next) {
  __shared__ LeafSmem<TW, MAXE> sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tt = threadIdx.x;
  const unsigned long long cnt = *(volatile const unsigned long long*)a.handoff_count;
  for (;;) {
    if (tt == 0) sm.leaf = (int64_t)atomicAdd(next, 1ull);
    team_sync<TW>(0);
    const int64_t i = sm.leaf;
    if ((unsigned long long)i >= cnt) break;
    const ShkHandoff h = a.handoff[i];
    const LeafOut o{h.seed_slot, -1};
    solve_rotate<TW, WIDE>(a, sm, h.k0, h.n, o, 0, warp, lane, tt, h.next_base, h.evals, h.passes, h.aev);
  }
}

// One CTA per bucket: copy its plan's nodes into the global node table.
__global__ void expand_nodes_kernel(const ShkPlanNode* pn, const int64_t* plan_off, const int32_t* bucket_plan,
                                    const int64_t* node_base, const int64_t* key_start, const int64_t* root_pos,
                                    int64_t nbuckets, ShkTreeNode* nodes, int32_t* node_g, uint8_t* node_kind,
                                    int64_t* queue) {
  for (int64_t bu = blockIdx.x; bu < nbuckets; bu += gridDim.x) {
    const int32_t plan = bucket_plan[bu];
    if (plan < 0) continue;
    const int64_t pa = plan_off[plan], cnt = plan_off[plan + 1] - pa;
    const int64_t nb = node_base[bu], ks = key_start[bu];
    if (threadIdx.x == 0) queue[root_pos[bu]] = nb;
    for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
      const ShkPlanNode p = pn[pa + j];
      ShkTreeNode t;
      t.start = ks + p.off;
      t.m = p.m;
      t.kind = p.kind != 0;
      t.fanout = p.kind == 0 ? p.fanout : 0;
      t.pad = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        t.sizes[k] = p.sizes[k];
        t.child[k] = (p.kind == 0 && k < p.fanout) ? nb + p.child[k] : -1;
      }
      nodes[nb + j] = t;
      node_g[nb + j] = p.g;
      node_kind[nb + j] = (uint8_t)(p.kind != 0);
    }
  }
}

}  // namespace shk

using namespace shk;

int shk_launch_expand_nodes(const ShkPlanNode* plan_nodes, const int64_t* plan_off, const int32_t* bucket_plan,
                            const int64_t* node_base, const int64_t* key_start, const int64_t* root_pos,
                            int64_t nbuckets, ShkTreeNode* nodes, int32_t* node_g, uint8_t* node_kind, int64_t* queue,
                            cudaStream_t st) {
  if (nbuckets <= 0) return 0;
  int64_t g = nbuckets < 148 * 16 ? nbuckets : 148 * 16;
  expand_nodes_kernel<<<(unsigned)g, 128, 0, st>>>(plan_nodes, plan_off, bucket_plan, node_base, key_start, root_pos,
                                                   nbuckets, nodes, node_g, node_kind, queue);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_tree(const ShkTreeLaunch& p, cudaStream_t st) {
  if (p.nnodes <= 0) return 0;
  TreeArgs t;
  t.keys = reinterpret_cast<ulonglong2*>(p.keys);
  t.tmp = reinterpret_cast<ulonglong2*>(p.tmp);
  t.nodes = p.nodes;
  t.nnodes = p.nnodes;
  t.queue = p.queue;
  t.head = p.head;
  t.tail = p.tail;
  t.nsplit = p.nsplit;
  t.max_seed = p.max_seed;
  t.seeds = p.seeds;
  t.exhausted = p.exhausted;
  t.dup_flag = p.dup_flag;
  LeafArgs& a = t.leaf;
  a = LeafArgs{};
  a.hi = p.keys;
  a.lo = p.keys + 1;
  a.stride = 2;
  a.pre = 1;
  a.max_seed = p.max_seed;
  a.mode = p.mode;
  a.cache_k = p.cache_k;
  a.cache_min_leaf = p.cache_min_leaf;
  a.seed_out = p.seeds;
  a.choice_out = p.choice_out;
  a.stats_acc = p.stats_acc;
  a.exhausted = p.exhausted;
  a.place_out = p.place_out;
  a.abort_flag = p.abort_flag;
  a.handoff = reinterpret_cast<ShkHandoff*>(p.handoff);
  a.handoff_count = p.handoff_count;
  t.set_abort = p.mode != 0 && p.handoff_tw > 0 && p.abort_flag != nullptr && p.handoff_count && p.handoff_next;
  const bool wide = p.max_n > 32;
  const bool small = p.max_n <= 40;
  void (*kfn)(TreeArgs);
  if (p.mode == 0) {
    if (small)
      kfn = wide ? tree_kernel<true, 0, 40, SHK_TREE_MINB> : tree_kernel<false, 0, 40, SHK_TREE_MINB>;
    else
      kfn = tree_kernel<true, 0, 64, 8>;
  } else {
    if (small)
      kfn = wide ? tree_kernel<true, 1, 40, SHK_TREE_MINB> : tree_kernel<false, 1, 40, SHK_TREE_MINB>;
    else
      kfn = tree_kernel<true, 1, 64, 8>;
  }
  int occ = 0;
  SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 128, 0));
  if (occ < 1) occ = 1;
  const int sms = p.num_sms > 0 ? p.num_sms : 148;
  t.slow_wid = p.slow_wid > 0 ? p.slow_wid : (occ * 4) / 2;
  t.idle_wid = p.idle_wid > 0 ? p.idle_wid : 1 << 30;
  // -1: one leaf per fast warp (the slots below slow_wid on every SM)
  t.tail_reserve = p.tail_reserve >= 0 ? p.tail_reserve : (int64_t)sms * (t.slow_wid < occ * 4 ? t.slow_wid : occ * 4);
  if (p.mode != 0 && p.abort_flag == nullptr) {
    shk_set_error("tree launch: the rotate search needs the hand-off flag and buffer");
    return 3;
  }
  if ((int64_t)sms * occ * 4 > p.handoff_cap && p.mode != 0) {
    shk_set_error("tree launch: hand-off buffer smaller than the resident warps");
    return 3;
  }
  kfn<<<(unsigned)(sms * occ), 128, 0, st>>>(t);
  SHK_LAUNCHED();
  if (t.set_abort) {
    // resume teams: launched whatever the count (the count is on the device);
    // with no stopped leaf every CTA exits after one atomic
    void (*rfn)(LeafArgs, unsigned long long*);
#define SHK_RESUME_FN(TW) \
  (small ? (wide ? tree_resume_kernel<TW, true, 40> : tree_resume_kernel<TW, false, 40>) : tree_resume_kernel<TW, true, 64>)
    switch (p.handoff_tw) {
      case 1: rfn = SHK_RESUME_FN(1); break;
      case 2: rfn = SHK_RESUME_FN(2); break;
      case 4: rfn = SHK_RESUME_FN(4); break;
      case 8: rfn = SHK_RESUME_FN(8); break;
      default: shk_set_error("hand-off team size must be 1, 2, 4 or 8"); return 3;
    }
#undef SHK_RESUME_FN
    int rocc = 0;
    SHK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rocc, rfn, p.handoff_tw * 32, 0));
    if (rocc < 1) rocc = 1;
    rfn<<<(unsigned)(sms * rocc), p.handoff_tw * 32, 0, st>>>(a, p.handoff_next);
    SHK_LAUNCHED();
  }
  return 0;
}

#ifdef SHK_TREE_TRACE
extern "C" int shk_debug_tree_trace(unsigned long long* out, int64_t n) {
  if (n > (1 << 20)) n = 1 << 20;
  SHK_CUDA(cudaMemcpyFromSymbol(out, g_tree_trace, (size_t)n * 16));
  return 0;
}
extern "C" int shk_debug_tree_trace_m(unsigned int* out, int64_t n) {
  if (n > (1 << 20)) n = 1 << 20;
  SHK_CUDA(cudaMemcpyFromSymbol(out, g_tree_trace_m, (size_t)n * 4));
  return 0;
}
#endif
#ifdef SHK_SPLIT_WORK
extern "C" int shk_debug_split_work(unsigned long long* out, int reset) {
  SHK_CUDA(cudaMemcpyFromSymbol(out, g_split_work, 16));
  if (reset) {
    const unsigned long long z[2] = {0, 0};
    SHK_CUDA(cudaMemcpyToSymbol(g_split_work, z, 16));
  }
  return 0;
}
#endif
