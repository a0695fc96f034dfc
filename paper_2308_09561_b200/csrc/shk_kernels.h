// Internal launch interface between the C-ABI layer (shk_capi.cu) and the
// kernel translation units.  Everything here takes DEVICE pointers and a
// stream; nothing synchronizes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

void shk_set_error(const char* fmt, ...);

struct ShkLeafLaunch {
  const uint64_t* hi;
  const uint64_t* lo;
  const int64_t* off;
  int64_t L;
  int max_n;
  uint64_t max_seed;
  int mode;  // 0 plain, 1 rotate
  int cache_k;
  int cache_min_leaf;
  int64_t* seed_out;
  uint64_t* fbits_out;
  uint8_t* choice_out;
  int64_t* stats_out;
  int* counter;
  int* error;
  int team_warps;  // 0 = heuristic
  int num_sms;
  int stride;                     // 1: separate hi/lo arrays; 2: interleaved pairs (lo = hi + 1)
  const int64_t* seed_slot;       // optional scatter index for seed_out
  unsigned long long* stats_acc;  // optional [4] totals (evals, passes, checks, a_evals)
  int* exhausted;                 // optional flag
  int64_t* place_out;             // optional [N] global slot per key
  int pre;                        // keys' high words are already premix_hi'ed
};
int shk_launch_leaf_search(const ShkLeafLaunch& p, cudaStream_t st);
// Plain search with seed-block work stealing (shk_leaf_steal.cu): state is
// shk_leaf_steal_state_bytes(L) of device scratch, active max_active int64.
size_t shk_leaf_steal_state_bytes(int64_t L);
int shk_launch_int_peak(int kind, int iters, int num_sms, uint32_t* sink, int64_t* threads_out, int* ops_per_step,
                        cudaStream_t st);
int shk_launch_leaf_steal(const ShkLeafLaunch& p, void* state, long long* active, int max_active, int shared_counter,
                          cudaStream_t st);
int shk_launch_orient(const uint8_t* eu, const uint8_t* ev, const int64_t* off, int64_t L, uint64_t* fbits, int* ok,
                      cudaStream_t st);

// Split tasks: one per split node.  Keys of the node are [start, start + m)
// of the (bucket-sorted, partially partitioned) key arrays.
struct ShkSplitTask {
  int64_t start;
  int32_t m;
  int32_t fanout;
  int32_t sizes[4];
  int64_t seed_slot;  // index into the node seed array
};
struct ShkSplitLaunch {
  uint64_t* hi;      // interleaved (hi, lo) key pairs
  uint64_t* lo;      // unused (kept null)
  uint64_t* tmp_hi;  // scratch pairs, same size
  uint64_t* tmp_lo;  // unused
  const ShkSplitTask* tasks;
  int64_t ntasks;
  uint64_t max_seed;
  int64_t* seeds;      // per node
  int64_t* evals_out;  // per task or null
  int* counter;
  int num_sms;
  int partition;  // 1: stable-partition keys after the search
  int* exhausted; // optional flag: a node had no seed below max_seed
  unsigned long long* evals_acc;  // optional running total of split evals
  int exact_evals;  // 1: track the reference's exact `evals` (seam API); 0: fast verdict-only search
};
int shk_launch_split(const ShkSplitLaunch& p, cudaStream_t st);

// A node of a bucket-size plan (recsplit.flatten_plan + derived fields).
struct ShkPlanNode {
  int32_t kind, g, m, fanout;
  int32_t sizes[4];
  int32_t child[4];  // plan-local child indices
  int32_t off;       // key offset inside the bucket
  int32_t depth;
};
// Expand per-bucket plans into the global node table of a bucket range:
// nodes, Rice g / kind per node, and the root of every bucket in the queue.
int shk_launch_expand_nodes(const ShkPlanNode* plan_nodes, const int64_t* plan_off, const int32_t* bucket_plan,
                            const int64_t* node_base, const int64_t* key_start, const int64_t* root_pos,
                            int64_t nbuckets, struct ShkTreeNode* nodes, int32_t* node_g, uint8_t* node_kind,
                            int64_t* queue, cudaStream_t st);

// One node of a bucket range for the persistent construction kernel.
struct ShkTreeNode {
  int64_t start;     // first key (global index into the working key array)
  int32_t m;         // keys in the node
  int32_t kind;      // 0 split, 1 leaf
  int32_t fanout;    // split parts (kind 0)
  int32_t sizes[4];  // part sizes (kind 0)
  int32_t pad;
  int64_t child[4];  // global node ids of the parts (kind 0)
};
struct ShkTreeLaunch {
  uint64_t* keys;  // interleaved (hi, lo) pairs
  uint64_t* tmp;   // scratch pairs
  const ShkTreeNode* nodes;
  int64_t nnodes;
  int64_t* queue;  // [nnodes]: split region [0, nsplit) then leaf region; roots first in each; -1 = not yet published
  unsigned long long* head;  // [2] split head, leaf head
  unsigned long long* tail;  // [2] split tail, leaf tail
  int64_t nsplit;            // split nodes (size of the split region)
  int slow_wid;              // warps with %warpid >= slow_wid take leaves only; 0 = half the resident warps
  int idle_wid;              // warps with %warpid >= idle_wid take no work; 0 = none (A/B only)
  int64_t tail_reserve;      // leaf-only warps stop once fewer leaves remain (0 off, -1 auto)
  uint64_t max_seed;
  int64_t* seeds;  // per node
  int mode, cache_k, cache_min_leaf, max_n;
  uint8_t* choice_out;
  int64_t* place_out;
  unsigned long long* stats_acc;
  int* exhausted;
  int num_sms;
  const int* dup_flag;  // optional: the bucket sort's duplicate flag (nonzero: the kernel does nothing)
  // rotate search tail hand-off (required when mode != 0): the flag the kernel
  // raises once every leaf is handed out, a buffer of handoff_cap 56-byte
  // records (>= the resident warps), the count of records written and the
  // resume kernel's fetch counter (all zeroed by the caller); handoff_tw:
  // warps per resume team, 0 = no hand-off
  int* abort_flag;
  void* handoff;
  int64_t handoff_cap;
  unsigned long long* handoff_count;
  unsigned long long* handoff_next;
  int handoff_tw;
};
int shk_launch_tree(const ShkTreeLaunch& p, cudaStream_t st);

// Choice bits of build positions [k0, k1) moved to the keys' bucket-sorted
// positions (out[j - k0]); keys/sorted are interleaved pairs.
int shk_launch_choice_sorted(const uint64_t* keys, const uint64_t* sorted, const int64_t* prefix, int64_t nb,
                             const uint8_t* choice, int64_t k0, int64_t k1, uint8_t* out, cudaStream_t st);

// Bucketing.
// skeys: interleaved (hi, lo) pairs [2N], sorted by (bucket, hi, lo).
int shk_bucketize(const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nbuckets, uint64_t* skeys,
                  uint64_t* key_prefix /*[nb+1]*/, int* dup_flag, void* scratch, size_t scratch_bytes,
                  int64_t* max_bucket_out, cudaStream_t st,
                  uint64_t* h_prefix = nullptr /* host [nb+1]: early prefix, no wait for the sort */);
size_t shk_bucketize_scratch(int64_t N, int64_t nbuckets);

// Generic exclusive scan of int64 (n elements) -> out[n+1] (out[n] = total).
int shk_exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* scratch, size_t scratch_bytes,
                           cudaStream_t st);
size_t shk_scan_scratch(int64_t n);

// Rice: node seeds + g -> bit lengths; scan; scatter into zeroed words.
int shk_rice_lengths(const int64_t* seeds, const int32_t* g, int64_t nn, int64_t* len, cudaStream_t st);
int shk_rice_scatter(const int64_t* seeds, const int32_t* g, const int64_t* pos, int64_t nn, uint64_t* words,
                     cudaStream_t st);

// Ribbon.
struct ShkRibbon;
int shk_ribbon_create(ShkRibbon** out);
void shk_ribbon_destroy(ShkRibbon* r);
// rows from keys (seed) -> solve; words_out device [ceil(m/64)]; *consistent set.
// keys: interleaved (hi, lo) pairs [2N].
int shk_ribbon_solve_keys(ShkRibbon* r, const uint64_t* keys, const uint8_t* rhs, int64_t N, int64_t m,
                          uint64_t seed, uint64_t* words_out, int* consistent, cudaStream_t st);
// explicit rows
int shk_ribbon_solve_rows(ShkRibbon* r, const int64_t* starts, const uint64_t* p0, const uint64_t* p1,
                          const uint8_t* rhs, int64_t N, int64_t m, uint64_t* words_out, int* consistent,
                          cudaStream_t st);
// column-sharded solve (shk_ribbon.cu): rows are 24 bytes (p0, p1, start | rhs << 62)
int shk_ribbon_dist_begin(ShkRibbon* r, const uint64_t* keys, const uint8_t* rhs, int64_t N, int64_t m,
                          uint64_t seed, int64_t c0, int64_t c1, int64_t* n_export, int* bad, cudaStream_t st);
int shk_ribbon_dist_take_exports(ShkRibbon* r, void* rows_out, int64_t n, cudaStream_t st);
int shk_ribbon_dist_import(ShkRibbon* r, const void* rows_in, int64_t n, int64_t* n_export, int* bad,
                           cudaStream_t st);
int shk_ribbon_dist_backsub(ShkRibbon* r, const uint32_t* y_in, uint32_t* y_out, uint64_t* words_out,
                            cudaStream_t st);
int shk_ribbon_dist_map(ShkRibbon* r, uint32_t* map_out, cudaStream_t st);
int shk_ribbon_dist_finish(ShkRibbon* r, const uint32_t* y_in, uint64_t* words_out, cudaStream_t st);
int shk_launch_ribbon_rows(const uint64_t* hi, const uint64_t* lo, int stride, int64_t N, int64_t m, uint64_t seed,
                           int64_t* starts, uint64_t* p0, uint64_t* p1, cudaStream_t st);
// Split-hash part index of every key (split_parts seam).
int shk_launch_split_parts(const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed, const int64_t* sizes,
                           int fanout, int64_t* parts, cudaStream_t st);
// Pack separate hi/lo arrays into interleaved pairs.
int shk_launch_interleave(const uint64_t* hi, const uint64_t* lo, int64_t N, uint64_t* pairs, cudaStream_t st);
int shk_launch_deinterleave(const uint64_t* pairs, int64_t N, uint64_t* hi, uint64_t* lo, cudaStream_t st);
// premix_hi (inverse = 0) or unpremix_hi (inverse = 1) of the high words of
// interleaved key pairs, in place: the build's seed searches (split kernels,
// tree kernel, build-path leaves) take pre-mixed keys.
int shk_launch_premix(uint64_t* pairs, int64_t N, int inverse, cudaStream_t st);
int shk_launch_ribbon_query(const int64_t* starts, const uint64_t* p0, const uint64_t* p1, int64_t N,
                            const uint64_t* words, int64_t nwords, uint8_t* out, cudaStream_t st);

// Query.
struct ShkQueryDesc {
  int64_t nbuckets;
  int64_t n_keys;
  int mode;
  int64_t cache_k;
  const uint64_t* key_prefix;   // [nb+1]
  const int32_t* bucket_plan;   // [nb]  plan id (or -1 for empty)
  const int64_t* node_base;     // [nb]  first global node of the bucket
  const uint64_t* node_val;     // [total nodes] decoded node: split -> premixed seed mixer, leaf -> seed
  // query-side packed tables:
  //   bucketq[b]: {kp0 lo, kp0 hi8 | node_base hi8 << 8 | bad16 << 16, node_base lo,
  //                plan first node (0xFFFFFFFF: empty bucket)}
  //   planq[j]: {m | leaf << 15 | b1 << 16, b2 | b3 << 16, c0 | c1 << 16, c2 | c3 << 16}
  //             (b_k cumulative part bounds, 0xFFFF past the fanout; c_k plan-local children)
  const uint4* bucketq;
  const uint4* planq;
  const int32_t* bucket_bad;    // [nb]  first node whose decode overran (INT32_MAX none)
  const uint64_t* bit_offsets;  // [nb+1] stream bit offset of each bucket
  const uint64_t* stream;       // words
  int64_t stream_bit_len;
  int64_t stream_nwords;
  const int32_t* pn_kind;       // plan nodes, concatenated
  const int32_t* pn_g;
  const int32_t* pn_m;
  const int32_t* pn_child;      // [node][4] plan-local child index
  const int32_t* pn_sizes;      // [node][4]
  const int32_t* pn_fanout;
  const int64_t* plan_off;      // [nplans+1]
  uint64_t rib_seed;
  int64_t rib_m;
  const uint64_t* rib_words;
  int64_t rib_nwords;
};
int shk_launch_node_index(const ShkQueryDesc& d, uint64_t* node_val, int32_t* bucket_bad, cudaStream_t st);
int shk_launch_query(const ShkQueryDesc& d, const uint64_t* hi, const uint64_t* lo, int64_t Q, uint64_t* out,
                     int* err, int clamp, cudaStream_t st);
// Bijection check of Q values against [0, N): *offender = first index whose
// value is out of range or repeats an earlier one (all ones if none).
// first: N scratch slots.
int shk_launch_bijection(const uint64_t* v, int64_t Q, int64_t N, unsigned long long* first,
                         unsigned long long* offender, cudaStream_t st);

// Rice-decode a sequence of codes (test / seam parity).
int shk_launch_rice_decode(const uint64_t* words, int64_t bit_len, int64_t pos, const int32_t* g, int64_t count,
                           int64_t* values, int64_t* positions, int* err, cudaStream_t st);

// blake2b-128 master hash over CSR byte keys.
int shk_launch_blake2b(const uint8_t* blob, const int64_t* off, int64_t N, uint64_t salt, uint64_t* hi,
                       uint64_t* lo, cudaStream_t st);
int shk_launch_blake2b_fixed(const uint8_t* blob, int key_len, int64_t N, uint64_t salt, uint64_t* hi, uint64_t* lo,
                             cudaStream_t st);

// Analysis kernels (shk_experiments.cu).
int shk_launch_brute(const uint64_t* khi, const uint64_t* klo, int n, uint64_t base, uint64_t count,
                     unsigned long long* found, unsigned long long* evals, int num_sms, cudaStream_t st);
int shk_launch_mc_filter(const uint64_t* khi, const uint64_t* klo, int n, uint64_t count,
                         unsigned long long* passes, int num_sms, cudaStream_t st);
int shk_launch_enumerate(int n, unsigned long long* out, int num_sms, cudaStream_t st);
int shk_launch_route(const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                     const int64_t* bounds, int W, unsigned long long* counts_dev, unsigned long long* cursors_dev,
                     uint64_t* out, uint8_t* aux_out, int64_t* counts_host, cudaStream_t st);
int shk_launch_route_count(const uint64_t* keys, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                           const int64_t* bounds, int W, unsigned long long* counts_dev, int64_t* counts_host,
                           cudaStream_t st);
int shk_launch_route_p2p(const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                         const int64_t* bounds, int W, void* const* peer_bufs, const int64_t* peer_base, int64_t cap,
                         unsigned long long* cursors_dev, cudaStream_t st);
