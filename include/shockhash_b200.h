/*
 * shockhash_b200.h - C-ABI of the B200-native ShockHash hot path.
 *
 * The reference's drop-in seam for this path is the kernel module object
 * `shockhash._kernels.kernels` (/root/reference/pkg/src/shockhash/_kernels/
 * __init__.py:23), whose functions are defined in _core.pyx / _pure.py.  Every
 * batched entry point below replaces one of them (cited per function); the
 * orchestration entry points replace the per-bucket Python loop of
 * recsplit._build_hashed (recsplit.py:474-550) and MphfDescriptor.query_*
 * (recsplit.py:251-285).  Plain pointers and sizes only, no torch types.
 *
 * Conventions
 *   - Return value: SHK_OK (0) or an SHK_* code below; negative = CUDA error,
 *     text via shk_last_error().
 *   - flags & SHK_DEVICE: every array argument is a device pointer and the
 *     call is stream-ordered on the context's stream (no host sync).  Without
 *     it, arrays are host memory; the library copies them and returns when
 *     the outputs are written.
 *   - Keys are 128-bit master hash codes (hi, lo) as two uint64 arrays.
 *   - A context is single-owner and not thread-safe (one per host thread).
 *   - There is no CPU fallback: without a usable B200 every compute call
 *     fails with a negative code.
 */
#ifndef SHOCKHASH_B200_H
#define SHOCKHASH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SHK_OK = 0,
  SHK_EXHAUSTED = 1,  /* seed search hit max_seed -> ConstructionFailureError */
  SHK_FORMAT = 2,     /* bit-stream overrun -> FormatError */
  SHK_INVALID = 3,    /* bad parameter -> InvalidParameterError */
  SHK_UNSOLVABLE = 4, /* ribbon inconsistent for every tried seed */
  SHK_DUPLICATE = 5   /* equal 128-bit codes in a build */
};
#define SHK_DEVICE 1
/* shk_blake2b128_fixed only: the key blob is host memory (page-locked for
 * full speed), hi/lo are device pointers; the copy is pipelined in chunks
 * with the hashing (copy stream + main stream). */
#define SHK_BLOB_HOST 2
/* shk_build_create only: return as soon as the key prefix is on the host
 * (*dup = -1, unknown): the scatter and the sort keep running, and the caller
 * prepares run() meanwhile.  run() then waits for the duplicate flag just
 * before its first search kernel and returns SHK_DUPLICATE if it is set;
 * shk_build_duplicate reads it explicitly.  Device inputs (hi, lo) must stay
 * valid until one of those two calls returns (the scatter still reads them). */
#define SHK_BUILD_ASYNC 8

typedef struct shk_ctx shk_ctx;
typedef struct shk_build shk_build;
typedef struct shk_qdesc shk_qdesc;

const char* shk_last_error(void);
int shk_version(void);
int shk_device_count(int* n);
int shk_ctx_create(int device, shk_ctx** out);
int shk_ctx_destroy(shk_ctx* ctx);
int shk_ctx_sync(shk_ctx* ctx);
/* cudaStream_t of the context; shk_ctx_set_stream(ctx, NULL) restores the
 * context's own stream. */
void* shk_ctx_stream(shk_ctx* ctx);
int shk_ctx_set_stream(shk_ctx* ctx, void* stream);
int shk_ctx_num_sms(shk_ctx* ctx);
/* Tuning / instrumentation options of a context. */
enum {
  SHK_OPT_EXACT_SPLIT_EVALS = 0, /* 1: builds also count the reference's split `evals` (slower) */
  SHK_OPT_LEAF_TEAM_WARPS = 1,   /* warps per leaf in the per-level schedule (0 = heuristic) */
  SHK_OPT_SCHEDULE = 2,          /* 0: one persistent task-queue launch per build; 1: one launch per level */
  SHK_OPT_LEAF_FIXED_TEAMS = 3   /* 1: batched PLAIN leaf search with a fixed team per leaf (no seed-block
                                    stealing; A/B only) */
};
int shk_ctx_set_option(shk_ctx* ctx, int opt, int64_t value);
/* Fused route + all-to-all over peer memory (input-sharded build): count
 * the keys per owner rank (as shk_route), then store every key (and its aux
 * byte) straight into the owner's receive buffer -- peer_bufs[d] is this
 * process's mapping of rank d's buffer (CUDA IPC: shk_ipc_buffer_alloc +
 * shk_ipc_counter_open, which maps any IPC handle), laid out as cap keys of
 * 16 B then cap aux bytes; this rank's keys for d land at slots
 * [peer_base[d], peer_base[d] + count_d).  Synchronous; the caller orders
 * the receivers' reads after every sender's return (a barrier). */
int shk_route_count(shk_ctx* ctx, const uint64_t* keys, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                    const int64_t* bounds, int W, int64_t* counts_out);
int shk_route_p2p(shk_ctx* ctx, const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm,
                  uint64_t seed, const int64_t* bounds, int W, void* const* peer_bufs, const int64_t* peer_base,
                  int64_t cap);
int shk_ipc_buffer_alloc(shk_ctx* ctx, size_t bytes, void* handle_out, void** dev_ptr);
/* Cross-GPU leaf queue for the batched PLAIN leaf search (no reference
 * counterpart: the reference is single-threaded).  One rank allocates a
 * device counter and exports its CUDA IPC handle (64 bytes); every rank
 * opens it and sets it on its context; then every rank launches
 * shk_leaf_search over ALL leaves (device buffers pre-set: seeds to a value
 * < -1, fbits to 0) and the launches take leaves from the one counter (NVLink
 * system-scope atomics), so the ranks finish together however the per-leaf
 * seed counts fall.  Each leaf is written by exactly one rank; a MAX / SUM
 * all-reduce of the seed / f-bit arrays completes every rank's copy.  The
 * owner resets the counter (shk_ipc_counter_reset) before each batch. */
int shk_ipc_counter_alloc(shk_ctx* ctx, void* handle_out, void** dev_ptr);
int shk_ipc_counter_open(shk_ctx* ctx, const void* handle, void** dev_ptr);
int shk_ipc_counter_close(shk_ctx* ctx, void* dev_ptr, int owner);
int shk_ipc_counter_reset(shk_ctx* ctx, void* dev_ptr);
int shk_ctx_set_leaf_counter(shk_ctx* ctx, void* dev_ptr); /* NULL: the context's own counter */
/* Integer-issue microbenchmark (measurement only; the reference has no
 * counterpart): one timed launch of 8 independent 32-bit chains per thread,
 * 64 warps per SM.  kind 0: LOP3, 1: IMAD, 2: LOP3+IMAD 1:1, 3: SHF+LOP3+IMAD
 * 2:1:1.  Returns the device time and the int32 ops executed. */
int shk_int_peak(shk_ctx* ctx, int kind, int iters, double* ms_out, double* ops_out);
/* Device memory from the context's caching pool (bench / zero-copy users). */
int shk_dev_alloc(shk_ctx* ctx, size_t bytes, void** out);
/* Page-locked host memory (host<->device copies at full PCIe/C2C rate, and
 * asynchronous on the context stream). */
int shk_host_alloc(shk_ctx* ctx, size_t bytes, void** out);
int shk_host_free(shk_ctx* ctx, void* p);
int shk_dev_free(shk_ctx* ctx, void* p);
int shk_memcpy(shk_ctx* ctx, void* dst, const void* src, size_t bytes, int kind /*0 H2D 1 D2H 2 D2D*/);
/* Stream-ordered byte fill of device memory (value & 0xFF). */
int shk_memset(shk_ctx* ctx, void* dst, int value, size_t bytes);
/* Exclusive prefix sum of n int64 device values into out[0..n] (out[n] = the
 * total), stream-ordered, synchronous on return: the scan every build stage
 * uses (recsplit.py:485 key_prefix = cumsum(counts), the Rice code offsets,
 * the ribbon's chunk offsets). */
int shk_exclusive_scan(shk_ctx* ctx, const int64_t* in, int64_t* out, int64_t n);
/* Events on the context stream: elapsed milliseconds between two records. */
int shk_timer_start(shk_ctx* ctx);
int shk_timer_stop(shk_ctx* ctx, float* ms);
/* Number of kernels this library launched since context creation. */
int64_t shk_launch_count(shk_ctx* ctx);

/* ---- scalar hash family (__host__ __device__ source shared with kernels):
 * mix64 _core.pyx:45-48, seed_mixer :51-52, remix :55-56, hash_range :59-60,
 * leaf_pair :79-98, split_bit :101-102, leaf_cell :751-771 */
uint64_t shk_mix64(uint64_t z);
uint64_t shk_seed_mixer(uint64_t seed, uint64_t tag);
uint64_t shk_remix(uint64_t hi, uint64_t lo, uint64_t seed, uint64_t tag);
uint64_t shk_hash_range(uint64_t v, uint64_t m);
void shk_leaf_pair(uint64_t hi, uint64_t lo, uint64_t seed, int n, int* h0, int* h1);
int shk_split_bit(uint64_t hi, uint64_t lo, uint64_t seed);
int shk_leaf_cell(uint64_t hi, uint64_t lo, int64_t q, int mleaf, int mode, int64_t cache_k, int choice);

/* ---- leaf seed search, batched over L leaves in CSR form (leaf i = keys
 * [leaf_off[i], leaf_off[i+1]), 1..64 keys).  Replaces search_plain
 * (_core.pyx:186-229) for mode 0 and search_rotate(hi, lo, n, cache_k, ...)
 * (_core.pyx:238-334) for mode 1, plus the orientation of the found seed
 * (shockhash._finish -> pseudoforest.orient, pseudoforest.py:149-201).
 * cache_k applies to leaves with more than cache_min_leaf keys (0 = always,
 * matching the raw kernel; 32 = recsplit's rule, recsplit.py:577).
 * seed_out[L]: minimum seed / encoded rotate seed, -1 if none < max_seed.
 * fbits_out[L] (nullable): bit i = choice of key i.  stats_out[L*4]
 * (nullable): (hash_evals, filter_passes, exact_checks, a_evals).
 * team_warps: warps cooperating on one leaf (0 = heuristic, else 1/2/4/8). */
int shk_leaf_search(shk_ctx* ctx, int mode, int cache_k, int cache_min_leaf, const uint64_t* hi, const uint64_t* lo,
                    const int64_t* leaf_off, int64_t L, uint64_t max_seed, int team_warps, int64_t* seed_out,
                    uint64_t* fbits_out, int64_t* stats_out, int flags);

/* ---- canonical 1-orientation of L edge lists (pseudoforest.orient,
 * pseudoforest.py:149-201).  eu/ev: cells per edge, CSR leaf_off (n <= 64
 * edges on n cells).  ok_out[i] = 0 if list i is not a pseudoforest. */
int shk_orient(shk_ctx* ctx, const uint8_t* eu, const uint8_t* ev, const int64_t* leaf_off, int64_t L,
               uint64_t* fbits_out, int32_t* ok_out, int flags);

/* ---- split-seed search on one node (split_seed_search, _core.pyx:385-428)
 * and part indices (split_parts, _core.pyx:378-382).  fanout <= 4. */
int shk_split_search(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, int64_t m, const int64_t* sizes,
                     int fanout, uint64_t max_seed, int64_t* seed_out, int64_t* evals_out);
int shk_split_parts(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed,
                    const int64_t* sizes, int fanout, int64_t* parts_out);

/* ---- ribbon retrieval.  rows: ribbon_rows (_core.pyx:435-439); solve:
 * ribbon_solve (_core.pyx:442-524) -> *consistent = 0 when the system is
 * inconsistent (reference returns None); query: ribbon_query_many
 * (_core.pyx:548-568); build: the seed loop of retrieval_build_arrays
 * (retrieval.py:93-106) over seeds [0, max_tries). */
int shk_ribbon_rows(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t m, uint64_t seed,
                    int64_t* starts, uint64_t* pat0, uint64_t* pat1, int flags);
int shk_ribbon_solve(shk_ctx* ctx, const int64_t* starts, const uint64_t* pat0, const uint64_t* pat1,
                     const uint8_t* rhs, int64_t N, int64_t m, uint64_t* words_out, int* consistent, int flags);
int shk_ribbon_query(shk_ctx* ctx, const int64_t* starts, const uint64_t* pat0, const uint64_t* pat1, int64_t N,
                     const uint64_t* words, int64_t nwords, uint8_t* out, int flags);
int shk_ribbon_build(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, const uint8_t* rhs, int64_t N, int64_t m,
                     int max_tries, uint64_t* seed_out, uint64_t* words_out, int flags);

/* ---- Rice stream decode of `count` consecutive codes starting at bit pos
 * (rice_decode_stream, _core.pyx:626-635, applied repeatedly). */
int shk_rice_decode(shk_ctx* ctx, const uint64_t* words, int64_t nwords, int64_t bit_len, int64_t pos,
                    const int32_t* g, int64_t count, int64_t* values_out, int64_t* pos_out);

/* ---- master hash: blake2b-128 with salt (keys.master_hash_many,
 * keys.py:46-58).  Keys are a byte blob with CSR offsets off[N+1]. */
int shk_blake2b128(shk_ctx* ctx, const uint8_t* blob, int64_t blob_len, const int64_t* off, int64_t N, uint64_t salt,
                   uint64_t* hi, uint64_t* lo, int flags);
/* Same for N keys of key_len (1..128) bytes each, back to back (the
 * benchmark's 8-byte little-endian keys). */
int shk_blake2b128_fixed(shk_ctx* ctx, const uint8_t* blob, int key_len, int64_t N, uint64_t salt, uint64_t* hi,
                         uint64_t* lo, int flags);

/* ---- analysis entry points of the kernel seam (used by experiments.py).
 * search_bruteforce (_core.pyx:337-371): minimum seed in [0, max_seed) whose
 * single n-range hash is a bijection of the n keys (host hi/lo, n <= 64), or
 * -1; *evals_out = the reference's evals counter.
 * mc_filter_pass_count (_core.pyx:832-860): seeds in [0, trials) passing the
 * all-cells-hit filter on the synthetic key set derived from `entropy`.
 * enumerate_outcomes (_core.pyx:778-829): over all (n^2)^n ordered cell-pair
 * tuples, the pseudoforest count and the sum of 2^components (n <= 8). */
int shk_search_bruteforce(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, int n, uint64_t max_seed,
                          int64_t* seed_out, int64_t* evals_out);
int shk_mc_filter_pass_count(shk_ctx* ctx, int n, int64_t trials, uint64_t entropy, int64_t* passes_out);
int shk_enumerate_outcomes(shk_ctx* ctx, int n, uint64_t* pf_count_out, uint64_t* sum_2c_out);

/* ---- plan tables (recsplit.flatten_plan, recsplit.py:95-119), one per
 * distinct bucket size, concatenated: plan p covers nodes
 * [plan_off[p], plan_off[p+1]); node fields are the reference's arrays
 * (kind 0 split / 1 leaf, g, fanout, sizes_off into sizes_flat, subtree,
 * m_node).  sizes_off is plan-local (as flatten_plan returns it); each plan's
 * sizes start at sizes_base[p] in sizes_flat. */
typedef struct shk_plans {
  int64_t nplans;
  const int64_t* plan_m;     /* bucket size of each plan */
  const int64_t* plan_off;   /* [nplans+1] */
  const int64_t* sizes_base; /* [nplans] */
  const int64_t* kind;
  const int64_t* g;
  const int64_t* fanout;
  const int64_t* sizes_off;
  const int64_t* subtree;
  const int64_t* m_node;
  const int64_t* sizes_flat;
} shk_plans;

/* ---- MPHF construction (recsplit._build_hashed, recsplit.py:474-550).
 * create: bucket hash, sort by (bucket, hi, lo), key_prefix, duplicate flag
 *   (recsplit.py:475-483, :433-440).  *dup != 0 means equal 128-bit codes.
 * run: split-seed searches + stable partitions, leaf searches, orientation
 *   and the Rice stream for buckets [b0, b1) (recsplit.py:499-521).
 * ribbon: retrieval over ALL keys with the choice bits (recsplit.py:523);
 *   choice (nullable, host or device per flags) overrides the build's own.
 * stats_out[8] of run: hash_evals, filter_passes, exact_checks, a_evals,
 *   leaf_seed_bits, split_seed_bits, leaf_count (recsplit.py:539-547), and
 *   the number of leaves the persistent kernel handed to the resume teams
 *   at its tail (rotate modes; SHK_TREE_HANDOFF_TW, diagnostic only). */
int shk_build_create(shk_ctx* ctx, const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nbuckets, int flags,
                     shk_build** out, int* dup, int64_t* max_bucket);
int shk_build_duplicate(shk_build* b, int* dup /* 0 or 1; waits for the sort */);
int shk_build_key_prefix(shk_build* b, uint64_t* key_prefix /* [nb+1] host */);
int shk_build_sorted_keys(shk_build* b, uint64_t* hi, uint64_t* lo /* [N] host */);
int shk_build_run(shk_build* b, const shk_plans* plans, int mode, int cache_k, int cache_min_leaf, int64_t b0,
                  int64_t b1, uint64_t max_seed, int64_t* stats_out);
int shk_build_stream_size(shk_build* b, int64_t* bit_len, int64_t* nwords);
int shk_build_stream(shk_build* b, uint64_t* words /* [nwords] */, uint64_t* bit_offsets /* [b1-b0+1] */);
int shk_build_choice(shk_build* b, uint8_t* choice /* [N] host, sorted key order */);
/* record_placements (recsplit.py:493, :592-594): global slot of every sorted
 * key as placed at construction time; enable before shk_build_run. */
int shk_build_set_record_placements(shk_build* b, int on);
int shk_build_placements(shk_build* b, int64_t* out /* [N] host */);
/* Sharded builds (dist.py): a rank builds only its bucket range, so only that
 * range of its key array is permuted into leaf order.  With keep_sorted (set
 * before shk_build_run) the bucket-sorted keys are kept, choice_sorted returns
 * the choice bits of key positions [k0, k1) re-ordered to the sorted order,
 * and shk_build_ribbon with choice_flags & SHK_RIBBON_SORTED_KEYS builds the
 * ribbon rows from the sorted keys (choice given in sorted order).  The
 * ribbon solution does not depend on row order. */
#define SHK_RIBBON_SORTED_KEYS 4
int shk_build_set_keep_sorted(shk_build* b, int on);
int shk_build_choice_sorted(shk_build* b, int64_t k0, int64_t k1, uint8_t* out /* [k1-k0] */,
                            int flags /* SHK_DEVICE: out is a device pointer (no sync) */);
/* Column-sharded ribbon (SURVEY.md §8(e) option B) over the kept sorted keys:
 * this rank owns columns [c0, c1) (multiples of 8192 except c1 = m).
 * begin eliminates the rows that start in the range (choice_sorted: all N
 * choice bits in sorted order, host or, with flags & SHK_DEVICE, device); rows whose pivot leaves the range are
 * exported (24 bytes each: p0, p1, start | rhs << 62, global columns) for the
 * right neighbour, which imports them (and may export further).  *bad = 1:
 * the system is inconsistent (next seed).  When no rank exports, backsub runs
 * right to left across ranks: y_in = the right neighbour's first 127 solution
 * bits (4 words, zero for the last range), y_out = this range's, words_out =
 * its (c1 - c0 + 63) / 64 solution words (host). */
int shk_build_dribbon_begin(shk_build* b, const uint8_t* choice_sorted, int flags, int64_t m, uint64_t seed,
                            int64_t c0, int64_t c1, int64_t* n_export, int* bad);
/* Input-sharded multi-GPU build (dist.py; no reference counterpart): the
 * column-sharded ribbon fed with explicit keys (device, interleaved (hi, lo)
 * pairs) and rhs bytes that were routed to this rank, and the device
 * pointers of a finished build's keys in leaf order and their choice bytes. */
int shk_build_dribbon_begin_keys(shk_build* b, const uint64_t* keys_dev, const uint8_t* rhs_dev, int64_t n, int64_t m,
                                 uint64_t seed, int64_t c0, int64_t c1, int64_t* n_export, int* bad);
int shk_build_leaf_arrays(shk_build* b, void** keys_dev, void** choice_dev);
/* Partition n keys (device, interleaved pairs) by owner rank -- kind 0: the
 * rank owning the key's bucket (nbm = number of buckets), kind 1: the rank
 * owning its ribbon row's start column (nbm = m, seed = ribbon seed); rank r
 * owns values [bounds[r], bounds[r+1]) (host array of W+1).  keys_out /
 * aux_out (device) receive the keys (and the optional per-key byte aux)
 * grouped by rank; counts_out (host, W) the group sizes.  Synchronous. */
int shk_route(shk_ctx* ctx, const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
              const int64_t* bounds, int W, uint64_t* keys_out, uint8_t* aux_out, int64_t* counts_out);
int shk_build_dribbon_exports(shk_build* b, void* rows_out, int64_t n);
int shk_build_dribbon_import(shk_build* b, const void* rows_in, int64_t n, int64_t* n_export, int* bad);
int shk_build_dribbon_backsub(shk_build* b, const uint32_t* y_in, uint32_t* y_out, uint64_t* words_out);
/* Parallel form of the right-to-left pass: map computes this range's
 * back-substitution forms and returns its boundary map (map_out: 128 rows of
 * 4 words; row j < 127 = the range's first 127 solution bits when the 127
 * bits right of it are e_j, row 127 = when they are zero; the map is affine
 * over GF(2)).  Every rank composes the maps of the ranks to its right into
 * its own y_in (no serial hand-off), then finish runs the chain and the
 * final map (words_out as in backsub). */
int shk_build_dribbon_map(shk_build* b, uint32_t* map_out /* [128][4] host */);
int shk_build_dribbon_finish(shk_build* b, const uint32_t* y_in, uint64_t* words_out);
int shk_build_ribbon(shk_build* b, const uint8_t* choice, int choice_flags, int64_t m, int max_tries,
                     uint64_t* seed_out, uint64_t* words_out /* [ceil(m/64)] host */);
/* Device time of the last phases (CUDA events on the context stream), ms:
 * [0] bucketize [1] split searches [2] leaf searches [3] Rice stream
 * [4] ribbon; split_evals = the reference's split `evals` counter summed. */
int shk_build_phase_ms(shk_build* b, float* ms /* [5] */, int64_t* split_evals);
/* Device ms of each split level (one launch per tree depth) of the last run;
 * returns the number of levels written. */
int shk_build_level_ms(shk_build* b, float* ms, int32_t* depth, int max_levels);
int shk_build_destroy(shk_build* b);

/* ---- MPHF evaluation (MphfDescriptor.query_hashed_many ->
 * query_stream, _core.pyx:642-742).  create uploads the descriptor and builds
 * the per-node bit-position index; query returns SHK_FORMAT where the
 * reference raises FormatError.  clamp=1 applies min(out, N-1)
 * (recsplit.py:275). */
int shk_qdesc_create(shk_ctx* ctx, int64_t n_keys, int64_t nbuckets, int mode, int64_t cache_k,
                     const uint64_t* key_prefix, const uint64_t* bit_offsets, const uint64_t* stream_words,
                     int64_t stream_nwords, int64_t stream_bit_len, const shk_plans* plans, uint64_t rib_seed,
                     int64_t rib_m, const uint64_t* rib_words, int64_t rib_nwords, shk_qdesc** out);
int shk_query(shk_qdesc* d, const uint64_t* hi, const uint64_t* lo, int64_t Q, uint64_t* out, int clamp, int flags);
/* MphfDescriptor.query_many(keys) end to end (recsplit.py:270-275): N
 * fixed-length keys packed in a HOST buffer (page-locked for full PCIe
 * rate) -> indices in a host array.  Chunks are copied in, fingerprinted
 * (blake2b-128, salt) and queried on the device while the neighbouring
 * chunks' copies run (two copy streams).  clamp as shk_query. */
int shk_query_blob(shk_qdesc* q, const uint8_t* blob, int key_len, int64_t Q, uint64_t salt, uint64_t* out, int clamp);
/* MphfDescriptor.verify (recsplit.py:383-394) on the device: query the Q
 * hashed keys (clamped) and check the outputs form a bijection onto [0, N).
 * *ok = 1 iff so; otherwise *offender = the first input index whose output is
 * out of range or repeats an earlier input's (-1 when Q != N). */
int shk_verify(shk_qdesc* d, const uint64_t* hi, const uint64_t* lo, int64_t Q, int flags, int* ok,
               int64_t* offender);
int shk_qdesc_destroy(shk_qdesc* d);

#ifdef __cplusplus
}
#endif
#endif /* SHOCKHASH_B200_H */
