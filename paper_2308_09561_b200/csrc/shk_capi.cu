// C-ABI of the B200 ShockHash hot path (declared in include/shockhash_b200.h)
// plus the native build/query runtime: device memory pool, stream, plan
// tables, level-by-level split scheduling, leaf batches, Rice stream
// assembly and the ribbon seed loop.  Replaces the Python orchestration of
// recsplit._build_hashed (recsplit.py:474-594) and query_hashed_many
// (recsplit.py:251-275).
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../include/shockhash_b200.h"
#include "shk_common.cuh"
#include "shk_kernels.h"

// (analysis) SHK_HOST_TRACE=1: host timestamps of the build's stages, us
// since the build object was created, on stderr
static double host_now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static bool host_trace_on() {
  static const bool on = getenv("SHK_HOST_TRACE") != nullptr;
  return on;
}
static double g_host_t0 = 0;
#define HOST_TRACE(tag) \
  do { \
    if (host_trace_on()) fprintf(stderr, "host %-24s %9.1f us\n", tag, host_now_us() - g_host_t0); \
  } while (0)

// ---------------------------------------------------------------------------
// errors / launch counting

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void shk_set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

void shk_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

#define RC(x)            \
  do {                   \
    int rc_ = (x);       \
    if (rc_) return rc_; \
  } while (0)

// ---------------------------------------------------------------------------
// context + caching device pool

struct shk_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // side stream for pipelined host->device copies
  cudaStream_t copy_out = nullptr;  // side stream for pipelined device->host copies
  int num_sms = 148;
  std::multimap<size_t, void*> free_blocks;
  std::unordered_map<void*, size_t> live;
  int* d_counter = nullptr;  // scratch ints: [0] counter [1] flag [2] flag
  int* h_flags = nullptr;    // pinned host ints (a ring of per-build duplicate flags)
  unsigned flag_next = 0;
  ShkRibbon* rib = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int64_t opt[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // shk_ctx_set_option
  int* shared_leaf_counter = nullptr;  // shk_ctx_set_leaf_counter (cross-GPU leaf queue)
  struct PlanCache* plans = nullptr;   // the last build's plan tables, host and device (plan_cache)
  void* h_stage = nullptr;             // pinned staging for the per-build tables (one H2D copy)
  size_t h_stage_cap = 0;
};
static void plan_cache_free(shk_ctx* c);

static size_t round_up(size_t b) {
  if (b < 256) return 256;
  if (b < (1u << 20)) return (b + 255) & ~(size_t)255;
  return (b + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);
}

static int pool_alloc(shk_ctx* c, size_t bytes, void** out) {
  size_t b = round_up(bytes);
  auto it = c->free_blocks.lower_bound(b);
  if (it != c->free_blocks.end() && it->first <= b * 2) {
    *out = it->second;
    c->live[it->second] = it->first;
    c->free_blocks.erase(it);
    return 0;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, b);
  if (e != cudaSuccess) {
    // release cached blocks and retry once
    cudaGetLastError();
    for (auto& kv : c->free_blocks) cudaFree(kv.second);
    c->free_blocks.clear();
    SHK_CUDA(cudaMalloc(&p, b));
  }
  c->live[p] = b;
  *out = p;
  return 0;
}

static void pool_free(shk_ctx* c, void* p) {
  if (!p) return;
  auto it = c->live.find(p);
  if (it == c->live.end()) return;
  c->free_blocks.emplace(it->second, p);
  c->live.erase(it);
}

// RAII device buffer from the pool.
struct DBuf {
  shk_ctx* c = nullptr;
  void* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(shk_ctx* ctx) : c(ctx) {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (c && p) pool_free(c, p);
    p = nullptr;
    n = 0;
  }
  int alloc(size_t bytes) {
    release();
    n = bytes;
    return pool_alloc(c, bytes ? bytes : 1, &p);
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

static int h2d(shk_ctx* c, void* d, const void* h, size_t n) {
  if (n) SHK_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c->stream));
  return 0;
}
static int d2h(shk_ctx* c, void* h, const void* d, size_t n) {
  if (n) SHK_CUDA(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, c->stream));
  return 0;
}
static int csync(shk_ctx* c) {
  SHK_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

// Stage a possibly-host input array into device memory.
static int stage_in(shk_ctx* c, int flags, const void* src, size_t bytes, DBuf& tmp, const void** dev) {
  if (flags & SHK_DEVICE) {
    *dev = src;
    return 0;
  }
  RC(tmp.alloc(bytes));
  RC(h2d(c, tmp.p, src, bytes));
  *dev = tmp.p;
  return 0;
}
// Output: device pointer to write to (either the caller's or a temp).
static int stage_out(shk_ctx* c, int flags, void* dst, size_t bytes, DBuf& tmp, void** dev) {
  if (!dst) {
    *dev = nullptr;
    return 0;
  }
  if (flags & SHK_DEVICE) {
    *dev = dst;
    return 0;
  }
  RC(tmp.alloc(bytes));
  *dev = tmp.p;
  return 0;
}
static int finish_out(shk_ctx* c, int flags, void* dst, const DBuf& tmp, size_t bytes) {
  if (!dst || (flags & SHK_DEVICE)) return 0;
  return d2h(c, dst, tmp.p, bytes);
}

extern "C" {

const char* shk_last_error(void) { return g_err.c_str(); }
int shk_version(void) { return 10000; }
int64_t shk_launch_count(shk_ctx*) { return g_launches.load(); }

int shk_device_count(int* n) {
  int k = 0;
  cudaError_t e = cudaGetDeviceCount(&k);
  if (e != cudaSuccess) {
    cudaGetLastError();
    k = 0;
  }
  *n = k;
  return 0;
}

int shk_ctx_create(int device, shk_ctx** out) {
  int n = 0;
  shk_device_count(&n);
  if (n <= 0) {
    shk_set_error("no CUDA device available: the B200 path has no CPU fallback");
    return -1;
  }
  SHK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SHK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    shk_set_error("device %d is sm_%d%d; this library is built for sm_100a (B200)", device, prop.major, prop.minor);
    return -2;
  }
  shk_ctx* c = new shk_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  SHK_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  SHK_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  SHK_CUDA(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
  c->stream = c->own;
  SHK_CUDA(cudaMalloc(&c->d_counter, 256));
  SHK_CUDA(cudaMallocHost(&c->h_flags, 64 * sizeof(int)));
  SHK_CUDA(cudaEventCreate(&c->t0));
  SHK_CUDA(cudaEventCreate(&c->t1));
  shk_ribbon_create(&c->rib);
  *out = c;
  return 0;
}

int shk_ctx_destroy(shk_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->free_blocks) cudaFree(kv.second);
  for (auto& kv : c->live) cudaFree(kv.first);
  shk_ribbon_destroy(c->rib);
  plan_cache_free(c);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  cudaFree(c->d_counter);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  cudaEventDestroy(c->t0);
  cudaEventDestroy(c->t1);
  cudaStreamDestroy(c->own);
  cudaStreamDestroy(c->copy);
  cudaStreamDestroy(c->copy_out);
  delete c;
  return 0;
}

int shk_ctx_sync(shk_ctx* c) { return csync(c); }
void* shk_ctx_stream(shk_ctx* c) { return (void*)c->stream; }
int shk_ctx_set_stream(shk_ctx* c, void* s) {
  c->stream = s ? (cudaStream_t)s : c->own;
  return 0;
}
int shk_ctx_num_sms(shk_ctx* c) { return c->num_sms; }
int shk_ctx_set_option(shk_ctx* c, int opt, int64_t value) {
  if (opt < 0 || opt >= 8) {
    shk_set_error("unknown option %d", opt);
    return SHK_INVALID;
  }
  c->opt[opt] = value;
  return 0;
}

int shk_dev_alloc(shk_ctx* c, size_t bytes, void** out) { return pool_alloc(c, bytes, out); }
int shk_host_alloc(shk_ctx* c, size_t bytes, void** out) {
  (void)c;
  SHK_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  return 0;
}
int shk_host_free(shk_ctx* c, void* p) {
  (void)c;
  if (p) SHK_CUDA(cudaFreeHost(p));
  return 0;
}
int shk_dev_free(shk_ctx* c, void* p) {
  pool_free(c, p);
  return 0;
}
int shk_memcpy(shk_ctx* c, void* dst, const void* src, size_t bytes, int kind) {
  cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  SHK_CUDA(cudaMemcpyAsync(dst, src, bytes, k, c->stream));
  return csync(c);
}
int shk_memset(shk_ctx* c, void* dst, int value, size_t bytes) {
  SHK_CUDA(cudaMemsetAsync(dst, value, bytes, c->stream));
  return 0;
}
int shk_exclusive_scan(shk_ctx* c, const int64_t* in, int64_t* out, int64_t n) {
  if (n < 0) {
    shk_set_error("scan length must be >= 0");
    return SHK_INVALID;
  }
  const size_t ss = shk_scan_scratch(n);
  void* scratch = nullptr;
  RC(pool_alloc(c, ss, &scratch));
  const int rc = shk_exclusive_scan_i64(in, out, n, scratch, ss, c->stream);
  const int rs = csync(c);
  pool_free(c, scratch);
  return rc ? rc : rs;
}
int shk_timer_start(shk_ctx* c) {
  SHK_CUDA(cudaEventRecord(c->t0, c->stream));
  return 0;
}
int shk_timer_stop(shk_ctx* c, float* ms) {
  SHK_CUDA(cudaEventRecord(c->t1, c->stream));
  SHK_CUDA(cudaEventSynchronize(c->t1));
  SHK_CUDA(cudaEventElapsedTime(ms, c->t0, c->t1));
  return 0;
}

// ---- scalar API --------------------------------------------------------------
uint64_t shk_mix64(uint64_t z) { return shk::mix64(z); }
uint64_t shk_seed_mixer(uint64_t seed, uint64_t tag) { return shk::seed_mixer(seed, tag); }
uint64_t shk_remix(uint64_t hi, uint64_t lo, uint64_t seed, uint64_t tag) { return shk::remix(hi, lo, seed, tag); }
uint64_t shk_hash_range(uint64_t v, uint64_t m) { return shk::hash_range(v, m); }
void shk_leaf_pair(uint64_t hi, uint64_t lo, uint64_t seed, int n, int* h0, int* h1) {
  shk::leaf_pair(hi, lo, seed, n, *h0, *h1);
}
int shk_split_bit(uint64_t hi, uint64_t lo, uint64_t seed) { return shk::split_bit(hi, lo, seed); }
int shk_leaf_cell(uint64_t hi, uint64_t lo, int64_t q, int mleaf, int mode, int64_t cache_k, int choice) {
  return shk::leaf_cell(hi, lo, q, mleaf, mode, cache_k, choice);
}

// ---- leaf search -------------------------------------------------------------
int shk_leaf_search(shk_ctx* c, int mode, int cache_k, int cache_min_leaf, const uint64_t* hi, const uint64_t* lo,
                    const int64_t* leaf_off, int64_t L, uint64_t max_seed, int team_warps, int64_t* seed_out,
                    uint64_t* fbits_out, int64_t* stats_out, int flags) {
  if (L < 0 || (mode != 0 && mode != 1) || cache_k < 0) {
    shk_set_error("invalid leaf search parameters");
    return SHK_INVALID;
  }
  if (L == 0) return 0;
  // Validate leaf sizes (host copy of the offsets).
  std::vector<int64_t> hoff((size_t)L + 1);
  if (flags & SHK_DEVICE) {
    RC(d2h(c, hoff.data(), leaf_off, (L + 1) * 8));
    RC(csync(c));
  } else {
    memcpy(hoff.data(), leaf_off, (L + 1) * 8);
  }
  int max_n = 0;
  for (int64_t i = 0; i < L; ++i) {
    int64_t n = hoff[i + 1] - hoff[i];
    if (n < 1 || n > 64) {
      shk_set_error("leaf %lld has %lld keys; leaves hold 1..64 keys", (long long)i, (long long)n);
      return SHK_INVALID;
    }
    if (n > max_n) max_n = (int)n;
  }
  const int64_t N = hoff[L] - hoff[0];
  DBuf thi(c), tlo(c), toff(c), tseed(c), tfb(c), tst(c);
  const void *dhi, *dlo, *doff;
  void *dseed, *dfb, *dst;
  RC(stage_in(c, flags, hi, (size_t)(hoff[L]) * 8, thi, &dhi));
  RC(stage_in(c, flags, lo, (size_t)(hoff[L]) * 8, tlo, &dlo));
  RC(stage_in(c, flags, leaf_off, (size_t)(L + 1) * 8, toff, &doff));
  RC(stage_out(c, flags, seed_out, (size_t)L * 8, tseed, &dseed));
  RC(stage_out(c, flags, fbits_out, (size_t)L * 8, tfb, &dfb));
  RC(stage_out(c, flags, stats_out, (size_t)L * 32, tst, &dst));
  (void)N;
  ShkLeafLaunch p{};
  p.hi = (const uint64_t*)dhi;
  p.lo = (const uint64_t*)dlo;
  p.off = (const int64_t*)doff;
  p.L = L;
  p.max_n = max_n;
  p.max_seed = max_seed;
  p.mode = mode;
  p.cache_k = cache_k;
  p.cache_min_leaf = cache_min_leaf;
  p.seed_out = (int64_t*)dseed;
  p.fbits_out = (uint64_t*)dfb;
  p.choice_out = nullptr;
  p.stats_out = (int64_t*)dst;
  p.counter = c->d_counter;
  p.error = c->d_counter + 1;
  p.team_warps = team_warps;
  p.num_sms = c->num_sms;
  p.stride = 1;
  DBuf steal_state(c), steal_active(c);
  if (mode == 0 && team_warps == 0 && max_n > 24 && !stats_out && !c->opt[SHK_OPT_LEAF_FIXED_TEAMS]) {
    // plain search: every warp on its own, 32-seed blocks handed out per
    // leaf, idle warps join the last leaves (shk_leaf_steal.cu).  Leaves of
    // <= 24 keys need a few hundred seeds at most: one warp each, no
    // stealing (the fixed-team kernel).  Per-leaf counters (stats_out)
    // come from the fixed-team kernel too.
    const int max_active = c->num_sms * 64 + 1;
    RC(steal_state.alloc(shk_leaf_steal_state_bytes(L)));
    RC(steal_active.alloc((size_t)max_active * 8));
    int shared = 0;
    if (c->shared_leaf_counter) {  // leaves handed out by a counter shared with other GPUs / processes
      p.counter = c->shared_leaf_counter;
      shared = 1;
    }
    RC(shk_launch_leaf_steal(p, steal_state.p, steal_active.as<long long>(), max_active, shared, c->stream));
  } else {
    RC(shk_launch_leaf_search(p, c->stream));
  }
  RC(finish_out(c, flags, seed_out, tseed, (size_t)L * 8));
  RC(finish_out(c, flags, fbits_out, tfb, (size_t)L * 8));
  RC(finish_out(c, flags, stats_out, tst, (size_t)L * 32));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

// ---- routing to owner ranks (input-sharded build) ------------------------------
int shk_route(shk_ctx* c, const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
              const int64_t* bounds, int W, uint64_t* keys_out, uint8_t* aux_out, int64_t* counts_out) {
  if ((kind != 0 && kind != 1) || n < 0) {
    shk_set_error("route: kind 0 (bucket) or 1 (ribbon column)");
    return SHK_INVALID;
  }
  DBuf cnt(c), cur(c);
  RC(cnt.alloc(64 * 8));
  RC(cur.alloc(64 * 8));
  return shk_launch_route(keys, aux, n, kind, nbm, seed, bounds, W, cnt.as<unsigned long long>(),
                          cur.as<unsigned long long>(), keys_out, aux_out, counts_out, c->stream);
}

int shk_route_count(shk_ctx* c, const uint64_t* keys, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                    const int64_t* bounds, int W, int64_t* counts_out) {
  DBuf cnt(c);
  RC(cnt.alloc(64 * 8));
  return shk_launch_route_count(keys, n, kind, nbm, seed, bounds, W, cnt.as<unsigned long long>(), counts_out,
                                c->stream);
}
int shk_route_p2p(shk_ctx* c, const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm,
                  uint64_t seed, const int64_t* bounds, int W, void* const* peer_bufs, const int64_t* peer_base,
                  int64_t cap) {
  DBuf cur(c);
  RC(cur.alloc(64 * 8));
  return shk_launch_route_p2p(keys, aux, n, kind, nbm, seed, bounds, W, peer_bufs, peer_base, cap,
                              cur.as<unsigned long long>(), c->stream);
}
// IPC-shareable device buffers (the peer receive buffers of shk_route_p2p)
int shk_ipc_buffer_alloc(shk_ctx* c, size_t bytes, void* handle_out, void** dev_ptr) {
  void* p = nullptr;
  SHK_CUDA(cudaSetDevice(c->device));
  SHK_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
  cudaIpcMemHandle_t h;
  SHK_CUDA(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof(h));
  *dev_ptr = p;
  return 0;
}

// ---- cross-GPU leaf queue (CUDA IPC) ------------------------------------------
int shk_ipc_counter_alloc(shk_ctx* c, void* handle_out, void** dev_ptr) {
  int* p = nullptr;
  SHK_CUDA(cudaSetDevice(c->device));
  SHK_CUDA(cudaMalloc(&p, 256));
  SHK_CUDA(cudaMemset(p, 0, 256));
  cudaIpcMemHandle_t h;
  SHK_CUDA(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof(h));
  *dev_ptr = p;
  return 0;
}
int shk_ipc_counter_open(shk_ctx* c, const void* handle, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SHK_CUDA(cudaSetDevice(c->device));
  SHK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}
int shk_ipc_counter_close(shk_ctx* c, void* dev_ptr, int owner) {
  SHK_CUDA(cudaSetDevice(c->device));
  if (owner)
    SHK_CUDA(cudaFree(dev_ptr));
  else
    SHK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return 0;
}
int shk_ipc_counter_reset(shk_ctx* c, void* dev_ptr) {
  SHK_CUDA(cudaMemsetAsync(dev_ptr, 0, sizeof(int), c->stream));
  return csync(c);
}
int shk_ctx_set_leaf_counter(shk_ctx* c, void* dev_ptr) {
  c->shared_leaf_counter = (int*)dev_ptr;
  return 0;
}

int shk_int_peak(shk_ctx* c, int kind, int iters, double* ms_out, double* ops_out) {
  if (iters <= 0) {
    shk_set_error("iters must be positive");
    return SHK_INVALID;
  }
  DBuf sink(c);
  RC(sink.alloc(64));
  int64_t threads = 0;
  int per = 0;
  cudaEvent_t e0, e1;
  SHK_CUDA(cudaEventCreate(&e0));
  SHK_CUDA(cudaEventCreate(&e1));
  RC(shk_launch_int_peak(kind, iters, c->num_sms, sink.as<uint32_t>(), &threads, &per, c->stream));  // warm-up
  SHK_CUDA(cudaEventRecord(e0, c->stream));
  RC(shk_launch_int_peak(kind, iters, c->num_sms, sink.as<uint32_t>(), &threads, &per, c->stream));
  SHK_CUDA(cudaEventRecord(e1, c->stream));
  SHK_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  SHK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms;
  *ops_out = (double)threads * (double)iters * (double)per;
  return 0;
}

int shk_orient(shk_ctx* c, const uint8_t* eu, const uint8_t* ev, const int64_t* leaf_off, int64_t L,
               uint64_t* fbits_out, int32_t* ok_out, int flags) {
  if (L <= 0) return 0;
  std::vector<int64_t> hoff((size_t)L + 1);
  if (flags & SHK_DEVICE) {
    RC(d2h(c, hoff.data(), leaf_off, (L + 1) * 8));
    RC(csync(c));
  } else {
    memcpy(hoff.data(), leaf_off, (L + 1) * 8);
  }
  for (int64_t i = 0; i < L; ++i) {
    int64_t n = hoff[i + 1] - hoff[i];
    if (n < 1 || n > 64) {
      shk_set_error("edge list %lld has %lld edges; 1..64 supported", (long long)i, (long long)n);
      return SHK_INVALID;
    }
  }
  DBuf tu(c), tv(c), to(c), tf(c), tk(c);
  const void *du, *dv, *doff;
  void *df, *dk;
  RC(stage_in(c, flags, eu, (size_t)hoff[L], tu, &du));
  RC(stage_in(c, flags, ev, (size_t)hoff[L], tv, &dv));
  RC(stage_in(c, flags, leaf_off, (size_t)(L + 1) * 8, to, &doff));
  RC(stage_out(c, flags, fbits_out, (size_t)L * 8, tf, &df));
  RC(stage_out(c, flags, ok_out, (size_t)L * 4, tk, &dk));
  RC(shk_launch_orient((const uint8_t*)du, (const uint8_t*)dv, (const int64_t*)doff, L, (uint64_t*)df, (int*)dk,
                       c->stream));
  RC(finish_out(c, flags, fbits_out, tf, (size_t)L * 8));
  RC(finish_out(c, flags, ok_out, tk, (size_t)L * 4));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

// ---- split search (single node, seam parity) -----------------------------------
int shk_split_search(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, int64_t m, const int64_t* sizes, int fanout,
                     uint64_t max_seed, int64_t* seed_out, int64_t* evals_out) {
  if (fanout < 1 || fanout > 4 || m < 1 || m >= 32768) {
    shk_set_error("split search supports fanout 1..4 and 1 <= m < 32768 (got fanout %d, m %lld)", fanout,
                  (long long)m);
    return SHK_INVALID;
  }
  int64_t tot = 0;
  for (int j = 0; j < fanout; ++j) {
    if (sizes[j] < 0) {
      shk_set_error("negative part size");
      return SHK_INVALID;
    }
    tot += sizes[j];
  }
  if (tot != m) {
    shk_set_error("part sizes must sum to m");
    return SHK_INVALID;
  }
  DBuf keys(c), tmp(c), task(c), seeds(c), ev(c);
  RC(keys.alloc((size_t)m * 16));
  RC(tmp.alloc((size_t)m * 16));
  {
    DBuf th(c), tl(c);
    RC(th.alloc((size_t)m * 8));
    RC(tl.alloc((size_t)m * 8));
    RC(h2d(c, th.p, hi, (size_t)m * 8));
    RC(h2d(c, tl.p, lo, (size_t)m * 8));
    RC(shk_launch_interleave(th.as<uint64_t>(), tl.as<uint64_t>(), m, keys.as<uint64_t>(), c->stream));
    RC(shk_launch_premix(keys.as<uint64_t>(), m, 0, c->stream));
    RC(csync(c));
  }
  ShkSplitTask t{};
  t.start = 0;
  t.m = (int32_t)m;
  t.fanout = fanout;
  for (int j = 0; j < 4; ++j) t.sizes[j] = j < fanout ? (int32_t)sizes[j] : 0;
  t.seed_slot = 0;
  RC(task.alloc(sizeof t));
  RC(h2d(c, task.p, &t, sizeof t));
  RC(seeds.alloc(8));
  RC(ev.alloc(8));
  ShkSplitLaunch p{};
  p.hi = keys.as<uint64_t>();
  p.tmp_hi = tmp.as<uint64_t>();
  p.tasks = task.as<ShkSplitTask>();
  p.ntasks = 1;
  p.max_seed = max_seed;
  p.seeds = seeds.as<int64_t>();
  p.evals_out = ev.as<int64_t>();
  p.counter = c->d_counter;
  p.num_sms = c->num_sms;
  p.partition = 0;
  p.exact_evals = 1;
  RC(shk_launch_split(p, c->stream));
  RC(d2h(c, seed_out, seeds.p, 8));
  RC(d2h(c, evals_out, ev.p, 8));
  return csync(c);
}

int shk_split_parts(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed, const int64_t* sizes,
                    int fanout, int64_t* parts_out) {
  if (m <= 0) return 0;
  if (fanout < 1) {
    shk_set_error("fanout must be >= 1");
    return SHK_INVALID;
  }
  DBuf th(c), tl(c), ts(c), tp(c);
  RC(th.alloc((size_t)m * 8));
  RC(tl.alloc((size_t)m * 8));
  RC(ts.alloc((size_t)fanout * 8));
  RC(tp.alloc((size_t)m * 8));
  RC(h2d(c, th.p, hi, (size_t)m * 8));
  RC(h2d(c, tl.p, lo, (size_t)m * 8));
  RC(h2d(c, ts.p, sizes, (size_t)fanout * 8));
  RC(shk_launch_split_parts(th.as<uint64_t>(), tl.as<uint64_t>(), m, seed, ts.as<int64_t>(), fanout,
                            tp.as<int64_t>(), c->stream));
  RC(d2h(c, parts_out, tp.p, (size_t)m * 8));
  return csync(c);
}

// ---- ribbon ----------------------------------------------------------------------
int shk_ribbon_rows(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t m, uint64_t seed,
                    int64_t* starts, uint64_t* pat0, uint64_t* pat1, int flags) {
  if (m < 128) {
    shk_set_error("ribbon needs m >= 128");
    return SHK_INVALID;
  }
  if (N <= 0) return 0;
  DBuf th(c), tl(c), ts(c), t0(c), t1(c);
  const void *dh, *dl;
  void *ds, *d0, *d1;
  RC(stage_in(c, flags, hi, (size_t)N * 8, th, &dh));
  RC(stage_in(c, flags, lo, (size_t)N * 8, tl, &dl));
  RC(stage_out(c, flags, starts, (size_t)N * 8, ts, &ds));
  RC(stage_out(c, flags, pat0, (size_t)N * 8, t0, &d0));
  RC(stage_out(c, flags, pat1, (size_t)N * 8, t1, &d1));
  RC(shk_launch_ribbon_rows((const uint64_t*)dh, (const uint64_t*)dl, 1, N, m, seed, (int64_t*)ds, (uint64_t*)d0,
                            (uint64_t*)d1, c->stream));
  RC(finish_out(c, flags, starts, ts, (size_t)N * 8));
  RC(finish_out(c, flags, pat0, t0, (size_t)N * 8));
  RC(finish_out(c, flags, pat1, t1, (size_t)N * 8));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

int shk_ribbon_solve(shk_ctx* c, const int64_t* starts, const uint64_t* pat0, const uint64_t* pat1,
                     const uint8_t* rhs, int64_t N, int64_t m, uint64_t* words_out, int* consistent, int flags) {
  if (m < 128) {
    shk_set_error("ribbon needs m >= 128");
    return SHK_INVALID;
  }
  const int64_t nw = (m + 63) / 64;
  DBuf ts(c), t0(c), t1(c), tr(c), tw(c);
  const void *ds, *d0, *d1, *dr;
  void* dw;
  RC(stage_in(c, flags, starts, (size_t)N * 8, ts, &ds));
  RC(stage_in(c, flags, pat0, (size_t)N * 8, t0, &d0));
  RC(stage_in(c, flags, pat1, (size_t)N * 8, t1, &d1));
  RC(stage_in(c, flags, rhs, (size_t)N, tr, &dr));
  RC(stage_out(c, flags, words_out, (size_t)nw * 8, tw, &dw));
  // validate starts on the host side when given host arrays
  if (!(flags & SHK_DEVICE)) {
    for (int64_t i = 0; i < N; ++i)
      if (starts[i] < 0 || starts[i] > m - 128) {
        shk_set_error("row %lld start %lld outside [0, m-128]", (long long)i, (long long)starts[i]);
        return SHK_INVALID;
      }
  }
  RC(shk_ribbon_solve_rows(c->rib, (const int64_t*)ds, (const uint64_t*)d0, (const uint64_t*)d1, (const uint8_t*)dr,
                           N, m, (uint64_t*)dw, consistent, c->stream));
  if (*consistent) RC(finish_out(c, flags, words_out, tw, (size_t)nw * 8));
  return csync(c);
}

int shk_ribbon_query(shk_ctx* c, const int64_t* starts, const uint64_t* pat0, const uint64_t* pat1, int64_t N,
                     const uint64_t* words, int64_t nwords, uint8_t* out, int flags) {
  if (N <= 0) return 0;
  DBuf ts(c), t0(c), t1(c), tw(c), to(c);
  const void *ds, *d0, *d1, *dw;
  void* dout;
  RC(stage_in(c, flags, starts, (size_t)N * 8, ts, &ds));
  RC(stage_in(c, flags, pat0, (size_t)N * 8, t0, &d0));
  RC(stage_in(c, flags, pat1, (size_t)N * 8, t1, &d1));
  RC(stage_in(c, flags, words, (size_t)(nwords > 0 ? nwords : 1) * 8, tw, &dw));
  RC(stage_out(c, flags, out, (size_t)N, to, &dout));
  RC(shk_launch_ribbon_query((const int64_t*)ds, (const uint64_t*)d0, (const uint64_t*)d1, N, (const uint64_t*)dw,
                             nwords, (uint8_t*)dout, c->stream));
  RC(finish_out(c, flags, out, to, (size_t)N));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

static int ribbon_seed_loop(shk_ctx* c, const uint64_t* dkeys, const uint8_t* drhs, int64_t N, int64_t m,
                            int max_tries, uint64_t* seed_out, uint64_t* dwords) {
  for (int seed = 0; seed < max_tries; ++seed) {
    int ok = 0;
    RC(shk_ribbon_solve_keys(c->rib, dkeys, drhs, N, m, (uint64_t)seed, dwords, &ok, c->stream));
    if (ok) {
      *seed_out = (uint64_t)seed;
      return 0;
    }
  }
  shk_set_error("retrieval system unsolvable after %d seeds (n=%lld, m=%lld)", max_tries, (long long)N,
                (long long)m);
  return SHK_UNSOLVABLE;
}

int shk_ribbon_build(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, const uint8_t* rhs, int64_t N, int64_t m,
                     int max_tries, uint64_t* seed_out, uint64_t* words_out, int flags) {
  if (m < 128) {
    shk_set_error("ribbon needs m >= 128");
    return SHK_INVALID;
  }
  const int64_t nw = (m + 63) / 64;
  DBuf th(c), tl(c), tr(c), keys(c), tw(c);
  const void *dh, *dl, *dr;
  void* dw;
  RC(stage_in(c, flags, hi, (size_t)N * 8, th, &dh));
  RC(stage_in(c, flags, lo, (size_t)N * 8, tl, &dl));
  RC(stage_in(c, flags, rhs, (size_t)N, tr, &dr));
  RC(stage_out(c, flags, words_out, (size_t)nw * 8, tw, &dw));
  RC(keys.alloc((size_t)N * 16 + 16));
  RC(shk_launch_interleave((const uint64_t*)dh, (const uint64_t*)dl, N, keys.as<uint64_t>(), c->stream));
  RC(ribbon_seed_loop(c, keys.as<uint64_t>(), (const uint8_t*)dr, N, m, max_tries, seed_out, (uint64_t*)dw));
  RC(finish_out(c, flags, words_out, tw, (size_t)nw * 8));
  return csync(c);
}

int shk_rice_decode(shk_ctx* c, const uint64_t* words, int64_t nwords, int64_t bit_len, int64_t pos,
                    const int32_t* g, int64_t count, int64_t* values_out, int64_t* pos_out) {
  if (count <= 0) return 0;
  if (nwords * 64 < bit_len) {
    shk_set_error("bit_len exceeds the word array");
    return SHK_INVALID;
  }
  DBuf tw(c), tg(c), tv(c), tp(c);
  RC(tw.alloc((size_t)(nwords + 1) * 8));
  RC(tg.alloc((size_t)count * 4));
  RC(tv.alloc((size_t)count * 8));
  RC(tp.alloc((size_t)count * 8));
  RC(h2d(c, tw.p, words, (size_t)nwords * 8));
  RC(h2d(c, tg.p, g, (size_t)count * 4));
  int* err = c->d_counter + 2;
  SHK_CUDA(cudaMemsetAsync(err, 0, 4, c->stream));
  RC(shk_launch_rice_decode(tw.as<uint64_t>(), bit_len, pos, tg.as<int32_t>(), count, tv.as<int64_t>(),
                            tp.as<int64_t>(), err, c->stream));
  int herr = 0;
  RC(d2h(c, &herr, err, 4));
  RC(d2h(c, values_out, tv.p, (size_t)count * 8));
  RC(d2h(c, pos_out, tp.p, (size_t)count * 8));
  RC(csync(c));
  if (herr) {
    shk_set_error("bit stream overrun");
    return SHK_FORMAT;
  }
  return 0;
}

int shk_blake2b128(shk_ctx* c, const uint8_t* blob, int64_t blob_len, const int64_t* off, int64_t N, uint64_t salt,
                   uint64_t* hi, uint64_t* lo, int flags) {
  if (N <= 0) return 0;
  DBuf tb(c), to(c), th(c), tl(c);
  const void *db, *doff;
  void *dh, *dl;
  // Fixed-length fast path when every key has the same length (host offsets):
  // the offsets need not cross PCIe at all.
  int64_t L0 = 0;
  if (!(flags & SHK_DEVICE) && off[0] == 0 && blob_len == off[N]) {
    L0 = off[1] - off[0];
    if (L0 < 1 || L0 > 128 || L0 * N != blob_len) L0 = 0;
    for (int64_t i = 0; i < N && L0; ++i)
      if (off[i + 1] - off[i] != L0) L0 = 0;
  }
  RC(stage_in(c, flags, blob, (size_t)(blob_len > 0 ? blob_len : 1), tb, &db));
  RC(stage_out(c, flags, hi, (size_t)N * 8, th, &dh));
  RC(stage_out(c, flags, lo, (size_t)N * 8, tl, &dl));
  if (L0) {
    RC(shk_launch_blake2b_fixed((const uint8_t*)db, (int)L0, N, salt, (uint64_t*)dh, (uint64_t*)dl, c->stream));
  } else {
    RC(stage_in(c, flags, off, (size_t)(N + 1) * 8, to, &doff));
    RC(shk_launch_blake2b((const uint8_t*)db, (const int64_t*)doff, N, salt, (uint64_t*)dh, (uint64_t*)dl,
                          c->stream));
  }
  RC(finish_out(c, flags, hi, th, (size_t)N * 8));
  RC(finish_out(c, flags, lo, tl, (size_t)N * 8));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

// ---- analysis entry points (experiments seam) ----------------------------------
int shk_search_bruteforce(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, int n, uint64_t max_seed,
                          int64_t* seed_out, int64_t* evals_out) {
  if (n < 0 || n > 64) {
    shk_set_error("search_bruteforce supports 0 <= n <= 64 (got %d)", n);
    return SHK_INVALID;
  }
  DBuf kh(c), kl(c), st(c);
  RC(kh.alloc(64 * 8));
  RC(kl.alloc(64 * 8));
  RC(st.alloc(16));
  RC(h2d(c, kh.p, hi, (size_t)n * 8));
  RC(h2d(c, kl.p, lo, (size_t)n * 8));
  unsigned long long* found = st.as<unsigned long long>();
  unsigned long long* evals = found + 1;
  // Batches of doubling size; the batch holding the minimum bijective seed is
  // re-counted up to that seed, so evals match the scalar loop exactly.
  int64_t total = 0;
  uint64_t base = 0, batch = 1ull << 16;
  while (base < max_seed) {
    const uint64_t cnt = (max_seed - base < batch) ? max_seed - base : batch;
    const unsigned long long init[2] = {~0ull, 0ull};
    RC(h2d(c, found, init, 16));
    RC(shk_launch_brute(kh.as<uint64_t>(), kl.as<uint64_t>(), n, base, cnt, found, evals, c->num_sms, c->stream));
    unsigned long long res[2];
    RC(d2h(c, res, found, 16));
    RC(csync(c));
    if (res[0] != ~0ull) {
      RC(h2d(c, found, init, 16));
      RC(shk_launch_brute(kh.as<uint64_t>(), kl.as<uint64_t>(), n, base, res[0] - base + 1, found, evals,
                          c->num_sms, c->stream));
      unsigned long long res2[2];
      RC(d2h(c, res2, found, 16));
      RC(csync(c));
      *seed_out = (int64_t)res[0];
      *evals_out = total + (int64_t)res2[1];
      return SHK_OK;
    }
    total += (int64_t)res[1];
    base += cnt;
    if (batch < (1ull << 28)) batch <<= 1;
  }
  *seed_out = -1;
  *evals_out = total;
  return SHK_OK;
}

int shk_mc_filter_pass_count(shk_ctx* c, int n, int64_t trials, uint64_t entropy, int64_t* passes_out) {
  if (n > 64) {
    shk_set_error("mc_filter_pass_count supports n <= 64 (got %d)", n);
    return SHK_INVALID;
  }
  if (trials <= 0) {
    *passes_out = 0;
    return SHK_OK;
  }
  if (n <= 1) {  // every seed covers the (at most one) cell: _core.pyx:834-835
    *passes_out = trials;
    return SHK_OK;
  }
  uint64_t h[128];
  for (int j = 0; j < n; ++j) {  // the synthetic key set, _core.pyx:844-846
    h[j] = shk::mix64(entropy + 2ull * (uint64_t)j);
    h[64 + j] = shk::mix64(entropy + 2ull * (uint64_t)j + 1ull);
  }
  DBuf keys(c), cnt(c);
  RC(keys.alloc(128 * 8));
  RC(cnt.alloc(8));
  RC(h2d(c, keys.p, h, sizeof h));
  SHK_CUDA(cudaMemsetAsync(cnt.p, 0, 8, c->stream));
  RC(shk_launch_mc_filter(keys.as<uint64_t>(), keys.as<uint64_t>() + 64, n, (uint64_t)trials,
                          cnt.as<unsigned long long>(), c->num_sms, c->stream));
  unsigned long long r = 0;
  RC(d2h(c, &r, cnt.p, 8));
  RC(csync(c));
  *passes_out = (int64_t)r;
  return SHK_OK;
}

int shk_enumerate_outcomes(shk_ctx* c, int n, uint64_t* pf_count_out, uint64_t* sum_2c_out) {
  if (n > 8) {
    shk_set_error("enumeration limited to n <= 8");
    return SHK_INVALID;
  }
  if (n <= 0) {  // the empty tuple: one pseudoforest with 0 components
    *pf_count_out = 1;
    *sum_2c_out = 1;
    return SHK_OK;
  }
  DBuf out(c);
  RC(out.alloc(16));
  SHK_CUDA(cudaMemsetAsync(out.p, 0, 16, c->stream));
  RC(shk_launch_enumerate(n, out.as<unsigned long long>(), c->num_sms, c->stream));
  unsigned long long r[2];
  RC(d2h(c, r, out.p, 16));
  RC(csync(c));
  *pf_count_out = r[0];
  *sum_2c_out = r[1];
  return SHK_OK;
}

int shk_blake2b128_fixed(shk_ctx* c, const uint8_t* blob, int key_len, int64_t N, uint64_t salt, uint64_t* hi,
                         uint64_t* lo, int flags) {
  if (N <= 0) return 0;
  if (key_len < 1 || key_len > 128) {
    shk_set_error("fixed-length keys must be 1..128 bytes");
    return SHK_INVALID;
  }
  DBuf tb(c), th(c), tl(c);
  if (flags & SHK_BLOB_HOST) {
    // chunked: the H2D of chunk k+1 (copy stream) overlaps the hashing of
    // chunk k (context stream); host-blocking, like every host-input call
    const int64_t nchunk = 8;
    const int64_t per = (N + nchunk - 1) / nchunk;
    RC(tb.alloc((size_t)key_len * N));
    cudaEvent_t ev[8];
    for (int k = 0; k < nchunk; ++k) SHK_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    int rc = 0;
    for (int64_t k = 0; k < nchunk && !rc; ++k) {
      const int64_t a = k * per, b = (a + per < N) ? a + per : N;
      if (a >= b) break;
      const size_t off = (size_t)a * key_len, len = (size_t)(b - a) * key_len;
      cudaError_t e = cudaMemcpyAsync(tb.as<uint8_t>() + off, blob + off, len, cudaMemcpyHostToDevice, c->copy);
      if (e == cudaSuccess) e = cudaEventRecord(ev[k], c->copy);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, ev[k], 0);
      if (e != cudaSuccess) {
        shk_set_error("blake2b chunked copy: %s", cudaGetErrorString(e));
        rc = -1000 - (int)e;
        break;
      }
      rc = shk_launch_blake2b_fixed(tb.as<uint8_t>() + off, key_len, b - a, salt, hi + a, lo + a, c->stream);
    }
    cudaStreamSynchronize(c->copy);
    cudaStreamSynchronize(c->stream);
    for (int k = 0; k < nchunk; ++k) cudaEventDestroy(ev[k]);
    return rc;
  }
  const void* db;
  void *dh, *dl;
  RC(stage_in(c, flags, blob, (size_t)key_len * N, tb, &db));
  RC(stage_out(c, flags, hi, (size_t)N * 8, th, &dh));
  RC(stage_out(c, flags, lo, (size_t)N * 8, tl, &dl));
  RC(shk_launch_blake2b_fixed((const uint8_t*)db, key_len, N, salt, (uint64_t*)dh, (uint64_t*)dl, c->stream));
  RC(finish_out(c, flags, hi, th, (size_t)N * 8));
  RC(finish_out(c, flags, lo, tl, (size_t)N * 8));
  if (!(flags & SHK_DEVICE)) RC(csync(c));
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Plans: host tables derived from the reference's flattened plan arrays.

using PlanNode = ShkPlanNode;
struct PlanSet {
  std::vector<int64_t> plan_m;
  std::vector<int64_t> plan_off;  // nplans+1
  std::vector<PlanNode> nodes;
  std::unordered_map<int64_t, int32_t> by_size;
  int max_depth = 0;
};

static int load_plans(const shk_plans* P, PlanSet& S) {
  if (!P || P->nplans < 0) {
    shk_set_error("missing plan tables");
    return SHK_INVALID;
  }
  S.plan_m.assign(P->plan_m, P->plan_m + P->nplans);
  S.plan_off.assign(P->plan_off, P->plan_off + P->nplans + 1);
  const int64_t total = S.plan_off.empty() ? 0 : S.plan_off.back();
  S.nodes.resize((size_t)total);
  for (int64_t p = 0; p < P->nplans; ++p) {
    const int64_t a = S.plan_off[p], b = S.plan_off[p + 1];
    if (b <= a) {
      shk_set_error("empty plan %lld", (long long)p);
      return SHK_INVALID;
    }
    S.by_size[S.plan_m[p]] = (int32_t)p;
    for (int64_t j = a; j < b; ++j) {
      PlanNode& nd = S.nodes[j];
      nd.kind = (int32_t)P->kind[j];
      nd.g = (int32_t)P->g[j];
      nd.m = (int32_t)P->m_node[j];
      nd.fanout = nd.kind == 0 ? (int32_t)P->fanout[j] : 0;
      if (nd.g < 0 || nd.g > 63) {
        shk_set_error("Rice parameter out of range");
        return SHK_INVALID;
      }
      if (nd.kind == 0 && (nd.fanout < 1 || nd.fanout > 4)) {
        shk_set_error("split fanout %d unsupported (1..4)", nd.fanout);
        return SHK_INVALID;
      }
      for (int k = 0; k < 4; ++k) {
        nd.sizes[k] = (k < nd.fanout) ? (int32_t)P->sizes_flat[P->sizes_base[p] + P->sizes_off[j] + k] : 0;
        nd.child[k] = 0;
      }
    }
    // children (preorder: first child follows, next child after its subtree)
    for (int64_t j = a; j < b; ++j) {
      PlanNode& nd = S.nodes[j];
      if (nd.kind != 0) continue;
      int64_t cidx = j + 1;
      for (int k = 0; k < nd.fanout; ++k) {
        if (cidx >= b) {
          shk_set_error("malformed plan subtree counts");
          return SHK_INVALID;
        }
        nd.child[k] = (int32_t)(cidx - a);
        cidx += P->subtree[cidx];
      }
    }
    // offsets and depths (walk in preorder)
    S.nodes[a].off = 0;
    S.nodes[a].depth = 0;
    for (int64_t j = a; j < b; ++j) {
      PlanNode& nd = S.nodes[j];
      if (nd.kind != 0) continue;
      int32_t o = nd.off;
      for (int k = 0; k < nd.fanout; ++k) {
        PlanNode& ch = S.nodes[a + nd.child[k]];
        ch.off = o;
        ch.depth = nd.depth + 1;
        if (ch.depth > S.max_depth) S.max_depth = ch.depth;
        o += nd.sizes[k];
      }
    }
  }
  return 0;
}

// The plan tables of repeated builds over one key set (or any sets with the
// same bucket sizes) are identical: the context keeps the last PlanSet and its
// device copy, reused when the incoming arrays are equal (a content compare,
// ~1 MB at C4, instead of parsing 18k nodes into freshly faulted pages and
// re-uploading them: ~0.25 ms of host time before the first search).
struct PlanCache {
  std::vector<int64_t> src;  // the input arrays the tables were built from
  PlanSet S;
  ShkPlanNode* d_nodes = nullptr;
  int64_t* d_off = nullptr;
  size_t d_nodes_n = 0, d_off_n = 0;
  bool valid = false;
};

static void plan_cache_free(shk_ctx* c) {
  if (!c->plans) return;
  cudaFree(c->plans->d_nodes);
  cudaFree(c->plans->d_off);
  delete c->plans;
  c->plans = nullptr;
}

// Walk the input arrays in a fixed order: fn(ptr, count) per array.
template <class F>
static void plans_arrays(const shk_plans* P, F&& fn) {
  const int64_t np = P->nplans;
  const int64_t total = np > 0 ? P->plan_off[np] : 0;
  int64_t flat = 0;  // sizes_flat entries read by load_plans
  for (int64_t p = 0; p < np; ++p)
    for (int64_t j = P->plan_off[p]; j < P->plan_off[p + 1]; ++j)
      if (P->kind[j] == 0) {
        const int64_t need = P->sizes_base[p] + P->sizes_off[j] + P->fanout[j];
        if (need > flat) flat = need;
      }
  fn(&np, 1);
  fn(P->plan_m, np);
  fn(P->plan_off, np + 1);
  fn(P->sizes_base, np);
  fn(P->kind, total);
  fn(P->g, total);
  fn(P->fanout, total);
  fn(P->sizes_off, total);
  fn(P->subtree, total);
  fn(P->m_node, total);
  fn(&flat, 1);
  fn(P->sizes_flat, flat);
}

static int plan_cache_get(shk_ctx* c, const shk_plans* P, const PlanSet** out) {
  if (!P || P->nplans < 0) {
    shk_set_error("missing plan tables");
    return SHK_INVALID;
  }
  if (!c->plans) c->plans = new PlanCache();
  PlanCache& pc = *c->plans;
  if (pc.valid) {
    bool same = true;
    size_t o = 0;
    plans_arrays(P, [&](const int64_t* a, int64_t n) {
      if (!same) return;
      if (o + (size_t)n > pc.src.size() || (n && memcmp(pc.src.data() + o, a, (size_t)n * 8) != 0)) same = false;
      o += (size_t)n;
    });
    if (same && o == pc.src.size()) {
      *out = &pc.S;
      return 0;
    }
  }
  pc.valid = false;
  pc.S = PlanSet();
  RC(load_plans(P, pc.S));
  pc.src.clear();
  plans_arrays(P, [&](const int64_t* a, int64_t n) { pc.src.insert(pc.src.end(), a, a + n); });
  const size_t nn = pc.S.nodes.size() + 1, no = pc.S.plan_off.size() + 1;
  if (pc.d_nodes_n < nn) {
    cudaFree(pc.d_nodes);
    pc.d_nodes = nullptr;
    SHK_CUDA(cudaMalloc(&pc.d_nodes, nn * sizeof(ShkPlanNode)));
    pc.d_nodes_n = nn;
  }
  if (pc.d_off_n < no) {
    cudaFree(pc.d_off);
    pc.d_off = nullptr;
    SHK_CUDA(cudaMalloc(&pc.d_off, no * 8));
    pc.d_off_n = no;
  }
  SHK_CUDA(cudaMemcpy(pc.d_nodes, pc.S.nodes.data(), pc.S.nodes.size() * sizeof(ShkPlanNode), cudaMemcpyHostToDevice));
  SHK_CUDA(cudaMemcpy(pc.d_off, pc.S.plan_off.data(), pc.S.plan_off.size() * 8, cudaMemcpyHostToDevice));
  pc.valid = true;
  *out = &pc.S;
  return 0;
}

// Pinned host staging of `bytes` (grown on demand; the previous contents
// must have been consumed: every build syncs before it returns).
static int host_stage(shk_ctx* c, size_t bytes, void** out) {
  if (c->h_stage_cap < bytes) {
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->h_stage_cap = 0;
    SHK_CUDA(cudaMallocHost(&c->h_stage, bytes));
    c->h_stage_cap = bytes;
  }
  *out = c->h_stage;
  return 0;
}

// ---------------------------------------------------------------------------
// Build object.

struct shk_build {
  shk_ctx* c = nullptr;
  int64_t N = 0, nb = 0, max_bucket = 0;
  DBuf keys, tmp, prefix, choice;
  std::vector<uint64_t> h_prefix;
  // results of run()
  int64_t b0 = 0, b1 = 0;
  int64_t nnodes = 0;
  DBuf words;
  int64_t bit_len = 0, nwords = 0;
  std::vector<uint64_t> bit_off;  // [b1-b0+1] relative to the range start
  bool ran = false;
  bool record = false;
  DBuf place;
  // bucket-sorted copy of the keys (kept when a sharded build asks for it:
  // run() permutes `keys` in place only inside the rank's bucket range)
  bool keep_sorted = false;
  DBuf sorted;
  DBuf drhs;            // choice bits (sorted order) of a column-sharded ribbon
  int64_t dcols = 0;    // its local column count
  // phase timing (CUDA events on the context stream): 0 bucketize, 1 splits,
  // 2 leaves, 3 rice, 4 ribbon (last run)
  cudaEvent_t ev[12] = {};
  float phase_ms[6] = {0, 0, 0, 0, 0, 0};
  int64_t split_evals = 0;
  // asynchronous bucketize (SHK_BUILD_ASYNC): the duplicate flag lands in
  // pinned memory behind the sort; run() (or shk_build_duplicate) reads it
  int* h_dup = nullptr;
  bool dup_pending = false;
  int dup_value = 0;
  int take_dup() {
    if (dup_pending) {
      cudaEventSynchronize(ev[1]);
      dup_value = *h_dup;
      dup_pending = false;
      phase_ms[0] = span(0, 1);
    }
    return dup_value;
  }
  explicit shk_build(shk_ctx* ctx)
      : c(ctx), keys(ctx), tmp(ctx), prefix(ctx), choice(ctx), words(ctx), place(ctx), sorted(ctx), drhs(ctx) {}
  ~shk_build() {
    if (dup_pending) cudaEventSynchronize(ev[1]);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    level_reset();
  }
  void mark(int i) {
    if (!ev[i]) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[i], c->stream);
  }
  // per split level (depth) timing
  std::vector<cudaEvent_t> lev;
  std::vector<int> lev_depth;
  void level_mark(int depth) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    lev.push_back(e);
    lev_depth.push_back(depth);
  }
  void level_reset() {
    for (auto e : lev) cudaEventDestroy(e);
    lev.clear();
    lev_depth.clear();
  }
  float span(int a, int z) {
    float ms = 0;
    if (ev[a] && ev[z] && cudaEventElapsedTime(&ms, ev[a], ev[z]) == cudaSuccess) return ms;
    cudaGetLastError();
    return 0;
  }
};

__global__ void gather_bitoff_kernel(const int64_t* pos, const int64_t* node_base, int64_t nb, uint64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nb; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint64_t)pos[node_base[i]];
}

__global__ void seed_bits_kernel(const int64_t* len, const uint8_t* kind, int64_t nn, unsigned long long* acc) {
  unsigned long long a = 0, b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    if (kind[i])
      a += (unsigned long long)len[i];
    else
      b += (unsigned long long)len[i];
  }
  a = shk::warp_sum(a);
  b = shk::warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], a);
    atomicAdd(&acc[1], b);
  }
}

extern "C" {

int shk_build_create(shk_ctx* c, const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nbuckets, int flags,
                     shk_build** out, int* dup, int64_t* max_bucket) {
  if (N < 1 || nbuckets < 1) {
    shk_set_error("build needs N >= 1 and nbuckets >= 1");
    return SHK_INVALID;
  }
  g_host_t0 = host_now_us();
  HOST_TRACE("create");
  shk_build* b = new shk_build(c);
  b->N = N;
  b->nb = nbuckets;
  DBuf th(c), tl(c), scratch(c);
  const void *dh, *dl;
  int rc = 0;
  do {
    if ((rc = stage_in(c, flags, hi, (size_t)N * 8, th, &dh))) break;
    if ((rc = stage_in(c, flags, lo, (size_t)N * 8, tl, &dl))) break;
    if ((rc = b->keys.alloc((size_t)N * 16))) break;
    if ((rc = b->tmp.alloc((size_t)N * 16))) break;
    if ((rc = b->prefix.alloc((size_t)(nbuckets + 1) * 8))) break;
    if ((rc = b->choice.alloc((size_t)N))) break;
    size_t ss = shk_bucketize_scratch(N, nbuckets);
    if ((rc = scratch.alloc(ss))) break;
    int* ddup = c->d_counter + 3;
    b->mark(0);
    b->h_prefix.resize((size_t)nbuckets + 1);
    const bool async = (flags & SHK_BUILD_ASYNC) != 0;
    if ((rc = shk_bucketize((const uint64_t*)dh, (const uint64_t*)dl, N, nbuckets, b->keys.as<uint64_t>(),
                            b->prefix.as<uint64_t>(), ddup, scratch.p, ss, &b->max_bucket, c->stream,
                            async ? b->h_prefix.data() : nullptr)))
      break;
    HOST_TRACE("bucketize enqueued");
    if (async) {
      // the prefix is on the host already; the scatter and the sort are
      // still running: the duplicate flag follows them into pinned memory
      b->h_dup = c->h_flags + (c->flag_next++ & 63u);
      SHK_CUDA(cudaMemcpyAsync(b->h_dup, ddup, 4, cudaMemcpyDeviceToHost, c->stream));
      b->mark(1);
      b->dup_pending = true;
      *dup = -1;
      // host inputs were staged into pool buffers freed on return: finish now
      if (!(flags & SHK_DEVICE)) *dup = b->take_dup();
    } else {
      if ((rc = d2h(c, b->h_prefix.data(), b->prefix.p, (size_t)(nbuckets + 1) * 8))) break;
      int hd = 0;
      if ((rc = d2h(c, &hd, ddup, 4))) break;
      b->mark(1);
      if ((rc = csync(c))) break;
      b->phase_ms[0] = b->span(0, 1);
      *dup = hd;
    }
    if (max_bucket) *max_bucket = b->max_bucket;
  } while (0);
  if (rc) {
    delete b;
    return rc;
  }
  *out = b;
  HOST_TRACE("create return");
  return 0;
}

int shk_build_duplicate(shk_build* b, int* dup) {
  *dup = b->take_dup();
  return 0;
}

int shk_build_key_prefix(shk_build* b, uint64_t* out) {
  memcpy(out, b->h_prefix.data(), (size_t)(b->nb + 1) * 8);
  return 0;
}

int shk_build_sorted_keys(shk_build* b, uint64_t* hi, uint64_t* lo) {
  shk_ctx* c = b->c;
  DBuf th(c), tl(c);
  RC(th.alloc((size_t)b->N * 8));
  RC(tl.alloc((size_t)b->N * 8));
  RC(shk_launch_deinterleave(b->keys.as<uint64_t>(), b->N, th.as<uint64_t>(), tl.as<uint64_t>(), c->stream));
  RC(d2h(c, hi, th.p, (size_t)b->N * 8));
  RC(d2h(c, lo, tl.p, (size_t)b->N * 8));
  return csync(c);
}

int shk_build_run(shk_build* b, const shk_plans* plans, int mode, int cache_k, int cache_min_leaf, int64_t b0,
                  int64_t b1, uint64_t max_seed, int64_t* stats_out) {
  shk_ctx* c = b->c;
  if (b0 < 0 || b1 > b->nb || b0 > b1 || (mode != 0 && mode != 1)) {
    shk_set_error("invalid bucket range or mode");
    return SHK_INVALID;
  }
  HOST_TRACE("run");
  const PlanSet* SP = nullptr;
  RC(plan_cache_get(c, plans, &SP));
  const PlanSet& S = *SP;
  HOST_TRACE("plans loaded");
  const int64_t nbr = b1 - b0;
  // ---- per-bucket plan ids and global node numbering
  std::vector<int64_t> node_base((size_t)nbr + 1);
  std::vector<int32_t> bplan((size_t)nbr);
  int64_t nn = 0;
  for (int64_t i = 0; i < nbr; ++i) {
    const int64_t bu = b0 + i;
    const int64_t m = (int64_t)(b->h_prefix[bu + 1] - b->h_prefix[bu]);
    node_base[i] = nn;
    if (m == 0) {
      bplan[i] = -1;
      continue;
    }
    auto it = S.by_size.find(m);
    if (it == S.by_size.end()) {
      shk_set_error("no plan for bucket size %lld", (long long)m);
      return SHK_INVALID;
    }
    bplan[i] = it->second;
    nn += S.plan_off[it->second + 1] - S.plan_off[it->second];
  }
  node_base[nbr] = nn;
  b->nnodes = nn;
  // ---- per-plan facts: leaf count, largest leaf, validation
  const bool use_tree = c->opt[SHK_OPT_SCHEDULE] == 0 && !c->opt[SHK_OPT_EXACT_SPLIT_EVALS];
  const int64_t nplans = (int64_t)S.plan_m.size();
  std::vector<int64_t> plan_leaves((size_t)nplans, 0);
  std::vector<char> plan_used((size_t)nplans, 0);
  for (int64_t i = 0; i < nbr; ++i)
    if (bplan[i] >= 0) plan_used[bplan[i]] = 1;
  int max_leaf = 0;
  for (int64_t pl = 0; pl < nplans; ++pl) {
    if (!plan_used[pl]) continue;
    for (int64_t j = S.plan_off[pl]; j < S.plan_off[pl + 1]; ++j) {
      const PlanNode& nd = S.nodes[j];
      if (nd.kind == 0 && nd.m >= 32768) {
        shk_set_error("split node of %d keys exceeds the 32767-key split kernel limit", nd.m);
        return SHK_INVALID;
      }
      if (nd.kind != 0) {
        if (nd.m < 1 || nd.m > 64) {
          shk_set_error("leaf of %d keys outside 1..64", nd.m);
          return SHK_INVALID;
        }
        ++plan_leaves[pl];
        if (nd.m > max_leaf) max_leaf = nd.m;
      }
    }
  }
  int64_t n_leaves = 0;
  for (int64_t i = 0; i < nbr; ++i)
    if (bplan[i] >= 0) n_leaves += plan_leaves[bplan[i]];
  // ---- node tables: on the device for the persistent schedule, on the host
  // (split tasks per depth + leaf CSR) for the per-level schedule
  std::vector<int32_t> ng;
  std::vector<uint8_t> nkind;
  std::vector<std::vector<ShkSplitTask>> tasks((size_t)S.max_depth + 1);
  std::vector<int64_t> leaf_off, leaf_slot;
  std::vector<int64_t> kstart_v, root_pos;
  // persistent schedule: split roots open the split region [0, nsplit) of the
  // queue, leaf roots the leaf region [nsplit, nn) (shk_tree.cu)
  const int64_t nsplit = nn - n_leaves;
  int64_t nroots_split = 0, nroots_leaf = 0;
  if (use_tree) {
    kstart_v.resize((size_t)nbr);
    root_pos.resize((size_t)nbr);
    for (int64_t i = 0; i < nbr; ++i) {
      kstart_v[i] = (int64_t)b->h_prefix[b0 + i];
      if (bplan[i] < 0) {
        root_pos[i] = -1;
      } else if (S.nodes[S.plan_off[bplan[i]]].kind == 0) {
        root_pos[i] = nroots_split++;
      } else {
        root_pos[i] = nsplit + nroots_leaf++;
      }
    }
  } else {
    ng.resize((size_t)nn);
    nkind.resize((size_t)nn);
    leaf_off.reserve((size_t)n_leaves + 1);
    for (int64_t i = 0; i < nbr; ++i) {
      if (bplan[i] < 0) continue;
      const int64_t kstart = (int64_t)b->h_prefix[b0 + i];
      const int64_t pa = S.plan_off[bplan[i]], pb = S.plan_off[bplan[i] + 1];
      for (int64_t j = pa; j < pb; ++j) {
        const PlanNode& nd = S.nodes[j];
        const int64_t slot = node_base[i] + (j - pa);
        ng[slot] = nd.g;
        nkind[slot] = (uint8_t)(nd.kind != 0);
        if (nd.kind == 0) {
          ShkSplitTask t{};
          t.start = kstart + nd.off;
          t.m = nd.m;
          t.fanout = nd.fanout;
          for (int k = 0; k < 4; ++k) t.sizes[k] = nd.sizes[k];
          t.seed_slot = slot;
          tasks[nd.depth].push_back(t);
        } else {
          leaf_off.push_back(kstart + nd.off);
          leaf_slot.push_back(slot);
        }
      }
    }
    leaf_off.push_back((int64_t)b->h_prefix[b1]);  // leaves are contiguous: CSR end = range end
  }
  int64_t L = use_tree ? 0 : (int64_t)leaf_slot.size();
  HOST_TRACE("node numbering");
  // ---- device tables
  DBuf dseeds(c), dg(c), dkind(c), dtasks(c), dloff(c), dlslot(c), dlen(c), dpos(c), dnb(c), dbo(c), dacc(c),
      dscan(c);
  RC(dseeds.alloc((size_t)(nn + 1) * 8));
  RC(dg.alloc((size_t)(nn + 1) * 4));
  RC(dkind.alloc((size_t)(nn + 1)));
  RC(dacc.alloc(64));
  SHK_CUDA(cudaMemsetAsync(dacc.p, 0, 64, c->stream));
  int* exh = c->d_counter + 4;
  SHK_CUDA(cudaMemsetAsync(exh, 0, 4, c->stream));
  if (!use_tree) {
    RC(h2d(c, dg.p, ng.data(), (size_t)nn * 4));
    RC(h2d(c, dkind.p, nkind.data(), (size_t)nn));
    size_t ntask_total = 0;
    for (auto& v : tasks) ntask_total += v.size();
    RC(dtasks.alloc((ntask_total + 1) * sizeof(ShkSplitTask)));
    size_t o = 0;
    for (auto& v : tasks) {
      RC(h2d(c, dtasks.as<char>() + o * sizeof(ShkSplitTask), v.data(), v.size() * sizeof(ShkSplitTask)));
      o += v.size();
    }
    RC(dloff.alloc((size_t)(L + 1) * 8));
    RC(dlslot.alloc((size_t)(L + 1) * 8));
    RC(h2d(c, dloff.p, leaf_off.data(), (size_t)(L + 1) * 8));
    RC(h2d(c, dlslot.p, leaf_slot.data(), (size_t)L * 8));
  }
  if (b->keep_sorted && !b->sorted.p) {
    RC(b->sorted.alloc((size_t)b->N * 16));
    SHK_CUDA(cudaMemcpyAsync(b->sorted.p, b->keys.p, (size_t)b->N * 16, cudaMemcpyDeviceToDevice, c->stream));
  }
  b->mark(2);
  b->level_reset();
  // an asynchronous bucketize is checked here, after the host-side
  // preparation (which overlapped the sort) and before the first search --
  // by the construction kernel itself on the persistent schedule (it reads
  // the sort's device flag and does nothing when it is set; the host checks
  // once the kernel is done), so the launch is enqueued while the sort runs
  HOST_TRACE("tables");
  if (!use_tree && b->take_dup()) {
    shk_set_error("equal 128-bit codes in the input");
    return SHK_DUPLICATE;
  }
  HOST_TRACE("dup flag");
  // the seed searches take pre-mixed key high words (shk_hash.cuh premix_hi);
  // undone right after the leaves
  RC(shk_launch_premix(b->keys.as<uint64_t>(), b->N, 0, c->stream));
  // dtab: queue counters + hand-off words (64 B), then node_base, key starts,
  // root slots and bucket plans
  constexpr size_t kTabNodeBase = 64;
  DBuf dnodes(c), dqueue(c), dtab(c), dhand(c);
  if (use_tree && nn > 0) {
    // ---- node table expanded on the device from the (small) plan tables:
    // the plan nodes are the cached device copy; the per-bucket tables and
    // the queue counters go up in ONE copy from pinned staging
    RC(dnodes.alloc((size_t)nn * sizeof(ShkTreeNode)));
    RC(dqueue.alloc((size_t)nn * 8));
    const size_t o_qc = 0, o_nb = kTabNodeBase, o_ks = o_nb + (size_t)(nbr + 1) * 8, o_rp = o_ks + (size_t)(nbr + 1) * 8,
                 o_bp = o_rp + (size_t)(nbr + 1) * 8, tab_bytes = o_bp + (size_t)(nbr + 1) * 4;
    RC(dtab.alloc(tab_bytes));
    void* hs = nullptr;
    RC(host_stage(c, tab_bytes, &hs));
    char* H = (char*)hs;
    // split head, leaf head, split tail, leaf tail
    // then the hand-off flag, records written, resume fetch counter
    const unsigned long long qc[8] = {0ull, (unsigned long long)nsplit, (unsigned long long)nroots_split,
                                      (unsigned long long)(nsplit + nroots_leaf), 0ull, 0ull, 0ull, 0ull};
    memcpy(H + o_qc, qc, 64);
    memcpy(H + o_nb, node_base.data(), (size_t)(nbr + 1) * 8);
    memcpy(H + o_ks, kstart_v.data(), (size_t)nbr * 8);
    memcpy(H + o_rp, root_pos.data(), (size_t)nbr * 8);
    memcpy(H + o_bp, bplan.data(), (size_t)nbr * 4);
    RC(h2d(c, dtab.p, hs, tab_bytes));
    char* D = dtab.as<char>();
    SHK_CUDA(cudaMemsetAsync(dqueue.p, 0xFF, (size_t)nn * 8, c->stream));
    RC(shk_launch_expand_nodes(c->plans->d_nodes, c->plans->d_off, (const int32_t*)(D + o_bp),
                               (const int64_t*)(D + o_nb), (const int64_t*)(D + o_ks), (const int64_t*)(D + o_rp), nbr,
                               dnodes.as<ShkTreeNode>(), dg.as<int32_t>(), dkind.as<uint8_t>(), dqueue.as<int64_t>(),
                               c->stream));
    // ---- one persistent launch for every split node and leaf (shk_tree.cu)
    ShkTreeLaunch p{};
    p.keys = b->keys.as<uint64_t>();
    p.tmp = b->tmp.as<uint64_t>();
    p.nodes = dnodes.as<ShkTreeNode>();
    p.nnodes = nn;
    p.queue = dqueue.as<int64_t>();
    p.head = (unsigned long long*)(D + o_qc);
    p.tail = (unsigned long long*)(D + o_qc) + 2;
    p.dup_flag = b->dup_pending ? c->d_counter + 3 : nullptr;
    p.nsplit = nsplit;
    {
      // A/B of the slot-aware schedule: SHK_TREE_SLOT_AWARE=0 lets every warp
      // take split nodes; SHK_TREE_SLOW_WID=k sets the first leaf-only slot
      const char* e = getenv("SHK_TREE_SLOT_AWARE");
      const char* w = getenv("SHK_TREE_SLOW_WID");
      p.slow_wid = (e && e[0] == '0') ? (1 << 30) : (w ? atoi(w) : 0);
      const char* iw = getenv("SHK_TREE_IDLE_WID");
      p.idle_wid = iw ? atoi(iw) : 0;
      // leaf tail: slow-slot warps take no new leaf once fewer than
      // tail_reserve leaves remain (-1: one per fast warp)
      const char* tr = getenv("SHK_TREE_TAIL_RESERVE");
      p.tail_reserve = tr ? atoll(tr) : 0;
    }
    p.max_seed = max_seed;
    p.seeds = dseeds.as<int64_t>();
    p.mode = mode;
    p.cache_k = cache_k;
    p.cache_min_leaf = cache_min_leaf;
    p.max_n = max_leaf;
    p.choice_out = b->choice.as<uint8_t>();
    if (b->record) {
      RC(b->place.alloc((size_t)b->N * 8));
      p.place_out = b->place.as<int64_t>();
    }
    p.stats_acc = dacc.as<unsigned long long>();
    p.exhausted = exh;
    p.num_sms = c->num_sms;
    // rotate tail hand-off (shk_tree.cu): SHK_TREE_HANDOFF_TW = warps per
    // resume team (0 = off: the flag is never raised)
    if (mode != 0) {
      const char* ht = getenv("SHK_TREE_HANDOFF_TW");
      p.handoff_tw = ht ? atoi(ht) : 8;
      p.handoff_cap = (int64_t)(c->num_sms > 0 ? c->num_sms : 148) * 64;
      RC(dhand.alloc((size_t)p.handoff_cap * 56));
      p.handoff = dhand.p;
      p.abort_flag = (int*)(D + o_qc + 32);
      p.handoff_count = dacc.as<unsigned long long>() + 7;  // read back with the stats
      p.handoff_next = (unsigned long long*)(D + o_qc + 40);
    }
    RC(shk_launch_tree(p, c->stream));
    HOST_TRACE("tree launched");
    b->mark(3);
  }
  // ---- splits, level by level (every node of one depth in one launch)
  if (!use_tree) {
    size_t o = 0;
    for (auto& v : tasks) {
      if (!v.empty()) {
        ShkSplitLaunch p{};
        p.hi = b->keys.as<uint64_t>();
        p.tmp_hi = b->tmp.as<uint64_t>();
        p.tasks = dtasks.as<ShkSplitTask>() + o;
        p.ntasks = (int64_t)v.size();
        p.max_seed = max_seed;
        p.seeds = dseeds.as<int64_t>();
        p.evals_out = nullptr;
        p.counter = c->d_counter;
        p.num_sms = c->num_sms;
        p.partition = 1;
        p.exhausted = exh;
        p.evals_acc = dacc.as<unsigned long long>() + 6;
        p.exact_evals = c->opt[SHK_OPT_EXACT_SPLIT_EVALS] ? 1 : 0;
        b->level_mark((int)(&v - &tasks[0]));
        RC(shk_launch_split(p, c->stream));
      }
      o += v.size();
    }
    b->level_mark((int)tasks.size());
  }
  // ---- leaves
  b->mark(3);
  if (L > 0) {
    ShkLeafLaunch p{};
    p.hi = b->keys.as<uint64_t>();
    p.lo = b->keys.as<uint64_t>() + 1;
    p.stride = 2;
    p.pre = 1;
    p.off = dloff.as<int64_t>();
    p.L = L;
    p.max_n = max_leaf;
    p.max_seed = max_seed;
    p.mode = mode;
    p.cache_k = cache_k;
    p.cache_min_leaf = cache_min_leaf;
    p.seed_out = dseeds.as<int64_t>();
    p.seed_slot = dlslot.as<int64_t>();
    p.fbits_out = nullptr;
    p.choice_out = b->choice.as<uint8_t>();
    p.stats_out = nullptr;
    p.stats_acc = dacc.as<unsigned long long>();
    p.counter = c->d_counter;
    p.error = c->d_counter + 1;
    p.exhausted = exh;
    p.num_sms = c->num_sms;
    p.team_warps = (int)c->opt[SHK_OPT_LEAF_TEAM_WARPS];
    if (b->record) {
      RC(b->place.alloc((size_t)b->N * 8));
      p.place_out = b->place.as<int64_t>();
    }
    RC(shk_launch_leaf_search(p, c->stream));
  }
  RC(shk_launch_premix(b->keys.as<uint64_t>(), b->N, 1, c->stream));
  b->mark(4);
  // ---- Rice stream: lengths -> scan -> scatter.  The lengths are computed
  // before the host has seen the exhaustion flag (one round trip instead of
  // two): with an exhausted search they are garbage and the flag, read with
  // the total, stops the build before anything is sized from them.
  int hex = 0;
  RC(d2h(c, &hex, exh, 4));
  RC(dlen.alloc((size_t)(nn + 1) * 8));
  RC(dpos.alloc((size_t)(nn + 2) * 8));
  RC(shk_rice_lengths(dseeds.as<int64_t>(), dg.as<int32_t>(), nn, dlen.as<int64_t>(), c->stream));
  size_t ss = shk_scan_scratch(nn);
  RC(dscan.alloc(ss));
  RC(shk_exclusive_scan_i64(dlen.as<int64_t>(), dpos.as<int64_t>(), nn, dscan.p, ss, c->stream));
  seed_bits_kernel<<<64, 256, 0, c->stream>>>(dlen.as<int64_t>(), dkind.as<uint8_t>(), nn,
                                               dacc.as<unsigned long long>() + 4);
  SHK_LAUNCHED();
  int64_t total_bits = 0;
  RC(d2h(c, &total_bits, dpos.as<int64_t>() + nn, 8));
  RC(csync(c));
  HOST_TRACE("tree done + rice length");
  if (b->take_dup()) {  // the persistent schedule checks the flag on the device (above)
    shk_set_error("equal 128-bit codes in the input");
    return SHK_DUPLICATE;
  }
  if (hex) {
    shk_set_error("seed search exhausted (max_seed %llu)", (unsigned long long)max_seed);
    return SHK_EXHAUSTED;
  }
  b->bit_len = total_bits;
  b->nwords = (total_bits + 63) / 64;
  RC(b->words.alloc((size_t)(b->nwords + 1) * 8));
  SHK_CUDA(cudaMemsetAsync(b->words.p, 0, (size_t)(b->nwords + 1) * 8, c->stream));
  RC(shk_rice_scatter(dseeds.as<int64_t>(), dg.as<int32_t>(), dpos.as<int64_t>(), nn, b->words.as<uint64_t>(),
                      c->stream));
  // per-bucket bit offsets: pos[node_base[i]]
  // (the persistent schedule's device copy of node_base is still in dtab)
  const int64_t* d_nb = dtab.p ? (const int64_t*)(dtab.as<char>() + kTabNodeBase) : nullptr;
  if (!d_nb) {
    RC(dnb.alloc((size_t)(nbr + 1) * 8));
    RC(h2d(c, dnb.p, node_base.data(), (size_t)(nbr + 1) * 8));
    d_nb = dnb.as<int64_t>();
  }
  RC(dbo.alloc((size_t)(nbr + 1) * 8));
  gather_bitoff_kernel<<<(unsigned)((nbr + 256) / 256), 256, 0, c->stream>>>(dpos.as<int64_t>(), d_nb, nbr,
                                                                              dbo.as<uint64_t>());
  SHK_LAUNCHED();
  b->bit_off.resize((size_t)nbr + 1);
  RC(d2h(c, b->bit_off.data(), dbo.p, (size_t)(nbr + 1) * 8));
  unsigned long long acc[8];
  RC(d2h(c, acc, dacc.p, 64));
  b->mark(5);
  RC(csync(c));
  b->phase_ms[1] = b->span(2, 3);
  b->phase_ms[2] = b->span(3, 4);
  b->phase_ms[3] = b->span(4, 5);
  b->split_evals = (int64_t)acc[6];
  if (stats_out) {
    stats_out[0] = (int64_t)acc[0];
    stats_out[1] = (int64_t)acc[1];
    stats_out[2] = (int64_t)acc[2];
    stats_out[3] = (int64_t)acc[3];
    stats_out[4] = (int64_t)acc[4];  // leaf seed bits
    stats_out[5] = (int64_t)acc[5];  // split seed bits
    stats_out[6] = n_leaves;
    stats_out[7] = (int64_t)acc[7];  // leaves the tree kernel handed off to the resume teams
  }
  b->b0 = b0;
  b->b1 = b1;
  b->ran = true;
  HOST_TRACE("run return");
  return 0;
}

int shk_build_stream_size(shk_build* b, int64_t* bit_len, int64_t* nwords) {
  if (!b->ran) {
    shk_set_error("shk_build_run first");
    return SHK_INVALID;
  }
  *bit_len = b->bit_len;
  *nwords = b->nwords;
  return 0;
}

int shk_build_stream(shk_build* b, uint64_t* words, uint64_t* bit_offsets) {
  if (!b->ran) {
    shk_set_error("shk_build_run first");
    return SHK_INVALID;
  }
  if (words) RC(d2h(b->c, words, b->words.p, (size_t)b->nwords * 8));
  if (bit_offsets) memcpy(bit_offsets, b->bit_off.data(), b->bit_off.size() * 8);
  return csync(b->c);
}

int shk_build_set_record_placements(shk_build* b, int on) {
  b->record = on != 0;
  return 0;
}

int shk_build_set_keep_sorted(shk_build* b, int on) {
  b->keep_sorted = on != 0;
  return 0;
}

// ---- column-sharded ribbon over the build's sorted keys ---------------------
int shk_build_dribbon_begin(shk_build* b, const uint8_t* choice_sorted, int flags, int64_t m, uint64_t seed,
                            int64_t c0, int64_t c1, int64_t* n_export, int* bad) {
  shk_ctx* c = b->c;
  if (!b->sorted.p) {
    shk_set_error("sorted keys were not kept (shk_build_set_keep_sorted)");
    return SHK_INVALID;
  }
  if (!b->drhs.p) {
    RC(b->drhs.alloc((size_t)b->N));
  }
  if (flags & SHK_DEVICE)
    SHK_CUDA(cudaMemcpyAsync(b->drhs.p, choice_sorted, (size_t)b->N, cudaMemcpyDeviceToDevice, c->stream));
  else
    RC(h2d(c, b->drhs.p, choice_sorted, (size_t)b->N));
  b->dcols = c1 - c0;
  b->mark(6);  // ribbon phase: from here to the end of backsub (exchanges included)
  return shk_ribbon_dist_begin(c->rib, b->sorted.as<uint64_t>(), b->drhs.as<uint8_t>(), b->N, m, seed, c0, c1,
                               n_export, bad, c->stream);
}

// Column-sharded ribbon from explicit rows' keys (device, interleaved
// (hi, lo) pairs) and their rhs bytes: the input-sharded build routes every
// key with its choice bit to the owner of its row's start column first.
int shk_build_dribbon_begin_keys(shk_build* b, const uint64_t* keys_dev, const uint8_t* rhs_dev, int64_t n, int64_t m,
                                 uint64_t seed, int64_t c0, int64_t c1, int64_t* n_export, int* bad) {
  shk_ctx* c = b->c;
  b->dcols = c1 - c0;
  b->mark(6);
  return shk_ribbon_dist_begin(c->rib, keys_dev, rhs_dev, n, m, seed, c0, c1, n_export, bad, c->stream);
}

// Device pointers of the build's keys in leaf order (interleaved pairs) and
// their choice bytes, valid until the build is destroyed (after run()).
int shk_build_leaf_arrays(shk_build* b, void** keys_dev, void** choice_dev) {
  if (!b->ran) {
    shk_set_error("leaf arrays need a finished run()");
    return SHK_INVALID;
  }
  *keys_dev = b->keys.p;
  *choice_dev = b->choice.p;
  return 0;
}

int shk_build_dribbon_exports(shk_build* b, void* rows_out, int64_t n) {
  return shk_ribbon_dist_take_exports(b->c->rib, rows_out, n, b->c->stream);
}

int shk_build_dribbon_import(shk_build* b, const void* rows_in, int64_t n, int64_t* n_export, int* bad) {
  return shk_ribbon_dist_import(b->c->rib, rows_in, n, n_export, bad, b->c->stream);
}

int shk_build_dribbon_backsub(shk_build* b, const uint32_t* y_in, uint32_t* y_out, uint64_t* words_out) {
  shk_ctx* c = b->c;
  const int64_t nw = (b->dcols + 63) / 64;
  DBuf tw(c);
  RC(tw.alloc((size_t)nw * 8));
  RC(shk_ribbon_dist_backsub(c->rib, y_in, y_out, tw.as<uint64_t>(), c->stream));
  RC(d2h(c, words_out, tw.p, (size_t)nw * 8));
  b->mark(7);
  RC(csync(c));
  b->phase_ms[4] = b->span(6, 7);
  return 0;
}

int shk_build_dribbon_map(shk_build* b, uint32_t* map_out) {
  return shk_ribbon_dist_map(b->c->rib, map_out, b->c->stream);
}

int shk_build_dribbon_finish(shk_build* b, const uint32_t* y_in, uint64_t* words_out) {
  shk_ctx* c = b->c;
  const int64_t nw = (b->dcols + 63) / 64;
  DBuf tw(c);
  RC(tw.alloc((size_t)nw * 8));
  RC(shk_ribbon_dist_finish(c->rib, y_in, tw.as<uint64_t>(), c->stream));
  RC(d2h(c, words_out, tw.p, (size_t)nw * 8));
  b->mark(7);
  RC(csync(c));
  b->phase_ms[4] = b->span(6, 7);
  return 0;
}

int shk_build_choice_sorted(shk_build* b, int64_t k0, int64_t k1, uint8_t* out, int flags) {
  shk_ctx* c = b->c;
  if (!b->sorted.p || !b->ran) {
    shk_set_error("choice_sorted needs shk_build_set_keep_sorted before shk_build_run");
    return SHK_INVALID;
  }
  if (k0 < 0 || k1 > b->N || k0 > k1) {
    shk_set_error("bad key range");
    return SHK_INVALID;
  }
  if (k1 == k0) return 0;
  if (flags & SHK_DEVICE) {  // straight into the caller's (collective) buffer
    RC(shk_launch_choice_sorted(b->keys.as<uint64_t>(), b->sorted.as<uint64_t>(), b->prefix.as<int64_t>(), b->nb,
                                b->choice.as<uint8_t>(), k0, k1, out, c->stream));
    return csync(c);
  }
  DBuf d(c);
  RC(d.alloc((size_t)(k1 - k0)));
  RC(shk_launch_choice_sorted(b->keys.as<uint64_t>(), b->sorted.as<uint64_t>(), b->prefix.as<int64_t>(), b->nb,
                              b->choice.as<uint8_t>(), k0, k1, d.as<uint8_t>(), c->stream));
  RC(d2h(c, out, d.p, (size_t)(k1 - k0)));
  return csync(c);
}

int shk_build_placements(shk_build* b, int64_t* out) {
  if (!b->ran || !b->record) {
    shk_set_error("placements were not recorded");
    return SHK_INVALID;
  }
  RC(d2h(b->c, out, b->place.p, (size_t)b->N * 8));
  return csync(b->c);
}

int shk_build_choice(shk_build* b, uint8_t* choice) {
  RC(d2h(b->c, choice, b->choice.p, (size_t)b->N));
  return csync(b->c);
}

int shk_build_ribbon(shk_build* b, const uint8_t* choice, int choice_flags, int64_t m, int max_tries,
                     uint64_t* seed_out, uint64_t* words_out) {
  shk_ctx* c = b->c;
  HOST_TRACE("ribbon");
  if (m < 128) {
    shk_set_error("ribbon needs m >= 128");
    return SHK_INVALID;
  }
  const uint8_t* drhs = b->choice.as<uint8_t>();
  DBuf tr(c);
  if (choice) {
    const void* d;
    RC(stage_in(c, choice_flags, choice, (size_t)b->N, tr, &d));
    drhs = (const uint8_t*)d;
  }
  const int64_t nw = (m + 63) / 64;
  DBuf tw(c);
  RC(tw.alloc((size_t)nw * 8));
  // SHK_RIBBON_SORTED_KEYS: rows from the bucket-sorted copy (choice given in
  // that order), as a sharded build's rank 0 does
  const uint64_t* rkeys = b->keys.as<uint64_t>();
  if (choice_flags & 4) {
    if (!b->sorted.p) {
      shk_set_error("sorted keys were not kept (shk_build_set_keep_sorted)");
      return SHK_INVALID;
    }
    rkeys = b->sorted.as<uint64_t>();
  }
  b->mark(6);
  HOST_TRACE("ribbon start");
  RC(ribbon_seed_loop(c, rkeys, drhs, b->N, m, max_tries, seed_out, tw.as<uint64_t>()));
  HOST_TRACE("ribbon solved");
  b->mark(7);
  RC(d2h(c, words_out, tw.p, (size_t)nw * 8));
  RC(csync(c));
  b->phase_ms[4] = b->span(6, 7);
  return 0;
}

int shk_build_level_ms(shk_build* b, float* ms, int32_t* depth, int max_levels) {
  int k = 0;
  for (size_t i = 0; i + 1 < b->lev.size() && k < max_levels; ++i, ++k) {
    float t = 0;
    if (cudaEventElapsedTime(&t, b->lev[i], b->lev[i + 1]) != cudaSuccess) cudaGetLastError();
    ms[k] = t;
    if (depth) depth[k] = b->lev_depth[i];
  }
  return k;
}

int shk_build_phase_ms(shk_build* b, float* ms, int64_t* split_evals) {
  for (int i = 0; i < 5; ++i) ms[i] = b->phase_ms[i];
  if (split_evals) *split_evals = b->split_evals;
  return 0;
}

int shk_build_destroy(shk_build* b) {
  delete b;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Query descriptor.

struct shk_qdesc {
  shk_ctx* c;
  ShkQueryDesc d{};
  DBuf kp, bo, sw, rw, bplan, nbase, npos, bbad, kind, g, mm, child, sizes, fan, poff, planq, bucketq;
  int64_t nnodes = 0;
  explicit shk_qdesc(shk_ctx* ctx)
      : c(ctx), kp(ctx), bo(ctx), sw(ctx), rw(ctx), bplan(ctx), nbase(ctx), npos(ctx), bbad(ctx), kind(ctx), g(ctx),
        mm(ctx), child(ctx), sizes(ctx), fan(ctx), poff(ctx), planq(ctx), bucketq(ctx) {}
};

extern "C" {

int shk_qdesc_create(shk_ctx* c, int64_t n_keys, int64_t nbuckets, int mode, int64_t cache_k,
                     const uint64_t* key_prefix, const uint64_t* bit_offsets, const uint64_t* stream_words,
                     int64_t stream_nwords, int64_t stream_bit_len, const shk_plans* plans, uint64_t rib_seed,
                     int64_t rib_m, const uint64_t* rib_words, int64_t rib_nwords, shk_qdesc** out) {
  if (nbuckets < 1 || nbuckets > 0xFFFFFFFFll) {
    shk_set_error("invalid bucket count");
    return SHK_INVALID;
  }
  if (stream_nwords * 64 < stream_bit_len) {
    shk_set_error("stream bit length exceeds the word array");
    return SHK_INVALID;
  }
  if (rib_m != 0 && (rib_m < shk::RIBBON_W || rib_m > (1ll << 40))) {
    shk_set_error("invalid retrieval column count %lld", (long long)rib_m);
    return SHK_INVALID;
  }
  PlanSet S;
  RC(load_plans(plans, S));
  shk_qdesc* q = new shk_qdesc(c);
  std::unique_ptr<shk_qdesc> guard(q);
  std::vector<int32_t> bplan((size_t)nbuckets);
  std::vector<int64_t> nbase((size_t)nbuckets + 1);
  int64_t nn = 0;
  for (int64_t bu = 0; bu < nbuckets; ++bu) {
    const int64_t m = (int64_t)(key_prefix[bu + 1] - key_prefix[bu]);
    nbase[bu] = nn;
    if (m <= 0) {
      bplan[bu] = -1;
      continue;
    }
    auto it = S.by_size.find(m);
    if (it == S.by_size.end()) {
      shk_set_error("no plan for bucket size %lld", (long long)m);
      return SHK_INVALID;
    }
    bplan[bu] = it->second;
    nn += S.plan_off[it->second + 1] - S.plan_off[it->second];
  }
  nbase[nbuckets] = nn;
  q->nnodes = nn;
  const size_t np = S.nodes.size();
  std::vector<int32_t> kind(np), g(np), mm(np), child(np * 4), sizes(np * 4), fan(np);
  std::vector<uint32_t> planq(np * 4, 0u);
  for (size_t j = 0; j < np; ++j) {
    kind[j] = S.nodes[j].kind;
    g[j] = S.nodes[j].g;
    mm[j] = S.nodes[j].m;
    fan[j] = S.nodes[j].fanout;
    for (int k = 0; k < 4; ++k) {
      child[4 * j + k] = S.nodes[j].child[k];
      sizes[4 * j + k] = S.nodes[j].sizes[k];
    }
    // one uint4 of 16-bit fields (m < 32768, plan-local child ids < 65536):
    // {m | leaf << 15 | b1 << 16, b2 | b3 << 16, c0 | c1 << 16, c2 | c3 << 16}
    // with b_k the cumulative part bounds (0xFFFF past the fanout: r < m
    // never reaches them), so part = #(b_k <= r), the offset is lane `part`
    // of (0, b1, b2, b3) and the child is lane `part` of (c0, c1, c2, c3)
    auto u16 = [](int32_t v) { return (uint32_t)v & 0xFFFFu; };
    uint32_t bnd[4] = {0, 0xFFFFu, 0xFFFFu, 0xFFFFu};
    if (kind[j] == 0) {
      uint32_t acc = 0;
      for (int k = 1; k < fan[j]; ++k) {
        acc += (uint32_t)sizes[4 * j + k - 1];
        bnd[k] = acc;
      }
    }
    uint32_t* e = &planq[4 * j];
    e[0] = u16(mm[j]) | ((kind[j] != 0 ? 1u : 0u) << 15) | (bnd[1] << 16);
    e[1] = bnd[2] | (bnd[3] << 16);
    e[2] = u16(child[4 * j]) | (u16(child[4 * j + 1]) << 16);
    e[3] = u16(child[4 * j + 2]) | (u16(child[4 * j + 3]) << 16);
  }
  // one uint4 per bucket (a query's first random load is a single 16-byte
  // gather): {kp0 lo, kp0 hi8 | node_base hi8 << 8 | bad << 16, node_base lo,
  // first plan node or 0xFFFFFFFF for an empty bucket}; bad = the first
  // undecodable plan-local node (0xFFFF: none; plan nodes are < 65535), set on
  // the device by node_index_kernel.  Key prefixes and node counts < 2^40.
  if (key_prefix[nbuckets] >= (1ull << 40) || nn >= (1ll << 40) || S.plan_off.back() >= 0xFFFFFFFFll) {
    shk_set_error("descriptor too large for the query tables");
    return SHK_INVALID;
  }
  std::vector<uint32_t> bucketq((size_t)nbuckets * 4, 0u);
  for (int64_t bu = 0; bu < nbuckets; ++bu) {
    uint32_t* e = &bucketq[4 * bu];
    const uint64_t kp0 = key_prefix[bu], nb0 = (uint64_t)nbase[bu];
    e[0] = (uint32_t)kp0;
    e[1] = (uint32_t)(kp0 >> 32) | ((uint32_t)(nb0 >> 32) << 8) | (0xFFFFu << 16);
    e[2] = (uint32_t)nb0;
    e[3] = bplan[bu] >= 0 ? (uint32_t)S.plan_off[bplan[bu]] : 0xFFFFFFFFu;
  }
  const int64_t rnw = rib_nwords > 0 ? rib_nwords : 0;
  RC(q->kp.alloc((size_t)(nbuckets + 1) * 8));
  RC(q->bo.alloc((size_t)(nbuckets + 1) * 8));
  RC(q->sw.alloc((size_t)(stream_nwords + 1) * 8));
  // zero padding past the words: the query's paired loads may read up to
  // word ceil(m / 64) + 1 (the reference reads zeros out of range)
  const int64_t rnw_alloc = (rnw > (rib_m + 63) / 64 ? rnw : (rib_m + 63) / 64) + 2;
  RC(q->rw.alloc((size_t)rnw_alloc * 8));
  RC(q->bplan.alloc((size_t)nbuckets * 4));
  RC(q->nbase.alloc((size_t)(nbuckets + 1) * 8));
  RC(q->npos.alloc((size_t)(nn + 1) * 8));
  RC(q->bbad.alloc((size_t)nbuckets * 4));
  RC(q->kind.alloc(np * 4 + 4));
  RC(q->g.alloc(np * 4 + 4));
  RC(q->mm.alloc(np * 4 + 4));
  RC(q->child.alloc(np * 16 + 16));
  RC(q->sizes.alloc(np * 16 + 16));
  RC(q->fan.alloc(np * 4 + 4));
  RC(q->poff.alloc(S.plan_off.size() * 8 + 8));
  RC(q->planq.alloc(np * 16 + 16));
  RC(q->bucketq.alloc((size_t)nbuckets * 16 + 16));
  RC(h2d(c, q->planq.p, planq.data(), np * 16));
  RC(h2d(c, q->bucketq.p, bucketq.data(), (size_t)nbuckets * 16));
  RC(h2d(c, q->kp.p, key_prefix, (size_t)(nbuckets + 1) * 8));
  RC(h2d(c, q->bo.p, bit_offsets, (size_t)(nbuckets + 1) * 8));
  SHK_CUDA(cudaMemsetAsync(q->sw.p, 0, (size_t)(stream_nwords + 1) * 8, c->stream));
  RC(h2d(c, q->sw.p, stream_words, (size_t)stream_nwords * 8));
  SHK_CUDA(cudaMemsetAsync(q->rw.p, 0, (size_t)rnw_alloc * 8, c->stream));
  if (rnw) RC(h2d(c, q->rw.p, rib_words, (size_t)rnw * 8));
  RC(h2d(c, q->bplan.p, bplan.data(), (size_t)nbuckets * 4));
  RC(h2d(c, q->nbase.p, nbase.data(), (size_t)(nbuckets + 1) * 8));
  RC(h2d(c, q->kind.p, kind.data(), np * 4));
  RC(h2d(c, q->g.p, g.data(), np * 4));
  RC(h2d(c, q->mm.p, mm.data(), np * 4));
  RC(h2d(c, q->child.p, child.data(), np * 16));
  RC(h2d(c, q->sizes.p, sizes.data(), np * 16));
  RC(h2d(c, q->fan.p, fan.data(), np * 4));
  RC(h2d(c, q->poff.p, S.plan_off.data(), S.plan_off.size() * 8));
  ShkQueryDesc& d = q->d;
  d.nbuckets = nbuckets;
  d.n_keys = n_keys;
  d.mode = mode;
  d.cache_k = cache_k;
  d.key_prefix = q->kp.as<uint64_t>();
  d.bucket_plan = q->bplan.as<int32_t>();
  d.node_base = q->nbase.as<int64_t>();
  d.node_val = q->npos.as<uint64_t>();
  d.planq = q->planq.as<uint4>();
  d.bucketq = q->bucketq.as<uint4>();
  d.bucket_bad = q->bbad.as<int32_t>();
  d.bit_offsets = q->bo.as<uint64_t>();
  d.stream = q->sw.as<uint64_t>();
  d.stream_bit_len = stream_bit_len;
  d.stream_nwords = stream_nwords;
  d.pn_kind = q->kind.as<int32_t>();
  d.pn_g = q->g.as<int32_t>();
  d.pn_m = q->mm.as<int32_t>();
  d.pn_child = q->child.as<int32_t>();
  d.pn_sizes = q->sizes.as<int32_t>();
  d.pn_fanout = q->fan.as<int32_t>();
  d.plan_off = q->poff.as<int64_t>();
  d.rib_seed = rib_seed;
  d.rib_m = rib_m;
  d.rib_words = q->rw.as<uint64_t>();
  d.rib_nwords = rnw;
  RC(shk_launch_node_index(d, q->npos.as<uint64_t>(), q->bbad.as<int32_t>(), c->stream));
  RC(csync(c));
  *out = guard.release();
  return 0;
}

int shk_query(shk_qdesc* q, const uint64_t* hi, const uint64_t* lo, int64_t Q, uint64_t* out, int clamp, int flags) {
  shk_ctx* c = q->c;
  if (Q <= 0) return 0;
  DBuf th(c), tl(c), to(c);
  const void *dh, *dl;
  void* dout;
  RC(stage_in(c, flags, hi, (size_t)Q * 8, th, &dh));
  RC(stage_in(c, flags, lo, (size_t)Q * 8, tl, &dl));
  RC(stage_out(c, flags, out, (size_t)Q * 8, to, &dout));
  int* err = c->d_counter + 5;
  SHK_CUDA(cudaMemsetAsync(err, 0, 4, c->stream));
  RC(shk_launch_query(q->d, (const uint64_t*)dh, (const uint64_t*)dl, Q, (uint64_t*)dout, err, clamp, c->stream));
  RC(finish_out(c, flags, out, to, (size_t)Q * 8));
  int herr = 0;
  RC(d2h(c, &herr, err, 4));
  RC(csync(c));
  if (herr) {
    shk_set_error("bit stream overrun");
    return SHK_FORMAT;
  }
  return 0;
}

// query_many(keys) end to end from a host buffer of fixed-length keys:
// chunks of the key blob go H2D on the copy stream, are fingerprinted on the
// context stream and queried on a third stream, and the outputs come back D2H
// on a second copy stream, so the PCIe transfers of chunk k+1 (in) and k-1
// (out) overlap the kernels of chunk k.  Host-blocking.  (recsplit.py:270-275:
// master_hash_many + query_hashed_many.)
int shk_query_blob(shk_qdesc* q, const uint8_t* blob, int key_len, int64_t Q, uint64_t salt, uint64_t* out, int clamp) {
  shk_ctx* c = q->c;
  if (Q <= 0) return 0;
  if (key_len < 1 || key_len > 128) {
    shk_set_error("fixed-length keys must be 1..128 bytes");
    return SHK_INVALID;
  }
  const int64_t CH = (int64_t)1 << 22;  // keys per chunk
  const int64_t per = Q < CH ? Q : CH;
  // Four stages on four streams, every buffer double: H2D (copy stream) ->
  // fingerprints (context stream) -> query (its own stream) -> D2H (second
  // copy stream).  The fingerprint kernel is ALU-bound and the query kernel
  // gather-bound, so chunk k's query runs beside chunk k+1's fingerprints
  // and the PCIe transfers bound the call (back to back on one stream the two
  // kernels of a chunk took longer than its H2D).
  DBuf kb[2] = {DBuf(c), DBuf(c)}, ob[2] = {DBuf(c), DBuf(c)}, hh[2] = {DBuf(c), DBuf(c)}, ll[2] = {DBuf(c), DBuf(c)};
  for (int k = 0; k < 2; ++k) {
    RC(kb[k].alloc((size_t)per * key_len));
    RC(ob[k].alloc((size_t)per * 8));
    RC(hh[k].alloc((size_t)per * 8));
    RC(ll[k].alloc((size_t)per * 8));
  }
  int* err = c->d_counter + 5;
  SHK_CUDA(cudaMemsetAsync(err, 0, 4, c->stream));
  const int64_t nch = (Q + per - 1) / per;
  cudaStream_t qs = nullptr;
  SHK_CUDA(cudaStreamCreateWithFlags(&qs, cudaStreamNonBlocking));
  cudaEvent_t in_done[2], hash_done[2], query_done[2], out_done[2];
  for (int k = 0; k < 2; ++k) {
    SHK_CUDA(cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming));
    SHK_CUDA(cudaEventCreateWithFlags(&hash_done[k], cudaEventDisableTiming));
    SHK_CUDA(cudaEventCreateWithFlags(&query_done[k], cudaEventDisableTiming));
    SHK_CUDA(cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming));
  }
  int rc = 0;
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess && !rc) {
      shk_set_error("query pipeline: %s", cudaGetErrorString(e));
      rc = -1000 - (int)e;
    }
    return e == cudaSuccess;
  };
  for (int64_t k = 0; k < nch && !rc; ++k) {
    const int s = (int)(k & 1);
    const int64_t a = k * per, n = (a + per < Q) ? per : Q - a;
    // H2D: the key buffer is free once chunk k-2 was fingerprinted
    if (k >= 2 && !ck(cudaStreamWaitEvent(c->copy, hash_done[s], 0))) break;
    if (!ck(cudaMemcpyAsync(kb[s].p, blob + (size_t)a * key_len, (size_t)n * key_len, cudaMemcpyHostToDevice, c->copy)))
      break;
    if (!ck(cudaEventRecord(in_done[s], c->copy))) break;
    // fingerprints: the code buffers are free once chunk k-2 was queried
    if (!ck(cudaStreamWaitEvent(c->stream, in_done[s], 0))) break;
    if (k >= 2 && !ck(cudaStreamWaitEvent(c->stream, query_done[s], 0))) break;
    rc = shk_launch_blake2b_fixed(kb[s].as<uint8_t>(), key_len, n, salt, hh[s].as<uint64_t>(), ll[s].as<uint64_t>(),
                                  c->stream);
    if (rc) break;
    if (!ck(cudaEventRecord(hash_done[s], c->stream))) break;
    // query: the output buffer is free once chunk k-2 was copied out
    if (!ck(cudaStreamWaitEvent(qs, hash_done[s], 0))) break;
    if (k >= 2 && !ck(cudaStreamWaitEvent(qs, out_done[s], 0))) break;
    rc = shk_launch_query(q->d, hh[s].as<uint64_t>(), ll[s].as<uint64_t>(), n, ob[s].as<uint64_t>(), err, clamp, qs);
    if (rc) break;
    if (!ck(cudaEventRecord(query_done[s], qs))) break;
    // D2H
    if (!ck(cudaStreamWaitEvent(c->copy_out, query_done[s], 0))) break;
    if (!ck(cudaMemcpyAsync(out + a, ob[s].p, (size_t)n * 8, cudaMemcpyDeviceToHost, c->copy_out))) break;
    if (!ck(cudaEventRecord(out_done[s], c->copy_out))) break;
  }
  cudaStreamSynchronize(c->copy);
  cudaStreamSynchronize(c->stream);
  cudaStreamSynchronize(qs);
  cudaStreamSynchronize(c->copy_out);
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(in_done[k]);
    cudaEventDestroy(hash_done[k]);
    cudaEventDestroy(query_done[k]);
    cudaEventDestroy(out_done[k]);
  }
  cudaStreamDestroy(qs);
  if (rc) return rc;
  int herr = 0;
  RC(d2h(c, &herr, err, 4));
  RC(csync(c));
  if (herr) {
    shk_set_error("bit stream overrun");
    return SHK_FORMAT;
  }
  return 0;
}

int shk_verify(shk_qdesc* q, const uint64_t* hi, const uint64_t* lo, int64_t Q, int flags, int* ok,
               int64_t* offender) {
  shk_ctx* c = q->c;
  *ok = 0;
  *offender = -1;
  const int64_t N = q->d.n_keys;
  if (Q != N) return 0;  // not a bijection onto [0, N); no offender (recsplit.py:388-389)
  if (N <= 0) {
    *ok = 1;
    return 0;
  }
  DBuf th(c), tl(c), vals(c), first(c), off(c);
  const void *dh, *dl;
  RC(stage_in(c, flags, hi, (size_t)Q * 8, th, &dh));
  RC(stage_in(c, flags, lo, (size_t)Q * 8, tl, &dl));
  RC(vals.alloc((size_t)Q * 8));
  RC(first.alloc((size_t)N * 8));
  RC(off.alloc(8));
  int* err = c->d_counter + 5;
  SHK_CUDA(cudaMemsetAsync(err, 0, 4, c->stream));
  RC(shk_launch_query(q->d, (const uint64_t*)dh, (const uint64_t*)dl, Q, vals.as<uint64_t>(), err, 1, c->stream));
  RC(shk_launch_bijection(vals.as<uint64_t>(), Q, N, first.as<unsigned long long>(), off.as<unsigned long long>(),
                          c->stream));
  int herr = 0;
  unsigned long long hoff = 0;
  RC(d2h(c, &herr, err, 4));
  RC(d2h(c, &hoff, off.p, 8));
  RC(csync(c));
  if (herr) {
    shk_set_error("bit stream overrun");
    return SHK_FORMAT;
  }
  if (hoff == ~0ull) {
    *ok = 1;
  } else {
    *offender = (int64_t)hoff;
  }
  return 0;
}

int shk_qdesc_destroy(shk_qdesc* q) {
  delete q;
  return 0;
}

}  // extern "C"
