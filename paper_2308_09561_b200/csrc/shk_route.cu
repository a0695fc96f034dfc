// Routing keys to the rank that owns them (input-sharded multi-GPU build,
// dist.py): by bucket (recsplit.py:475-483's bucket hash; rank r owns the
// bucket range shard_range(nb, r, W)) or by ribbon start column
// (_core.pyx:435-439's row start; rank r owns column_range(m, r, W)).  The
// reference is single-threaded; this is the partition step in front of one
// all-to-all.  Keys are interleaved (hi, lo) pairs; an optional byte per key
// (the choice bit) travels with its key.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

constexpr int RT_MAXW = 64;
struct RouteBounds {
  int64_t b[RT_MAXW + 1];  // owner r of value v: b[r] <= v < b[r + 1]
};

SHK_D int route_dest(ulonglong2 k, int kind, uint64_t nbm, u2 x, const RouteBounds& B, int W) {
  const u2 v = remix_d(split64(k.x), split64(k.y), x);
  int64_t val;
  if (kind == 0)
    val = (int64_t)__umulhi(v.hi, (uint32_t)nbm);  // bucket (nb < 2^32)
  else
    val = (int64_t)(((uint64_t)v.hi * (nbm - RIBBON_W + 1)) >> 32);  // ribbon start column
  int r = 0;
  while (r + 1 < W && val >= B.b[r + 1]) ++r;
  return r;
}

__global__ void route_count_kernel(const ulonglong2* keys, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                                   RouteBounds B, int W, unsigned long long* counts) {
  __shared__ unsigned int c[RT_MAXW];
  for (int i = threadIdx.x; i < W; i += blockDim.x) c[i] = 0;
  __syncthreads();
  const u2 x = split64(seed_mixer(seed, kind == 0 ? TAG_BUCKET : TAG_RSTART));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&c[route_dest(keys[i], kind, nbm, x, B, W)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < W; i += blockDim.x)
    if (c[i]) atomicAdd(&counts[i], (unsigned long long)c[i]);
}

// cursors[r] start at the destination offsets; warp-aggregated reservations
// (one atomic per destination present in the warp)
__global__ void route_scatter_kernel(const ulonglong2* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm,
                                     uint64_t seed, RouteBounds B, int W, unsigned long long* cursors,
                                     ulonglong2* out, uint8_t* aux_out) {
  const u2 x = split64(seed_mixer(seed, kind == 0 ? TAG_BUCKET : TAG_RSTART));
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool in = i < n;
    ulonglong2 k = make_ulonglong2(0, 0);
    int d = -1;
    if (in) {
      k = keys[i];
      d = route_dest(k, kind, nbm, x, B, W);
    }
    const unsigned peers = __match_any_sync(FULL_WARP, d);
    const int leader = __ffs(peers) - 1;
    unsigned long long pos = 0;
    if (in && lane == leader) pos = atomicAdd(&cursors[d], (unsigned long long)__popc(peers));
    pos = __shfl_sync(FULL_WARP, pos, leader);
    if (in) {
      const unsigned long long p = pos + __popc(peers & ((1u << lane) - 1u));
      out[p] = k;
      if (aux) aux_out[p] = aux[i];
    }
  }
}

// Fused route + all-to-all over peer memory: every key is stored straight
// into the receive buffer of the rank that owns it (CUDA IPC mappings of the
// peers' buffers: NVLink stores on a multi-GPU node), at that rank's slot
// for this source (peer_base[d]) plus a warp-aggregated local cursor.  The
// receive buffer holds cap keys (16 B) followed by cap aux bytes.
struct PeerPtrs {
  unsigned char* p[RT_MAXW];
  int64_t base[RT_MAXW];
};

__global__ void route_p2p_kernel(const ulonglong2* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm,
                                 uint64_t seed, RouteBounds B, int W, PeerPtrs P, int64_t cap,
                                 unsigned long long* cursors) {
  const u2 x = split64(seed_mixer(seed, kind == 0 ? TAG_BUCKET : TAG_RSTART));
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool in = i < n;
    ulonglong2 k = make_ulonglong2(0, 0);
    int d = -1;
    if (in) {
      k = keys[i];
      d = route_dest(k, kind, nbm, x, B, W);
    }
    const unsigned peers = __match_any_sync(FULL_WARP, d);
    const int leader = __ffs(peers) - 1;
    unsigned long long pos = 0;
    if (in && lane == leader) pos = atomicAdd(&cursors[d], (unsigned long long)__popc(peers));
    pos = __shfl_sync(FULL_WARP, pos, leader);
    if (in) {
      const int64_t slot = P.base[d] + (int64_t)(pos + __popc(peers & ((1u << lane) - 1u)));
      reinterpret_cast<ulonglong2*>(P.p[d])[slot] = k;  // NVLink store into the owner's buffer
      if (aux) P.p[d][cap * 16 + slot] = aux[i];
    }
  }
  __threadfence_system();
}

}  // namespace shk

using namespace shk;

int shk_launch_route(const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                     const int64_t* bounds, int W, unsigned long long* counts_dev, unsigned long long* cursors_dev,
                     uint64_t* out, uint8_t* aux_out, int64_t* counts_host, cudaStream_t st) {
  if (W < 1 || W > RT_MAXW) {
    shk_set_error("route: 1..%d ranks", RT_MAXW);
    return 3;
  }
  RouteBounds B;
  for (int r = 0; r <= W; ++r) B.b[r] = bounds[r];
  SHK_CUDA(cudaMemsetAsync(counts_dev, 0, (size_t)W * 8, st));
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  if (n > 0) {
    route_count_kernel<<<(unsigned)g, 256, 0, st>>>((const ulonglong2*)keys, n, kind, nbm, seed, B, W, counts_dev);
    SHK_LAUNCHED();
  }
  unsigned long long hc[RT_MAXW] = {0};
  SHK_CUDA(cudaMemcpyAsync(hc, counts_dev, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  unsigned long long off[RT_MAXW];
  unsigned long long acc = 0;
  for (int r = 0; r < W; ++r) {
    off[r] = acc;
    acc += hc[r];
    counts_host[r] = (int64_t)hc[r];
  }
  SHK_CUDA(cudaMemcpyAsync(cursors_dev, off, (size_t)W * 8, cudaMemcpyHostToDevice, st));
  if (n > 0) {
    route_scatter_kernel<<<(unsigned)g, 256, 0, st>>>((const ulonglong2*)keys, aux, n, kind, nbm, seed, B, W,
                                                      cursors_dev, (ulonglong2*)out, aux_out);
    SHK_LAUNCHED();
  }
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int shk_launch_route_count(const uint64_t* keys, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                           const int64_t* bounds, int W, unsigned long long* counts_dev, int64_t* counts_host,
                           cudaStream_t st) {
  if (W < 1 || W > RT_MAXW) {
    shk_set_error("route: 1..%d ranks", RT_MAXW);
    return 3;
  }
  RouteBounds B;
  for (int r = 0; r <= W; ++r) B.b[r] = bounds[r];
  SHK_CUDA(cudaMemsetAsync(counts_dev, 0, (size_t)W * 8, st));
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  if (n > 0) {
    route_count_kernel<<<(unsigned)g, 256, 0, st>>>((const ulonglong2*)keys, n, kind, nbm, seed, B, W, counts_dev);
    SHK_LAUNCHED();
  }
  unsigned long long hc[RT_MAXW] = {0};
  SHK_CUDA(cudaMemcpyAsync(hc, counts_dev, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < W; ++r) counts_host[r] = (int64_t)hc[r];
  return 0;
}

int shk_launch_route_p2p(const uint64_t* keys, const uint8_t* aux, int64_t n, int kind, uint64_t nbm, uint64_t seed,
                         const int64_t* bounds, int W, void* const* peer_bufs, const int64_t* peer_base, int64_t cap,
                         unsigned long long* cursors_dev, cudaStream_t st) {
  if (W < 1 || W > RT_MAXW) {
    shk_set_error("route: 1..%d ranks", RT_MAXW);
    return 3;
  }
  RouteBounds B;
  PeerPtrs P;
  for (int r = 0; r <= W; ++r) B.b[r] = bounds[r];
  for (int r = 0; r < W; ++r) {
    P.p[r] = (unsigned char*)peer_bufs[r];
    P.base[r] = peer_base[r];
  }
  SHK_CUDA(cudaMemsetAsync(cursors_dev, 0, (size_t)W * 8, st));
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  if (n > 0) {
    route_p2p_kernel<<<(unsigned)g, 256, 0, st>>>((const ulonglong2*)keys, aux, n, kind, nbm, seed, B, W, P, cap,
                                                  cursors_dev);
    SHK_LAUNCHED();
  }
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}
