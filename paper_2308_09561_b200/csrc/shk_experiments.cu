// The analysis entry points of the kernel seam:
//   search_bruteforce     _core.pyx:337-371   (single-hash bijection retry)
//   mc_filter_pass_count  _core.pyx:832-860   (all-cells-hit filter rate)
//   enumerate_outcomes    _core.pyx:778-829   (exact pseudoforest census)
// They are what experiments.py (:31-49, :124-148, :180-226) calls.  All three
// are order-independent reductions over seeds / edge tuples, so they map onto
// one thread per seed / per tuple prefix with warp + atomic reductions.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

// ---------------------------------------------------------------------------
// Brute force: for every seed in [base, base + count), the evals the
// reference's scalar loop spends on it (index of the first colliding key + 1,
// or n when the single hash is a bijection) and the minimum bijective seed.
__global__ void brute_kernel(const uint64_t* __restrict__ khi, const uint64_t* __restrict__ klo, int n,
                             uint64_t base, uint64_t count, unsigned long long* found,
                             unsigned long long* evals) {
  __shared__ u2 sh[64], sl[64];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sh[i] = split64(khi[i]);
    sl[i] = split64(klo[i]);
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = base + t;
    const u2 x = seed_mixer_d(s, TAG_LEAF);
    uint32_t m0 = 0, m1 = 0;
    int e = n;
    bool bij = true;
    for (int i = 0; i < n; ++i) {
      const u2 v = remix_d(sh[i], sl[i], x);
      const uint32_t h = __umulhi(v.hi, (uint32_t)n);
      const uint32_t b0 = shl_clamp(1u, h), b1 = shl_clamp(1u, h - 32u);
      if ((m0 & b0) | (m1 & b1)) {
        e = i + 1;
        bij = false;
        break;
      }
      m0 |= b0;
      m1 |= b1;
    }
    acc += (unsigned long long)e;
    if (bij) atomicMin(found, (unsigned long long)s);  // n distinct cells of n: full
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(evals, acc);
}

// Filter pass count: seeds whose leaf_pair cells cover all n cells.
__global__ void mc_filter_kernel(const uint64_t* __restrict__ khi, const uint64_t* __restrict__ klo, int n,
                                 uint64_t count, unsigned long long* passes) {
  __shared__ u2 sh[64], sl[64];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sh[i] = split64(khi[i]);
    sl[i] = split64(klo[i]);
  }
  __syncthreads();
  const uint32_t full0 = n >= 32 ? 0xFFFFFFFFu : (1u << n) - 1u;
  const uint32_t full1 = n >= 64 ? 0xFFFFFFFFu : n > 32 ? (1u << (n - 32)) - 1u : 0u;
  unsigned long long acc = 0;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count; s += (uint64_t)gridDim.x * blockDim.x) {
    const u2 x = seed_mixer_d(s, TAG_LEAF);
    uint32_t m0 = 0, m1 = 0;
    for (int i = 0; i < n; ++i) {
      uint32_t h0, h1;
      leaf_pair_d(remix_d(sh[i], sl[i], x), (uint32_t)n, (uint32_t)(n - 1), h0, h1);
      m0 |= shl_clamp(1u, h0) | shl_clamp(1u, h1);
      m1 |= shl_clamp(1u, h0 - 32u) | shl_clamp(1u, h1 - 32u);
    }
    acc += (m0 == full0 && m1 == full1) ? 1ull : 0ull;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(passes, acc);
}

// ---------------------------------------------------------------------------
// Exact enumeration over all (n^2)^n tuples of ordered cell pairs, n <= 8.
// State of a partial multigraph: CM byte i = node mask of i's component, EC
// nibble r = edge count of the component whose lowest node is r.  A component
// is valid (<= one cycle) iff edges <= nodes, and a tuple is a pseudoforest iff
// every component is valid, the same predicate as the reference's union-find
// (cycle into a cyclic component, or merging two cyclic ones, fails).
// Threads own prefixes of n-2 edges, loop over the ordered component pairs
// edge n-1 can join (weighted by their vertex-pair counts) and count edge n
// in closed form from the component sizes.

SHK_D uint64_t byte_spread(uint32_t mask8) {
  // byte i = 0xFF iff bit i of mask8
  const uint64_t t = ((uint64_t)mask8 * 0x0101010101010101ull) & 0x8040201008040201ull;
  const uint32_t lo = __vcmpne4((uint32_t)t, 0u), hi = __vcmpne4((uint32_t)(t >> 32), 0u);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

SHK_D bool add_edge(uint64_t& CM, uint32_t& EC, int& comps, uint32_t u, uint32_t v) {
  const uint32_t cu = (uint32_t)(CM >> (8 * u)) & 0xFFu, cv = (uint32_t)(CM >> (8 * v)) & 0xFFu;
  const uint32_t ru = __ffs(cu) - 1, rv = __ffs(cv) - 1;
  if (cu == cv) {
    const uint32_t e = ((EC >> (4 * ru)) & 15u) + 1u;
    if (e > (uint32_t)__popc(cu)) return false;
    EC += 1u << (4 * ru);
    return true;
  }
  const uint32_t merged = cu | cv;
  const uint32_t e = ((EC >> (4 * ru)) & 15u) + ((EC >> (4 * rv)) & 15u) + 1u;
  if (e > (uint32_t)__popc(merged)) return false;
  const uint32_t r = ru < rv ? ru : rv;
  EC = (EC & ~(15u << (4 * r))) | (e << (4 * r));
  const uint64_t M = byte_spread(merged);
  CM = (CM & ~M) | (((uint64_t)merged * 0x0101010101010101ull) & M);
  --comps;
  return true;
}

// Completions of a valid state by one more edge: (pseudoforest count, sum 2^c).
template <int N>
SHK_D void close_last(uint64_t CM, uint32_t EC, int comps, unsigned long long& pf, unsigned long long& s2) {
  uint32_t sumsq = 0, okin = 0, sf = 0, sumsqf = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t c = (uint32_t)(CM >> (8 * i)) & 0xFFu;
    if ((c & ((2u << i) - 1u)) == (1u << i)) {  // i is the lowest node: the representative
      const uint32_t s = __popc(c), e = (EC >> (4 * i)) & 15u;
      sumsq += s * s;
      if (e < s) {
        okin += s * s;
      } else {
        sf += s;
        sumsqf += s * s;
      }
    }
  }
  const uint32_t okx = (N * N - sumsq) - (sf * sf - sumsqf);
  pf += okin + okx;
  s2 += ((unsigned long long)okin << comps) + (comps > 0 ? ((unsigned long long)okx << (comps - 1)) : 0ull);
}

template <int N>
__global__ void enum_kernel(uint64_t nprefix, unsigned long long* out) {
  constexpr int P = N >= 2 ? N - 2 : 0;   // prefix edges per thread
  constexpr int LOOP = N >= 2 ? 1 : 0;    // edges enumerated in the loop
  constexpr uint32_t T = N * N;
  unsigned long long pf = 0, s2 = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nprefix; t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t CM = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) CM |= (uint64_t)(1u << i) << (8 * i);
    uint32_t EC = 0;
    int comps = N;
    bool ok = true;
    uint64_t r = t;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint32_t e = (uint32_t)(r % T);
      r /= T;
      if (ok) ok = add_edge(CM, EC, comps, e / N, e % N);
    }
    if (!ok) continue;
    if (LOOP) {
      // edge n-1 only matters through the components of its endpoints: loop
      // over ordered component pairs (C, D), weight |C| |D| vertex pairs
      uint32_t reps = 0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const uint32_t c = (uint32_t)(CM >> (8 * i)) & 0xFFu;
        if ((c & ((2u << i) - 1u)) == (1u << i)) reps |= 1u << i;
      }
      for (uint32_t ru = reps; ru; ru &= ru - 1) {
        const uint32_t u = __ffs(ru) - 1, su = __popc((uint32_t)(CM >> (8 * u)) & 0xFFu);
        for (uint32_t rv = reps; rv; rv &= rv - 1) {
          const uint32_t v = __ffs(rv) - 1, sv = __popc((uint32_t)(CM >> (8 * v)) & 0xFFu);
          uint64_t CM2 = CM;
          uint32_t EC2 = EC;
          int c2 = comps;
          if (add_edge(CM2, EC2, c2, u, v)) {
            unsigned long long p1 = 0, q1 = 0;
            close_last<N>(CM2, EC2, c2, p1, q1);
            pf += p1 * (su * sv);
            s2 += q1 * (su * sv);
          }
        }
      }
    } else {
      close_last<N>(CM, EC, comps, pf, s2);
    }
  }
  pf = warp_sum(pf);
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) {
    if (pf) atomicAdd(out, pf);
    if (s2) atomicAdd(out + 1, s2);
  }
}

}  // namespace shk

using namespace shk;

static int exp_grid(uint64_t work, int num_sms) {
  uint64_t g = (work + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int shk_launch_brute(const uint64_t* khi, const uint64_t* klo, int n, uint64_t base, uint64_t count,
                     unsigned long long* found, unsigned long long* evals, int num_sms, cudaStream_t st) {
  brute_kernel<<<exp_grid(count, num_sms), 256, 0, st>>>(khi, klo, n, base, count, found, evals);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_mc_filter(const uint64_t* khi, const uint64_t* klo, int n, uint64_t count,
                         unsigned long long* passes, int num_sms, cudaStream_t st) {
  mc_filter_kernel<<<exp_grid(count, num_sms), 256, 0, st>>>(khi, klo, n, count, passes);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_enumerate(int n, unsigned long long* out, int num_sms, cudaStream_t st) {
  uint64_t nprefix = 1;
  for (int k = 0; k < n - 2; ++k) nprefix *= (uint64_t)n * n;
  const int g = exp_grid(nprefix, num_sms);
  switch (n) {
#define SHK_ENUM_CASE(K)                                        \
  case K:                                                       \
    enum_kernel<K><<<g, 256, 0, st>>>(nprefix, out);            \
    break;
    SHK_ENUM_CASE(1)
    SHK_ENUM_CASE(2)
    SHK_ENUM_CASE(3)
    SHK_ENUM_CASE(4)
    SHK_ENUM_CASE(5)
    SHK_ENUM_CASE(6)
    SHK_ENUM_CASE(7)
    SHK_ENUM_CASE(8)
#undef SHK_ENUM_CASE
    default:
      shk_set_error("enumeration limited to 1 <= n <= 8");
      return 3;
  }
  SHK_LAUNCHED();
  return 0;
}
