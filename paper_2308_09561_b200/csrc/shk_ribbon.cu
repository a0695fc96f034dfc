// 1-bit retrieval: banded GF(2) system with a 128-bit band ("ribbon").
//
// Restates _core.pyx:435-568 (ribbon_rows, ribbon_solve, window128,
// parity128, ribbon_query_many) and retrieval.py:93-106.
//
// The reference eliminates rows on the fly in key order into one slot per
// pivot column, then back-substitutes right to left with free columns = 0.
// That solution is unique given the row space, and so is
// consistency, so ANY elimination order gives the reference's words.  GPU
// scheme:
//   1. rows (start, 128-bit pattern, rhs) are generated and counting-sorted
//      by elimination chunk (CE columns);
//   2. one warp per chunk eliminates its rows into its slots in shared memory
//      (32 rows in flight, lock-step claim protocol: XOR with the occupied
//      slot, shift to the next set bit); rows whose pivot walks past the chunk end are
//      emitted as overflow and inserted by the next pass into the chunk they
//      reached; passes repeat until no row overflows;
//   3. back substitution over back-chunks of CB columns runs in parallel
//      with the solution of the 127 columns right of each chunk as symbolic
//      unknowns: a CTA carries 128 bit-sliced affine forms (one per lane), so
//      each chunk yields the affine map from its right neighbour's first 127
//      bits to its own first 127 bits;
//   4. a single warp walks the chunks right to left evaluating those maps
//      (the only sequential step: 127x128 GF(2) mat-vec per chunk);
//   5. every column's solution bit is then parity(its affine form & its
//      chunk's boundary), a fully parallel map (step 3 stored the forms).
#include <cuda_pipeline.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

// Elimination chunk (columns).  Measured at C4: 512 -> ribbon 4.9 ms, 1024 ->
// 5.2, 256 -> 5.6, 2048 -> 7.1 (smaller chunks: more resident warps per SM,
// more rows overflowing into later passes).
#ifndef SHK_RIBBON_CE
#define SHK_RIBBON_CE 512
#endif
constexpr int CE = SHK_RIBBON_CE;
#ifndef SHK_RIBBON_CB
#define SHK_RIBBON_CB 8192
#endif
constexpr int CB = SHK_RIBBON_CB;
#define RIB_SPAN_DEFAULT "1,2"
// Rows per chunk bin of the emitted rows (a 512-column chunk gets ~488 rows
// on average at eps = 0.05, sd ~22; a full bin spills to the overflow list).
constexpr int64_t RIB_BIN_CAP = 576;  // back-substitution chunk (columns), multiple of CE and 64

struct RRow {
  uint64_t p0, p1;
  int64_t s;  // start column; bit 62 = rhs
};
constexpr int64_t RHS_BIT = 1ll << 62;
constexpr int64_t S_MASK = RHS_BIT - 1;

// ---------------------------------------------------------------------------
// Row generation (ribbon_rows) + chunk histogram.
__global__ void ribbon_rows_kernel(const uint64_t* hi, const uint64_t* lo, int stride, int64_t N, int64_t m,
                                   uint64_t seed, int64_t* starts, uint64_t* p0, uint64_t* p1) {
  const u2 xs = split64(seed_mixer(seed, TAG_RSTART));
  const u2 x0 = split64(seed_mixer(seed, TAG_RPAT0));
  const u2 x1 = split64(seed_mixer(seed, TAG_RPAT1));
  const uint64_t span = (uint64_t)(m - RIBBON_W + 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    u2 kh = split64(hi[i * stride]), kl = split64(lo[i * stride]);
    u2 v = remix_d(kh, kl, xs);
    starts[i] = (int64_t)(((uint64_t)v.hi * span) >> 32);
    u2 a = remix_d(kh, kl, x0);
    u2 b = remix_d(kh, kl, x1);
    p0[i] = join64(a.lo | 1u, a.hi);
    p1[i] = join64(b.lo, b.hi);
  }
}

// Rows from keys directly into chunk buckets (fused generation + histogram).
// Only rows starting in columns [c0, c1) are kept, re-based to c0 (a
// column-sharded solve; the single-GPU solve passes the whole range).
__global__ void ribbon_keyrows_hist_kernel(const ulonglong2* keys, int64_t N, int64_t m, uint64_t seed,
                                           int64_t* hist, int64_t c0, int64_t c1) {
  const u2 xs = split64(seed_mixer(seed, TAG_RSTART));
  const uint64_t span = (uint64_t)(m - RIBBON_W + 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 k = keys[i];
    u2 v = remix_d(split64(k.x), split64(k.y), xs);
    int64_t s = (int64_t)(((uint64_t)v.hi * span) >> 32);
    if (s >= c0 && s < c1) atomicAdd((unsigned long long*)&hist[(s - c0) / CE], 1ull);
  }
}

__global__ void ribbon_keyrows_scatter_kernel(const ulonglong2* keys, const uint8_t* rhs, int64_t N, int64_t m,
                                              uint64_t seed, int64_t* cursor, RRow* rows, int64_t c0, int64_t c1) {
  const u2 xs = split64(seed_mixer(seed, TAG_RSTART));
  const u2 x0 = split64(seed_mixer(seed, TAG_RPAT0));
  const u2 x1 = split64(seed_mixer(seed, TAG_RPAT1));
  const uint64_t span = (uint64_t)(m - RIBBON_W + 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 k = keys[i];
    u2 kh = split64(k.x), kl = split64(k.y);
    u2 v = remix_d(kh, kl, xs);
    int64_t s = (int64_t)(((uint64_t)v.hi * span) >> 32);
    if (s < c0 || s >= c1) continue;
    s -= c0;
    u2 a = remix_d(kh, kl, x0);
    u2 b = remix_d(kh, kl, x1);
    int64_t pos = (int64_t)atomicAdd((unsigned long long*)&cursor[s / CE], 1ull);
    RRow r;
    r.p0 = join64(a.lo | 1u, a.hi);
    r.p1 = join64(b.lo, b.hi);
    r.s = s | ((rhs[i] & 1) ? RHS_BIT : 0);
    rows[pos] = r;
  }
}

// Rows from keys straight into per-chunk bins of `cap` rows (no histogram
// pass): a row's slot is one atomicAdd on its chunk's count; rows past a full
// bin go to the overflow list, which the second elimination pass takes with
// the first pass's own overflow (single-GPU solve over all columns).
__global__ void ribbon_keyrows_bins_kernel(const ulonglong2* keys, const uint8_t* rhs, int64_t N, int64_t m,
                                           uint64_t seed, unsigned long long* bcnt, int64_t cap, RRow* bins,
                                           RRow* ovf, unsigned long long* ovf_cnt) {
  const u2 xs = split64(seed_mixer(seed, TAG_RSTART));
  const u2 x0 = split64(seed_mixer(seed, TAG_RPAT0));
  const u2 x1 = split64(seed_mixer(seed, TAG_RPAT1));
  const uint64_t span = (uint64_t)(m - RIBBON_W + 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 k = keys[i];
    u2 kh = split64(k.x), kl = split64(k.y);
    u2 v = remix_d(kh, kl, xs);
    const int64_t s = (int64_t)(((uint64_t)v.hi * span) >> 32);
    const int64_t ch = s / CE;
    const unsigned long long pos = atomicAdd(bcnt + ch, 1ull);
    u2 a = remix_d(kh, kl, x0);
    u2 b = remix_d(kh, kl, x1);
    RRow r;
    r.p0 = join64(a.lo | 1u, a.hi);
    r.p1 = join64(b.lo, b.hi);
    r.s = s | ((rhs[i] & 1) ? RHS_BIT : 0);
    RRow* dst = pos < (unsigned long long)cap ? bins + ch * cap + (int64_t)pos : ovf + atomicAdd(ovf_cnt, 1ull);
    *dst = r;
  }
}

// Explicit rows (ribbon_solve seam).
__global__ void ribbon_rows_hist_kernel(const int64_t* starts, int64_t N, int64_t* hist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&hist[starts[i] / CE], 1ull);
}

__global__ void ribbon_rows_scatter_kernel(const int64_t* starts, const uint64_t* p0, const uint64_t* p1,
                                           const uint8_t* rhs, int64_t N, int64_t* cursor, RRow* rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = starts[i];
    int64_t pos = (int64_t)atomicAdd((unsigned long long*)&cursor[s / CE], 1ull);
    RRow r;
    r.p0 = p0[i];
    r.p1 = p1[i];
    r.s = s | ((rhs[i] & 1) ? RHS_BIT : 0);
    rows[pos] = r;
  }
}

// ---------------------------------------------------------------------------
// Elimination pass: one warp per chunk with pending rows; all 32 lanes insert
// rows concurrently.  Slot state (pivot row per column, occupancy and rhs
// bitmaps) lives in shared memory for the pass and in global memory between
// passes.  Lock-step protocol per iteration: (A) every lane reads the slot at
// its row's current pivot column; __syncwarp; (B) a lane that saw the slot
// occupied XORs the stored row into its own and moves to the next set bit; a
// lane that saw it empty claims it with atomicOr on the occupancy word and,
// if it won, stores its row there (same phase), else it retries next
// iteration (then it sees the winner's row).  A set occupancy bit therefore
// always refers to data written before the previous __syncwarp.  Any
// insertion order yields the same final solution.
// S: elimination chunks merged per warp (1 for the first pass; later passes
// take S consecutive chunks so a row can walk S chunks in one pass).
// Bin mode (bcnt != nullptr, S = 1): chunk c's rows are rows[c cap, c cap +
// min(bcnt[c], cap)) (rows emitted by the construction kernel) instead of the
// CSR range row_off[c], row_off[c + 1].
template <int S, bool RING>
__global__ void __launch_bounds__(32) ribbon_elim_kernel(const RRow* rows, const int64_t* row_off,
                                                         const unsigned long long* bcnt, int64_t cap, int64_t nchunks,
                                                         int64_t m, uint64_t* sp0, uint64_t* sp1, uint32_t* occ,
                                                         uint32_t* sbit, RRow* ovf, int64_t* ovf_count,
                                                         int* inconsistent, int first_pass) {
  constexpr int CEs = CE * S;
  __shared__ uint64_t q0s[CEs], q1s[CEs];
  __shared__ uint32_t occs[CEs / 32], sbs[CEs / 32];
  const int64_t c = blockIdx.x;
  if (c * S >= nchunks) return;
  int64_t r0, r1;
  if (bcnt) {
    r0 = c * cap;
    const unsigned long long k = bcnt[c];
    r1 = r0 + (k < (unsigned long long)cap ? (int64_t)k : cap);
  } else {
    r0 = row_off[c * S];
    r1 = row_off[(c + 1) * S < nchunks ? (c + 1) * S : nchunks];
  }
  if (r0 == r1) return;
  const int lane = threadIdx.x;
  const int64_t base = c * CEs;
  const int64_t cols = (m - base < CEs) ? (m - base) : CEs;
  const int64_t nrows = r1 - r0;
  const int64_t wbase = base / 32;
  if (first_pass) {  // slots start empty: no global state to load
    for (int j = lane; j < CEs / 32; j += 32) occs[j] = sbs[j] = 0;
  } else {
    for (int j = lane; j < CEs; j += 32) {
      const bool in = j < cols;
      q0s[j] = in ? sp0[base + j] : 0;
      q1s[j] = in ? sp1[base + j] : 0;
    }
    for (int j = lane; j < CEs / 32; j += 32) {
      const bool in = (j * 32) < cols;
      occs[j] = in ? occ[wbase + j] : 0;
      sbs[j] = in ? sbit[wbase + j] : 0;
    }
  }
  __syncwarp();
  bool active = false, bad = false;
  uint64_t a0 = 0, a1 = 0;
  uint32_t b = 0;
  int j = 0;
  // RING (the first pass: ~490 rows per chunk): rows are handed out in order
  // from a 64-row shared ring -- the lanes whose row finished take the next
  // ones at the top of an iteration (ballot rank) -- refilled 32 rows at a
  // time from a register stage whose global loads were issued one refill
  // earlier, so no lane waits on a global load for its next row (with one
  // row prefetched per lane, a lane whose rows claim a slot at once -- the
  // first rows of a chunk -- stalled the warp for a global round trip almost
  // every iteration: C4 pass 0 0.95 -> 0.66 ms, C2 0.23 -> 0.13 ms).  The
  // later passes hold a few rows per warp that walk long; there lane i takes
  // rows i, i + 32, ... with one row prefetched (the ring's per-iteration
  // bookkeeping sits on their walk's critical path).
  __shared__ RRow ring[RING ? 64 : 1];
  const unsigned lt = (1u << lane) - 1u;
  int64_t head = 0, filled = 0;  // RING, warp-uniform: rows handed out / stored in the ring
  RRow stage{0, 0, 0};
  int64_t next = lane;  // !RING: this lane's next row
  if (lane < nrows) stage = rows[r0 + lane];
  if (!RING) next += 32;
  auto refill = [&]() {
    const int64_t k = nrows - filled < 32 ? nrows - filled : 32;
    if (lane < k) ring[(filled + lane) & 63] = stage;
    filled += k;
    if (filled + lane < nrows) stage = rows[r0 + filled + lane];
    __syncwarp();
  };
  auto start = [&](const RRow& r) {
    active = true;
    a0 = r.p0;
    a1 = r.p1;
    b = (r.s & RHS_BIT) ? 1u : 0u;
    j = (int)((r.s & S_MASK) - base);
  };
  auto take = [&]() {
    if constexpr (RING) {
      if (filled - head < 32 && filled < nrows) refill();
      const unsigned need = __ballot_sync(FULL_WARP, !active);
      if (!active) {
        const int64_t idx = head + __popc(need & lt);
        if (idx < filled) start(ring[idx & 63]);
      }
      head += __popc(need);
      if (head > filled) head = filled;
    } else {
      if (!active && next - 32 < nrows) {
        start(stage);
        if (next < nrows) stage = rows[r0 + next];
        next += 32;
      }
    }
  };
  take();
  while (__any_sync(FULL_WARP, active)) {
    // phase A: read the slot at the current pivot
    const bool esc = active && j >= CEs;
    uint32_t w = 0, sw = 0;
    uint64_t q0 = 0, q1 = 0;
    if (active && !esc) {
      w = occs[j >> 5];
      sw = sbs[j >> 5];
      q0 = q0s[j];
      q1 = q1s[j];
    }
    __syncwarp();
    // phase B: act
    if (active) {
      if (esc) {
        const int64_t kk = (int64_t)atomicAdd((unsigned long long*)ovf_count, 1ull);
        RRow o;
        o.p0 = a0;
        o.p1 = a1;
        o.s = (base + j) | (b ? RHS_BIT : 0);
        ovf[kk] = o;
        active = false;
      } else {
        const uint32_t bitm = 1u << (j & 31);
        if (w & bitm) {
          a0 ^= q0;
          a1 ^= q1;
          b ^= (sw >> (j & 31)) & 1u;
          if ((a0 | a1) == 0) {
            if (b) bad = true;
            active = false;
          } else {
            int t;
            if (a0) {
              t = __ffsll((long long)a0) - 1;
              a0 = (a0 >> t) | (t ? (a1 << (64 - t)) : 0);
              a1 >>= t;
            } else {
              t = 63 + __ffsll((long long)a1);  // 64 + ctz(a1)
              a0 = a1 >> (t - 64);
              a1 = 0;
            }
            j += t;
          }
        } else {
          const uint32_t old = atomicOr(&occs[j >> 5], bitm);
          if (!(old & bitm)) {
            q0s[j] = a0;
            q1s[j] = a1;
            if (b) atomicOr(&sbs[j >> 5], bitm);
            active = false;
          }
        }
      }
    }
    __syncwarp();
    take();
  }
  if (__any_sync(FULL_WARP, bad) && lane == 0) atomicOr(inconsistent, 1);
  __syncwarp();
  for (int jj = lane; jj < cols; jj += 32) {
    sp0[base + jj] = q0s[jj];
    sp1[base + jj] = q1s[jj];
  }
  for (int jj = lane; jj < CEs / 32; jj += 32) {
    if ((jj * 32) < cols) {
      occ[wbase + jj] = occs[jj];
      sbit[wbase + jj] = sbs[jj];
    }
  }
}

// ---------------------------------------------------------------------------
// Symbolic back substitution (affine forms), one CTA of 4 warps per
// back-chunk.  Warp q, lane L owns unknown u = 4L + q (u = 127 is the
// constant term) and tracks W_u: a 128-bit window whose bit k is the
// coefficient of u in sol[c + 1 + k].  forms_out[chunk][u] = W_u after the
// chunk's first column.  Every column's own affine form is also written
// (coef[col], word q bit L = coefficient of unknown 4L + q, i.e. warp q's
// new bits of that column across its lanes), so the final pass is a
// parallel map instead of a second sequential walk.  A lane collects its own
// bits of a 32-column group in N anyway, so the words come from one 32 x 32
// bit transpose per group (no per-column ballot or store).
//
// The window is not shifted per column.  Columns go in aligned groups of 32
// (right to left); within a group the window at the column k steps below
// the group's top is (Wg << k) | N, Wg = the window at the group's top and
// N = the k bits produced since.  So parity(W & p) = parity(Wg & (p >> k))
// ^ parity(N & low_k(p)): the CTA stages each column's pattern pre-shifted
// by its k (k = 31 - col % 32, fixed per staging thread) plus its low k bits,
// and a warp's per-column step is LDS.128 + LDS, 5 AND/XOR, POPC, ballot and
// N = 2N + bit; the 4-word window moves once per group (a word rename).
// Window bit 127 (sol[c + 128], never used by a 127-bit pattern) is pinned to
// 1 for the constant term and 0 for the unknowns, and the staged pattern
// carries the column's rhs in that bit, so the constant lane's parity picks up
// the rhs with no branch (the pre-shifted pattern is zero in bits 127-k..126,
// which pair with the bits of Wg that have left the window).
__global__ void __launch_bounds__(128) ribbon_forms_kernel(int64_t m, int64_t nbchunks, int cb, const uint64_t* sp0,
                                                           const uint64_t* sp1, const uint32_t* occ,
                                                           const uint32_t* sbit, uint4* forms, uint4* coef) {
  // double-buffered 256-column tiles: while the warps walk tile k, each
  // thread's global loads for tile k+1 are in flight, and the finished
  // coefficients of tile k-1 are written out; one barrier per tile
  __shared__ uint4 tpw[2][256];
  __shared__ uint32_t tlo[2][256];
  __shared__ uint32_t tcoef[2][256][4];
  const int64_t c = blockIdx.x;
  if (c >= nbchunks) return;
  const int tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
  const int u = 4 * lane + q;
  const int64_t s0 = c * cb;
  const int64_t e = (s0 + cb < m) ? s0 + cb : m;
  const uint32_t kmask = (u == 127) ? 0x80000000u : 0u;
  // initial window e_u (bit 127 = kmask) split at the top column's group
  // offset k0 (tiles and groups are 32-aligned; k0 > 0 only at the system end)
  const int k0 = 31 - (int)((e - 1) & 31);
  uint32_t W0 = 0, W1 = 0, W2 = 0, W3 = kmask, N = 0;
  if (u < 127) {
    if (u < k0) {
      N = 1u << u;
    } else {
      const int v = u - k0;
      const uint32_t b = 1u << (v & 31);
      W0 = (v >> 5) == 0 ? b : 0u;
      W1 = (v >> 5) == 1 ? b : 0u;
      W2 = (v >> 5) == 2 ? b : 0u;
      W3 |= (v >> 5) == 3 ? b : 0u;
    }
  }
  // tiles from the top: tile 0 is [tstart(e-1), e), tile k+1 ends where tile k starts
  auto tile_start = [&](int64_t col) { return (col / 256) * 256 > s0 ? (col / 256) * 256 : s0; };
  // per-thread prefetch registers: columns tid and tid + 128 of a tile
  uint64_t pa0[2], pa1[2];
  uint32_t prhs[2];
  auto prefetch = [&](int64_t ts, int nt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + 128 * h;
      pa0[h] = pa1[h] = 0ull;
      prhs[h] = 0;
      if (j < nt) {
        const int64_t cc = ts + j;
        if ((occ[cc >> 5] >> (cc & 31)) & 1u) {
          pa0[h] = sp0[cc];
          pa1[h] = sp1[cc];
          prhs[h] = (sbit[cc >> 5] >> (cc & 31)) & 1u;  // rhs (free columns: 0)
        }
      }
    }
  };
  const int ks = 31 - lane;  // group offset of this thread's staged columns (tid and tid + 128)
  auto stash = [&](int buf, int nt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + 128 * h;
      if (j < nt) {
        const uint64_t a0 = pa0[h], a1 = pa1[h];
        // p >> 1 as four 32-bit words (127 bits)
        const uint32_t x = (uint32_t)(a0 >> 1) | ((uint32_t)(a0 >> 32) << 31);
        const uint32_t y = (uint32_t)(a0 >> 33) | ((uint32_t)a1 << 31);
        const uint32_t z = (uint32_t)(a1 >> 1) | ((uint32_t)(a1 >> 32) << 31);
        const uint32_t w = (uint32_t)(a1 >> 33);
        tpw[buf][j] = make_uint4(__funnelshift_r(x, y, ks), __funnelshift_r(y, z, ks), __funnelshift_r(z, w, ks),
                                 (w >> ks) | (prhs[h] << 31));
        tlo[buf][j] = x & ((1u << ks) - 1u);
      }
    }
  };
  auto step = [&](int buf, int j) {
    const uint4 p = tpw[buf][j];
    const uint32_t nb = __popc((W0 & p.x) ^ (W1 & p.y) ^ (W2 & p.z) ^ (W3 & p.w) ^ (N & tlo[buf][j])) & 1u;
    N = 2u * N + nb;
  };
  // End of a group whose lowest column is tile index gb and which made cnt
  // columns: bit t of N (t < cnt) is this lane's unknown's coefficient in
  // column gb + t.  A 32 x 32 bit transpose across the warp (5 shuffle
  // stages) gives lane t the column's word (bit L = unknown 4L + q), stored
  // once per group instead of a ballot and a store per column.
  auto flush = [&](int buf, int gb, int cnt) {
    uint32_t x = N;
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      const uint32_t M = sft == 16 ? 0x0000FFFFu : sft == 8 ? 0x00FF00FFu : sft == 4 ? 0x0F0F0F0Fu
                         : sft == 2 ? 0x33333333u : 0x55555555u;
      const uint32_t y = __shfl_xor_sync(FULL_WARP, x, sft);
      x = (lane & sft) ? ((x & ~M) | ((y >> sft) & M)) : ((x & M) | ((y << sft) & ~M));
    }
    if (lane < cnt) tcoef[buf][gb + lane][q] = x;
  };
  auto next_group = [&]() {
    W3 = (W2 & 0x7FFFFFFFu) | kmask;
    W2 = W1;
    W1 = W0;
    W0 = N;
    N = 0;
  };
  int64_t col = e - 1;
  int64_t ts = tile_start(col);
  int nt = (int)(col - ts + 1);
  prefetch(ts, nt);
  stash(0, nt);
  __syncthreads();
  int64_t prev_ts = -1;
  int prev_nt = 0, buf = 0;
  for (int k = 0;; ++k) {
    buf = k & 1;
    const int64_t nts = ts - 1 >= s0 ? tile_start(ts - 1) : -1;
    const int nnt = nts >= 0 ? (int)(ts - nts) : 0;
    if (nnt) prefetch(nts, nnt);
    int j = nt - 1;
    if ((j & 31) != 31) {  // partial top group (the system's last columns only)
      const int gb = j & ~31, cnt = j - gb + 1;
      for (; j >= gb; --j) step(buf, j);
      flush(buf, gb, cnt);
      next_group();
    }
    for (; j >= 0; j -= 32) {
#pragma unroll
      for (int t = 0; t < 32; ++t) step(buf, j - t);
      flush(buf, j - 31, 32);
      next_group();
    }
    if (nnt) stash(buf ^ 1, nnt);
    // coefficients of the previous tile (complete since the last barrier)
    if (prev_nt)
      for (int j = tid; j < prev_nt; j += 128)
        coef[prev_ts + j] =
            make_uint4(tcoef[buf ^ 1][j][0], tcoef[buf ^ 1][j][1], tcoef[buf ^ 1][j][2], tcoef[buf ^ 1][j][3]);
    __syncthreads();
    prev_ts = ts;
    prev_nt = nt;
    if (!nnt) break;
    ts = nts;
    nt = nnt;
  }
  // the last tile's coefficients (complete after the final barrier)
  for (int j = tid; j < prev_nt; j += 128)
    coef[prev_ts + j] = make_uint4(tcoef[buf][j][0], tcoef[buf][j][1], tcoef[buf][j][2], tcoef[buf][j][3]);
  forms[c * 128 + u] = make_uint4(W0, W1, W2, W3);
}

// Right-to-left chain over back-chunks: y = first 127 solution bits of chunk
// c + 1 (right boundary of chunk c); chunk c's forms map it to chunk c's
// first bits (an affine GF(2) map: sum of the forms of the set bits of y plus
// the constant's form).  One warp per chain; the next chunk's forms are
// loaded while the current one is evaluated.  The chunks are cut in groups
// of G consecutive chunks (group g = chunks [gG, gG + G)) so the serial
// chain is two-level (rib_chain_final): the groups' maps in parallel, then a
// short chain over the group maps, then every group's own chain in parallel.
//   RUN mode (lin < 0): block g runs group g from y = ybound[g] (or *y_io when
//     ybound is null); ysel[c] (may be null) gets chunk c's right boundary in
//     the coef layout (word q bit L = y bit 4L + q; bit 127 = 1 for the
//     constant), yplain[c] (may be null) the same boundary as plain bits;
//     with ybound null, *y_io gets the final y (chunk c_lo's first bits).
//   MAP mode (lin >= 0): block (j, g) runs group g from y = e_j (j < 127) or
//     y = 0 (j = 127) and writes y_io[128 g + j].  lin = 0: images of the basis
//     (the affine map as the column-sharded solve composes it); lin = 1: the
//     constant is left out of the chains of j < 127, giving the linear part
//     L e_j and, at j = 127, the constant -- the same layout as a chunk's
//     forms, so the group maps chain with this kernel too.
__global__ void __launch_bounds__(32) ribbon_chain_kernel(int64_t nbchunks, int64_t G, const uint4* forms,
                                                          uint4* ysel, uint4* yplain, uint4* y_io,
                                                          const uint4* ybound, int lin) {
  // D-deep cp.async ring: the forms of chunk c - D are in flight while chunk
  // c is evaluated (each lane copies and later reads only its own 64 bytes).
  constexpr int D = 8;
  __shared__ uint4 ring[D][128];
  const int lane = threadIdx.x;
  const bool map = lin >= 0;
  const int j = map ? (int)blockIdx.x : 0;
  const int64_t g = map ? (int64_t)blockIdx.y : (int64_t)blockIdx.x;
  const int64_t c_lo = g * G;
  const int64_t c_hi = (c_lo + G < nbchunks) ? c_lo + G : nbchunks;
  if (c_lo >= c_hi) return;
  uint4 y;
  uint32_t cst = 1u;
  if (!map) {
    y = ybound ? ybound[g] : *y_io;
  } else {
    const uint32_t b = (j < 127) ? 1u << (j & 31) : 0u;
    y = make_uint4((j >> 5) == 0 ? b : 0u, (j >> 5) == 1 ? b : 0u, (j >> 5) == 2 ? b : 0u, (j >> 5) == 3 ? b : 0u);
    if (lin > 0 && j < 127) cst = 0u;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const int64_t cc = c_hi - 1 - k;
    if (cc >= c_lo) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        __pipeline_memcpy_async(&ring[k][4 * lane + q], forms + cc * 128 + 4 * lane + q, sizeof(uint4));
    }
    __pipeline_commit();
  }
  int slot = 0;
  for (int64_t c = c_hi - 1; c >= c_lo; --c) {
    __pipeline_wait_prior(D - 1);
    uint4 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = ring[slot][4 * lane + q];
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    uint32_t sel[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int u = 4 * lane + q;
      uint32_t yw = (u >> 5) == 0 ? y.x : (u >> 5) == 1 ? y.y : (u >> 5) == 2 ? y.z : y.w;
      sel[q] = (u == 127) ? cst : ((yw >> (u & 31)) & 1u);
      const uint32_t msk = 0u - sel[q];
      acc0 ^= w[q].x & msk;
      acc1 ^= w[q].y & msk;
      acc2 ^= w[q].z & msk;
      acc3 ^= w[q].w & msk;
    }
    // refill the slot just consumed (after its values were used)
    if (c - D >= c_lo) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        __pipeline_memcpy_async(&ring[slot][4 * lane + q], forms + (c - D) * 128 + 4 * lane + q, sizeof(uint4));
    }
    __pipeline_commit();
    slot = (slot + 1 == D) ? 0 : slot + 1;
    if (ysel) {
      const uint32_t s0 = __ballot_sync(FULL_WARP, sel[0]), s1 = __ballot_sync(FULL_WARP, sel[1]);
      const uint32_t s2 = __ballot_sync(FULL_WARP, sel[2]), s3 = __ballot_sync(FULL_WARP, sel[3]);
      if (lane == 0) ysel[c] = make_uint4(s0, s1, s2, s3);
    }
    if (yplain && lane == 0) yplain[c] = y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc0 ^= __shfl_xor_sync(FULL_WARP, acc0, o);
      acc1 ^= __shfl_xor_sync(FULL_WARP, acc1, o);
      acc2 ^= __shfl_xor_sync(FULL_WARP, acc2, o);
      acc3 ^= __shfl_xor_sync(FULL_WARP, acc3, o);
    }
    y = make_uint4(acc0, acc1, acc2, acc3 & 0x7FFFFFFFu);  // 127 bits
  }
  if (lane == 0) {
    if (map)
      y_io[g * 128 + j] = y;
    else if (!ybound)
      *y_io = y;
  }
}

// Final back substitution, a parallel map: sol[col] = parity(coef[col] &
// ysel[chunk]); one warp per 64-bit solution word (two ballots).
__global__ void ribbon_final_kernel(int64_t m, int64_t nwords, int cb, const uint4* __restrict__ coef,
                                    const uint4* __restrict__ ysel, uint64_t* words) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nwords; wi += nwarps) {
    uint32_t bits[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t cc = wi * 64 + h * 32 + lane;
      uint32_t bit = 0;
      if (cc < m) {
        const uint4 a = __ldcs(coef + cc);
        const uint4 y = __ldg(ysel + cc / cb);
        bit = __popc((a.x & y.x) ^ (a.y & y.y) ^ (a.z & y.z) ^ (a.w & y.w)) & 1u;
      }
      bits[h] = __ballot_sync(FULL_WARP, bit);
    }
    if (lane == 0) words[wi] = (uint64_t)bits[0] | ((uint64_t)bits[1] << 32);
  }
}

__global__ void ribbon_query_kernel(const int64_t* starts, const uint64_t* p0, const uint64_t* p1, int64_t N,
                                    const uint64_t* words, int64_t nwords, uint8_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = starts[i];
    int64_t wi = s >> 6;
    int sh = (int)(s & 63);
    uint64_t v0 = 0, v1 = 0;
    uint64_t a = wi < nwords ? words[wi] : 0;
    uint64_t b = wi + 1 < nwords ? words[wi + 1] : 0;
    uint64_t c = wi + 2 < nwords ? words[wi + 2] : 0;
    if (sh) {
      v0 = (a >> sh) | (b << (64 - sh));
      v1 = (b >> sh) | (c << (64 - sh));
    } else {
      v0 = a;
      v1 = b;
    }
    out[i] = (uint8_t)((__popcll(v0 & p0[i]) + __popcll(v1 & p1[i])) & 1);
  }
}

// Overflow rows of a pass, regrouped by the chunk they reached.  Rows past the
// local column range [0, M) (a column-sharded solve: they belong to the next
// rank) are appended to `exp` in global columns (+ c0) instead.
__global__ void ribbon_ovf_hist_kernel(const RRow* o, const int64_t* np, int64_t* hist, int64_t M) {
  const int64_t n = *np;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = o[i].s & S_MASK;
    if (s < M) atomicAdd((unsigned long long*)&hist[s / CE], 1ull);
  }
}
__global__ void ribbon_ovf_scatter_kernel(const RRow* o, const int64_t* np, int64_t* cursor, RRow* out, int64_t M,
                                          RRow* exp, int64_t* exp_count, int64_t c0) {
  const int64_t n = *np;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    RRow r = o[i];
    const int64_t s = r.s & S_MASK;
    if (s < M) {
      int64_t p = (int64_t)atomicAdd((unsigned long long*)&cursor[s / CE], 1ull);
      out[p] = r;
    } else {
      const int64_t k = (int64_t)atomicAdd((unsigned long long*)exp_count, 1ull);
      r.s = (s + c0) | (r.s & RHS_BIT);
      exp[k] = r;
    }
  }
}

// Imported rows (global columns) re-based to this rank's first column.
__global__ void ribbon_rebase_kernel(RRow* o, int64_t n, int64_t c0) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = o[i].s;
    o[i].s = ((s & S_MASK) - c0) | (s & RHS_BIT);
  }
}

}  // namespace shk

using namespace shk;

// Byte offsets of the solver's buffers inside ShkRibbon::buf.
struct RibLayout {
  size_t off_rows, off_rows2, off_ovf, off_exp, off_hist, off_rowoff, off_cursor, off_sp0, off_sp1, off_occ, off_sb,
      off_forms, off_coef, off_y, off_yio, off_ymap, off_gmap, off_ygrp, off_cnt, off_scan, off_bins, off_bcnt,
      total;
};

struct ShkRibbon {
  // device buffers, grown on demand
  void* buf = nullptr;
  size_t cap = 0;
  // column-sharded solve state (shk_ribbon_dist_*): rows capacity, local
  // column count, first global column
  RibLayout dL{};
  int64_t dN = 0, dM = 0, dc0 = 0;
};

int shk_ribbon_create(ShkRibbon** out) {
  *out = new ShkRibbon();
  return 0;
}

void shk_ribbon_destroy(ShkRibbon* r) {
  if (!r) return;
  if (r->buf) cudaFree(r->buf);
  delete r;
}

namespace {

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// Back-substitution chunk for M columns: the forms pass costs ~cb column
// steps on one CTA (latency-bound when there are few chunks) and the chain
// ~M / cb sequential mat-vecs, so small systems take short chunks (a power
// of two in [256, CB], ~sqrt(11.5 M)); large ones CB (throughput-bound).
int rib_cb(int64_t M) {
  const double want = sqrt((double)M * 11.5);
  int cb = 256;
  while (cb < want && cb < CB) cb <<= 1;
  return cb;
}

// Two-level chain over nbc back-chunks: groups of G ~ sqrt(nbc) chunks
// (ribbon_chain_kernel); short systems keep the single chain.
constexpr int64_t CHAIN_FLAT = 48;
int64_t chain_group(int64_t nbc) {
  int64_t G = 1;
  while (G * G < nbc) ++G;
  return G;
}
int64_t chain_groups(int64_t nbc) {
  if (nbc <= CHAIN_FLAT) return 1;
  const int64_t G = chain_group(nbc);
  return (nbc + G - 1) / G;
}

RibLayout layout(int64_t N, int64_t m, bool bins = false) {
  RibLayout L;
  int64_t nch = (m + CE - 1) / CE;
  int64_t nbc = (m + rib_cb(m) - 1) / rib_cb(m);
  int64_t nw32 = (m + 31) / 32 + CE / 32;
  size_t o = 0;
  L.off_rows = o;
  o += al((size_t)(N + 1) * sizeof(RRow));
  L.off_rows2 = o;
  o += al((size_t)(N + 1) * sizeof(RRow));
  L.off_ovf = o;
  o += al((size_t)(N + 1) * sizeof(RRow));
  L.off_exp = o;
  o += al((size_t)(N + 1) * sizeof(RRow));
  L.off_hist = o;
  o += al((size_t)(nch + 1) * 8);
  L.off_rowoff = o;
  o += al((size_t)(nch + 2) * 8);
  L.off_cursor = o;
  o += al((size_t)(nch + 1) * 8);
  L.off_sp0 = o;
  o += al((size_t)(m + 64) * 8);
  L.off_sp1 = o;
  o += al((size_t)(m + 64) * 8);
  L.off_occ = o;
  o += al((size_t)nw32 * 4);
  L.off_sb = o;
  o += al((size_t)nw32 * 4);
  L.off_forms = o;
  o += al((size_t)nbc * 128 * 16);
  L.off_coef = o;
  o += al((size_t)m * 16);
  L.off_y = o;
  o += al((size_t)nbc * 16);
  L.off_yio = o;
  o += 256;
  L.off_ymap = o;
  o += 128 * 16;
  {
    const int64_t ng = chain_groups(nbc);
    L.off_gmap = o;
    o += al((size_t)ng * 128 * 16);
    L.off_ygrp = o;
    o += al((size_t)ng * 16);
  }
  L.off_cnt = o;
  o += 256;
  L.off_scan = o;
  o += al(shk_scan_scratch(nch));
  L.off_bins = L.off_bcnt = 0;
  if (bins) {  // rows emitted by the construction kernel
    L.off_bins = o;
    o += al((size_t)nch * RIB_BIN_CAP * sizeof(RRow));
    L.off_bcnt = o;
    o += al((size_t)nch * 8);
  }
  L.total = o;
  return L;
}

int ensure(ShkRibbon* r, size_t bytes) {
  if (r->cap >= bytes) return 0;
  if (r->buf) cudaFree(r->buf);
  r->buf = nullptr;
  r->cap = 0;
  SHK_CUDA(cudaMalloc(&r->buf, bytes));
  r->cap = bytes;
  return 0;
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

// Views of the solver buffers.
struct RibBufs {
  RRow *rows, *rows2, *ovf, *exp;
  int64_t *hist, *rowoff, *cursor, *cnt;  // cnt: [0] ovf count, [1] inconsistent flag (int), [2] export count
  uint64_t *sp0, *sp1;
  uint32_t *occ, *sb;
  uint4 *forms, *coef, *yb, *yio, *ymap, *gmap, *ygrp;
  void* scan;
  RibBufs(ShkRibbon* R, const RibLayout& L) {
    char* B = (char*)R->buf;
    rows = (RRow*)(B + L.off_rows);
    rows2 = (RRow*)(B + L.off_rows2);
    ovf = (RRow*)(B + L.off_ovf);
    exp = (RRow*)(B + L.off_exp);
    hist = (int64_t*)(B + L.off_hist);
    rowoff = (int64_t*)(B + L.off_rowoff);
    cursor = (int64_t*)(B + L.off_cursor);
    cnt = (int64_t*)(B + L.off_cnt);
    sp0 = (uint64_t*)(B + L.off_sp0);
    sp1 = (uint64_t*)(B + L.off_sp1);
    occ = (uint32_t*)(B + L.off_occ);
    sb = (uint32_t*)(B + L.off_sb);
    forms = (uint4*)(B + L.off_forms);
    coef = (uint4*)(B + L.off_coef);
    yb = (uint4*)(B + L.off_y);
    yio = (uint4*)(B + L.off_yio);
    ymap = (uint4*)(B + L.off_ymap);
    gmap = (uint4*)(B + L.off_gmap);
    ygrp = (uint4*)(B + L.off_ygrp);
    scan = B + L.off_scan;
  }
};

// Empty slot table for M columns.
int rib_clear(ShkRibbon* R, const RibLayout& L, int64_t M, cudaStream_t st) {
  RibBufs b(R, L);
  const int64_t nw32 = (M + 31) / 32 + CE / 32;
  SHK_CUDA(cudaMemsetAsync(b.sp0, 0, (size_t)(M + 64) * 8, st));
  SHK_CUDA(cudaMemsetAsync(b.sp1, 0, (size_t)(M + 64) * 8, st));
  SHK_CUDA(cudaMemsetAsync(b.occ, 0, (size_t)nw32 * 4, st));
  SHK_CUDA(cudaMemsetAsync(b.sb, 0, (size_t)nw32 * 4, st));
  SHK_CUDA(cudaMemsetAsync(b.cnt, 0, 256, st));
  return 0;
}

// Regroup `n` rows at `src` (local columns) by elimination chunk into
// rows2 / rowoff; rows past column M go to the export buffer (global
// columns, + c0).
// Regroups the *np rows (count read on the device) at `src`.
int rib_regroup(const RibBufs& b, const RRow* src, const int64_t* np, int64_t M, int64_t c0, cudaStream_t st) {
  const int64_t nch = (M + CE - 1) / CE;
  SHK_CUDA(cudaMemsetAsync(b.hist, 0, (size_t)(nch + 1) * 8, st));
  ribbon_ovf_hist_kernel<<<148 * 4, 256, 0, st>>>(src, np, b.hist, M);
  SHK_LAUNCHED();
  int rc = shk_exclusive_scan_i64(b.hist, b.rowoff, nch, b.scan, shk_scan_scratch(nch), st);
  if (rc) return rc;
  SHK_CUDA(cudaMemcpyAsync(b.cursor, b.rowoff, (size_t)nch * 8, cudaMemcpyDeviceToDevice, st));
  ribbon_ovf_scatter_kernel<<<148 * 4, 256, 0, st>>>(src, np, b.cursor, b.rows2, M, b.exp, b.cnt + 2, c0);
  SHK_LAUNCHED();
  return 0;
}

// Chunks per warp of elimination pass `pass` (SHK_RIBBON_SPAN="1,1,4": a
// list per pass, the last entry repeats).  The first passes hold rows in
// every chunk and need one warp per chunk for parallelism; the late passes
// hold a few rows that walk several chunks, so merging chunks saves passes.
int rib_span(int pass) {
  static const std::vector<int> spans = [] {
    std::vector<int> v;
    const char* e = getenv("SHK_RIBBON_SPAN");
    std::string str = e ? e : RIB_SPAN_DEFAULT;
    size_t i = 0;
    while (i < str.size()) {
      const int x = atoi(str.c_str() + i);
      v.push_back((x == 2 || x == 4) ? x : 1);
      const size_t j = str.find(',', i);
      if (j == std::string::npos) break;
      i = j + 1;
    }
    if (v.empty()) v.push_back(1);
    return v;
  }();
  return spans[(size_t)pass < spans.size() ? (size_t)pass : spans.size() - 1];
}

// Elimination passes over the chunk-grouped rows at `cur` (offsets in
// rowoff) into the slot table of M local columns, until no row is left
// inside the range.  first: the slot table is known empty.  Rows leaving the
// range accumulate in the export buffer (count cnt[2]).  *bad: inconsistent.
// Passes run in batches without host round trips (every count stays on the
// device; a pass with nothing pending costs one near-empty launch); the host
// checks for completion once per batch.
int rib_passes(ShkRibbon* R, const RibLayout& L, RRow* cur, int64_t M, int64_t c0, int first, int* bad_out,
               cudaStream_t st, const unsigned long long* bins_cnt = nullptr) {
  RibBufs b(R, L);
  const int64_t nch = (M + CE - 1) / CE;
  int* bad = (int*)(b.cnt + 1);
  *bad_out = 0;
  constexpr int BATCH = 4;
  for (int pass = 0;;) {
    for (int k = 0; k < BATCH; ++k, ++pass) {
      // bin mode: the first pass's overflow list already holds the rows that
      // did not fit their bins (its count is cnt[0])
      const unsigned long long* bc = pass == 0 ? bins_cnt : nullptr;
      if (!bc) SHK_CUDA(cudaMemsetAsync(b.cnt, 0, 8, st));
      static const bool trace = getenv("SHK_RIBBON_TRACE") != nullptr;  // analysis: per-pass counts + times
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (trace) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
      }
      // first pass: one warp per 512-column chunk (all chunks hold rows);
      // later passes: 4 chunks per warp (few chunks hold rows, and a row may
      // walk 4 chunks before it overflows: ~3 passes after the first instead
      // of ~11)
      const int S = bc ? 1 : rib_span(pass);
      RRow* src = pass == 0 ? cur : b.rows2;
      const int fp = (first && pass == 0) ? 1 : 0;
      const unsigned g = (unsigned)((nch + S - 1) / S);
      if (S == 1 && pass == 0)
        ribbon_elim_kernel<1, true>
            <<<g, 32, 0, st>>>(src, b.rowoff, bc, RIB_BIN_CAP, nch, M, b.sp0, b.sp1, b.occ, b.sb, b.ovf, b.cnt, bad, fp);
      else if (S == 1)
        ribbon_elim_kernel<1, false>
            <<<g, 32, 0, st>>>(src, b.rowoff, bc, RIB_BIN_CAP, nch, M, b.sp0, b.sp1, b.occ, b.sb, b.ovf, b.cnt, bad, fp);
      else if (S == 2)
        ribbon_elim_kernel<2, false>
            <<<g, 32, 0, st>>>(src, b.rowoff, bc, RIB_BIN_CAP, nch, M, b.sp0, b.sp1, b.occ, b.sb, b.ovf, b.cnt, bad, fp);
      else
        ribbon_elim_kernel<4, false>
            <<<g, 32, 0, st>>>(src, b.rowoff, bc, RIB_BIN_CAP, nch, M, b.sp0, b.sp1, b.occ, b.sb, b.ovf, b.cnt, bad, fp);
      SHK_LAUNCHED();
      if (trace) {
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        int64_t h2[2];
        cudaMemcpy(h2, b.cnt, 16, cudaMemcpyDeviceToHost);
        fprintf(stderr, "ribbon pass %d: elim %.1f us, rows overflowing %lld\n", pass, ms * 1e3, (long long)h2[0]);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      }
      int rc = rib_regroup(b, b.ovf, b.cnt, M, c0, st);
      if (rc) return rc;
    }
    int64_t h[2];
    SHK_CUDA(cudaMemcpyAsync(h, b.cnt, 16, cudaMemcpyDeviceToHost, st));
    SHK_CUDA(cudaStreamSynchronize(st));
    if ((int)h[1]) {
      *bad_out = 1;
      return 0;
    }
    if (!h[0]) return 0;  // the last pass left nothing to regroup
    if (pass > 100000) {
      shk_set_error("ribbon elimination did not converge");
      return -1;
    }
  }
}

// Back substitution of the M local columns given the 127 solution bits right
// of them (y_in, host); y_out (host, may be null) gets the range's first 127
// bits; words_out (device) gets ceil(M/64) solution words.
int rib_forms(ShkRibbon* R, const RibLayout& L, int64_t M, cudaStream_t st) {
  RibBufs b(R, L);
  const int cb = rib_cb(M);
  const int64_t nbc = (M + cb - 1) / cb;
  ribbon_forms_kernel<<<(unsigned)nbc, 128, 0, st>>>(M, nbc, cb, b.sp0, b.sp1, b.occ, b.sb, b.forms, b.coef);
  SHK_LAUNCHED();
  return 0;
}

// forms must be current; chain from y_in, final map.
int rib_chain_final(ShkRibbon* R, const RibLayout& L, int64_t M, const uint32_t* y_in, uint32_t* y_out,
                    uint64_t* words_out, cudaStream_t st) {
  RibBufs b(R, L);
  const int cb = rib_cb(M);
  const int64_t nbc = (M + cb - 1) / cb;
  const uint4 y0 = y_in ? make_uint4(y_in[0], y_in[1], y_in[2], y_in[3]) : make_uint4(0, 0, 0, 0);
  SHK_CUDA(cudaMemcpyAsync(b.yio, &y0, 16, cudaMemcpyHostToDevice, st));
  if (nbc <= CHAIN_FLAT) {
    ribbon_chain_kernel<<<1, 32, 0, st>>>(nbc, nbc, b.forms, b.yb, nullptr, b.yio, nullptr, -1);
    SHK_LAUNCHED();
  } else {
    // group maps (linear part + constant) in parallel, the chain over the
    // group maps (each group's right boundary), then every group's chain
    const int64_t G = chain_group(nbc), ng = chain_groups(nbc);
    ribbon_chain_kernel<<<dim3(128, (unsigned)ng), 32, 0, st>>>(nbc, G, b.forms, nullptr, nullptr, b.gmap, nullptr,
                                                                1);
    SHK_LAUNCHED();
    ribbon_chain_kernel<<<1, 32, 0, st>>>(ng, ng, b.gmap, nullptr, b.ygrp, b.yio, nullptr, -1);
    SHK_LAUNCHED();
    ribbon_chain_kernel<<<(unsigned)ng, 32, 0, st>>>(nbc, G, b.forms, b.yb, nullptr, nullptr, b.ygrp, -1);
    SHK_LAUNCHED();
  }
  const int64_t nwords = (M + 63) / 64;
  int64_t fb = (nwords + 7) / 8;
  if (fb > 148 * 8) fb = 148 * 8;
  ribbon_final_kernel<<<(unsigned)fb, 256, 0, st>>>(M, nwords, cb, b.coef, b.yb, words_out);
  SHK_LAUNCHED();
  if (y_out) {
    SHK_CUDA(cudaMemcpyAsync(y_out, b.yio, 16, cudaMemcpyDeviceToHost, st));
    SHK_CUDA(cudaStreamSynchronize(st));
  }
  return 0;
}

int rib_backsub(ShkRibbon* R, const RibLayout& L, int64_t M, const uint32_t* y_in, uint32_t* y_out, uint64_t* words_out,
                cudaStream_t st) {
  int rc = rib_forms(R, L, M, st);
  if (rc) return rc;
  return rib_chain_final(R, L, M, y_in, y_out, words_out, st);
}

// Shared single-system driver once rows are in r->buf at off_rows with the
// chunk offsets in off_rowoff.
int solve_sorted(ShkRibbon* R, const RibLayout& L, int64_t N, int64_t m, uint64_t* words_out, int* consistent,
                 cudaStream_t st) {
  int rc = rib_clear(R, L, m, st);
  if (rc) return rc;
  int bad = 0;
  (void)N;
  rc = rib_passes(R, L, RibBufs(R, L).rows, m, 0, 1, &bad, st);
  if (rc) return rc;
  if (bad) {
    *consistent = 0;
    return 0;
  }
  *consistent = 1;
  return rib_backsub(R, L, m, nullptr, nullptr, words_out, st);
}

}  // namespace


namespace {
// Rows of the keys whose start column lies in [c0, c0 + M), chunk-grouped at
// off_rows / off_rowoff in local columns.
int gen_keyrows(ShkRibbon* R, const RibLayout& L, const ulonglong2* keys, const uint8_t* rhs, int64_t N, int64_t m,
                uint64_t seed, int64_t c0, int64_t M, cudaStream_t st) {
  RibBufs b(R, L);
  const int64_t nch = (M + CE - 1) / CE;
  const int64_t c1 = c0 + M;
  SHK_CUDA(cudaMemsetAsync(b.hist, 0, (size_t)(nch + 1) * 8, st));
  if (N > 0) {
    ribbon_keyrows_hist_kernel<<<grid_for(N), 256, 0, st>>>(keys, N, m, seed, b.hist, c0, c1);
    SHK_LAUNCHED();
  }
  int rc = shk_exclusive_scan_i64(b.hist, b.rowoff, nch, b.scan, shk_scan_scratch(nch), st);
  if (rc) return rc;
  SHK_CUDA(cudaMemcpyAsync(b.cursor, b.rowoff, (size_t)nch * 8, cudaMemcpyDeviceToDevice, st));
  if (N > 0) {
    ribbon_keyrows_scatter_kernel<<<grid_for(N), 256, 0, st>>>(keys, rhs, N, m, seed, b.cursor, b.rows, c0, c1);
    SHK_LAUNCHED();
  }
  return 0;
}
}  // namespace

int shk_ribbon_solve_keys(ShkRibbon* R, const uint64_t* keys_u64, const uint8_t* rhs, int64_t N, int64_t m,
                          uint64_t seed, uint64_t* words_out, int* consistent, cudaStream_t st) {
  const ulonglong2* keys = reinterpret_cast<const ulonglong2*>(keys_u64);
  if (m < RIBBON_W) {
    shk_set_error("ribbon needs m >= 128");
    return 3;
  }
  static const bool csr = [] {
    const char* e = getenv("SHK_RIBBON_BINS");  // A/B: 0 = histogram + scan + CSR scatter
    return e && e[0] == '0';
  }();
  if (csr) {
    RibLayout L = layout(N, m);
    int rc = ensure(R, L.total);
    if (rc) return rc;
    rc = gen_keyrows(R, L, keys, rhs, N, m, seed, 0, m, st);
    if (rc) return rc;
    return solve_sorted(R, L, N, m, words_out, consistent, st);
  }
  RibLayout L = layout(N, m, true);
  int rc = ensure(R, L.total);
  if (rc) return rc;
  rc = rib_clear(R, L, m, st);  // also zeroes the overflow count cnt[0]
  if (rc) return rc;
  RibBufs b(R, L);
  char* B = (char*)R->buf;
  const int64_t nch = (m + CE - 1) / CE;
  unsigned long long* bcnt = (unsigned long long*)(B + L.off_bcnt);
  RRow* bins = (RRow*)(B + L.off_bins);
  SHK_CUDA(cudaMemsetAsync(bcnt, 0, (size_t)nch * 8, st));
  if (N > 0) {
    ribbon_keyrows_bins_kernel<<<grid_for(N), 256, 0, st>>>(keys, rhs, N, m, seed, bcnt, RIB_BIN_CAP, bins, b.ovf,
                                                            (unsigned long long*)b.cnt);
    SHK_LAUNCHED();
  }
  int bad = 0;
  rc = rib_passes(R, L, bins, m, 0, 1, &bad, st, bcnt);
  if (rc) return rc;
  if (bad) {
    *consistent = 0;
    return 0;
  }
  *consistent = 1;
  return rib_backsub(R, L, m, nullptr, nullptr, words_out, st);
}

// ---------------------------------------------------------------------------
// Column-sharded solve (SURVEY.md §8(e) option B): this rank owns columns
// [c0, c1) (c0 a multiple of CB).  begin: rows starting in the range,
// eliminated locally; rows whose pivot walks past c1 are exported (global
// columns) for the right neighbour, which imports them and may export
// further.  When no rank exports any more, backsub runs right to left
// across ranks: each takes the first 127 solution bits of its right
// neighbour and hands its own first 127 bits to its left neighbour.  The
// solution is the single-system one.
int shk_ribbon_dist_begin(ShkRibbon* R, const uint64_t* keys_u64, const uint8_t* rhs, int64_t N, int64_t m,
                          uint64_t seed, int64_t c0, int64_t c1, int64_t* n_export, int* bad, cudaStream_t st) {
  if (m < RIBBON_W || c0 < 0 || c1 > m || c0 >= c1 || (c0 % CB) != 0 || (c1 != m && (c1 % CB) != 0)) {
    shk_set_error("bad column range [%lld, %lld) of %lld", (long long)c0, (long long)c1, (long long)m);
    return 3;
  }
  const int64_t M = c1 - c0;
  RibLayout L = layout(N, M);
  int rc = ensure(R, L.total);
  if (rc) return rc;
  R->dL = L;
  R->dN = N;
  R->dM = M;
  R->dc0 = c0;
  rc = rib_clear(R, L, M, st);
  if (rc) return rc;
  rc = gen_keyrows(R, L, reinterpret_cast<const ulonglong2*>(keys_u64), rhs, N, m, seed, c0, M, st);
  if (rc) return rc;
  RibBufs b(R, L);
  rc = rib_passes(R, L, b.rows, M, c0, 1, bad, st);
  if (rc) return rc;
  SHK_CUDA(cudaMemcpyAsync(n_export, b.cnt + 2, 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// Copy out (host, 24 bytes per row: p0, p1, start | rhs << 62) and clear the
// exported rows.
int shk_ribbon_dist_take_exports(ShkRibbon* R, void* rows_out, int64_t n, cudaStream_t st) {
  RibBufs b(R, R->dL);
  if (n > 0) SHK_CUDA(cudaMemcpyAsync(rows_out, b.exp, (size_t)n * sizeof(RRow), cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaMemsetAsync(b.cnt + 2, 0, 8, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// Insert rows exported by the left neighbour (global columns >= c0).
int shk_ribbon_dist_import(ShkRibbon* R, const void* rows_in, int64_t n, int64_t* n_export, int* bad,
                           cudaStream_t st) {
  RibBufs b(R, R->dL);
  *bad = 0;
  if (n > R->dN) {
    shk_set_error("too many imported rows");
    return 3;
  }
  if (n > 0) {
    SHK_CUDA(cudaMemcpyAsync(b.ovf, rows_in, (size_t)n * sizeof(RRow), cudaMemcpyHostToDevice, st));
    ribbon_rebase_kernel<<<grid_for(n), 256, 0, st>>>(b.ovf, n, R->dc0);
    SHK_LAUNCHED();
    SHK_CUDA(cudaMemcpyAsync(b.cnt + 3, &n, 8, cudaMemcpyHostToDevice, st));
    int rc = rib_regroup(b, b.ovf, b.cnt + 3, R->dM, R->dc0, st);
    if (rc) return rc;
    rc = rib_passes(R, R->dL, b.rows2, R->dM, R->dc0, 0, bad, st);
    if (rc) return rc;
  }
  SHK_CUDA(cudaMemcpyAsync(n_export, b.cnt + 2, 8, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// y_in: the right neighbour's first 127 solution bits (zero for the last
// range); y_out: this range's first 127 bits; words_out (device): its
// (c1 - c0 + 63) / 64 solution words.
int shk_ribbon_dist_backsub(ShkRibbon* R, const uint32_t* y_in, uint32_t* y_out, uint64_t* words_out,
                            cudaStream_t st) {
  return rib_backsub(R, R->dL, R->dM, y_in, y_out, words_out, st);
}

// Parallel back substitution across ranks, step 1: this range's forms and
// its boundary map (map_out, host, [128][4] words: rows j < 127 = the first
// 127 bits for y_in = e_j, row 127 = for y_in = 0).
int shk_ribbon_dist_map(ShkRibbon* R, uint32_t* map_out, cudaStream_t st) {
  RibBufs b(R, R->dL);
  int rc = rib_forms(R, R->dL, R->dM, st);
  if (rc) return rc;
  const int64_t nbc = (R->dM + rib_cb(R->dM) - 1) / rib_cb(R->dM);
  if (nbc <= CHAIN_FLAT) {
    ribbon_chain_kernel<<<dim3(128, 1), 32, 0, st>>>(nbc, nbc, b.forms, nullptr, nullptr, b.ymap, nullptr, 0);
  } else {  // the range's map composed from its group maps
    const int64_t G = chain_group(nbc), ng = chain_groups(nbc);
    ribbon_chain_kernel<<<dim3(128, (unsigned)ng), 32, 0, st>>>(nbc, G, b.forms, nullptr, nullptr, b.gmap, nullptr,
                                                                1);
    SHK_LAUNCHED();
    ribbon_chain_kernel<<<dim3(128, 1), 32, 0, st>>>(ng, ng, b.gmap, nullptr, nullptr, b.ymap, nullptr, 0);
  }
  SHK_LAUNCHED();
  SHK_CUDA(cudaMemcpyAsync(map_out, b.ymap, 128 * 16, cudaMemcpyDeviceToHost, st));
  SHK_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// Step 2: chain from the composed y_in and the final map (forms from step 1).
int shk_ribbon_dist_finish(ShkRibbon* R, const uint32_t* y_in, uint64_t* words_out, cudaStream_t st) {
  return rib_chain_final(R, R->dL, R->dM, y_in, nullptr, words_out, st);
}

int shk_ribbon_solve_rows(ShkRibbon* R, const int64_t* starts, const uint64_t* p0, const uint64_t* p1,
                          const uint8_t* rhs, int64_t N, int64_t m, uint64_t* words_out, int* consistent,
                          cudaStream_t st) {
  if (m < RIBBON_W) {
    shk_set_error("ribbon needs m >= 128");
    return 3;
  }
  RibLayout L = layout(N, m);
  int rc = ensure(R, L.total);
  if (rc) return rc;
  char* B = (char*)R->buf;
  const int64_t nch = (m + CE - 1) / CE;
  int64_t* hist = (int64_t*)(B + L.off_hist);
  int64_t* rowoff = (int64_t*)(B + L.off_rowoff);
  int64_t* cursor = (int64_t*)(B + L.off_cursor);
  SHK_CUDA(cudaMemsetAsync(hist, 0, (size_t)(nch + 1) * 8, st));
  if (N > 0) {
    ribbon_rows_hist_kernel<<<grid_for(N), 256, 0, st>>>(starts, N, hist);
    SHK_LAUNCHED();
  }
  rc = shk_exclusive_scan_i64(hist, rowoff, nch, B + L.off_scan, shk_scan_scratch(nch), st);
  if (rc) return rc;
  SHK_CUDA(cudaMemcpyAsync(cursor, rowoff, (size_t)nch * 8, cudaMemcpyDeviceToDevice, st));
  if (N > 0) {
    ribbon_rows_scatter_kernel<<<grid_for(N), 256, 0, st>>>(starts, p0, p1, rhs, N, cursor, (RRow*)(B + L.off_rows));
    SHK_LAUNCHED();
  }
  return solve_sorted(R, L, N, m, words_out, consistent, st);
}

int shk_launch_ribbon_rows(const uint64_t* hi, const uint64_t* lo, int stride, int64_t N, int64_t m, uint64_t seed,
                           int64_t* starts, uint64_t* p0, uint64_t* p1, cudaStream_t st) {
  if (N <= 0) return 0;
  ribbon_rows_kernel<<<grid_for(N), 256, 0, st>>>(hi, lo, stride, N, m, seed, starts, p0, p1);
  SHK_LAUNCHED();
  return 0;
}

int shk_launch_ribbon_query(const int64_t* starts, const uint64_t* p0, const uint64_t* p1, int64_t N,
                            const uint64_t* words, int64_t nwords, uint8_t* out, cudaStream_t st) {
  if (N <= 0) return 0;
  ribbon_query_kernel<<<grid_for(N), 256, 0, st>>>(starts, p0, p1, N, words, nwords, out);
  SHK_LAUNCHED();
  return 0;
}
