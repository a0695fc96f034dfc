// ShockHash hash family, shared by every kernel and by the scalar host API.
//
// Bit-exact restatement of the reference hash family
//   /root/reference/pkg/src/shockhash/_kernels/_pure.py:17-72
//   /root/reference/pkg/src/shockhash/_kernels/_core.pyx:24-102
// (SplitMix64 finalizer, per-(seed, tag) mixer, remix, 32-bit multiply-shift
// range reduction, leaf_pair with h1 drawn from the n-1 cells != h0).
//
// Device versions are written in 32-bit halves so the 64-bit multiplies map to
// IMAD.WIDE / IMAD on the FMA pipe and the constant right shifts of the high
// word map to IMAD.HI (also FMA pipe), balancing the ALU (LOP3/SHF) and FMA
// pipes, which is where the integer issue roofline of the seed searches is set.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SHK_HD __host__ __device__ __forceinline__
#define SHK_D __device__ __forceinline__
#else
#define SHK_HD inline
#endif

namespace shk {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t MUL1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MUL2 = 0x94D049BB133111EBull;

enum Tag : uint64_t {
  TAG_LEAF = 1,
  TAG_SPLITBIT = 2,
  TAG_SPLIT = 3,
  TAG_BUCKET = 4,
  TAG_RSTART = 5,
  TAG_RPAT0 = 6,
  TAG_RPAT1 = 7,
};

constexpr int RIBBON_W = 128;

// ---------------------------------------------------------------------------
// Portable definitions (host scalar API; also valid device code).

SHK_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MUL1;
  z = (z ^ (z >> 27)) * MUL2;
  return z ^ (z >> 31);
}

SHK_HD uint64_t seed_mixer(uint64_t seed, uint64_t tag) { return mix64(seed + tag * GOLDEN); }

SHK_HD uint64_t remix_x(uint64_t hi, uint64_t lo, uint64_t x) { return mix64(mix64(hi ^ x) ^ lo); }

SHK_HD uint64_t remix(uint64_t hi, uint64_t lo, uint64_t seed, uint64_t tag) {
  return remix_x(hi, lo, seed_mixer(seed, tag));
}

SHK_HD uint64_t hash_range(uint64_t v, uint64_t m) { return ((v >> 32) * m) >> 32; }

// Cells of a key in a leaf of n cells from one remixed word (n == 1 -> (0, 0)).
SHK_HD void leaf_pair_v(uint64_t v, int n, int& h0, int& h1) {
  int a = (int)(((v >> 32) * (uint64_t)n) >> 32);
  int b = (int)(((v & 0xFFFFFFFFull) * (uint64_t)(n - 1)) >> 32);
  b += (b >= a);
  h0 = a;
  h1 = b;
}

SHK_HD void leaf_pair(uint64_t hi, uint64_t lo, uint64_t seed, int n, int& h0, int& h1) {
  if (n == 1) {
    h0 = 0;
    h1 = 0;
    return;
  }
  leaf_pair_v(remix(hi, lo, seed, TAG_LEAF), n, h0, h1);
}

SHK_HD int split_bit(uint64_t hi, uint64_t lo, uint64_t seed) {
  return (int)(remix(hi, lo, seed, TAG_SPLITBIT) >> 63);
}

// Query-side cell of a key inside its leaf: _core.pyx:751-767 / _pure.py:553-569.
SHK_HD int leaf_cell(uint64_t hi, uint64_t lo, int64_t q, int mleaf, int mode, int64_t cache_k, int choice) {
  int h0, h1;
  if (mode == 0) {
    leaf_pair(hi, lo, (uint64_t)q, mleaf, h0, h1);
    return choice ? h1 : h0;
  }
  int64_t base = q / mleaf;
  int64_t r = q % mleaf;
  int64_t sa = (mode == 2 && cache_k && mleaf > 32) ? base - (base % cache_k) : base;
  if (split_bit(hi, lo, (uint64_t)sa) == 0) {
    leaf_pair(hi, lo, (uint64_t)sa, mleaf, h0, h1);
    return choice ? h1 : h0;
  }
  leaf_pair(hi, lo, (uint64_t)base, mleaf, h0, h1);
  return (int)(((int64_t)(choice ? h1 : h0) + r) % mleaf);
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// Device fast paths (bit-identical to the portable definitions).

struct u2 {
  uint32_t lo, hi;
};

SHK_D u2 split64(uint64_t v) {
  u2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(r.lo), "=r"(r.hi) : "l"(v));
  return r;
}

SHK_D uint64_t join64(uint32_t lo, uint32_t hi) {
  uint64_t v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(lo), "r"(hi));
  return v;
}

// z ^= z >> S in 32-bit halves; the high-word shift goes to the FMA pipe as
// IMAD.HI(hi, 2^(32-S)).
#ifndef SHK_ALU_SHIFTS
#define SHK_ALU_SHIFTS 0
#endif
template <int S>
SHK_D u2 xorshr_alu(u2 z);
template <int S>
SHK_D u2 xorshr(u2 z) {
  if (SHK_ALU_SHIFTS) return xorshr_alu<S>(z);
  uint32_t lo_sh = __funnelshift_r(z.lo, z.hi, S);       // (z >> S) low word
  uint32_t hi_sh = __umulhi(z.hi, 1u << (32 - S));        // (z >> S) high word
  u2 r;
  r.lo = z.lo ^ lo_sh;
  r.hi = z.hi ^ hi_sh;
  return r;
}

// Same with the high-word shift on the ALU pipe (SHF): the split search's
// loop is FMA-pipe bound (IMAD.WIDE), measured +7% (tools/remix_variants.cu).
template <int S>
SHK_D u2 xorshr_alu(u2 z) {
  uint32_t lo_sh = __funnelshift_r(z.lo, z.hi, S);
  uint32_t hi_sh;
  asm("shr.b32 %0, %1, %2;" : "=r"(hi_sh) : "r"(z.hi), "n"(S));
  u2 r;
  r.lo = z.lo ^ lo_sh;
  r.hi = z.hi ^ hi_sh;
  return r;
}

// z * C (mod 2^64) in halves: one IMAD.WIDE.U32 + two chained IMAD (written
// in PTX: left to itself the compiler sums the cross terms separately and
// spends a fourth FMA-pipe instruction on the add).
template <uint64_t C>
SHK_D u2 mulc(u2 z) {
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  u2 r;
  asm("{\n\t.reg .u64 w;\n\t.reg .u32 wh, t;\n\t"
      "mul.wide.u32 w, %2, %4;\n\t"
      "mov.b64 {%0, wh}, w;\n\t"
      "mad.lo.u32 t, %2, %5, wh;\n\t"
      "mad.lo.u32 %1, %3, %4, t;\n\t"
      "}"
      : "=r"(r.lo), "=r"(r.hi)
      : "r"(z.lo), "r"(z.hi), "n"(cl), "n"(ch));
  return r;
}

// High word of z * C (mod 2^64): IMAD.HI + two chained IMAD.
template <uint64_t C>
SHK_D uint32_t mulc_hi(u2 z) {
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "mul.hi.u32 t, %1, %3;\n\t"
      "mad.lo.u32 t, %1, %4, t;\n\t"
      "mad.lo.u32 %0, %2, %3, t;\n\t"
      "}"
      : "=r"(r)
      : "r"(z.lo), "r"(z.hi), "n"(cl), "n"(ch));
  return r;
}

SHK_D u2 mix64_d(u2 z) {
  z = mulc<MUL1>(xorshr<30>(z));
  z = mulc<MUL2>(xorshr<27>(z));
  return xorshr<31>(z);
}

// remix with a precomputed seed mixer x = seed_mixer(seed, tag).
SHK_D u2 remix_d(u2 k_hi, u2 k_lo, u2 x) {
  u2 z;
  z.lo = k_hi.lo ^ x.lo;
  z.hi = k_hi.hi ^ x.hi;
  z = mix64_d(z);
  z.lo ^= k_lo.lo;
  z.hi ^= k_lo.hi;
  return mix64_d(z);
}


// ---------------------------------------------------------------------------
// Pre-mixed keys.  The first xor-shift of remix distributes over the seed
// xor:  (hi ^ x) ^ ((hi ^ x) >> 30) = (hi ^ (hi >> 30)) ^ (x ^ (x >> 30)),
// so the seed searches store every key's high word as hp = premix(hi) once
// and every candidate seed's mixer as xp = premix(x) once, and drop one
// xor-shift (4 ALU instructions) from every (key, seed) evaluation.  Results
// are bit-identical to remix(); unpremix inverts premix.
SHK_HD uint64_t premix_hi(uint64_t h) { return h ^ (h >> 30); }
SHK_HD uint64_t unpremix_hi(uint64_t h) { return h ^ (h >> 30) ^ (h >> 60); }

SHK_D u2 seed_mixer_pre_d(uint64_t seed, uint64_t tag) { return split64(premix_hi(seed_mixer(seed, tag))); }

// First mix64 from pre-mixed operands, then the second one (full remix).
// AM bit i: xor-shift i (27, 31, 30, 27, 31 in order) takes its high-word
// shift on the ALU pipe (SHF) instead of the FMA pipe (IMAD.HI), to balance
// the two pipes per kernel (the plain leaf search is FMA-heavy: ncu
// profiles/r01_ncu_full_leaf_c3_v17.csv).
template <int S, int AM, int I>
SHK_D u2 xs_sel(u2 z) {
  return ((AM >> I) & 1) ? xorshr_alu<S>(z) : xorshr<S>(z);
}
template <int AM = 0>
SHK_D u2 remix_pre_d(u2 kp, u2 k_lo, u2 xp) {
  u2 z;
  z.lo = kp.lo ^ xp.lo;
  z.hi = kp.hi ^ xp.hi;
  z = mulc<MUL1>(z);
  z = mulc<MUL2>(xs_sel<27, AM, 0>(z));
  z = xs_sel<31, AM, 1>(z);
  z.lo ^= k_lo.lo;
  z.hi ^= k_lo.hi;
  z = mulc<MUL1>(xs_sel<30, AM, 2>(z));
  z = mulc<MUL2>(xs_sel<27, AM, 3>(z));
  return xs_sel<31, AM, 4>(z);
}

// AM bit i: xor-shift i (27, 31, 30, 27) takes its high-word shift on the
// ALU pipe (SHF) instead of the FMA pipe (IMAD.HI, two FMA issue slots).
template <int AM = 0>
SHK_D uint32_t remix_top_pre_d(u2 kp, u2 k_lo, u2 xp) {
  u2 z;
  z.lo = kp.lo ^ xp.lo;
  z.hi = kp.hi ^ xp.hi;
  z = mulc<MUL1>(z);
  z = mulc<MUL2>(xs_sel<27, AM, 0>(z));
  z = xs_sel<31, AM, 1>(z);
  z.lo ^= k_lo.lo;
  z.hi ^= k_lo.hi;
  z = mulc<MUL1>(xs_sel<30, AM, 2>(z));
  return mulc_hi<MUL2>(xs_sel<27, AM, 3>(z)) >> 31;
}


SHK_D void leaf_pair_d(u2 v, uint32_t n, uint32_t nm1, uint32_t& h0, uint32_t& h1) {
  uint32_t a = __umulhi(v.hi, n);
  uint32_t b = __umulhi(v.lo, nm1);
  b += (b >= a) ? 1u : 0u;
  h0 = a;
  h1 = b;
}

SHK_D u2 seed_mixer_d(uint64_t seed, uint64_t tag) { return split64(seed_mixer(seed, tag)); }

// PTX shl.b32 clamps shift amounts >= 32 to a zero result, which gives cheap
// 64-bit cell masks split in two 32-bit words.
SHK_D uint32_t shl_clamp(uint32_t v, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
  return r;
}

// v << (s mod 32) (SHF.L.W).
SHK_D uint32_t shl_wrap(uint32_t v, uint32_t s) { return __funnelshift_l(0u, v, s); }
#endif

}  // namespace shk
