// Microbenchmark: throughput of the split-search inner loop (remix hi word +
// 3 threshold counts) with different ALU/FMA formulations of the xor-shifts.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/remix_variants.cu -o tools/remix_variants
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
struct u2 { uint32_t lo, hi; };
__constant__ uint32_t P2[33];
template <uint64_t C> __device__ __forceinline__ u2 mulc(u2 z) {
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  uint64_t w = (uint64_t)z.lo * cl; u2 r{(uint32_t)w, (uint32_t)(w >> 32)};
  r.hi = r.hi + z.lo * ch + z.hi * cl; return r;
}
template <uint64_t C> __device__ __forceinline__ u2 mulc2(u2 z) {  // no IMAD.WIDE
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  u2 r; r.lo = z.lo * cl; r.hi = __umulhi(z.lo, cl) + z.lo * ch + z.hi * cl; return r;
}
template <uint64_t C> __device__ __forceinline__ u2 mulc3(u2 z) {  // IMAD.WIDE with the cross terms as addend
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  uint32_t t = z.lo * ch + z.hi * cl;
  uint64_t w = (uint64_t)z.lo * cl + ((uint64_t)t << 32);
  return u2{(uint32_t)w, (uint32_t)(w >> 32)};
}
template <uint64_t C> __device__ __forceinline__ u2 mulc5(u2 z) {
  constexpr uint32_t cl = (uint32_t)C, ch = (uint32_t)(C >> 32);
  u2 r;
  asm("{\n\t.reg .u64 w;\n\t.reg .u32 wh, t;\n\t"
      "mul.wide.u32 w, %2, %4;\n\t"
      "mov.b64 {%0, wh}, w;\n\t"
      "mad.lo.u32 t, %2, %5, wh;\n\t"
      "mad.lo.u32 %1, %3, %4, t;\n\t"
      "}" : "=r"(r.lo), "=r"(r.hi) : "r"(z.lo), "r"(z.hi), "n"(cl), "n"(ch));
  return r;
}
template <uint64_t C, int W> __device__ __forceinline__ u2 mulv(u2 z) {
  return W == 1 ? mulc2<C>(z) : W == 2 ? mulc5<C>(z) : mulc<C>(z);
}
template <int S, bool F> __device__ __forceinline__ u2 xs(u2 z) {
  uint32_t lo_sh;
  if (F) lo_sh = __umulhi(z.lo, P2[32 - S]) + z.hi * P2[32 - S];
  else lo_sh = __funnelshift_r(z.lo, z.hi, S);
  uint32_t hi_sh = __umulhi(z.hi, 1u << (32 - S));
  return u2{z.lo ^ lo_sh, z.hi ^ hi_sh};
}
template <int S> __device__ __forceinline__ u2 xsa(u2 z) {  // all-ALU variant
  uint32_t lo_sh = __funnelshift_r(z.lo, z.hi, S);
  uint32_t hi_sh;
  asm("shr.b32 %0, %1, %2;" : "=r"(hi_sh) : "r"(z.hi), "n"(S));
  return u2{z.lo ^ lo_sh, z.hi ^ hi_sh};
}
template <int S, int A> __device__ __forceinline__ u2 xsv(u2 z) { return A ? xsa<S>(z) : xs<S, false>(z); }
template <int M> __device__ __forceinline__ uint32_t remix_hi(u2 h, u2 l, u2 x) {
  u2 z{h.lo ^ x.lo, h.hi ^ x.hi};
  z = mulv<0xBF58476D1CE4E5B9ull, (M & 64) ? 1 : (M & 1024) ? 2 : 0>(xsv<30, (M & 1)>(z));
  z = mulv<0x94D049BB133111EBull, (M & 128) ? 1 : (M & 2048) ? 2 : 0>(xsv<27, (M & 2)>(z));
  z = xsv<31, (M & 4)>(z);
  z.lo ^= l.lo; z.hi ^= l.hi;
  z = mulv<0xBF58476D1CE4E5B9ull, (M & 256) ? 1 : (M & 4096) ? 2 : 0>(xsv<30, (M & 8)>(z));
  z = mulv<0x94D049BB133111EBull, (M & 512) ? 1 : (M & 8192) ? 2 : 0>(xsv<27, (M & 16)>(z));
  uint32_t hs; if (M & 32) asm("shr.b32 %0, %1, 31;" : "=r"(hs) : "r"(z.hi)); else hs = __umulhi(z.hi, 2u);
  return z.hi ^ hs;
}
template <int M> __global__ void kern(const ulonglong2* keys, int m, int iters, uint32_t T0, uint32_t T1, uint32_t T2, int* out) {
  int g1 = 0, g2 = 0, g3 = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t s = (uint64_t)it * 1000003 + blockIdx.x * blockDim.x + threadIdx.x;
    u2 x{(uint32_t)(s * 0x9E3779B97F4A7C15ull), (uint32_t)((s * 0x9E3779B97F4A7C15ull) >> 32)};
#pragma unroll 8
    for (int i = 0; i < m; ++i) {
      ulonglong2 k = __ldg(keys + i);
      uint32_t vh = remix_hi<M>(u2{(uint32_t)k.x, (uint32_t)(k.x >> 32)}, u2{(uint32_t)k.y, (uint32_t)(k.y >> 32)}, x);
      g1 += vh >= T0; g2 += vh >= T1; g3 += vh >= T2;
    }
  }
  if (g1 + g2 + g3 == 0x7fffffff) out[0] = 1;
}
template <int M> void run(const ulonglong2* keys, int* out) {
  int m = 160, iters = 64;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern<M>, 256, 0);
  dim3 grid(148 * occ);
  kern<M><<<grid, 256>>>(keys, m, 4, 1 << 30, 2u << 30, 3u << 30, out);
  cudaEventRecord(a);
  kern<M><<<grid, 256>>>(keys, m, iters, 1 << 30, 2u << 30, 3u << 30, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double evals = (double)grid.x * 256 * iters * m;
  printf("mask %4d occ %d: %.3f ms  %.1f Geval/s  (%.1f Tops/s at 46 ops/eval)\n", M, occ, ms, evals / ms / 1e6, evals * 46 / ms / 1e9);
}
int main() {
  uint32_t p[33]; for (int i = 0; i < 33; ++i) p[i] = i < 32 ? (1u << i) : 0;
  cudaMemcpyToSymbol(P2, p, sizeof p);
  ulonglong2* keys; cudaMalloc(&keys, 4096 * 16); cudaMemset(keys, 7, 4096 * 16);
  int* out; cudaMalloc(&out, 4);
  run<63>(keys, out); run<63+64>(keys, out); run<63+64+128>(keys, out); run<63+512>(keys, out); run<0>(keys, out); run<960>(keys, out);
  run<63+1024+2048+4096+8192>(keys, out); run<0+1024+2048+4096+8192>(keys, out); run<63+1024+2048+4096>(keys, out);
  run<63+960>(keys, out); run<31+960>(keys, out); run<32+1+2+4+960>(keys, out); run<32+1+2+4+15360>(keys, out);
  run<32+8+16+4+15360>(keys, out); run<32+4+15360>(keys, out);
  return 0;
}
