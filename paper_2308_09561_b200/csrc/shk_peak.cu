// Integer-issue peak microbenchmark: the measured denominator beside the
// nominal 128 int32 ops/clk/SM of the seed searches' roofline (SURVEY.md
// §8(d)).  Not part of the reference's path (it has no counterpart); bench.py
// runs it once per process and reports it next to the nominal figure.
//
// Every thread runs 8 independent dependency chains of 32-bit integer
// instructions (inline PTX, so ptxas emits exactly one SASS instruction per
// PTX op: LOP3.LUT for lop3.b32, IMAD for mad.lo.u32, SHF for shf.r.wrap):
//   kind 0: LOP3 only         (ALU pipe)
//   kind 1: IMAD only         (FMA-heavy pipe)
//   kind 2: LOP3 + IMAD, 1:1  (both pipes: the ideal split of the searches)
//   kind 3: SHF + LOP3 + IMAD, 2:1:1 (the remix's own mix: xor-shifts on
//           SHF/LOP3, multiplies on IMAD)
// Pipe costs of the multiply forms the hash uses (analysis, tools/int_peak.py;
// two ops per chain step each):
//   kind 4: IMAD.WIDE only   kind 5: IMAD.HI only
//   kind 6: IMAD.WIDE + LOP3 1:1   kind 7: IMAD.HI + LOP3 1:1
//   kind 8: IMAD by a power of two (a shift on the FMA pipe) + LOP3 1:1
// ops = threads x iters x 8 chains x ops per chain step; the grid fills every
// SM with 64 warps.
#include "shk_common.cuh"
#include "shk_kernels.h"

namespace shk {

template <int KIND>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t* sink, int iters, uint32_t seed) {
  uint32_t x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = seed ^ (threadIdx.x * 0x9E3779B9u + j * 0x85EBCA6Bu + blockIdx.x);
  const uint32_t y = seed * 3u + 1u, z = seed ^ 0x5bd1e995u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(y), "r"(z));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(x[j]) : "r"(z), "r"(y));
      } else if (KIND == 1) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(y), "r"(z));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(z), "r"(y));
      } else if (KIND == 2) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(y), "r"(z));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(z), "r"(y));
      } else if (KIND == 4 || KIND == 6) {
        uint32_t lo, hi;
        asm volatile("{\n\t.reg .u64 w;\n\tmul.wide.u32 w, %2, %3;\n\tmov.b64 {%0, %1}, w;\n\t}"
                     : "=r"(lo), "=r"(hi)
                     : "r"(x[j]), "r"(y));
        if (KIND == 4) {
          asm volatile("{\n\t.reg .u64 w;\n\tmul.wide.u32 w, %2, %3;\n\tmov.b64 {%0, %1}, w;\n\t}"
                       : "=r"(x[j]), "=r"(hi)
                       : "r"(lo), "r"(z));
        } else {
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(x[j]) : "r"(lo), "r"(hi), "r"(z));
        }
      } else if (KIND == 5 || KIND == 7) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[j]) : "r"(y));
        if (KIND == 5)
          asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[j]) : "r"(z));
        else
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(z), "r"(y));
      } else if (KIND == 8) {
        asm volatile("mad.lo.u32 %0, %0, 8192, %1;" : "+r"(x[j]) : "r"(y));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(z), "r"(y));
      } else {
        uint32_t t;
        asm volatile("shf.r.wrap.b32 %0, %1, %1, 13;" : "=r"(t) : "r"(x[j]));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(t), "r"(y));
        asm volatile("shf.r.wrap.b32 %0, %1, %1, 7;" : "=r"(t) : "r"(x[j]));
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(x[j]) : "r"(t), "r"(z));
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= x[j];
  if (acc == 0x12345678u) sink[0] = acc;  // keeps the chains alive
}

}  // namespace shk

using namespace shk;

int shk_launch_int_peak(int kind, int iters, int num_sms, uint32_t* sink, int64_t* threads_out, int* ops_per_step,
                        cudaStream_t st) {
  const int blocks = num_sms * 8;  // 8 x 256 threads = 64 warps per SM
  *threads_out = (int64_t)blocks * 256;
  *ops_per_step = 8 * (kind == 3 ? 4 : 2);
  switch (kind) {
    case 0: int_peak_kernel<0><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 1: int_peak_kernel<1><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 2: int_peak_kernel<2><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 3: int_peak_kernel<3><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 4: int_peak_kernel<4><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 5: int_peak_kernel<5><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 6: int_peak_kernel<6><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 7: int_peak_kernel<7><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    case 8: int_peak_kernel<8><<<blocks, 256, 0, st>>>(sink, iters, 0x1234567u); break;
    default: shk_set_error("int peak kind must be 0..8"); return 3;
  }
  SHK_LAUNCHED();
  return 0;
}
