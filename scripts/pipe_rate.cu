// ALU pipe probe: clocks per warp-instruction for FFMA, FFMA2, FADD2, MUFU.EX2,
// F2FP, IMAD with one warp per SM sub-partition and 8 independent chains.
#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
  uint64_t b[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 0.001f + i;
    b[i] = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i] + 1);
  }
  const uint64_t c2 = (uint64_t(__float_as_uint(0.999f)) << 32) | __float_as_uint(0.999f);
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fmaf(a[i], 0.999f, 0.001f);
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(b[i]) : "l"(c2));
      if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(c2));
      if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 4) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        a[i] = __uint_as_float(r);
      }
      if (OP == 5) {
        uint32_t r = __float_as_uint(a[i]);
        asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(r) : "r"(r));
        a[i] = __uint_as_float(r);
      }
      if (OP == 6) a[i] = fmaxf(a[i], -126.0f) + 0.f;
      if (OP == 7) {  // ex2.approx.f16x2 (SASS: MUFU.EX2.F16 per half?)
        uint32_t r = __float_as_uint(a[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r));
        a[i] = __uint_as_float(r);
      }
      if (OP == 8) {  // ex2.approx.f16 (scalar)
        unsigned short r = (unsigned short)__float_as_uint(a[i]);
        asm volatile("ex2.approx.f16 %0, %0;" : "+h"(r));
        a[i] = __uint_as_float(r);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(uint32_t(b[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaMalloc(&c, 8);
  const char* names[9] = {"FFMA", "FFMA2", "FADD2", "MUFU.EX2", "F2FP(cvt bf16x2)", "IMAD",
                          "FMNMX+FADD", "ex2.approx.f16x2", "ex2.approx.f16"};
  for (int w : {1, 2, 4})
    for (int op = 0; op < 9; ++op) {
      const int iters = 4096;
      auto launch = [&] {
        switch (op) {
          case 0: k<0><<<148, 128 * w>>>(o, iters, c); break;
          case 1: k<1><<<148, 128 * w>>>(o, iters, c); break;
          case 2: k<2><<<148, 128 * w>>>(o, iters, c); break;
          case 3: k<3><<<148, 128 * w>>>(o, iters, c); break;
          case 4: k<4><<<148, 128 * w>>>(o, iters, c); break;
          case 5: k<5><<<148, 128 * w>>>(o, iters, c); break;
          case 6: k<6><<<148, 128 * w>>>(o, iters, c); break;
          case 7: k<7><<<148, 128 * w>>>(o, iters, c); break;
          case 8: k<8><<<148, 128 * w>>>(o, iters, c); break;
        }
      };
      launch();
      launch();
      long long clk = 0;
      cudaMemcpy(&clk, c, 8, cudaMemcpyDeviceToHost);
      printf("%d warp/SMSP %-18s %6.2f clk per warp-instr per SMSP\n", w, names[op],
             double(clk) / (double(iters) * 8 * w));
    }
  return 0;
}
