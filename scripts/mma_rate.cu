// tcgen05 MMA issue-rate probe: clocks per 128 x N x 16 MMA for the operand
// forms the attention kernel uses (SS K-major, SS with MN-major B, TS with A
// in TMEM), one CTA per SM, operands garbage (rate only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2410_05004_b200/csrc
//        scripts/mma_rate.cu -o build/mma_rate
#include <cstdio>

#include "sm100.cuh"

using namespace hc;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

__global__ void probe(int mode, int n, int iters, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {  // warp-uniform issue loop, one elected lane issues
    uint32_t id = umma_idesc_f16(128, n, true);
    if (mode == 1 || mode == 2) id |= 1u << 16;  // B MN-major
    const uint64_t da = umma_desc_sw128(smem_u32(sm));
    const uint64_t db = umma_desc_sw128(smem_u32(sm + 65536));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
      if (elect_one()) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (mode == 2)
            umma_ts(tmem + 256, tmem + uint32_t(u * 8), db, id, 1);
          else
            umma_f16(tmem + uint32_t((u % nacc) * (512 / nacc)), da + uint64_t(u & 3) * 2, db + uint64_t(u & 3) * 2, id, 1);
        }
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[3] = {"SS K-major", "SS B MN-major", "TS (A in TMEM)"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {64, 128, 256}) {
      if (mode == 2 && n > 256) continue;
      for (int nacc = 1; nacc <= 512 / n; nacc *= 2) {
        if (mode == 2 && nacc > 1) break;
        const int iters = 4096;
        probe<<<148, 128, 200 * 1024>>>(mode, n, iters, nacc, d);
        probe<<<148, 128, 200 * 1024>>>(mode, n, iters, nacc, d);
        unsigned long long c = 0;
        cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-16s N=%3d acc=%d: %6.1f clk/MMA  -> %6.0f FLOP/clk/SM (%s)\n", names[mode], n,
               nacc, double(c) / iters, 2.0 * 128 * n * 16 * iters / double(c), cudaGetErrorString(e));
      }
    }
  return 0;
}
