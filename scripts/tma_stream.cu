// Weight-streaming microbenchmark: how fast can one CTA per SM pull a
// row-major [N x 4096] bf16 matrix through a TMA ring (no MMA), as a
// function of the box shape (rows x 64 columns) and of how many consecutive
// K boxes one stage covers (the decode GEMMs stream weights like this).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -Ipaper_2410_05004_b200/csrc scripts/tma_stream.cu
//        paper_2410_05004_b200/csrc/tma.cpp -lcuda -o /tmp/tma_stream
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"

using namespace hc;

constexpr int kK = 4096;

__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap tm, int n_rows, int box_rows, int bps,
                  int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t stage_bytes = uint32_t(box_rows) * 128u * uint32_t(bps);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(stages) * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int groups = n_rows / box_rows;
  const int kb_per_group = kK / 64 / bps;
  if (warp == 0 && lane == 0) {
    int it = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x)
      for (int kb = 0; kb < kb_per_group; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        for (int b = 0; b < bps; ++b)
          tma_load_2d(smem + size_t(s) * stage_bytes + size_t(b) * box_rows * 128, &tm, &full[s],
                      (kb * bps + b) * 64, g * box_rows);
      }
  } else if (warp == 1 && lane == 0) {
    int it = 0;
    unsigned long long acc = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x)
      for (int kb = 0; kb < kb_per_group; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        acc += smem[size_t(s) * stage_bytes + (it & 127)];
        mbar_arrive(&empty[s]);
      }
    if (acc == 0x12345) *sink = acc;
  }
}

int main(int argc, char** argv) {
  const int n_rows = 131072;  // 1 GiB: far beyond L2
  const size_t bytes = size_t(n_rows) * kK * 2;
  void* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct V {
    int box_rows, bps, ring_kb, ctas_per_sm;
  } vs[] = {{64, 1, 200, 1}, {64, 2, 200, 1}, {64, 4, 200, 1}, {64, 8, 200, 1},
            {128, 1, 200, 1}, {128, 2, 200, 1}, {128, 4, 192, 1}, {256, 1, 192, 1},
            {32, 4, 200, 1}, {16, 8, 200, 1}, {64, 1, 96, 2}, {64, 4, 96, 2},
            {64, 1, 64, 1}, {64, 4, 64, 1}, {64, 4, 128, 1}};
  printf("box_rows bps ring_kb ctas/sm  GB/s\n");
  for (const V& v : vs) {
    CUtensorMap tm;
    if (!make_tmap_kmajor(&tm, w, kK, n_rows, kK * 2, uint32_t(v.box_rows))) {
      printf("tmap fail\n");
      return 1;
    }
    const uint32_t stage_bytes = uint32_t(v.box_rows) * 128u * uint32_t(v.bps);
    const int stages = int(size_t(v.ring_kb) * 1024 / stage_bytes);
    if (stages < 2) continue;
    const size_t smem = size_t(stages) * stage_bytes + 16 * size_t(stages) + 64;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = sms * v.ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i)
      stream_kernel<<<grid, 64, smem>>>(tm, n_rows, v.box_rows, v.bps, stages, sink);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; ++i)
      stream_kernel<<<grid, 64, smem>>>(tm, n_rows, v.box_rows, v.bps, stages, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%8d %3d %7d %7d  %7.1f  %s (stages %d)\n", v.box_rows, v.bps, v.ring_kb,
           v.ctas_per_sm, bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(e), stages);
  }
  return 0;
}
