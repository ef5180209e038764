// Per-CTA timeline of the CTA-pair GEMM (one 4096-token N=4096 projection):
// globaltimer stamps of every unit's MMA issue and epilogue, SM busy fraction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -DHC_PAIR_TRACE -Ipaper_2410_05004_b200/csrc scripts/pair_trace.cu
//        paper_2410_05004_b200/csrc/tma.cpp -lcuda -o gpurun_out/pair_trace
//   gpurun_out/pair_trace [M N K [tail 0|1 [mode 0 KV+RoPE | 1 RESID | 2 GELU]]]
#include "../paper_2410_05004_b200/csrc/k1_restore_kv.cu"

#include <algorithm>
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 4096, N = argc > 2 ? atoi(argv[2]) : 4096,
            K = argc > 3 ? atoi(argv[3]) : 4096;
  const bool split = argc > 4 ? atoi(argv[4]) != 0 : true;
  const int mode = argc > 5 ? atoi(argv[5]) : hc::kEpiResid;
  void *a, *b, *xb;
  float* x;
  cudaMalloc(&a, size_t(M) * K * 2);
  cudaMalloc(&b, size_t(N) * K * 2);
  cudaMalloc(&xb, size_t(M) * N * 2);
  cudaMalloc(&x, size_t(M) * N * 4);
  cudaMemset(a, 0x3c, size_t(M) * K * 2);
  cudaMemset(b, 0x3c, size_t(N) * K * 2);
  cudaMemset(x, 0, size_t(M) * N * 4);
  CUtensorMap ta, tb;
  hc::make_tmap_kmajor(&ta, a, K, M, uint64_t(K) * 2, 128);
  hc::make_tmap_kmajor(&tb, b, K, N, uint64_t(K) * 2, 128);
  hc::GemmOut g;
  g.x = x;
  g.xb = xb;
  g.ldo = N;
  const int ctas = 148, slots = hc::kPairTraceSlots;
  unsigned long long *h_tr = nullptr, *d_tr = nullptr;
  cudaHostAlloc(&h_tr, sizeof(unsigned long long) * ctas * slots, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&d_tr, h_tr, 0);
  // KV mode: dense K/V rows (N/2 each), LN fold, RoPE on the K half
  void *kout, *vout, *rope;
  float *stats, *colsum;
  cudaMalloc(&kout, size_t(M) * N);
  cudaMalloc(&vout, size_t(M) * N);
  cudaMalloc(&rope, size_t(M) * 64 * 8);
  cudaMalloc(&stats, size_t(M) * 8);
  cudaMalloc(&colsum, size_t(N) * 4);
  cudaMemset(rope, 0, size_t(M) * 64 * 8);
  cudaMemset(stats, 0, size_t(M) * 8);
  cudaMemset(colsum, 0, size_t(N) * 4);
  hc::KvOut kv;
  kv.k_base = kout;
  kv.v_base = vout;
  kv.d_kv = N / 2;
  hc::EpiArgs epi;
  if (mode != hc::kEpiResid) {
    epi.row_mean = stats;
    epi.row_rstd = stats + M;
    epi.colsum = colsum;
  }
  if (mode == hc::kEpiKv) {
    epi.rope = static_cast<const float2*>(rope);
    epi.d_head = 128;
    epi.rope_rows = M;
  }
  auto run = [&] {
    if (mode == hc::kEpiKv)
      return hc::launch_restore_kv(ta, tb, 128, M, N, K, true, kv, epi, 148, 0, split);
    return hc::launch_gemm_dense(ta, tb, 128, mode, M, N, K, g, epi, 148, 0, split);
  };
  for (int i = 0; i < 20; ++i) run();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 50;
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  memset(h_tr, 0, sizeof(unsigned long long) * ctas * slots);
  cudaMemcpyToSymbol(hc::g_pair_trace, &d_tr, sizeof(d_tr));
  for (int i = 0; i < 3; ++i) run();  // traced (last one kept), back to back
  cudaError_t err = cudaDeviceSynchronize();
  printf("mode %d M=%d N=%d K=%d tail_split=%d: %s, %.1f us/launch (untraced, %d reps)\n", mode, M, N, K,
         int(split), cudaGetErrorString(err), ms * 1e3 / reps, reps);
  (void)mode;
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int c = 0; c < ctas; ++c) {
    t0 = std::min(t0, h_tr[c * slots + 0]);
    t1 = std::max(t1, h_tr[c * slots + 1]);
  }
  double mma_ns = 0, epi_ns = 0;
  for (int c = 0; c < ctas; c += 2) {  // leader CTAs (MMA issue stamps)
    const unsigned long long* r = h_tr + size_t(c) * slots;
    printf("cta %3d start %6.1f end %6.1f |", c, (r[0] - t0) * 1e-3, (r[1] - t0) * 1e-3);
    for (int u = 0; u < 9; ++u) {
      const unsigned long long* q = r + 2 + 4 * u;
      if (!q[0] && !q[2]) continue;
      printf(" u%d mma %6.1f-%6.1f epi %6.1f-%6.1f |", u, (q[0] - t0) * 1e-3, (q[1] - t0) * 1e-3,
             (q[2] - t0) * 1e-3, (q[3] - t0) * 1e-3);
      if (q[1] > q[0]) mma_ns += double(q[1] - q[0]);
      if (q[3] > q[2]) epi_ns += double(q[3] - q[2]);
    }
    printf("\n");
  }
  printf("kernel span %.1f us; mean per leader CTA: MMA issue %.1f us, epilogue %.1f us\n",
         (t1 - t0) * 1e-3, mma_ns * 1e-3 / (ctas / 2), epi_ns * 1e-3 / (ctas / 2));
  return 0;
}
