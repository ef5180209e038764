// Pipeline trace of the two-Q-tile attention kernel: SM clocks of the MMA
// issues and softmax hand-offs of one CTA (n=4096, 32 heads, dense).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -DHC_FA_TRACE -Ipaper_2410_05004_b200/csrc scripts/fa_trace.cu
//        paper_2410_05004_b200/csrc/tma.cpp -o gpurun_out/fa_trace
#include "../paper_2410_05004_b200/csrc/attention_tc.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096, heads = 32, dh = 128;
  const size_t sz = size_t(n) * heads * dh * 2;
  void *q, *k, *v, *o;
  cudaMalloc(&q, sz);
  cudaMalloc(&k, sz);
  cudaMalloc(&v, sz);
  cudaMalloc(&o, sz);
  std::vector<uint16_t> h(sz / 2);
  uint64_t x = 1;
  for (auto& e : h) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const float f = float(int((x >> 33) & 0xFFFF) - 32768) / 32768.0f;
    uint32_t b;
    memcpy(&b, &f, 4);
    e = uint16_t(b >> 16);
  }
  cudaMemcpy(q, h.data(), sz, cudaMemcpyHostToDevice);
  cudaMemcpy(k, h.data(), sz, cudaMemcpyHostToDevice);
  cudaMemcpy(v, h.data(), sz, cudaMemcpyHostToDevice);
  hc::KvOut kv;
  kv.k_base = k;
  kv.v_base = v;
  kv.d_kv = heads * dh;
  unsigned long long* h_tr = nullptr;
  cudaHostAlloc(&h_tr, sizeof(unsigned long long) * 10 * 2 * 64, cudaHostAllocMapped);
  memset(h_tr, 0, sizeof(unsigned long long) * 10 * 2 * 64);
  unsigned long long* d_tr = nullptr;
  cudaHostGetDevicePointer(&d_tr, h_tr, 0);
  cudaMemcpyToSymbol(hc::g_fa_trace, &d_tr, sizeof(d_tr));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = argc > 3 ? atoi(argv[3]) : 10;
  for (int i = 0; i < (reps > 1 ? 3 : 0); ++i) hc::launch_attention_tc(q, n, heads, heads, dh, kv, n, o, 0);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) hc::launch_attention_tc(q, n, heads, heads, dh, kv, n, o, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("status %s, %.1f us/launch\n", cudaGetErrorString(err), ms * 1e3 / reps);
  unsigned long long(&tr)[10][2][64] = *reinterpret_cast<unsigned long long(*)[10][2][64]>(h_tr);
  const unsigned long long t0 = tr[4][0][0];
  const char* names[10] = {"QKi", "PVi", "S", "P", "QKw", "PVw", "Sld", "max", "exp", "st"};
  const int nt = argc > 2 ? atoi(argv[2]) : (n + 127) / 128;
  for (int j = 0; j < nt; ++j)
    for (int t = 0; t < 2; ++t) {
      printf("j=%2d t=%d", j, t);
      for (int ev = 0; ev < 10; ++ev) printf(" %s %6lld", names[ev], (long long)(tr[ev][t][j] - t0));
      printf("\n");
    }
  return 0;
}
