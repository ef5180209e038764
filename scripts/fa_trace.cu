// Pipeline trace of the two-Q-tile attention kernel: SM clocks of the MMA
// issues and softmax hand-offs of one CTA (n=4096, 32 heads, dense).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -DHC_FA_TRACE -Ipaper_2410_05004_b200/csrc scripts/fa_trace.cu
//        paper_2410_05004_b200/csrc/tma.cpp -o gpurun_out/fa_trace
#include "../paper_2410_05004_b200/csrc/attention_tc.cu"

#include <cstdio>
#include <algorithm>
#include <vector>

namespace hc {
bool pdl_enabled() { return false; }  // (defined in k1_restore_kv.cu in the library)
}

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
  const int n_ctas = ((n + 255) / 256) * heads;
  unsigned long long* h_cta = nullptr;
  cudaHostAlloc(&h_cta, sizeof(unsigned long long) * 4 * n_ctas, cudaHostAllocMapped);
  memset(h_cta, 0, sizeof(unsigned long long) * 4 * n_ctas);
  unsigned long long* d_cta = nullptr;
  cudaHostGetDevicePointer(&d_cta, h_cta, 0);
  cudaMemcpyToSymbol(hc::g_fa_cta, &d_cta, sizeof(d_cta));
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
  // per-CTA spans of the last launch: duration = a + b * steps (least squares),
  // SM occupancy = sum of CTA spans / (SMs x kernel span)
  unsigned long long t_lo = ~0ull, t_hi = 0;
  double sx = 0, sy = 0, sxx = 0, sxy = 0, busy = 0;
  int sm_max = 0;
  for (int c = 0; c < n_ctas; ++c) {
    const unsigned long long* r = h_cta + 4 * c;
    t_lo = std::min(t_lo, r[0]);
    t_hi = std::max(t_hi, r[1]);
    const double d = double(r[1] - r[0]), x = double(r[3]);
    sx += x; sy += d; sxx += x * x; sxy += x * d; busy += d;
    sm_max = std::max(sm_max, int(r[2]));
  }
  const double b = (n_ctas * sxy - sx * sy) / (n_ctas * sxx - sx * sx), a = (sy - b * sx) / n_ctas;
  printf("kernel span %.1f us; CTA span = %.2f us + %.3f us/step; SM busy %.1f %%\n",
         (t_hi - t_lo) * 1e-3, a * 1e-3, b * 1e-3, 100.0 * busy / ((sm_max + 1) * double(t_hi - t_lo)));
  for (int c = 0; c < n_ctas; c += n_ctas / 16) {
    const unsigned long long* r = h_cta + 4 * c;
    printf("cta %3d sm %3llu steps %2llu start %7.1f end %7.1f us\n", c, r[2], r[3],
           (r[0] - t_lo) * 1e-3, (r[1] - t_lo) * 1e-3);
  }
  return 0;
}
