// peer.cu -- the head-sharded restore's all-gather fused into K1 over peer
// memory (SURVEY 8e on B200 terms).
//
// Each rank holds only its own token range of a layer's hidden states (fetched
// over its own PCIe link). Instead of all-gathering the ranges into a full
// n x d copy on every GPU (NCCL, the baseline), every rank's K1 reads the A
// tiles of each range straight from the owning rank's buffer -- mapped into
// this process with CUDA IPC, reached over NVLink -- so the transfer overlaps
// the MMAs tile by tile and no gathered copy is ever written. Row statistics
// for the LayerNorm fold read the ranges the same way.
//
// Cross-GPU ordering uses flags in device memory: an owner announces a filled
// staging slot by storing an epoch into every consumer's flag array
// (system-scope release stores over NVLink), a consumer announces it is done
// with a slot the same way; each side waits only on its own memory
// (cuStreamWaitValue32, or a one-thread polling kernel where stream memory
// operations are unavailable).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "common.h"
#include "kernels.h"
#include "weights.h"

namespace hc {

CUtensorMap weight_map(const hc_weights::Layer& L, int bn, int d, int rows);
KvOut kv_out_pages(const hc_kv_pages* pages, int layer, const int32_t* page_table,
                   int table_stride, const int32_t* cu_seqlens, int n_seqs);
void validate_pages(const hc_weights* w, const hc_kv_pages* pages, int d_kv_expected);

namespace {

__global__ void signal_kernel(uint32_t* const* addrs, int n, uint32_t value) {
  __threadfence_system();  // everything this stream did before is visible first
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    asm volatile("st.global.release.sys.u32 [%0], %1;" ::"l"(addrs[i]), "r"(value) : "memory");
}

__global__ void wait_kernel(const uint32_t* addr, uint32_t value) {
  uint32_t v = 0;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.global.acquire.sys.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
    if (v >= value) break;
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60000000000ull) asm volatile("trap;");  // watchdog: a peer gone for 60 s
  }
}

__global__ void append_rows_kernel(const uint4* __restrict__ step, int rows_in_step, int h0, int d,
                                   const AppendDst* __restrict__ dsts) {
  const int b = blockIdx.x, l = blockIdx.y;
  const int vec = d / 8;
  const uint4* src = step + (size_t(h0 + l) * rows_in_step + b) * vec;
  uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(dsts[b].dst) + size_t(l) * dsts[b].pitch);
  for (int i = threadIdx.x; i < vec; i += blockDim.x) dst[i] = __ldg(src + i);
}

__global__ void convert_f32_kernel(const float4* __restrict__ src, uint2* __restrict__ dst,
                                   int64_t n4) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = __ldg(src + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    dst[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

__global__ void convert_f16_kernel(const uint2* src, uint2* dst, int64_t n4) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint2 u = src[i];
    const __half2 h0 = *reinterpret_cast<const __half2*>(&u.x);
    const __half2 h1 = *reinterpret_cast<const __half2*>(&u.y);
    const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
    __nv_bfloat162 a = __floats2bfloat162_rn(f0.x, f0.y), b = __floats2bfloat162_rn(f1.x, f1.y);
    dst[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

// LayerNorm statistics of a head-sharded layer: every owner computed the
// mean/rstd of its own token range into its staging slot; a consumer copies
// them (8 B per row, over NVLink) into one contiguous array for K1's
// epilogue instead of re-reading the owners' rows.
__global__ void gather_stats_kernel(StatSources src, float* __restrict__ mean,
                                    float* __restrict__ rstd) {
  const int s = blockIdx.y;
  if (s >= src.n) return;
  const int64_t b = src.row0[s], rows = src.row0[s + 1] - b;
  const float* m = src.mean[s];
  const float* r = src.rstd[s];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += int64_t(gridDim.x) * blockDim.x) {
    mean[b + i] = m[i];
    rstd[b + i] = r[i];
  }
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitFn wait_value_fn() {
  static WaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitFn>(p);
  });
  return fn;
}

}  // namespace

cudaError_t launch_convert_to_bf16(const void* src, int src_dtype, void* dst, int64_t n,
                                   cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n % 4) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const unsigned grid = unsigned(std::min<int64_t>((n4 + 255) / 256, 148 * 16));
  if (src_dtype == HC_DTYPE_F32)
    convert_f32_kernel<<<grid, 256, 0, stream>>>(static_cast<const float4*>(src),
                                                 static_cast<uint2*>(dst), n4);
  else if (src_dtype == HC_DTYPE_F16)
    convert_f16_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint2*>(src),
                                                 static_cast<uint2*>(dst), n4);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_signal_flags(uint32_t* const* d_flag_ptrs, int n, uint32_t value,
                                cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  signal_kernel<<<1, 32, 0, stream>>>(d_flag_ptrs, n, value);
  return cudaGetLastError();
}

cudaError_t launch_gather_stats(const StatSources& src, int64_t max_rows, float* mean, float* rstd,
                                cudaStream_t stream) {
  if (src.n <= 0 || max_rows <= 0) return cudaSuccess;
  const unsigned gx = unsigned(std::min<int64_t>((max_rows + 255) / 256, 64));
  gather_stats_kernel<<<dim3(gx, unsigned(src.n)), 256, 0, stream>>>(src, mean, rstd);
  return cudaGetLastError();
}

cudaError_t wait_flag_geq(cudaStream_t stream, const uint32_t* d_flag, uint32_t value) {
  static const bool use_kernel = getenv("HC_WAIT_KERNEL") != nullptr;
  WaitFn fn = use_kernel ? nullptr : wait_value_fn();
  if (fn && fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(d_flag), value,
               CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS)
    return cudaSuccess;
  wait_kernel<<<1, 1, 0, stream>>>(d_flag, value);
  return cudaGetLastError();
}

cudaError_t launch_append_rows(const void* step_rows, int rows_in_step, int h0, int nh, int d,
                               const AppendDst* d_dsts, int n_rows, cudaStream_t stream) {
  if (n_rows <= 0 || nh <= 0) return cudaSuccess;
  if (d % 8) return cudaErrorInvalidValue;
  append_rows_kernel<<<dim3(unsigned(n_rows), unsigned(nh)), 128, 0, stream>>>(
      static_cast<const uint4*>(step_rows), rows_in_step, h0, d, d_dsts);
  return cudaGetLastError();
}

}  // namespace hc

using namespace hc;

extern "C" {

hc_status hc_stream_wait_flag(void* stream, const uint32_t* d_flag, uint32_t value) {
  return guard([&] {
    if (!d_flag) fail(HC_EINVAL, "wait_flag: null flag");
    HC_CUDA(wait_flag_geq(as_stream(stream), d_flag, value));
  });
}

hc_status hc_stream_signal_flags(void* stream, uint32_t* const* d_flag_ptrs, int32_t n,
                                 uint32_t value) {
  return guard([&] {
    if (n < 0 || n > 64 || (n > 0 && !d_flag_ptrs)) fail(HC_EINVAL, "signal_flags: bad argument");
    if (n == 0) return;
    cudaStream_t s = as_stream(stream);
    StreamScratch ptrs(sizeof(uint32_t*) * size_t(n), s);
    HC_CUDA(cudaMemcpyAsync(ptrs.ptr, d_flag_ptrs, sizeof(uint32_t*) * size_t(n),
                            cudaMemcpyHostToDevice, s));
    signal_kernel<<<1, 32, 0, s>>>(static_cast<uint32_t* const*>(ptrs.ptr), n, value);
    HC_CUDA(cudaGetLastError());
  });
}

hc_status hc_project_multi_source(const hc_weights* w, int32_t layer, int32_t n_src,
                                  const void* const* d_src, const int64_t* row_begin,
                                  const hc_kv_pages* pages, const int32_t* d_page_table,
                                  int32_t start_pos, void* stream) {
  return guard([&] {
    if (!w || !d_src || !row_begin || !d_page_table) fail(HC_EINVAL, "project_multi: null argument");
    if (n_src < 1 || n_src > kMaxASrc) fail(HC_EINVAL, "project_multi: 1..8 sources");
    if (layer < 0 || layer >= w->cfg.n_layers) fail(HC_EINVAL, "project: layer out of range");
    const auto& L = w->layers[size_t(layer)];
    if (!L.ready) fail(HC_EINVAL, "project: layer weights not set");
    validate_pages(w, pages, w->d_kv);
    if (row_begin[0] != 0) fail(HC_EINVAL, "project_multi: row_begin[0] must be 0");
    for (int s = 0; s < n_src; ++s) {
      if (row_begin[s + 1] < row_begin[s]) fail(HC_EINVAL, "project_multi: ranges must ascend");
      if (row_begin[s + 1] < row_begin[n_src] && row_begin[s + 1] % 128)
        fail(HC_EINVAL, "project_multi: source boundaries must be multiples of 128 rows");
      if (row_begin[s + 1] > row_begin[s] && !d_src[s]) fail(HC_EINVAL, "project_multi: null source");
    }
    const int64_t n = row_begin[n_src];
    if (n <= 0) return;
    if (w->cfg.rope_enabled && int64_t(start_pos) + n > w->rope_rows)
      fail(HC_EINVAL, "project: positions exceed max_seq");
    DeviceGuard dg(w->device);
    cudaStream_t s = as_stream(stream);
    const int d = w->cfg.d_hidden, N = 2 * w->d_kv;
    const bool norm = w->cfg.norm_enabled != 0;
    const bool center = norm && ln_center_enabled();
    StreamScratch stats(size_t(n) * 2 * sizeof(float) + 16, s);
    float* mean = static_cast<float*>(stats.ptr);
    float* rstd = mean + n;
    int32_t* flag = reinterpret_cast<int32_t*>(rstd + n);
    // the LayerNorm fold's guard for rows with |mean| >> sigma, as in the
    // single-GPU path: the statistics raise one flag for the matrix, and the
    // mean-shifted rows of every source are written into a local copy that K1
    // reads instead (the sources are other GPUs' buffers: never written here;
    // the copy is only touched when the flag is set)
    StreamScratch centered(center ? size_t(n) * size_t(d) * 2 : 0, s);
    if (center) HC_CUDA(launch_zero_i32(flag, 1, s));
    AMaps am;
    am.n = 0;
    const uint32_t abox = uint32_t(gemm_a_box(n));
    for (int i = 0; i < n_src; ++i) {
      const int64_t rows = row_begin[i + 1] - row_begin[i];
      if (rows == 0) continue;  // empty range (more ranks than row blocks)
      if (center)
        HC_CUDA(launch_row_stats_flagged(d_src[i], rows, d, d, true, mean + row_begin[i],
                                         rstd + row_begin[i], flag, s));
      else if (norm)
        HC_CUDA(launch_row_stats(d_src[i], rows, d, d, true, mean + row_begin[i],
                                 rstd + row_begin[i], s));
      if (!make_tmap_kmajor(&am.m[am.n], d_src[i], uint64_t(d), uint64_t(rows), uint64_t(d) * 2,
                            abox))
        fail(HC_ECUDA, "cuTensorMapEncodeTiled failed for a peer range");
      am.row0[am.n] = int(row_begin[i]);
      ++am.n;
    }
    am.row0[am.n] = 0x7fffffff;
    if (center) {
      // (after every statistics launch: the flag is final)
      for (int i = 0; i < n_src; ++i) {
        const int64_t rows = row_begin[i + 1] - row_begin[i];
        if (rows == 0) continue;
        HC_CUDA(launch_center_rows(d_src[i], rows, d, d, mean + row_begin[i], flag,
                                   static_cast<char*>(centered.ptr) + size_t(row_begin[i]) * d * 2,
                                   s));
      }
      if (!make_tmap_kmajor(&am.m[am.n], centered.ptr, uint64_t(d), uint64_t(n), uint64_t(d) * 2,
                            abox))
        fail(HC_ECUDA, "cuTensorMapEncodeTiled failed (centered rows)");
      am.alt_flag = flag;
    }
    const int sms = device_sm_count(w->device);
    const int bn = gemm_pick_bn(n, N, sms);
    KvOut out = kv_out_pages(pages, layer, d_page_table, 0, nullptr, 1);
    out.start_pos = start_pos;
    HC_CUDA(launch_restore_kv_multi(am, weight_map(L, bn, d, N), bn, int(n), N, d, true, out,
                                    epi_for(w, L.colsum, norm ? mean : nullptr,
                                            norm ? rstd : nullptr),
                                    sms, s));
  });
}

}  // extern "C"
