// attention.cu -- K6 pieces: causal prefill attention over the paged KV cache,
// embedding gather and greedy argmax (RECOMPUTE complement, model.cpp:67-92,
// 237-288).
//
// Attention is a flash-attention-2 style kernel: 64 queries per CTA (16 per
// warp), 64-key tiles double-buffered in swizzled shared memory with
// cp.async (rows gathered through the page table), S = Q K^T and O = P V on
// bf16 tensor-core MMAs (m16n8k16, fp32 accumulate), online softmax in fp32
// with exp2. Causal blocks are scheduled heaviest first.
#include <cuda_bf16.h>

#include <cmath>

#include "kernels.h"

namespace hc {

namespace {

constexpr int kQ = 64;  // queries per CTA
constexpr int kK = 64;  // keys per tile
constexpr int kAttnThreads = 128;

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// row-major tile of DH bf16 per row, 16-byte chunks XOR-swizzled by row
template <int DH>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + uint32_t(row * DH * 2) + (uint32_t(chunk ^ (row & 7)) << 4);
}

// Prefill from position 0 (cu_q == nullptr: one sequence of n rows) or the
// batched continuation (cu_q != nullptr: blockIdx.z = sequence, its rows
// [cu_q[z], cu_q[z+1]) at positions seq_start[z] + i, page-table row z).
template <int DH>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ q, int n, int n_heads, int group, KvOut kv,
                    __nv_bfloat16* __restrict__ out, float scale_log2,
                    const int32_t* __restrict__ cu_q, const int32_t* __restrict__ seq_start) {
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = s_u32(smem);
  const uint32_t sK0 = sQ + kQ * DH * 2;
  const uint32_t sV0 = sK0 + 2 * kK * DH * 2;
  const int qb = int(gridDim.x) - 1 - int(blockIdx.x);  // heaviest causal blocks first
  const int h = blockIdx.y, hk = h / group;
  const int ld = n_heads * DH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = qb * kQ;
  int row0 = 0, p0 = 0;  // first query row of this sequence, its position
  const int32_t* table = kv.page_table;
  if (cu_q) {
    const int z = blockIdx.z;
    row0 = __ldg(cu_q + z);
    n = __ldg(cu_q + z + 1) - row0;
    p0 = __ldg(seq_start + z);
    if (table) table += int64_t(z) * kv.table_stride;
  }
  if (q0 >= n) return;
  const int n_keys = p0 + min(n, q0 + kQ);  // keys [0, n_keys) reach this query tile
  q += size_t(row0) * ld;
  out += size_t(row0) * ld;

  for (int i = tid; i < kQ * CH; i += kAttnThreads) {
    const int r = i / CH, c = i % CH, row = q0 + r;
    const bool ok = row < n;
    cp_async16(swz<DH>(sQ, r, c), q + size_t(ok ? row : 0) * ld + h * DH + c * 8, ok);
  }
  auto load_kv = [&](int kb, int st) {
    const uint32_t sk = sK0 + uint32_t(st * kK * DH * 2), sv = sV0 + uint32_t(st * kK * DH * 2);
    for (int i = tid; i < kK * CH; i += kAttnThreads) {
      const int r = i / CH, c = i % CH, key = kb * kK + r;
      const bool ok = key < n_keys;
      int64_t orow = ok ? key : 0;
      if (ok && table)
        orow = int64_t(__ldg(table + key / kv.page_size)) * kv.page_size + key % kv.page_size;
      const size_t off = size_t(orow) * kv.d_kv + size_t(hk) * DH + size_t(c) * 8;
      cp_async16(swz<DH>(sk, r, c), static_cast<const __nv_bfloat16*>(kv.k_base) + off, ok);
      cp_async16(swz<DH>(sv, r, c), static_cast<const __nv_bfloat16*>(kv.v_base) + off, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const int n_kb = (n_keys + kK - 1) / kK;  // causal: key tiles up to the diagonal
  float o[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qf[DH / 16][4];
  const int r_lo = q0 + warp * 16 + (lane >> 2);  // this thread's rows: r_lo, r_lo + 8

  for (int kb = 0; kb < n_kb; ++kb) {
    if (kb + 1 < n_kb) {
      load_kv(kb + 1, (kb + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk)
        ldsm_x4(swz<DH>(sQ, warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), 2 * kk + (lane >> 4)),
                qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    const uint32_t sk = sK0 + uint32_t((kb & 1) * kK * DH * 2);
    const uint32_t sv = sV0 + uint32_t((kb & 1) * kK * DH * 2);
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(swz<DH>(sk, 16 * np + (lane & 7) + 8 * (lane >> 4), 2 * kk + ((lane >> 3) & 1)),
                b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // scale, causal + length mask, online softmax (rows r_lo and r_lo + 8)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * kK + 8 * j + 2 * (lane & 3) + (e & 1);
        const int row = r_lo + 8 * (e >> 1);
        float v = s[j][e] * scale_log2;
        if (key > p0 + row || key >= n_keys) v = -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2], sum[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float m_new = fmaxf(m_run[r], mx[r]);
      corr[r] = exp2f(m_run[r] - m_new);
      m_run[r] = m_new;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(s[j][e] - m_run[e >> 1]);
        s[j][e] = p;
        sum[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], 1);
      sum[r] += __shfl_xor_sync(0xffffffffu, sum[r], 2);
      l_run[r] = l_run[r] * corr[r] + sum[r];
    }
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                             pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                             pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(swz<DH>(sv, 16 * kk + (lane & 7) + 8 * ((lane >> 3) & 1), 2 * dp + (lane >> 4)),
                  b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();  // the next iteration's prefetch overwrites this stage
  }
  const float inv[2] = {1.f / l_run[0], 1.f / l_run[1]};
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = r_lo + 8 * r;
    if (row >= n) continue;
    __nv_bfloat16* dst = out + size_t(row) * ld + h * DH + 2 * (lane & 3);
#pragma unroll
    for (int j = 0; j < DH / 8; ++j)
      *reinterpret_cast<uint32_t*>(dst + 8 * j) =
          pack2(o[j][2 * r] * inv[r], o[j][2 * r + 1] * inv[r]);
  }
}

__global__ void embed_kernel(const int32_t* __restrict__ tokens, int64_t n, const uint4* __restrict__ emb,
                             int d, float* __restrict__ x, uint4* __restrict__ xb) {
  const int vec = d / 8;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * vec;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / vec;
    const int c = int(i % vec);
    const uint4 u = __ldg(emb + int64_t(__ldg(tokens + row)) * vec + c);
    xb[i] = u;
    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&u);
    float4* x4 = reinterpret_cast<float4*>(x + i * 8);
    x4[0] = make_float4(__bfloat162float(hv[0]), __bfloat162float(hv[1]), __bfloat162float(hv[2]),
                        __bfloat162float(hv[3]));
    x4[1] = make_float4(__bfloat162float(hv[4]), __bfloat162float(hv[5]), __bfloat162float(hv[6]),
                        __bfloat162float(hv[7]));
  }
}

__global__ void argmax_logits_kernel(const __nv_bfloat16* __restrict__ emb, int vocab, int d,
                                     const float* __restrict__ h, unsigned long long* best) {
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= vocab) return;
  float acc = 0.f;
  for (int c = lane; c < d; c += 32) acc += __bfloat162float(emb[size_t(t) * d + c]) * h[c];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    // order-preserving float key; ties resolve to the smallest token id like
    // the reference's strict '>' scan (model.cpp:71-78)
    uint32_t u = __float_as_uint(acc);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    atomicMax(best, (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - uint32_t(t)));
  }
}

// blockIdx.y = sequence: logits of its last row (cu[s+1]-1)
__global__ void argmax_rows_kernel(const __nv_bfloat16* __restrict__ emb, int vocab, int d,
                                   const float* __restrict__ x, const int32_t* __restrict__ cu,
                                   unsigned long long* best) {
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= vocab) return;
  const int s = blockIdx.y;
  const float* h = x + size_t(__ldg(cu + s + 1) - 1) * d;
  float acc = 0.f;
  for (int c = lane; c < d; c += 32) acc += __bfloat162float(emb[size_t(t) * d + c]) * h[c];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    uint32_t u = __float_as_uint(acc);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    atomicMax(best + s, (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - uint32_t(t)));
  }
}

__global__ void argmax_rows_finish_kernel(const unsigned long long* best, int n, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int32_t(0xFFFFFFFFu - uint32_t(best[i] & 0xFFFFFFFFull));
}

__global__ void argmax_finish_kernel(const unsigned long long* best, int32_t* out) {
  *out = int32_t(0xFFFFFFFFu - uint32_t(*best & 0xFFFFFFFFull));
}

}  // namespace

namespace {

cudaError_t attention_launch(const void* q, int n, dim3 grid, const int32_t* cu_q,
                             const int32_t* seq_start, int n_heads, int n_kv_heads, int dh,
                             const KvOut& kv, void* out, cudaStream_t stream) {
  const float scale_log2 = (1.0f / sqrtf(float(dh))) * 1.4426950408889634f;
  const int group = n_heads / n_kv_heads;
  if (dh != 128 && dh != 64) return cudaErrorInvalidValue;
  const size_t sm = size_t(kQ + 4 * kK) * size_t(dh) * 2;
  auto kern = dh == 128 ? attn_fwd_kernel<128> : attn_fwd_kernel<64>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  if (e != cudaSuccess) return e;
  kern<<<grid, kAttnThreads, sm, stream>>>(static_cast<const __nv_bfloat16*>(q), n, n_heads,
                                           group, kv, static_cast<__nv_bfloat16*>(out),
                                           scale_log2, cu_q, seq_start);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(const void* q, int n, int n_heads, int n_kv_heads, int dh,
                             const KvOut& kv, void* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  return attention_launch(q, n, dim3((n + kQ - 1) / kQ, n_heads, 1), nullptr, nullptr, n_heads,
                          n_kv_heads, dh, kv, out, stream);
}

cudaError_t launch_attention_extend(const void* q, int n_seqs, int max_new, const int32_t* cu_q,
                                    const int32_t* seq_start, int n_heads, int n_kv_heads,
                                    int dh, const KvOut& kv, void* out, cudaStream_t stream) {
  if (n_seqs <= 0 || max_new <= 0) return cudaSuccess;
  if (!cu_q || !seq_start) return cudaErrorInvalidValue;
  return attention_launch(q, 0, dim3((max_new + kQ - 1) / kQ, n_heads, n_seqs), cu_q, seq_start,
                          n_heads, n_kv_heads, dh, kv, out, stream);
}

cudaError_t launch_embed(const int32_t* tokens, int64_t n, const void* emb, int d, float* x,
                         void* xb, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n * (d / 8) + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  embed_kernel<<<unsigned(blocks), 256, 0, stream>>>(tokens, n, static_cast<const uint4*>(emb), d,
                                                     x, static_cast<uint4*>(xb));
  return cudaGetLastError();
}

cudaError_t launch_argmax_logits(const void* emb, int vocab, int d, const float* h,
                                 int32_t* out_token, cudaStream_t stream) {
  unsigned long long* best = nullptr;
  cudaError_t e = cudaMallocAsync(&best, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(best, 0, sizeof(unsigned long long), stream);
  argmax_logits_kernel<<<unsigned((vocab + 7) / 8), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(emb), vocab, d, h, best);
  argmax_finish_kernel<<<1, 1, 0, stream>>>(best, out_token);
  cudaFreeAsync(best, stream);
  return cudaGetLastError();
}

cudaError_t launch_argmax_rows(const void* emb, int vocab, int d, const float* h,
                               const int32_t* cu, int n_seqs, int32_t* out_tokens,
                               cudaStream_t stream) {
  if (n_seqs <= 0) return cudaSuccess;
  unsigned long long* best = nullptr;
  cudaError_t e = cudaMallocAsync(&best, sizeof(unsigned long long) * size_t(n_seqs), stream);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(best, 0, sizeof(unsigned long long) * size_t(n_seqs), stream);
  argmax_rows_kernel<<<dim3(unsigned((vocab + 7) / 8), unsigned(n_seqs)), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(emb), vocab, d, h, cu, best);
  argmax_rows_finish_kernel<<<unsigned((n_seqs + 127) / 128), 128, 0, stream>>>(best, n_seqs,
                                                                               out_tokens);
  cudaFreeAsync(best, stream);
  return cudaGetLastError();
}

}  // namespace hc
