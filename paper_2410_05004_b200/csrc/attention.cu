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

#include <algorithm>
#include <cstdlib>

#include <algorithm>
#include <cmath>

#include "kernels.h"
#include "sm100.cuh"

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

// ---------------------------------------------------------------- decode
// One query row per sequence (decode_step, model.cpp:332-347): split-KV
// flash-decoding on the CUDA cores -- the step is HBM-bound on the K/V pages,
// so every SM streams a slice of one sequence's keys for one KV head.
// grid (n_kv_heads, n_seqs, n_splits), 128 threads: DH/8 lanes share a key
// (16 B of K and V each), 4 keys per warp-pass x 4 in flight per lane group.
// Each (warp, lane-group) keeps an online-softmax state; the CTA merges them
// and writes this split's (max, sum, acc) for the combine kernel.
constexpr int kDecThreads = 128;

template <int DH>
__global__ void __launch_bounds__(kDecThreads)
    attn_decode_kernel(const __nv_bfloat16* __restrict__ q, int n_heads, int group, KvOut kv,
                       const int32_t* __restrict__ cu_q, const int32_t* __restrict__ seq_start,
                       int n_splits, float scale_log2, float* __restrict__ part) {
  pdl_wait();  // Q / K / V of this step (programmatic dependent launch)
  pdl_trigger();
  constexpr int LPK = DH / 8;            // lanes per key
  constexpr int KPW = 32 / LPK;          // keys per warp pass
  constexpr int KPB = KPW * (kDecThreads / 32);  // keys per block pass
  constexpr int UNROLL = 4;
  const int hk = blockIdx.x, z = blockIdx.y, split = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane / LPK, li = lane % LPK;  // key slot in the warp, lane in the key
  const int row = __ldg(cu_q + z);
  const int n_keys = __ldg(seq_start + z) + 1;
  const int per = (n_keys + n_splits - 1) / n_splits;
  const int k_begin = split * per, k_end = min(n_keys, k_begin + per);
  const int32_t* table = kv.page_table ? kv.page_table + int64_t(z) * kv.table_stride : nullptr;
  const int ld = n_heads * DH;
  __shared__ float red_m[kDecThreads / LPK], red_l[kDecThreads / LPK];
  __shared__ float red_acc[kDecThreads / LPK][DH];

  for (int g = 0; g < group; ++g) {
    const int h = hk * group + g;
    float qf[8];
    {
      const uint4 u = *reinterpret_cast<const uint4*>(q + size_t(row) * ld + h * DH + li * 8);
      const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) qf[e] = __bfloat162float(hv[e]) * scale_log2;
    }
    float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    // warp-uniform trip count: the key-group shuffles below need every lane
    for (int k0 = k_begin + warp * KPW; k0 < k_end; k0 += KPB * UNROLL) {
      uint4 kr[UNROLL], vr[UNROLL];
      bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int key = k0 + sub + u * KPB;
        ok[u] = key < k_end;
        int64_t orow = key;
        if (ok[u] && table)
          orow = int64_t(__ldg(table + key / kv.page_size)) * kv.page_size + key % kv.page_size;
        const size_t off = size_t(ok[u] ? orow : 0) * kv.d_kv + size_t(hk) * DH + size_t(li) * 8;
        kr[u] = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(kv.k_base) + off));
        vr[u] = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(kv.v_base) + off));
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const __nv_bfloat16* kh = reinterpret_cast<const __nv_bfloat16*>(&kr[u]);
        float sc = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) sc += qf[e] * __bfloat162float(kh[e]);
#pragma unroll
        for (int o = LPK / 2; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
        if (!ok[u]) continue;  // uniform across the key's lanes
        const float m_new = fmaxf(m, sc);
        const float corr = exp2f(m - m_new), p = exp2f(sc - m_new);
        const __nv_bfloat16* vh = reinterpret_cast<const __nv_bfloat16*>(&vr[u]);
        l = l * corr + p;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = acc[e] * corr + p * __bfloat162float(vh[e]);
        m = m_new;
      }
    }
    // merge the kDecThreads / LPK key-slot states of the block
    const int slot = tid / LPK;
    if (li == 0) {
      red_m[slot] = m;
      red_l[slot] = l;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red_acc[slot][li * 8 + e] = acc[e];
    __syncthreads();
    if (tid < DH) {
      float M = -INFINITY;
      for (int s2 = 0; s2 < kDecThreads / LPK; ++s2) M = fmaxf(M, red_m[s2]);
      float L = 0.f, A = 0.f;
      for (int s2 = 0; s2 < kDecThreads / LPK; ++s2) {
        const float c = red_m[s2] == -INFINITY ? 0.f : exp2f(red_m[s2] - M);
        L += red_l[s2] * c;
        A += red_acc[s2][tid] * c;
      }
      float* dst = part + ((size_t(z) * n_heads + h) * n_splits + split) * (DH + 2);
      dst[2 + tid] = A;
      if (tid == 0) {
        dst[0] = M;
        dst[1] = L;
      }
    }
    __syncthreads();
  }
}

// out[row(z), h] = sum_s acc_s * 2^(m_s - M) / sum_s l_s * 2^(m_s - M)
template <int DH>
__global__ void attn_decode_combine_kernel(const float* __restrict__ part, int n_heads,
                                           int n_splits, const int32_t* __restrict__ cu_q,
                                           __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int h = blockIdx.x, z = blockIdx.y, t = threadIdx.x;
  const float* base = part + (size_t(z) * n_heads + h) * n_splits * (DH + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, base[s * (DH + 2)]);
  float L = 0.f, A = 0.f;
  for (int s = 0; s < n_splits; ++s) {
    const float* p = base + s * (DH + 2);
    const float c = p[0] == -INFINITY ? 0.f : exp2f(p[0] - M);
    L += p[1] * c;
    A += p[2 + t] * c;
  }
  out[size_t(__ldg(cu_q + z)) * n_heads * DH + h * DH + t] = __float2bfloat16(A / L);
}

__global__ void embed_kernel(const int32_t* __restrict__ tokens, int64_t n, const uint4* __restrict__ emb,
                             int d, float* __restrict__ x, uint4* __restrict__ xb) {
  pdl_wait();
  pdl_trigger();
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

// Greedy tokens of up to kArgSeqs sequences per block (blockIdx.y = group of
// sequences): their last rows (fp32) are staged in shared memory, then each
// warp scores vocabulary rows, reading every embedding row ONCE per group.
constexpr int kArgSeqs = 8;

__global__ void argmax_rows_kernel(const __nv_bfloat16* __restrict__ emb, int vocab, int d,
                                   const float* __restrict__ x, const int32_t* __restrict__ cu,
                                   int n_seqs, int per_block, unsigned long long* best) {
  extern __shared__ float hs[];  // [per_block][d]
  const int s0 = blockIdx.y * per_block, ns = min(per_block, n_seqs - s0);
  for (int i = threadIdx.x; i < ns * d; i += blockDim.x) {
    const int s = i / d, c = i % d;
    hs[i] = x[size_t(__ldg(cu + s0 + s + 1) - 1) * d + c];
  }
  __syncthreads();
  // each warp scores kRows vocabulary rows at a time, so every h element read
  // from shared memory feeds kRows FMAs
  constexpr int kRows = 4;
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int t0 = (blockIdx.x * warps + (threadIdx.x >> 5)) * kRows; t0 < vocab;
       t0 += gridDim.x * warps * kRows) {
    float acc[kRows][kArgSeqs];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
#pragma unroll
      for (int s = 0; s < kArgSeqs; ++s) acc[r][s] = 0.f;
    for (int c8 = lane; c8 < d / 8; c8 += 32) {
      float ev[kRows][8];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int t = min(t0 + r, vocab - 1);
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(emb + size_t(t) * d) + c8);
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int e = 0; e < 8; ++e) ev[r][e] = __bfloat162float(hv[e]);
      }
#pragma unroll
      for (int s = 0; s < kArgSeqs; ++s) {
        if (s >= ns) break;
        const float4 h0 = *reinterpret_cast<const float4*>(hs + s * d + c8 * 8);
        const float4 h1 = *reinterpret_cast<const float4*>(hs + s * d + c8 * 8 + 4);
        const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[r][s] += ev[r][e] * hv[e];
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int t = t0 + r;
#pragma unroll
      for (int s = 0; s < kArgSeqs; ++s) {
        if (s >= ns) break;
        float a = acc[r][s];
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0 && t < vocab) {
          uint32_t u = __float_as_uint(a);
          u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
          atomicMax(best + s0 + s,
                    (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - uint32_t(t)));
        }
      }
    }
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
  static thread_local int attr_dev[2] = {-1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev[dh == 128] != dev) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return e;
    attr_dev[dh == 128] = dev;
  }
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
  if (max_new == 1 && (dh == 128 || dh == 64)) {
    // decode: split the keys so ~4 CTAs (16 warps) per SM stream K/V -- at 2
    // per SM the kernel was latency-bound at 41 % of HBM bandwidth (ncu), at 8
    // the per-split merge overhead dominates (B=16: 5.8 TB/s at 4K context)
    const int group = n_heads / n_kv_heads;
    static const int per_sm = [] {
      const char* e = getenv("HC_DECODE_CTAS_PER_SM");
      return e ? std::max(1, atoi(e)) : 4;
    }();
    int splits = (per_sm * 148 + n_kv_heads * n_seqs - 1) / (n_kv_heads * n_seqs);
    splits = splits < 1 ? 1 : splits > 64 ? 64 : splits;
    float* part = nullptr;
    const size_t pb = size_t(n_seqs) * n_heads * splits * (dh + 2) * sizeof(float);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&part), pb, stream);
    if (e != cudaSuccess) return e;
    const float scale_log2 = (1.0f / sqrtf(float(dh))) * 1.4426950408889634f;
    const dim3 grid{unsigned(n_kv_heads), unsigned(n_seqs), unsigned(splits)};
    if (dh == 128) {
      e = launch_pdl(attn_decode_kernel<128>, grid, dim3(kDecThreads), 0, stream,
                     static_cast<const __nv_bfloat16*>(q), n_heads, group, kv, cu_q, seq_start,
                     splits, scale_log2, part);
      if (e == cudaSuccess)
        e = launch_pdl(attn_decode_combine_kernel<128>, dim3(unsigned(n_heads), unsigned(n_seqs)),
                       dim3(128), 0, stream, static_cast<const float*>(part), n_heads, splits, cu_q,
                       static_cast<__nv_bfloat16*>(out));
    } else {
      e = launch_pdl(attn_decode_kernel<64>, grid, dim3(kDecThreads), 0, stream,
                     static_cast<const __nv_bfloat16*>(q), n_heads, group, kv, cu_q, seq_start,
                     splits, scale_log2, part);
      if (e == cudaSuccess)
        e = launch_pdl(attn_decode_combine_kernel<64>, dim3(unsigned(n_heads), unsigned(n_seqs)),
                       dim3(64), 0, stream, static_cast<const float*>(part), n_heads, splits, cu_q,
                       static_cast<__nv_bfloat16*>(out));
    }
    cudaFreeAsync(part, stream);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  return attention_launch(q, 0, dim3((max_new + kQ - 1) / kQ, n_heads, n_seqs), cu_q, seq_start,
                          n_heads, n_kv_heads, dh, kv, out, stream);
}

cudaError_t launch_embed(const int32_t* tokens, int64_t n, const void* emb, int d, float* x,
                         void* xb, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n * (d / 8) + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_pdl(embed_kernel, dim3(unsigned(blocks)), dim3(256), 0, stream, tokens, n,
                    static_cast<const uint4*>(emb), d, x, static_cast<uint4*>(xb));
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
  if (d % 8) return cudaErrorInvalidValue;
  const int per_block = std::max(1, std::min(kArgSeqs, int((200u << 10) / (unsigned(d) * 4u))));
  const size_t sm = size_t(per_block) * size_t(d) * sizeof(float);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(argmax_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  unsigned long long* best = nullptr;
  cudaError_t e = cudaMallocAsync(&best, sizeof(unsigned long long) * size_t(n_seqs), stream);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(best, 0, sizeof(unsigned long long) * size_t(n_seqs), stream);
  const unsigned groups = unsigned((n_seqs + per_block - 1) / per_block);
  argmax_rows_kernel<<<dim3(148, groups), 512, sm, stream>>>(
      static_cast<const __nv_bfloat16*>(emb), vocab, d, h, cu, n_seqs, per_block, best);
  argmax_rows_finish_kernel<<<unsigned((n_seqs + 127) / 128), 128, 0, stream>>>(best, n_seqs,
                                                                               out_tokens);
  cudaFreeAsync(best, stream);
  return cudaGetLastError();
}

namespace {

// hl rows: [s] = bf16(h_s), [B + s] = bf16(h_s - bf16(h_s)) for the last row
// h_s of every sequence -- E.hi + E.lo reproduces the fp32 logits to ~2^-17.
__global__ void hilo_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ cu,
                                 int n_seqs, int d, __nv_bfloat16* __restrict__ hl) {
  const int s = blockIdx.y;
  const float* h = x + size_t(__ldg(cu + s + 1) - 1) * d;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x) {
    const float v = h[c];
    const __nv_bfloat16 hi = __float2bfloat16(v);
    hl[size_t(s) * d + c] = hi;
    hl[size_t(n_seqs + s) * d + c] = __float2bfloat16(v - __bfloat162float(hi));
  }
}

// out[s] = argmax_t logits[t][s] + logits[t][B + s], ties to the smallest t
// (argmax_token's strict '>' scan, model.cpp:67-80). One block per sequence.
__global__ void argmax_pairs_kernel(const float* __restrict__ logits, int vocab, int ld, int n_seqs,
                                    int32_t* __restrict__ out) {
  const int s = blockIdx.x;
  float best = -INFINITY;
  int arg = 0x7fffffff;
  for (int t = threadIdx.x; t < vocab; t += blockDim.x) {
    const float v = logits[size_t(t) * ld + s] + logits[size_t(t) * ld + n_seqs + s];
    if (v > best) {
      best = v;
      arg = t;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ov > best || (ov == best && oi < arg)) {
      best = ov;
      arg = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = best;
    si[warp] = arg;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    arg = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ov > best || (ov == best && oi < arg)) {
        best = ov;
        arg = oi;
      }
    }
    if (lane == 0) out[s] = arg == 0x7fffffff ? 0 : arg;  // all-NaN logits: token 0
  }
}

}  // namespace

cudaError_t launch_hilo_rows(const float* x, const int32_t* cu, int n_seqs, int d, void* hl,
                             cudaStream_t stream) {
  if (n_seqs <= 0) return cudaSuccess;
  hilo_rows_kernel<<<dim3(unsigned((d + 255) / 256), unsigned(n_seqs)), 256, 0, stream>>>(
      x, cu, n_seqs, d, static_cast<__nv_bfloat16*>(hl));
  return cudaGetLastError();
}

cudaError_t launch_argmax_pairs(const float* logits, int vocab, int ld, int n_seqs, int32_t* out,
                                cudaStream_t stream) {
  if (n_seqs <= 0) return cudaSuccess;
  argmax_pairs_kernel<<<unsigned(n_seqs), 1024, 0, stream>>>(logits, vocab, ld, n_seqs, out);
  return cudaGetLastError();
}

}  // namespace hc
