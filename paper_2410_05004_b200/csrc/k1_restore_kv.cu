// k1_restore_kv.cu -- K1, the restoration kernel: hidden states -> paged K/V.
//
// Replaces the reference's project_hidden_to_kv (proj/src/model.cpp:219-235):
//   A = LayerNorm(H)               (model.cpp:43-61, unit scale, eps 1e-5)
//   K = A W_k^T, V = A W_v^T       (matmul_wt, proj/src/matrix.cpp:8-21)
//   RoPE(K) at positions start+i   (apply_rope, model.cpp:196-217, interleaved)
// as ONE persistent, warp-specialised tcgen05 GEMM over [W_k ; W_v]:
//   warp 0     TMA producer: A (128x64) and B (BNx64) tiles, 128B swizzle,
//              STAGES-deep smem ring (mbarrier full/empty).
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//              (M=128, N=BN, K=16 per instruction, fp32 accumulators in TMEM,
//              two accumulator buffers so the epilogue overlaps the next tile).
//   warps 2-5  epilogue: tcgen05.ld -> LayerNorm fold
//              K = rstd * (H W^T - mean * colsum(W)) -> RoPE from the host-built
//              (cos, sin) table (bit-identical coefficients to the reference)
//              -> bf16 -> vectorised stores straight into the paged KV cache.
// LayerNorm is folded into the epilogue so the A operand is the stored bf16 H
// exactly as it arrived over PCIe (no normalised copy is materialised).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <map>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"
#include "sm100.cuh"

namespace hc {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 192;
constexpr int kGroupM = 16;

template <int BN>
struct K1Cfg {
  static constexpr int kStages = BN == 256 ? 4 : BN == 128 ? 6 : 8;
  static constexpr uint32_t kABytes = kBM * kBK * 2;
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = 2 * BN;  // two fp32 accumulator buffers
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 /*bars*/ + 1024 /*align*/;
};

__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& m_blk,
                                            int& n_blk) {
  // grouped raster: kGroupM consecutive M tiles sweep all N tiles together so
  // concurrently resident CTAs share A rows and B columns through L2.
  int per_group = kGroupM * num_n;
  int group = tile / per_group;
  int first_m = group * kGroupM;
  int gm = min(num_m - first_m, kGroupM);
  int local = tile - group * per_group;
  m_blk = first_m + local % gm;
  n_blk = local / gm;
}

// The tensor map holding A row `row` and the row's coordinate within it.
__device__ __forceinline__ const CUtensorMap* amap(const AMaps& am, int row, int& local,
                                                   bool alt = false) {
  if (alt) {  // the mean-shifted copy of the whole matrix, after the sources
    local = row;
    return &am.m[am.n];
  }
  int s = 0;
  while (s + 1 < am.n && row >= am.row0[s + 1]) ++s;
  local = row - am.row0[s];
  return &am.m[s];
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Per-element epilogue arithmetic with explicit rounding (no FMA contraction):
// every epilogue -- the row-per-thread ones, the CTA pair's transposed one,
// the split-K reduction -- computes bit-identical values, so K/V written by a
// decode-sized forward and by a restore's K1 match exactly.
__device__ __forceinline__ float ln_fold(float acc, float mean, float colsum, float rstd) {
  return __fmul_rn(rstd, __fsub_rn(acc, __fmul_rn(mean, colsum)));
}
__device__ __forceinline__ void rope_rotate(float& a, float& b, float c, float s) {
  const float a0 = a;
  a = __fsub_rn(__fmul_rn(a0, c), __fmul_rn(b, s));
  b = __fadd_rn(__fmul_rn(a0, s), __fmul_rn(b, c));
}
__device__ __forceinline__ float gelu_ref(float v) {  // model.cpp:38-40
  return __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, erff(__fmul_rn(v, 0.70710678118654752f))));
}

// One thread = one output row; handles 32 consecutive columns [col0, col0+32).
// Columns [0, q_cols) are Q (fused Q/K/V projection), then K, then V.
__device__ __forceinline__ void epilogue_chunk(float (&f)[32], int col0, const KvOut& out,
                                               const EpiArgs& epi, float mean, float rstd,
                                               int pos, char* krow, char* vrow, char* qrow) {
  if (epi.row_mean) {
    const float4* cs = reinterpret_cast<const float4*>(epi.colsum + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 c = __ldg(cs + i);
      f[4 * i + 0] = ln_fold(f[4 * i + 0], mean, c.x, rstd);
      f[4 * i + 1] = ln_fold(f[4 * i + 1], mean, c.y, rstd);
      f[4 * i + 2] = ln_fold(f[4 * i + 2], mean, c.z, rstd);
      f[4 * i + 3] = ln_fold(f[4 * i + 3], mean, c.w, rstd);
    }
  }
  const bool is_q = col0 < out.q_cols;
  const int ckv = col0 - out.q_cols;
  const bool is_k = !is_q && ckv < out.d_kv;
  const int ocol = is_q ? col0 : is_k ? ckv : ckv - out.d_kv;
  if ((is_k || is_q) && epi.rope) {
    const int half = epi.d_head >> 1;
    const float2* row_cs = epi.rope + size_t(pos) * half;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int t = ((ocol + 2 * i) % epi.d_head) >> 1;
      float2 cs = __ldg(row_cs + t);
      rope_rotate(f[2 * i], f[2 * i + 1], cs.x, cs.y);
    }
  }
  char* dst = is_q ? qrow : is_k ? krow : vrow;
  if (out.out_f32 && !is_q) {
    float4* d4 = reinterpret_cast<float4*>(dst + size_t(ocol) * 4);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      d4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
  } else {
    uint4* d4 = reinterpret_cast<uint4*>(dst + size_t(ocol) * 2);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      d4[i] = make_uint4(pack_bf16(f[8 * i + 0], f[8 * i + 1]), pack_bf16(f[8 * i + 2], f[8 * i + 3]),
                         pack_bf16(f[8 * i + 4], f[8 * i + 5]), pack_bf16(f[8 * i + 6], f[8 * i + 7]));
  }
}

// RESID: x[row, col] += acc (fp32 residual stream), xb = bf16(x).
// GELU:  xb[row, col] = bf16(gelu(fold(acc))) (reference gelu, model.cpp:38-40).
__device__ __forceinline__ void epilogue_chunk_dense(float (&f)[32], int mode, int row, int col0,
                                                     const GemmOut& g, const EpiArgs& epi,
                                                     float mean, float rstd) {
  const size_t off = size_t(row) * size_t(g.ldo) + size_t(col0);
  if (mode == kEpiResid) {
    float4* x4 = reinterpret_cast<float4*>(g.x + off);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 x = x4[i];
      x.x = __fadd_rn(x.x, f[4 * i + 0]);
      x.y = __fadd_rn(x.y, f[4 * i + 1]);
      x.z = __fadd_rn(x.z, f[4 * i + 2]);
      x.w = __fadd_rn(x.w, f[4 * i + 3]);
      x4[i] = x;
      f[4 * i + 0] = x.x;
      f[4 * i + 1] = x.y;
      f[4 * i + 2] = x.z;
      f[4 * i + 3] = x.w;
    }
  } else {
    if (epi.row_mean) {
      const float4* cs = reinterpret_cast<const float4*>(epi.colsum + col0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 c = __ldg(cs + i);
        f[4 * i + 0] = ln_fold(f[4 * i + 0], mean, c.x, rstd);
        f[4 * i + 1] = ln_fold(f[4 * i + 1], mean, c.y, rstd);
        f[4 * i + 2] = ln_fold(f[4 * i + 2], mean, c.z, rstd);
        f[4 * i + 3] = ln_fold(f[4 * i + 3], mean, c.w, rstd);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] = gelu_ref(f[i]);
  }
  uint4* d4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(g.xb) + off);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    d4[i] = make_uint4(pack_bf16(f[8 * i + 0], f[8 * i + 1]), pack_bf16(f[8 * i + 2], f[8 * i + 3]),
                       pack_bf16(f[8 * i + 4], f[8 * i + 5]), pack_bf16(f[8 * i + 6], f[8 * i + 7]));
}

// Per-row epilogue metadata: LN stats, RoPE position and the K/V row pointers
// (dense or paged; ragged batches via cu_seqlens / seq_start).
struct RowMeta {
  float mean = 0.f, rstd = 1.f;
  int pos = 0;
  char* krow = nullptr;
  char* vrow = nullptr;
  char* qrow = nullptr;  // fused Q/K/V: this row's dense Q
};

template <int MODE>
__device__ __forceinline__ RowMeta row_meta(int row, const KvOut& out, const EpiArgs& epi) {
  RowMeta r;
  r.pos = out.start_pos;
  if (MODE == kEpiKv) {
    int seq = 0, local = row;
    if (out.cu_seqlens) {
      int lo = 0, hi = out.n_seqs - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(out.cu_seqlens + mid) <= row) lo = mid;
        else hi = mid - 1;
      }
      seq = lo;
      local = row - __ldg(out.cu_seqlens + seq);
    }
    r.pos = (out.seq_start ? __ldg(out.seq_start + seq) : out.start_pos) + local;
    int64_t orow;
    if (out.page_table) {
      int page = __ldg(out.page_table + int64_t(seq) * out.table_stride + r.pos / out.page_size);
      orow = int64_t(page) * out.page_size + r.pos % out.page_size;
    } else {
      orow = row;
    }
    const size_t esz = out.out_f32 ? 4 : 2;
    r.krow = static_cast<char*>(out.k_base) + size_t(orow) * out.d_kv * esz;
    r.vrow = static_cast<char*>(out.v_base) + size_t(orow) * out.d_kv * esz;
    if (out.q_base) r.qrow = static_cast<char*>(out.q_base) + size_t(row) * size_t(out.q_cols) * 2;
  }
  if (epi.row_mean) {
    r.mean = __ldg(epi.row_mean + row);
    r.rstd = __ldg(epi.row_rstd + row);
  }
  return r;
}

template <int MODE>
__device__ __forceinline__ void apply_chunk(float (&f)[32], int row, int col0, const RowMeta& r,
                                            const KvOut& out, const GemmOut& gout,
                                            const EpiArgs& epi) {
  if (MODE == kEpiKv)
    epilogue_chunk(f, col0, out, epi, r.mean, r.rstd, r.pos, r.krow, r.vrow, r.qrow);
  else epilogue_chunk_dense(f, MODE, row, col0, gout, epi, r.mean, r.rstd);
}

// Epilogue of one accumulator tile for one thread (= one TMEM lane = one
// output row): BN/32 chunks of tcgen05.ld + math + stores. Shared by the
// single-CTA and the CTA-pair kernels. With a split-K workspace (part) the
// raw fp32 accumulators of this K slice are stored instead
// (part[(split * M + row) * N + col]) for splitk_epilogue_kernel.
template <int BN, int MODE>
__device__ __forceinline__ void epilogue_tile(int row, int n_blk, int M, int N, const KvOut& out,
                                              const GemmOut& gout, const EpiArgs& epi,
                                              uint32_t tbase, int lane, float* part = nullptr,
                                              int split = 0) {
  (void)lane;
  const bool row_ok = row < M;
  RowMeta meta;
  if (row_ok && !part) meta = row_meta<MODE>(row, out, epi);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tbase + uint32_t(c * 32), v);
    tmem_wait_ld();
    const int col0 = n_blk * BN + c * 32;
    if (row_ok && col0 < N) {
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
      if (part) {
        float4* d4 = reinterpret_cast<float4*>(part + (size_t(split) * M + row) * size_t(N) + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          d4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
      } else {
        apply_chunk<MODE>(f, row, col0, meta, out, gout, epi);
      }
    }
  }
}

// Split-K reduction + epilogue: one warp per (row, 32-column chunk), one
// column per lane. Lane c sums column c over the K slices in slice order
// (deterministic, coalesced) and applies the mode's epilogue to it -- the
// same arithmetic as epilogue_chunk / epilogue_chunk_dense, per column (RoPE
// pairs meet through a lane shuffle).
template <int MODE>
__global__ void splitk_epilogue_kernel(const float* __restrict__ part, int splits, int M, int N,
                                       KvOut out, GemmOut gout, EpiArgs epi) {
  pdl_wait();  // the GEMM's partials (programmatic dependent launch)
  pdl_trigger();
  const int chunks = N / 32;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(M) * chunks) return;  // warp-uniform
  const int row = int(w / chunks), col = int(w % chunks) * 32 + lane;
  float v = 0.f;
  for (int sp = 0; sp < splits; ++sp) v += __ldg(part + (size_t(sp) * M + row) * size_t(N) + col);
  const RowMeta r = row_meta<MODE>(row, out, epi);
  if (MODE == kEpiResid) {
    const size_t off = size_t(row) * size_t(gout.ldo) + size_t(col);
    const float x = __fadd_rn(gout.x[off], v);
    gout.x[off] = x;
    static_cast<__nv_bfloat16*>(gout.xb)[off] = __float2bfloat16(x);
    return;
  }
  if (epi.row_mean) v = ln_fold(v, r.mean, __ldg(epi.colsum + col), r.rstd);
  if (MODE == kEpiGelu) {
    v = gelu_ref(v);
    static_cast<__nv_bfloat16*>(gout.xb)[size_t(row) * size_t(gout.ldo) + size_t(col)] =
        __float2bfloat16(v);
    return;
  }
  // kEpiKv
  const bool is_k = col < out.d_kv;  // uniform per 32-column chunk (d_kv % 32 == 0)
  const int ocol = is_k ? col : col - out.d_kv;
  const float other = __shfl_xor_sync(0xffffffffu, v, 1);
  if (is_k && epi.rope) {
    const float2 cs = __ldg(epi.rope + size_t(r.pos) * (epi.d_head >> 1) + ((ocol % epi.d_head) >> 1));
    float a = (lane & 1) ? other : v, b = (lane & 1) ? v : other;
    rope_rotate(a, b, cs.x, cs.y);
    v = (lane & 1) ? b : a;
  }
  char* dst = is_k ? r.krow : r.vrow;
  if (out.out_f32) reinterpret_cast<float*>(dst)[ocol] = v;
  else reinterpret_cast<__nv_bfloat16*>(dst)[ocol] = __float2bfloat16(v);
}

// Shared-memory ring: stage s holds [A rows | B rows] at s * stride. a_rows =
// rows of the A TMA box (gemm_a_box): 128, or 32/64 when M is that small.
// In the compact ring (a_rows < 128) the stride is only a_rows*128 + BN*128
// bytes: the UMMA still reads a 128-row A tile, whose rows >= a_rows are
// whatever follows (the stage's B rows, the next stage, or the tail pad) --
// they only feed accumulator rows >= M, which the epilogue never stores. A
// decode-sized GEMM thus keeps 3-4x more weight bytes in flight per SM.
// There, `kbs` consecutive k-block slots share one full/empty barrier pair
// (one expect_tx, one commit): a weight-streaming CTA moves >= 32 KB per
// barrier round trip. Measured (scripts/tma_stream.cu, 148 CTAs, 200 KB
// ring): 8 KB per barrier streams 4.6 TB/s, 16 KB 6.5, 32 KB 6.8-7.1. The
// MMA order over K is unchanged, so results are bit-identical.
constexpr size_t kMaxRingSmem = 227 * 1024;

struct RingCfg {
  int stages;       // slots (a multiple of kbs)
  int kbs;          // k-block slots per barrier group
  uint32_t stride;  // bytes per slot
  uint32_t a_bytes;
  size_t smem;      // dynamic smem incl. tail pad, barriers, alignment slack
};

template <int BN>
RingCfg ring_cfg(int a_rows) {
  RingCfg r;
  r.a_bytes = uint32_t(a_rows) * kBK * 2;
  r.stride = r.a_bytes + K1Cfg<BN>::kBBytes;
  const uint32_t pad = K1Cfg<BN>::kABytes - r.a_bytes;  // garbage rows past the last stage
  r.stages = a_rows == kBM ? K1Cfg<BN>::kStages
                           : int(std::min<size_t>(32, (size_t(200) * 1024 - pad) / r.stride));
  r.kbs = a_rows == kBM ? 1 : std::max(1, int((32u << 10) / r.stride));
  if (const char* e = getenv("HC_RING_KBS")) r.kbs = std::max(1, atoi(e));  // experiments
  r.kbs = std::max(1, std::min(r.kbs, r.stages / 2));
  r.stages -= r.stages % r.kbs;
  r.smem = size_t(r.stages) * r.stride + pad + 1024 /*bars*/ + 1024 /*align*/;
  return r;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ AMaps am,
                   const __grid_constant__ CUtensorMap tmB, int M, int N, int K, KvOut out,
                   GemmOut gout, EpiArgs epi, uint32_t idesc, int S, int kbs, uint32_t stride,
                   uint32_t a_bytes, int k_splits, float* part) {
  using Cfg = K1Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;  // stage s: A at s*stride, B at s*stride + a_bytes
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * stride +
                                               (Cfg::kABytes - a_bytes));
  const int G = S / kbs;  // barrier groups of kbs slots
  uint64_t* empty = full + G;
  uint64_t* tfull = empty + G;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_mn = num_m * num_n;
  const int num_tiles = num_mn * k_splits;  // tile = (K slice, M/N tile)
  const int num_kb = (K + kBK - 1) / kBK;
  const int kb_per = (num_kb + k_splits - 1) / k_splits;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < am.n; ++i) tma_prefetch_desc(&am.m[i]);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < G; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      // the A-map choice is made once, outside the loop: a per-load runtime
      // select between maps cost 6 % of tensor-pipe activity (ncu A/B)
      auto produce = [&](auto alt_tag) {
        constexpr bool kAlt = decltype(alt_tag)::value;
        int grp = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
          int m_blk, n_blk;
          tile_coords(tile % num_mn, num_m, num_n, m_blk, n_blk);
          const int kb0 = (tile / num_mn) * kb_per, kb1 = min(num_kb, kb0 + kb_per);
          int a_row;
          const CUtensorMap* ma = amap(am, m_blk * kBM, a_row, kAlt);
          for (int kb = kb0; kb < kb1; kb += kbs) {
            const int nk = min(kbs, kb1 - kb);
            mbar_wait(&empty[grp], phase ^ 1);
            mbar_arrive_expect_tx(&full[grp], uint32_t(nk) * (a_bytes + Cfg::kBBytes));
            for (int i = 0; i < nk; ++i) {
              uint8_t* st = sA + size_t(grp * kbs + i) * stride;
              tma_load_2d(st, ma, &full[grp], (kb + i) * kBK, a_row);
              tma_load_2d(st + a_bytes, &tmB, &full[grp], (kb + i) * kBK, n_blk * BN);
            }
            if (++grp == G) {
              grp = 0;
              phase ^= 1;
            }
          }
        }
      };
      if (am.alt_flag && *reinterpret_cast<const volatile int32_t*>(am.alt_flag))
        produce(std::true_type{});
      else
        produce(std::false_type{});
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform loop, one elected lane issues) --
    {
      int grp = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        const int kb0 = (tile / num_mn) * kb_per, kb1 = min(num_kb, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; kb += kbs) {
          const int nk = min(kbs, kb1 - kb);
          mbar_wait(&full[grp], phase);
          tc_fence_after();
          if (elect_one()) {
            for (int i = 0; i < nk; ++i) {
              const uint8_t* st = sA + size_t(grp * kbs + i) * stride;
              const uint64_t adesc = umma_desc_sw128(smem_u32(st));
              const uint64_t bdesc = umma_desc_sw128(smem_u32(st + a_bytes));
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
                umma_f16(d_tmem, adesc + uint64_t(2 * k), bdesc + uint64_t(2 * k), idesc,
                         ((kb + i - kb0) | k) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[grp]);  // frees the group's slots when these MMAs retire
          }
          __syncwarp();
          if (++grp == G) {
            grp = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5, 128 threads = 128 TMEM lanes) ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int m_blk, n_blk;
      tile_coords(tile % num_mn, num_m, num_n, m_blk, n_blk);
      const int row = m_blk * kBM + q * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      epilogue_tile<BN, MODE>(row, n_blk, M, N, out, gout, epi,
                              tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN), lane,
                              part, tile / num_mn);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}


// ------------------------------------------------------------ CTA-pair variant
// cta_group::2: a cluster of two CTAs (one per SM of a TPC) computes a
// 256 x 256 tile with M=256 MMAs issued by the leader. Each CTA loads its own
// 128 rows of A and 128 of the 256 B rows, so per SM the operand traffic per
// k-block drops from 48 KB (128x256 single-CTA tile) to 32 KB while the MMA
// work per SM is unchanged. Accumulator rows 0-127 live in the leader's TMEM,
// 128-255 in the peer's; both run the same epilogue on their own lanes.
// Epilogue warps of the pair kernel: two per TMEM lane quadrant, each taking
// half of the tile's columns -- four of them, one per quadrant, left the last
// tile's epilogue (~11 us, latency-bound per warp) exposed at the end of every
// launch. (A 5-stage ring that left room for wider scratch starved the MMAs
// of RESID tiles: 21.5 -> 24.5 us per K=4096 tile.)
constexpr int kPairEpiWarps = 8;

constexpr int kPairThreads = 64 + 32 * kPairEpiWarps;
constexpr int kPairStages = 6;
constexpr uint32_t kPairHalfBytes = 128 * kBK * 2;             // 16 KB: A half or B half
constexpr uint32_t kPairStageBytes = 2 * kPairHalfBytes;       // per CTA per stage
// + the transposing epilogue's scratch (4 warps x kPairEpiWarpBytes, defined
// below with the epilogue)
constexpr size_t kPairEpiBytes = kPairEpiWarps * (32 * 16 * 4 + 32 * 32);
constexpr size_t kPairSmem = size_t(kPairStages) * kPairStageBytes + 1024 + kPairEpiBytes + 1024;

__device__ __forceinline__ void tile_coords_pair(int tile, int num_m, int num_n, int& m_blk,
                                                 int& n_blk) {
  tile_coords(tile, num_m, num_n, m_blk, n_blk);
}

// Tail split of the last, partial wave (summation-order-free callers only,
// split_acc). With T tiles over C clusters the persistent schedule runs
// floor(T/C) full waves and a last one of R = T mod C tiles that leaves C-R
// SM pairs idle (N=4096 GEMMs of a 4096-token layer: 256 tiles on 74 pairs,
// 3.46 waves run as 4). When 2R <= C the R tail tiles are each split into two
// K halves on two clusters: the first half's raw fp32 accumulators go to a
// workspace (through L2), the second adds them to its own and runs the
// epilogue -- the last wave takes half as long. The unit -> (tile, K range)
// map depends only on the schedule shape (Ms, N, K, C), so a GEMM and its
// row-truncated copy (Ms fixed, fewer valid rows M) sum every element in the
// same order.
struct PairUnit {
  int tile, kb0, kb1, half, slot;  // half: -1 whole tile, 0/1 K halves of tail tile `slot`
};

__device__ __forceinline__ PairUnit pair_unit(int u, int full_units, bool split, int num_kb) {
  PairUnit p;
  if (!split || u < full_units) {
    p.tile = u;
    p.kb0 = 0;
    p.kb1 = num_kb;
    p.half = -1;
    p.slot = -1;
  } else {
    const int t = (u - full_units) >> 1, kh = num_kb >> 1;
    p.tile = full_units + t;
    p.half = (u - full_units) & 1;
    p.kb0 = p.half ? kh : 0;
    p.kb1 = p.half ? num_kb : kh;
    p.slot = t;
  }
  return p;
}

// Host and device agree on the tail split from the schedule shape alone.
__host__ __device__ __forceinline__ int pair_full_units(int tiles, int clusters) {
  return (tiles / clusters) * clusters;
}
// The exchange (first half's epilogue writing 128 KB per CTA, the second's
// reading it) costs ~8 us: at K = 11008 the split saves 8 us per launch (223
// -> 215 us); at K = 4096 (a 9 us half tile) it measured no better than the
// idle tail in round 1 (scripts/pair_trace.cu: 88.6 vs 90.8 us) and 1 %
// better with the 8-warp epilogue (O projection 114.5 -> 113.4 us, K6 layer
// span -0.25 %, scripts/ab_tail.sh), so K loops of >= 32 k-blocks split.
#ifndef HC_TAIL_MIN_KB
#define HC_TAIL_MIN_KB 32
#endif
constexpr int kTailMinKb = HC_TAIL_MIN_KB;
__host__ __device__ __forceinline__ bool pair_tail_split(int tiles, int clusters, int num_kb) {
  const int tail = tiles - pair_full_units(tiles, clusters);
  return tail > 0 && 2 * tail <= clusters && num_kb >= kTailMinKb;
}

// Workspace of one tail slot and CTA: 128 rows x 256 fp32 accumulators,
// chunk-major ((c * 8 + i) * 128 + row) float4s so a warp's accesses are
// contiguous.
constexpr size_t kTailSlotFloats = 128 * 256;

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void epi_bar_sync(int n_threads) {  // the epilogue warps of a CTA
  asm volatile("bar.sync 1, %0;" ::"r"(n_threads) : "memory");
}

// Epilogue of the CTA pair, one warp = 32 accumulator rows. tcgen05.ld
// hands each lane one row (32 columns per load); storing from that layout
// makes every warp-wide 16-byte access touch 32 rows, i.e. 32 L1 wavefronts
// per instruction -- a RESID tile (x read + written, xb written) then spent
// as long in its epilogue (~20 us) as in its MMAs, and N=4096 projections
// ran at ~58 % of the tensor pipe (scripts/pair_trace.cu). So each 32-column
// chunk is transposed through shared memory in two 16-column halves: lane l
// then holds 4 consecutive columns of rows 8j + l/4 (j = 0..3), and every
// global access of a warp covers 8 rows x 64 contiguous bytes. The 16-byte
// units of a row are XOR-swizzled with (row/2) & 3 so both the row-wise
// writes and the transposed reads are bank-conflict free. Per-row metadata
// (LN statistics, RoPE position, K/V row pointers) is computed once per tile
// by the row's own lane and read back from shared memory. A chunk's global
// loads (x rows, RoPE coefficients) depend only on rows and columns, so the
// next chunk's are issued before this chunk is processed.
struct EpiRow {
  float mean, rstd;
  int pos, valid;
  char* krow;
  char* vrow;
};
constexpr uint32_t kPairEpiWarpBytes = 32 * 16 * 4 + 32 * sizeof(EpiRow);

__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  return make_uint2(pack_bf16(a, b), pack_bf16(c, d));
}
// float offset of 16-byte unit u (0..3) of transposed row r
__device__ __forceinline__ int tunit(int r, int u) { return r * 16 + ((u ^ ((r >> 1) & 3)) << 2); }

// QKV: the fused Q/K/V projection (first out.q_cols columns are Q). A
// separate instantiation: the routing, compiled into K1's epilogue, cost it
// ~3 % (scripts/ab_k1_alone.sh: 182.9 vs 177.9 us per 7B layer).
template <int MODE, int BN, bool QKV>
__device__ __forceinline__ void epilogue_tile_pair(int row_base, int lane, int n_blk, int M, int N,
                                                   const KvOut& out, const GemmOut& gout,
                                                   const EpiArgs& epi, uint32_t tbase, float* ws,
                                                   int half, float* tbuf, EpiRow* meta,
                                                   int c_begin, int c_end) {
  if (half != 0) {
    const int row = row_base + lane;
    EpiRow e{0.f, 1.f, 0, 0, nullptr, nullptr};
    if (row < M) {
      const RowMeta r = row_meta<MODE>(row, out, epi);
      e = EpiRow{r.mean, r.rstd, r.pos, 1, r.krow, r.vrow};
    }
    meta[lane] = e;
  }
  const int g = lane >> 2, u = lane & 3;  // transposed: rows 8j + g, columns 4u..4u+3
  __syncwarp();  // meta visible to the warp
  const bool rope_on = MODE == kEpiKv && epi.rope != nullptr;
  // loads of chunk c: index 4 * h2 + j (16-column half h2, row 8j + g)
  auto issue = [&](int c, float4 (&ld)[8]) {
    const int col0 = n_blk * BN + c * 32;
    const bool k_half = col0 < (QKV ? out.q_cols : 0) + out.d_kv;  // Q or K: rotated
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int h2 = i >> 2, j = i & 3;
      const EpiRow& e = meta[8 * j + g];
      const int col = col0 + 16 * h2 + 4 * u;
      ld[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!e.valid || half == 0 || col0 >= N) continue;
      if (MODE == kEpiResid)
        ld[i] = *reinterpret_cast<const float4*>(gout.x + size_t(row_base + 8 * j + g) *
                                                               size_t(gout.ldo) + col);
      else if (rope_on && k_half)
        ld[i] = __ldg(reinterpret_cast<const float4*>(
            epi.rope + size_t(e.pos) * size_t(epi.d_head >> 1) + ((col % epi.d_head) >> 1)));
    }
  };
  float4 ld[8], ld_next[8];
  issue(c_begin, ld_next);
#pragma unroll 1
  for (int c = c_begin; c < c_end; ++c) {
#pragma unroll
    for (int i = 0; i < 8; ++i) ld[i] = ld_next[i];
    if (c + 1 < c_end) issue(c + 1, ld_next);
    uint32_t v[32];
    tmem_ld_32x32b_x32(tbase + uint32_t(c * 32), v);
    tmem_wait_ld();
    float f[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
    float4* w4 = ws ? reinterpret_cast<float4*>(ws) + size_t(c) * 8 * 128 + (row_base & 127) + lane
                    : nullptr;
    if (half == 0) {  // first K half: raw accumulators to the workspace
#pragma unroll
      for (int i = 0; i < 8; ++i)
        __stcg(w4 + i * 128, make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]));
      continue;
    }
    if (half == 1) {  // second K half: first half's sums + this half's
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 p = __ldcg(w4 + i * 128);
        f[4 * i + 0] = __fadd_rn(p.x, f[4 * i + 0]);
        f[4 * i + 1] = __fadd_rn(p.y, f[4 * i + 1]);
        f[4 * i + 2] = __fadd_rn(p.z, f[4 * i + 2]);
        f[4 * i + 3] = __fadd_rn(p.w, f[4 * i + 3]);
      }
    }
    const int col0 = n_blk * BN + c * 32;
    if (col0 >= N) continue;  // warp-uniform
    const int qc = QKV ? out.q_cols : 0;
    const bool is_q = QKV && MODE == kEpiKv && col0 < qc;
    const bool is_k = MODE == kEpiKv && !is_q && col0 - qc < out.d_kv;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      __syncwarp();  // the previous reads of tbuf are done
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        *reinterpret_cast<float4*>(tbuf + tunit(lane, q4)) =
            make_float4(f[16 * h2 + 4 * q4], f[16 * h2 + 4 * q4 + 1], f[16 * h2 + 4 * q4 + 2],
                        f[16 * h2 + 4 * q4 + 3]);
      __syncwarp();
      const int col = col0 + 16 * h2 + 4 * u;  // this lane's 4 columns
      const int ocol = MODE == kEpiKv ? (is_q ? col : is_k ? col - qc : col - qc - out.d_kv) : col;
      float4 cs4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (MODE != kEpiResid && epi.row_mean)
        cs4 = __ldg(reinterpret_cast<const float4*>(epi.colsum + col));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = 8 * j + g;
        const EpiRow& e = meta[r];
        if (!e.valid) continue;
        const float4 a4 = *reinterpret_cast<const float4*>(tbuf + tunit(r, u));
        const float4 l4 = ld[4 * h2 + j];
        float a[4] = {a4.x, a4.y, a4.z, a4.w};
        if (MODE == kEpiResid) {
          float4 x = l4;
          x.x = __fadd_rn(x.x, a[0]);
          x.y = __fadd_rn(x.y, a[1]);
          x.z = __fadd_rn(x.z, a[2]);
          x.w = __fadd_rn(x.w, a[3]);
          const size_t off = size_t(row_base + r) * size_t(gout.ldo) + col;
          *reinterpret_cast<float4*>(gout.x + off) = x;
          *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(gout.xb) + off) =
              pack4_bf16(x.x, x.y, x.z, x.w);
          continue;
        }
        if (epi.row_mean) {
          a[0] = ln_fold(a[0], e.mean, cs4.x, e.rstd);
          a[1] = ln_fold(a[1], e.mean, cs4.y, e.rstd);
          a[2] = ln_fold(a[2], e.mean, cs4.z, e.rstd);
          a[3] = ln_fold(a[3], e.mean, cs4.w, e.rstd);
        }
        if (MODE == kEpiGelu) {
          *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(gout.xb) +
                                    size_t(row_base + r) * size_t(gout.ldo) + col) =
              pack4_bf16(gelu_ref(a[0]), gelu_ref(a[1]), gelu_ref(a[2]), gelu_ref(a[3]));
          continue;
        }
        if ((is_k || is_q) && rope_on) {
          rope_rotate(a[0], a[1], l4.x, l4.y);
          rope_rotate(a[2], a[3], l4.z, l4.w);
        }
        char* dst = is_q ? static_cast<char*>(out.q_base) + size_t(row_base + r) * size_t(qc) * 2
                         : is_k ? e.krow : e.vrow;
        if (out.out_f32 && !is_q)
          *reinterpret_cast<float4*>(dst + size_t(ocol) * 4) = make_float4(a[0], a[1], a[2], a[3]);
        else
          *reinterpret_cast<uint2*>(dst + size_t(ocol) * 2) = pack4_bf16(a[0], a[1], a[2], a[3]);
      }
    }
  }
}

// scripts/pair_trace.cu (-DHC_PAIR_TRACE): globaltimer stamps per CTA --
// [0] start, [1] end, then per unit i of the CTA: 2+4i MMA issue start, +1 MMA
// issue end, +2 epilogue start (accumulator ready), +3 epilogue end.
#ifdef HC_PAIR_TRACE
__device__ unsigned long long* g_pair_trace;
constexpr int kPairTraceSlots = 40;
#define PAIR_TRACE(slot)                                                                \
  do {                                                                                  \
    if (g_pair_trace && (slot) < kPairTraceSlots)                                       \
      g_pair_trace[size_t(blockIdx.x) * kPairTraceSlots + (slot)] = global_ns();        \
  } while (0)
#else
#define PAIR_TRACE(slot) \
  do {                   \
  } while (0)
#endif

template <int MODE, int BN, bool QKV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    tc_gemm_pair_kernel(const __grid_constant__ AMaps am,
                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K, KvOut out,
                        GemmOut gout, EpiArgs epi, uint32_t idesc, int Ms, float* tail_ws,
                        int32_t* tail_flags, uint32_t epoch) {
  // M: rows stored; Ms >= M: rows the schedule is laid out for (units whose
  // tile starts at or past M are skipped by every role)
  // BN = 256 or 192 output columns per pair tile; each CTA stages BN/2 B rows
  constexpr int S = kPairStages;
  constexpr uint32_t kBHalf = uint32_t(BN / 2) * kBK * 2;
  static_assert(BN == 256 || BN == 192, "pair tile width");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kPairHalfBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * kPairHalfBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi_smem = sB + S * kPairHalfBytes + 1024;
  static_assert(kPairEpiBytes == kPairEpiWarps * kPairEpiWarpBytes, "epilogue scratch size");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = int(blockIdx.x >> 1), n_clusters = int(gridDim.x >> 1);
  const int num_m = (Ms + 255) / 256;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBK - 1) / kBK;
  const bool split = tail_ws != nullptr && pair_tail_split(num_tiles, n_clusters, num_kb);
  const int full_units = split ? pair_full_units(num_tiles, n_clusters) : num_tiles;
  const int num_units = split ? num_tiles + (num_tiles - full_units) : num_tiles;

  if (threadIdx.x == 0) PAIR_TRACE(0);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < am.n; ++i) tma_prefetch_desc(&am.m[i]);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kPairEpiWarps);  // the epilogue warps of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();     // the previous kernel's outputs (A, statistics, flags) are ready
  pdl_trigger();  // every CTA is resident: the next kernel may launch its prologue

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes counted on the leader) ----
    if (lane == 0) {
      auto produce = [&](auto alt_tag) {  // A-map choice outside the loop (see above)
        constexpr bool kAlt = decltype(alt_tag)::value;
        int stage = 0;
        uint32_t phase = 0;
        for (int u = cluster; u < num_units; u += n_clusters) {
          const PairUnit pu = pair_unit(u, full_units, split, num_kb);
          int m_blk, n_blk;
          tile_coords_pair(pu.tile, num_m, num_n, m_blk, n_blk);
          if (m_blk * 256 >= M) continue;
          for (int kb = pu.kb0; kb < pu.kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (kPairHalfBytes + kBHalf));
            int a_row;
            const CUtensorMap* ma = amap(am, m_blk * 256 + int(rank) * 128, a_row, kAlt);
            tma_load_2d_pair(sA + stage * kPairHalfBytes, ma, &full[stage], kb * kBK, a_row);
            tma_load_2d_pair(sB + stage * kPairHalfBytes, &tmB, &full[stage], kb * kBK,
                             n_blk * BN + int(rank) * (BN / 2));
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      };
      if (am.alt_flag && *reinterpret_cast<const volatile int32_t*>(am.alt_flag))
        produce(std::true_type{});
      else
        produce(std::false_type{});
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA; warp-uniform loop, one elected
    // lane issues: a divergent lane-0 loop costs ~100 clk of R2UR/ELECT per MMA)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int ui = 0;
      for (int u = cluster; u < num_units; u += n_clusters, ++ui) {
        const PairUnit pu = pair_unit(u, full_units, split, num_kb);
        int m_blk, n_blk;
        tile_coords_pair(pu.tile, num_m, num_n, m_blk, n_blk);
        if (m_blk * 256 >= M) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) PAIR_TRACE(2 + 4 * ui);
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        for (int kb = pu.kb0; kb < pu.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * kPairHalfBytes));
            const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * kPairHalfBytes));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_f16_pair(d_tmem, adesc + uint64_t(2 * k), bdesc + uint64_t(2 * k), idesc,
                            ((kb - pu.kb0) | k) != 0 ? 1u : 0u);
            umma_commit_pair(&empty[stage], 0x3);  // frees the slot in both CTAs
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
        if (lane == 0) PAIR_TRACE(3 + 4 * ui);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs, their own 128 TMEM lanes) --------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int ew = warp - 2, n_epi = 32 * kPairEpiWarps;
    constexpr int kChunksPerWarp = (BN / 32) / (kPairEpiWarps / 4);
    const int c_begin = (ew / 4) * kChunksPerWarp, c_end = c_begin + kChunksPerWarp;
    const bool lead = ew == 0 && lane == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int ui = -1;
    for (int u = cluster; u < num_units; u += n_clusters) {
      ++ui;
      const PairUnit pu = pair_unit(u, full_units, split, num_kb);
      int m_blk, n_blk;
      tile_coords_pair(pu.tile, num_m, num_n, m_blk, n_blk);
      if (m_blk * 256 >= M) continue;
      const int row_base = m_blk * 256 + int(rank) * 128 + q * 32;
      float* ws = pu.half >= 0 ? tail_ws + (size_t(pu.slot) * 2 + rank) * kTailSlotFloats : nullptr;
      int32_t* flag = pu.half >= 0 ? tail_flags + pu.slot * 2 + int(rank) : nullptr;
      if (MODE == kEpiResid && pu.half != 0 && row_base + lane < M) {
        // the residual rows this tile reads, into L2 while its MMAs run
        const char* xr = reinterpret_cast<const char*>(gout.x + size_t(row_base + lane) *
                                                                    size_t(gout.ldo) + n_blk * BN);
        for (int i = c_begin; i < c_end; ++i)
          if (n_blk * BN + i * 32 < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + i * 128));
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (lead) PAIR_TRACE(4 + 4 * ui);
      if (pu.half == 1) {  // the first K half's sums must have landed
        if (lead)
          while (uint32_t(ld_acquire_gpu(flag)) != epoch) __nanosleep(32);
        epi_bar_sync(n_epi);
      }
      uint8_t* my = epi_smem + size_t(ew) * kPairEpiWarpBytes;
      epilogue_tile_pair<MODE, BN, QKV>(row_base, lane, n_blk, M, N, out, gout, epi,
                               tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN), ws,
                               pu.half, reinterpret_cast<float*>(my),
                               reinterpret_cast<EpiRow*>(my + 32 * 16 * 4), c_begin, c_end);
      if (pu.half == 0) {  // publish: every thread's stores, then one release
        __threadfence();
        epi_bar_sync(n_epi);
        if (lead) st_release_gpu(flag, int32_t(epoch));
      }
      if (lead) PAIR_TRACE(5 + 4 * ui);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x == 0) PAIR_TRACE(1);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

// ------------------------------------------------------------ row stats
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&x)[8]) {
  uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (sizeof(T) == 2 && std::is_same<T, __nv_bfloat16>::value)
      x[i] = __bfloat162float(h[i]);
    else
      x[i] = __half2float(h[i]);
  }
}

// One pass over the row, shifted by its first element c (robust when
// |mean| >> sigma): per 16-byte load the 8 values' sum and sum of squares of
// (x - c) in fp32, accumulated across loads in double; mean = c + S/n,
// var = Q/n - (S/n)^2 (the reference's two-pass double variance,
// model.cpp:43-61, to ~1e-7 relative). FP64 only once per 8 elements: the
// B200 FP64 / F2F.F64 rate made a per-element double accumulation the bound.
// One warp per row, eight 16-byte loads in flight per lane. HBM-bound: 2
// bytes per element read once.
template <typename T>
__device__ __forceinline__ void row_stats_row(const T* __restrict__ r, int cols, int lane,
                                              float* mean_out, float* rstd_out, int32_t* flag) {
  constexpr int U = 8;
  const float c0 = __shfl_sync(0xffffffffu, lane == 0 ? float(r[0]) : 0.f, 0);
  double s[2] = {0.0, 0.0}, q[2] = {0.0, 0.0};
  auto acc8 = [&](const float (&v)[8], int k) {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float x = v[i] - c0;
      a += x;
      b = fmaf(x, x, b);
    }
    s[k] += double(a);
    q[k] += double(b);
  };
  int c = lane * 8;
#pragma unroll 2
  for (; c + (U - 1) * 256 < cols; c += U * 256) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) load8(r + c + u * 256, v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc8(v[u], u & 1);
  }
  for (; c < cols; c += 256) {
    float v[8];
    load8(r + c, v);
    acc8(v, 0);
  }
  double ss = s[0] + s[1], qq = q[0] + q[1];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    qq += __shfl_xor_sync(0xffffffffu, qq, o);
  }
  if (lane == 0) {
    const double mu = ss / double(cols);  // mean of x - c0
    double var = qq / double(cols) - mu * mu;
    if (var < 0) var = 0;
    const float mean = float(double(c0) + mu), rstd = 1.0f / sqrtf(float(var) + 1e-5f);
    *mean_out = mean;
    *rstd_out = rstd;
    if (flag && fabsf(mean) * rstd > kCenterRatio) atomicOr(flag, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) row_stats_kernel(const T* __restrict__ x, int64_t rows,
                                                        int cols, int64_t row_stride,
                                                        float* __restrict__ mean_out,
                                                        float* __restrict__ rstd_out,
                                                        int32_t* flag) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5);
  if (row >= rows) return;
  row_stats_row(x + row * row_stride, cols, threadIdx.x & 31, mean_out + row, rstd_out + row,
                flag);
}

// launch_center_rows: one warp per row, 16-byte vectors; a no-op (every CTA
// returns at once) unless the statistics raised the matrix's flag.
// out may alias x (in-place centering: every element is read, then written,
// by the same thread)
__global__ void __launch_bounds__(256) center_rows_kernel(const __nv_bfloat16* x,
                                                          int64_t rows, int cols,
                                                          int64_t row_stride, float* mean,
                                                          const int32_t* flag,
                                                          __nv_bfloat16* out) {
  pdl_wait();
  pdl_trigger();
  if (*reinterpret_cast<const volatile int32_t*>(flag) == 0) return;
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5); row < rows;
       row += int64_t(gridDim.x) * warps) {
    const float m = mean[row];
    const float c = __bfloat162float(__float2bfloat16_rn(m));
    const uint4* src = reinterpret_cast<const uint4*>(x + row * row_stride);
    uint4* dst = reinterpret_cast<uint4*>(out + row * int64_t(cols));
    for (int i = lane; i < cols / 8; i += 32) {
      uint4 u = src[i];
      __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) h[e] = __float2bfloat16_rn(__bfloat162float(h[e]) - c);
      dst[i] = u;
    }
    __syncwarp();
    if (lane == 0) mean[row] = m - c;
  }
}

template <typename T>
__global__ void colsum_kernel(const T* __restrict__ w, int64_t rows, int cols,
                              float* __restrict__ out) {
  const int warps = blockDim.x >> 5;
  const int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T* r = w + row * int64_t(cols);
  double s = 0.0;
  for (int c = lane * 8; c < cols; c += 256) {
    float v[8];
    load8(r + c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += double(v[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = float(s);
}

// ------------------------------------------------------------ synthetic fill
// Zeroing of small flag arrays as a kernel: a cudaMemsetAsync issued while
// the copy engines stream hidden states waited ~40-55 us before it ran (CUPTI
// trace of the restore: every per-layer memset of the recompute prefix
// stalled its stream that long).
__global__ void zero_i32_kernel(int32_t* p, int64_t n, int32_t step) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = int32_t(i) * step;  // step 0: zeros; 1: 0, 1, 2, .. (identity page table)
}

__global__ void fill_symmetric_kernel(void* dst, int64_t n, uint64_t seed, uint64_t offset,
                                      float bound, int dtype) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = seed + (offset + uint64_t(i) + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    double u = double(z >> 11) * 0x1p-53;
    float f = float((2.0 * u - 1.0) * double(bound));
    if (dtype == 0) static_cast<float*>(dst)[i] = f;
    else if (dtype == 1) static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(f);
    else static_cast<__half*>(dst)[i] = __float2half_rn(f);
  }
}

// ------------------------------------------------------------ KV scatter (K4)
// One warp per row: [K_row | V_row] (2*d_kv bf16) -> K page slot, V page slot.
__global__ void kv_scatter_kernel(const uint4* __restrict__ rows, int64_t n_rows, KvOut out) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  int seq = 0, local = int(row);
  if (out.cu_seqlens) {
    int lo = 0, hi = out.n_seqs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (__ldg(out.cu_seqlens + mid) <= row) lo = mid;
      else hi = mid - 1;
    }
    seq = lo;
    local = int(row - __ldg(out.cu_seqlens + seq));
  }
  const int pos = (out.seq_start ? __ldg(out.seq_start + seq) : out.start_pos) + local;
  int64_t orow = row;
  if (out.page_table) {
    int page = __ldg(out.page_table + int64_t(seq) * out.table_stride + pos / out.page_size);
    orow = int64_t(page) * out.page_size + pos % out.page_size;
  }
  const int vec = out.d_kv / 8;  // uint4 = 8 bf16
  const uint4* src = rows + row * 2 * vec;
  uint4* kd = static_cast<uint4*>(out.k_base) + orow * vec;
  uint4* vd = static_cast<uint4*>(out.v_base) + orow * vec;
  for (int i = lane; i < vec; i += 32) {
    uint4 a = __ldg(src + i);
    uint4 b = __ldg(src + vec + i);
    kd[i] = a;
    vd[i] = b;
  }
}

// One warp per row: columns [col0, col0 + out.d_kv) of a dense all-heads K
// and V ([n_rows x src_ld] bf16 each) -> this GPU's pages (its heads only;
// the replicated RECOMPUTE prefix of a head-sharded restore).
__global__ void kv_slice_kernel(const uint4* __restrict__ k_src, const uint4* __restrict__ v_src,
                                int src_ld, int col0, int64_t n_rows, KvOut out) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  int64_t orow = row;
  if (out.page_table) {
    const int64_t pos = out.start_pos + row;
    orow = int64_t(__ldg(out.page_table + pos / out.page_size)) * out.page_size +
           pos % out.page_size;
  }
  const int vec = out.d_kv / 8;
  const int64_t so = (row * src_ld + col0) / 8;
  uint4* kd = static_cast<uint4*>(out.k_base) + orow * vec;
  uint4* vd = static_cast<uint4*>(out.v_base) + orow * vec;
  for (int i = lane; i < vec; i += 32) {
    kd[i] = __ldg(k_src + so + i);
    vd[i] = __ldg(v_src + so + i);
  }
}

// One warp per row: K page slot, V page slot -> [K_row | V_row].
__global__ void kv_gather_kernel(KvOut kv, int pos0, int64_t n_rows, uint4* __restrict__ rows) {
  const int warps = blockDim.x >> 5;
  const int64_t row = int64_t(blockIdx.x) * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int64_t pos = pos0 + row;
  int64_t orow = pos;
  if (kv.page_table)
    orow = int64_t(__ldg(kv.page_table + pos / kv.page_size)) * kv.page_size + pos % kv.page_size;
  const int vec = kv.d_kv / 8;
  const uint4* ks = static_cast<const uint4*>(kv.k_base) + orow * vec;
  const uint4* vs = static_cast<const uint4*>(kv.v_base) + orow * vec;
  uint4* dst = rows + row * 2 * vec;
  for (int i = lane; i < vec; i += 32) {
    dst[i] = __ldg(ks + i);
    dst[vec + i] = __ldg(vs + i);
  }
}

}  // namespace

// Tail-split workspace per (device, stream): stream order makes reuse safe
// without a per-launch allocation or a flag reset -- a launch's flags carry
// its epoch, every earlier value differs. (A cudaMallocAsync + flag reset per
// launch put ~20 us of stream gaps around every split GEMM of a restore.)
struct TailWs {
  float* ws = nullptr;
  int32_t* flags = nullptr;
  int slots = 0;
  uint32_t epoch = 0;
};
cudaError_t tail_ws_for(int dev, cudaStream_t stream, int slots, TailWs** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, TailWs> cache;
  std::lock_guard<std::mutex> lock(mu);
  TailWs& t = cache[{dev, stream}];
  if (t.slots < slots) {
    if (t.ws) {  // grow (first large launch on this stream): the old buffer may be in use
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return e;
      cudaFree(t.ws);
      t.ws = nullptr;
      t.slots = 0;
    }
    const size_t ws_bytes = size_t(slots) * 2 * kTailSlotFloats * sizeof(float);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&t.ws), ws_bytes + size_t(slots) * 8);
    if (e != cudaSuccess) return e;
    t.flags = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(t.ws) + ws_bytes);
    e = cudaMemset(t.flags, 0, size_t(slots) * 8);
    if (e != cudaSuccess) return e;
    t.slots = slots;
    t.epoch = 0;
  }
  *out = &t;
  return cudaSuccess;
}

template <int MODE, int BN, bool QKV>
cudaError_t launch_pair_bn(const AMaps& tmA, const CUtensorMap& tmB128, int M, int N, int K,
                           bool bf16_in, const KvOut& out, const GemmOut& g, const EpiArgs& epi,
                           int num_sms, cudaStream_t stream, int Ms, bool split_acc) {
  const uint32_t idesc = umma_idesc_f16(256, BN, bf16_in);
  const int tiles = ((Ms + 255) / 256) * ((N + BN - 1) / BN);
  int grid = 2 * (tiles < num_sms / 2 ? tiles : num_sms / 2);
  // tail split (summation order may change: split_acc callers only)
  static const bool tail_enabled = [] {
    const char* e = getenv("HC_PAIR_TAIL");
    return e ? atoi(e) != 0 : true;
  }();
  float* ws = nullptr;
  int32_t* flags = nullptr;
  uint32_t epoch = 0;
  const int num_kb = (K + kBK - 1) / kBK;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  // (not under graph capture: a replay would reuse the baked-in epoch)
  if (split_acc && tail_enabled && cap == cudaStreamCaptureStatusNone &&
      pair_tail_split(tiles, grid / 2, num_kb)) {
    TailWs* t = nullptr;
    cudaError_t e = tail_ws_for(dev, stream, tiles - pair_full_units(tiles, grid / 2), &t);
    if (e != cudaSuccess) return e;
    ws = t->ws;
    flags = t->flags;
    epoch = ++t->epoch;
  }
  static thread_local int attr_dev = -1;
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_pair_kernel<MODE, BN, QKV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kPairSmem));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  return launch_pdl(tc_gemm_pair_kernel<MODE, BN, QKV>, dim3(grid), dim3(kPairThreads), kPairSmem,
                    stream, tmA, tmB128, M, N, K, out, g, epi, idesc, Ms, ws, flags, epoch);
}

// bn = the B box rows the caller's tensor map has: 128 -> 256-column pair
// tiles, 96 -> 192-column pair tiles (gemm_pick_bn)
template <int MODE>
cudaError_t launch_pair(int bn, const AMaps& tmA, const CUtensorMap& tmB, int M, int N, int K,
                        bool bf16_in, const KvOut& out, const GemmOut& g, const EpiArgs& epi,
                        int num_sms, cudaStream_t stream, int Ms, bool split_acc) {
  if constexpr (MODE == kEpiKv) {
    if (out.q_cols)
      return bn == 96 ? launch_pair_bn<MODE, 192, true>(tmA, tmB, M, N, K, bf16_in, out, g, epi,
                                                        num_sms, stream, Ms, split_acc)
                      : launch_pair_bn<MODE, 256, true>(tmA, tmB, M, N, K, bf16_in, out, g, epi,
                                                        num_sms, stream, Ms, split_acc);
  }
  if (bn == 96)
    return launch_pair_bn<MODE, 192, false>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms,
                                            stream, Ms, split_acc);
  return launch_pair_bn<MODE, 256, false>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream,
                                          Ms, split_acc);
}

// Pair kernel when the problem has enough 256x256 tiles to fill the SM pairs
// (and HC_K1_PAIR != 0); B must then be described with a 128-row box.
bool use_pair(int M, int N, int num_sms) {
  static const int enabled = [] {
    const char* e = getenv("HC_K1_PAIR");
    return e ? atoi(e) : 1;
  }();
  return enabled && M >= 256 && ((M + 255) / 256) * ((N + 255) / 256) >= num_sms / 2;
}

template <int BN, int MODE>
cudaError_t launch_tc(const AMaps& tmA, const CUtensorMap& tmB, int M, int N, int K,
                      bool bf16_in, const KvOut& out, const GemmOut& g, const EpiArgs& epi,
                      int num_sms, cudaStream_t stream, bool split_acc = false, int Ms = 0) {
  if (Ms < M) Ms = M;
  const uint32_t idesc = umma_idesc_f16(kBM, BN, bf16_in);
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {  // once per thread and device: the largest ring any call uses
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kMaxRingSmem));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const RingCfg r = ring_cfg<BN>(gemm_a_box(Ms));  // the caller's A box follows Ms
  // Decode-sized M: a CTA's time is ~(its K blocks) x (a fixed per-MMA cost),
  // whatever the tile width, so the K loop is split over CTAs (fp32 partials
  // + splitk_epilogue_kernel). Not used where bit-identical K/V matter.
  int k_splits = 1;
  const int num_kb = (K + kBK - 1) / kBK;
  if (split_acc && Ms <= kBM && N % 32 == 0) {
    k_splits = std::max(1, std::min(num_sms / std::max(1, tiles), num_kb / 2));
    const int kb_per = (num_kb + k_splits - 1) / k_splits;
    k_splits = (num_kb + kb_per - 1) / kb_per;  // no empty K slice
  }
  float* part = nullptr;
  if (k_splits > 1) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&part),
                                    size_t(k_splits) * size_t(M) * size_t(N) * sizeof(float), stream);
    if (e != cudaSuccess) return e;
  }
  const int grid_k = std::min(num_sms, tiles * k_splits);
  {
    cudaError_t e = launch_pdl(tc_gemm_kernel<BN, MODE>, dim3(grid_k), dim3(kThreads), r.smem,
                               stream, tmA, tmB, M, N, K, out, g, epi, idesc, r.stages, r.kbs,
                               r.stride, r.a_bytes, k_splits, part);
    if (e != cudaSuccess) return e;
  }
  if (k_splits > 1) {
    const int64_t threads = int64_t(M) * (N / 32) * 32;
    cudaError_t e = launch_pdl(splitk_epilogue_kernel<MODE>, dim3(unsigned((threads + 255) / 256)),
                               dim3(256), 0, stream, static_cast<const float*>(part), k_splits,
                               M, N, out, g, epi);
    if (e != cudaSuccess) return e;
    cudaFreeAsync(part, stream);
  }
  (void)grid;
  return cudaGetLastError();
}

int gemm_a_box(int64_t M) {
  static const int forced = [] {  // HC_GEMM_ABOX=128: disable the compact ring (experiments)
    const char* e = getenv("HC_GEMM_ABOX");
    return e ? atoi(e) : 0;
  }();
  if (forced == 128) return 128;
  return M <= 32 ? 32 : M <= 64 ? 64 : 128;
}

int gemm_pick_bn(int64_t M, int N, int num_sms) {
  if (use_pair(int(M), N, num_sms)) {
    // pair kernel with 256-column tiles (B box of 128 rows). 192-column
    // tiles (B box of 96 rows; HC_PAIR_BN=192 for A/B runs) fill the last
    // wave better -- N=4096 at 4096 rows: 5 waves x 192 vs 4 x 256 columns
    // -- but measured slower per GEMM on the 7B layer (scripts/ab_pair_bn.sh:
    // QKV 290 -> 332 us, O 118 -> 126, FC2 280 -> 334), so 256 it is
    static const int forced = [] {
      const char* e = getenv("HC_PAIR_BN");
      return e ? atoi(e) : 0;
    }();
    return forced == 192 ? 96 : 128;
  }
  static const int forced_bn = [] {  // HC_GEMM_BN: force the small-M tile width (experiments)
    const char* e = getenv("HC_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  if (M <= kBM && (forced_bn == 32 || forced_bn == 64 || forced_bn == 128 || forced_bn == 256))
    return forced_bn;
  if (M <= kBM) {
    // one M tile (decode-sized): the GEMM streams W once, so spread its
    // columns over every SM -- fewest column-waves x tile width, ties to
    // the wider tile
    int best = 256;
    int64_t best_cost = INT64_MAX;
    for (int bn : {256, 128, 64, 32}) {
      const int64_t tiles = (N + bn - 1) / bn;
      const int64_t cost = ((tiles + num_sms - 1) / num_sms) * bn;
      if (cost < best_cost) {
        best_cost = cost;
        best = bn;
      }
    }
    return best;
  }
  return ((M + kBM - 1) / kBM) * ((N + 255) / 256) >= num_sms ? 256 : 128;
}

int gemm_pick_bn_skinny(int64_t M, int N, int num_sms) {
  if (M > kBM) return gemm_pick_bn(M, N, num_sms);
  return N >= 256 ? 256 : 128;  // wide tiles; the K split supplies the parallelism
}

namespace {

template <int MODE>
cudaError_t launch_tc_bn(int bn, const AMaps& tmA, const CUtensorMap& tmB, int M, int N,
                         int K, bool bf16_in, const KvOut& out, const GemmOut& g,
                         const EpiArgs& epi, int num_sms, cudaStream_t stream, bool split_acc,
                         int Ms) {
  switch (bn) {
    case 256:
      return launch_tc<256, MODE>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, split_acc,
                                     Ms);
    case 128:
      return launch_tc<128, MODE>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, split_acc,
                                     Ms);
    case 64:
      return launch_tc<64, MODE>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, split_acc,
                                     Ms);
    case 32:
      return launch_tc<32, MODE>(tmA, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, split_acc,
                                     Ms);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

namespace {
AMaps amaps_with_alt(const CUtensorMap& tmA, const AltA* alt) {
  AMaps am = single_amap(tmA);
  if (alt) {
    am.m[1] = alt->map;
    am.alt_flag = alt->flag;
  }
  return am;
}
}  // namespace

cudaError_t launch_restore_kv(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, int M,
                              int N, int K, bool bf16_in, const KvOut& out, const EpiArgs& epi,
                              int num_sms, cudaStream_t stream, bool split_acc, const AltA* alt,
                              int m_sched) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (out.q_cols) split_acc = false;  // K/V columns: the exact summation order
  const int Ms = std::max(M, m_sched);
  GemmOut g;
  const AMaps am = amaps_with_alt(tmA, alt);
  if ((bn == 128 || bn == 96) && use_pair(Ms, N, num_sms))  // a pair B box (128 / 96 rows)
    return launch_pair<kEpiKv>(bn, am, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, Ms,
                               split_acc);
  return launch_tc_bn<kEpiKv>(bn, am, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream,
                              split_acc, Ms);
}

cudaError_t launch_restore_kv_multi(const AMaps& am, const CUtensorMap& tmB, int bn, int M, int N,
                                    int K, bool bf16_in, const KvOut& out, const EpiArgs& epi,
                                    int num_sms, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (am.n < 1 || am.n > kMaxASrc) return cudaErrorInvalidValue;
  for (int i = 1; i < am.n; ++i)
    if (am.row0[i] % kBM) return cudaErrorInvalidValue;  // a tile reads one source
  GemmOut g;
  if ((bn == 128 || bn == 96) && use_pair(M, N, num_sms))
    return launch_pair<kEpiKv>(bn, am, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, M,
                               false);
  // (no K split: the multi-source path restores K/V, which stay exact)
  return launch_tc_bn<kEpiKv>(bn, am, tmB, M, N, K, bf16_in, out, g, epi, num_sms, stream, false,
                              M);
}

cudaError_t launch_gemm_dense(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, int mode,
                              int M, int N, int K, const GemmOut& g, const EpiArgs& epi,
                              int num_sms, cudaStream_t stream, bool split_acc, const AltA* alt,
                              int m_sched) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int Ms = std::max(M, m_sched);
  KvOut o;
  const AMaps am = amaps_with_alt(tmA, alt);
  if ((bn == 128 || bn == 96) && use_pair(Ms, N, num_sms))
    return mode == kEpiResid
               ? launch_pair<kEpiResid>(bn, am, tmB, M, N, K, true, o, g, epi, num_sms, stream, Ms,
                                        split_acc)
               : launch_pair<kEpiGelu>(bn, am, tmB, M, N, K, true, o, g, epi, num_sms, stream, Ms,
                                       split_acc);
  if (mode == kEpiResid)
    return launch_tc_bn<kEpiResid>(bn, am, tmB, M, N, K, true, o, g, epi, num_sms, stream,
                                   split_acc, Ms);
  return launch_tc_bn<kEpiGelu>(bn, am, tmB, M, N, K, true, o, g, epi, num_sms, stream,
                                split_acc, Ms);
}

cudaError_t launch_row_stats_flagged(const void* x, int64_t rows, int cols, int64_t row_stride,
                                     bool bf16_in, float* mean, float* rstd, int32_t* flag,
                                     cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int threads = 256, per_block = threads / 32;
  const unsigned grid = unsigned((rows + per_block - 1) / per_block);
  if (bf16_in)
    return launch_pdl(row_stats_kernel<__nv_bfloat16>, dim3(grid), dim3(threads), 0, stream,
                      static_cast<const __nv_bfloat16*>(x), rows, cols, row_stride, mean, rstd,
                      flag);
  return launch_pdl(row_stats_kernel<__half>, dim3(grid), dim3(threads), 0, stream,
                    static_cast<const __half*>(x), rows, cols, row_stride, mean, rstd, flag);
}

cudaError_t launch_row_stats(const void* x, int64_t rows, int cols, int64_t row_stride,
                             bool bf16_in, float* mean, float* rstd, cudaStream_t stream) {
  return launch_row_stats_flagged(x, rows, cols, row_stride, bf16_in, mean, rstd, nullptr,
                                  stream);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HC_PDL");
    return !e || atoi(e) != 0;
  }();
  return on;
}

bool qkv_fusion_enabled() {
  static const bool on = [] {
    const char* e = getenv("HC_QKV_FUSED");
    return !e || atoi(e) != 0;
  }();
  return on;
}

bool ln_center_enabled() {
  static const bool on = [] {  // HC_LN_CENTER=0: never center (A/B measurements only)
    const char* e = getenv("HC_LN_CENTER");
    return !e || atoi(e) != 0;
  }();
  return on;
}

cudaError_t launch_center_rows(const void* x, int64_t rows, int cols, int64_t row_stride,
                               float* mean, const int32_t* flag, void* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (cols % 8 != 0 || row_stride % 8 != 0) return cudaErrorInvalidValue;
  const int threads = 256, per_block = threads / 32;
  const int64_t blocks = std::min<int64_t>((rows + per_block - 1) / per_block, 148 * 2);
  return launch_pdl(center_rows_kernel, dim3(unsigned(blocks)), dim3(threads), 0, stream,
                    static_cast<const __nv_bfloat16*>(x), rows, cols, row_stride, mean, flag,
                    static_cast<__nv_bfloat16*>(out));
}

cudaError_t launch_colsum(const void* w, int64_t rows, int cols, bool bf16_in, float* out,
                          cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int threads = 256, per_block = threads / 32;
  const unsigned grid = unsigned((rows + per_block - 1) / per_block);
  if (bf16_in)
    colsum_kernel<__nv_bfloat16><<<grid, threads, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(w), rows, cols, out);
  else
    colsum_kernel<__half><<<grid, threads, 0, stream>>>(static_cast<const __half*>(w), rows, cols,
                                                       out);
  return cudaGetLastError();
}

cudaError_t launch_zero_i32(int32_t* p, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 1024));
  return launch_pdl(zero_i32_kernel, dim3(blocks), dim3(256), 0, stream, p, n, int32_t(0));
}
cudaError_t launch_iota_i32(int32_t* p, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 1024));
  return launch_pdl(zero_i32_kernel, dim3(blocks), dim3(256), 0, stream, p, n, int32_t(1));
}

cudaError_t launch_fill_symmetric(void* dst, int64_t n, uint64_t seed, uint64_t offset,
                                  float bound, int dtype, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  fill_symmetric_kernel<<<unsigned(blocks), 256, 0, stream>>>(dst, n, seed, offset, bound, dtype);
  return cudaGetLastError();
}

cudaError_t launch_kv_scatter(const void* rows, int64_t n_rows, const KvOut& out,
                              cudaStream_t stream) {
  if (n_rows <= 0) return cudaSuccess;
  const int threads = 256, per_block = threads / 32;
  const unsigned grid = unsigned((n_rows + per_block - 1) / per_block);
  return launch_pdl(kv_scatter_kernel, dim3(grid), dim3(threads), 0, stream,
                    static_cast<const uint4*>(rows), n_rows, out);
}

cudaError_t launch_kv_slice(const void* k_src, const void* v_src, int src_ld, int col0,
                            int64_t n_rows, const KvOut& out, cudaStream_t stream) {
  if (n_rows <= 0) return cudaSuccess;
  if (out.d_kv % 8 || src_ld % 8 || col0 % 8 || out.out_f32) return cudaErrorInvalidValue;
  const int warps = 8;
  return launch_pdl(kv_slice_kernel, dim3(unsigned((n_rows + warps - 1) / warps)),
                    dim3(32 * warps), 0, stream, static_cast<const uint4*>(k_src),
                    static_cast<const uint4*>(v_src), src_ld, col0, n_rows, out);
}

cudaError_t launch_kv_gather(const KvOut& kv, int pos0, int64_t n_rows, void* rows,
                             cudaStream_t stream) {
  if (n_rows <= 0) return cudaSuccess;
  const int threads = 256, per_block = threads / 32;
  const unsigned grid = unsigned((n_rows + per_block - 1) / per_block);
  kv_gather_kernel<<<grid, threads, 0, stream>>>(kv, pos0, n_rows, static_cast<uint4*>(rows));
  return cudaGetLastError();
}

}  // namespace hc
