// attention_tc.cu -- K6 causal prefill attention on tcgen05 (sm_100a).
//
// attention_forward (proj/src/model.cpp:237-288) per (query tile of 128,
// head): softmax(Q K^T / sqrt(dh)) V over the paged KV cache, causal.
//   warp 0      TMA: Q tile once; K and V tiles (128 keys) into a 2-stage
//               ring, gathered page by page through the page table.
//   warp 1      TMEM owner + single-thread MMA issuer:
//                 S_j = Q K_j^T   (M=128, N=128, K=dh)   -> TMEM S[j%2]
//                 O  += P_j V_j   (M=128, N=dh, K=128)   -> TMEM O
//               QK_{j+1} is issued before PV_j so the tensor core works on
//               the next tile while the softmax warps handle this one.
//   warps 2-9   softmax, each query row split over two threads (one per
//               64-key half, warps w and w+4 share a TMEM lane quadrant and
//               exchange only the row max through smem): tcgen05.ld of S,
//               scale + causal mask, online softmax in fp32 with exp2 and a
//               lazily updated row max (P <= 2^8, O rescaled in TMEM only
//               when the max grows by more than 8 in log2 units), bf16 P
//               written into the 128-byte-swizzled K-major layout the MMA
//               reads; finally O / l -> bf16 rows in global memory.
// V is consumed as an MN-major B operand straight from its TMA layout.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <vector>

#include "kernels.h"
#include "sm100.cuh"

namespace hc {

namespace {

constexpr int kAttnM = 128;  // queries per CTA
constexpr int kAttnN = 128;  // keys per tile
constexpr int kAttnStages = 2;
constexpr int kAttnThreads = 320;  // TMA, MMA, 8 softmax warps (2 per TMEM lane quadrant)

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// MN-major (N contiguous) 128-byte-swizzled operand: 64 N-elements per
// 128-byte row, K rows at 128 B within 8-row atoms; LBO = stride between
// 64-element N blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo_bytes) {
  return static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4) |
         (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

struct AttnArgs {
  int n;
  int n_heads;
  int group;  // q heads per KV head
  int page_size;
  int box_rows;  // rows per K/V TMA box (min(page_size, 128))
  const int32_t* page_table;  // nullptr: dense rows
  __nv_bfloat16* out;         // [n][n_heads*dh]
  float scale_log2;
  // ragged batch of sequences, each a prefill from position 0 (two-tile
  // kernel only): sequence blockIdx.y owns query rows [cu[y], cu[y+1]) and
  // page-table row y (stride table_stride); nullptr = one sequence of n rows
  const int32_t* cu = nullptr;
  int table_stride = 0;
  // two-tile kernel grid order: true = (heads, sequences, pair rank), false =
  // (pair rank, heads, sequences); see launch_attn_tc
  bool rank_major = false;
};

template <int DH>
struct AttnCfg {
  static constexpr uint32_t kQBytes = kAttnM * DH * 2;
  static constexpr uint32_t kKVBytes = kAttnN * DH * 2;  // one of K or V per stage
  static constexpr uint32_t kStageBytes = 2 * kKVBytes;
  static constexpr uint32_t kPBytes = kAttnM * kAttnN * 2;
  // (no alignment slack: the dynamic smem window starts 1 KB aligned; the
  // kernel traps otherwise)
  static constexpr size_t kSmem = size_t(kQBytes) + size_t(kAttnStages) * kStageBytes +
                                  2 * size_t(kPBytes) + 512 /*bars*/ + 4 * kAttnM * 4 /*xmax*/;
  static constexpr uint32_t kHalf = kAttnM * 64 * 2;  // one 64-column block of a 128-row tile
};

template <int DH>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmK2,
                   const __grid_constant__ CUtensorMap tmV2, AttnArgs a) {
  using Cfg = AttnCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) asm volatile("trap;");  // SW128 operands need 1 KB alignment
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + Cfg::kQBytes;  // stage s: K at s*kStageBytes, V at +kKVBytes
  uint8_t* sP = sKV + kAttnStages * Cfg::kStageBytes;  // two P buffers (tile parity)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * Cfg::kPBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;           // [stages] K tile landed
  uint64_t* k_empty = k_full + kAttnStages;  // [stages] QK done with the K tile
  uint64_t* v_full = k_empty + kAttnStages;  // [stages] V tile landed
  uint64_t* v_empty = v_full + kAttnStages;  // [stages] PV done with the V tile
  uint64_t* s_full = v_empty + kAttnStages;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;  // [2], per P buffer
  uint64_t* o_done = p_full + 2;   // [2], PV_j commits to o_done[j & 1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  uint64_t* v_fix = o_done + 3;    // the last V tile's stale rows are zeroed (see attn_fa_kernel)
  float* xmax = reinterpret_cast<float*>(bars + 32);  // past the barriers + TMEM slot  // [2 parity][2 halves][128 rows]
  // end-of-loop partial sums go into P buffer 0 once every PV has completed
  float* xsum = reinterpret_cast<float*>(sP);  // [2 halves][128 rows]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = int(gridDim.x) - 1 - int(blockIdx.x);  // heaviest causal tiles first
  const int h = blockIdx.y, hk = h / a.group;
  const int q0 = qt * kAttnM;
  const int n_tiles = min(qt + 1, (a.n + kAttnN - 1) / kAttnN);
  const int kv_tiles = (a.n + kAttnN - 1) / kAttnN;
  const int fix_tile = (a.n % kAttnN) && kv_tiles - 1 < n_tiles ? kv_tiles - 1 : -1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK2);
    tma_prefetch_desc(&tmV2);
    mbar_init(q_full, 1);
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&p_full[b], 8);
      mbar_init(&o_done[b], 1);
    }
    mbar_init(v_fix, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + 256;  // O accumulator columns [256, 256+DH)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
      for (int hb = 0; hb < DH / 64; ++hb)
        tma_load_2d(sQ + hb * Cfg::kHalf, &tmQ, q_full, h * DH + hb * 64, q0);
      // K tiles are released by QK, V tiles only by PV: V loads lag K by one
      // tile so a K load never waits behind a P V product
      auto load_tile = [&](int j, bool is_v) {
        const int st = j % kAttnStages;
        uint64_t* full = is_v ? &v_full[st] : &k_full[st];
        mbar_wait(is_v ? &v_empty[st] : &k_empty[st], ((j / kAttnStages) & 1) ^ 1);
        mbar_arrive_expect_tx(full, Cfg::kKVBytes);
        uint8_t* dst = sKV + st * Cfg::kStageBytes + (is_v ? Cfg::kKVBytes : 0);
        const CUtensorMap* map = is_v ? &tmV : &tmK;
        if (a.page_table && a.box_rows < kAttnN) {
          // pages of this tile consecutive in the pool (a freshly allocated
          // session): one 128-row box per head half instead of one per page
          const int last = (a.n - 1) / a.page_size;
          const int pg0 = min(j * kAttnN / a.page_size, last);
          const int per = kAttnN / a.page_size;
          const int base = __ldg(a.page_table + pg0);
          bool contig = pg0 + per - 1 <= last;
          for (int c = 1; c < per && contig; ++c) contig = __ldg(a.page_table + pg0 + c) == base + c;
          if (contig) {
            const CUtensorMap* map2 = is_v ? &tmV2 : &tmK2;
            for (int hb = 0; hb < DH / 64; ++hb)
              tma_load_2d(dst + hb * Cfg::kHalf, map2, full, hk * DH + hb * 64, base * a.page_size);
            return;
          }
        }
        for (int c = 0; c < kAttnN / a.box_rows; ++c) {
          const int key0 = j * kAttnN + c * a.box_rows;
          int row = key0;
          if (a.page_table) {
            const int last = (a.n - 1) / a.page_size;  // keys past n: any valid page (masked)
            const int pg = min(key0 / a.page_size, last);
            row = __ldg(a.page_table + pg) * a.page_size + key0 % a.page_size;
          }
          for (int hb = 0; hb < DH / 64; ++hb)
            tma_load_2d(dst + hb * Cfg::kHalf + c * a.box_rows * 128, map, full,
                        hk * DH + hb * 64, row);
        }
      };
      for (int j = 0; j <= n_tiles; ++j) {
        if (j < n_tiles) load_tile(j, false);
        if (j >= 1) load_tile(j - 1, true);
      }
    }
    __syncwarp();
    if (fix_tile >= 0) {  // zero the V rows past the sequence (attn_fa_kernel)
      const int st = fix_tile % kAttnStages;
      mbar_wait(&v_full[st], (fix_tile / kAttnStages) & 1);
      const int r0 = a.n - fix_tile * kAttnN;
      uint8_t* base = sKV + st * Cfg::kStageBytes + Cfg::kKVBytes;
      const int nvec = (kAttnN - r0) * 128 / 16;
      for (int hb = 0; hb < DH / 64; ++hb) {
        uint4* p = reinterpret_cast<uint4*>(base + hb * Cfg::kHalf + r0 * 128);
        for (int i = lane; i < nvec; i += 32) p[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(v_fix);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA
    if (lane == 0) {
      const uint32_t id_qk = umma_idesc_f16(kAttnM, kAttnN, true);
      const uint32_t id_pv = umma_idesc_f16(kAttnM, DH, true) | (1u << 16);  // B MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_qk = [&](int j) {
        const int st = j % kAttnStages, sb = j & 1;
        const uint32_t sK = smem_u32(sKV + st * Cfg::kStageBytes);
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = uint32_t((kk >> 2) * Cfg::kHalf + (kk & 3) * 32);
          umma_f16(tmem + uint32_t(sb * 128), umma_desc_sw128(smem_u32(sQ) + off),
                   umma_desc_sw128(sK + off), id_qk, kk != 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        umma_commit(&k_empty[st]);
      };
      auto issue_pv = [&](int j) {
        const int st = j % kAttnStages, pb = j & 1;
        const uint32_t sV = smem_u32(sKV + st * Cfg::kStageBytes + Cfg::kKVBytes);
        const uint32_t sPj = smem_u32(sP + pb * Cfg::kPBytes);
        for (int kk = 0; kk < kAttnN / 16; ++kk) {
          const uint64_t pd = umma_desc_sw128(sPj + uint32_t((kk >> 2) * Cfg::kHalf) +
                                              uint32_t((kk & 3) * 32));
          const uint64_t vd = umma_desc_sw128_mn(sV + uint32_t(kk * 2048), Cfg::kHalf);
          umma_f16(t_o, pd, vd, id_pv, (j | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&o_done[pb]);
        umma_commit(&v_empty[st]);
      };
      // event-driven issue: QK_j as soon as its K tile and S buffer are
      // free (up to two tiles ahead of the softmax), PV_j as soon as P_j and
      // V_j are ready -- neither queue blocks the other
      int next_qk = 0, next_pv = 0;
      uint32_t spins = 0;
      while (next_pv < n_tiles) {
        bool progressed = false;
        if (next_qk < n_tiles) {
          const int j = next_qk;
          if (mbar_test(&k_full[j % kAttnStages], (j / kAttnStages) & 1) &&
              mbar_test(&s_empty[j & 1], ((j >> 1) & 1) ^ 1)) {
            tc_fence_after();
            issue_qk(j);
            ++next_qk;
            progressed = true;
          }
        }
        if (next_pv < next_qk) {
          const int j = next_pv;
          if (mbar_test(&p_full[j & 1], (j >> 1) & 1) &&
              mbar_test(&v_full[j % kAttnStages], (j / kAttnStages) & 1) &&
              (j != fix_tile || mbar_test(v_fix, 0))) {
            tc_fence_after();
            issue_pv(j);
            ++next_pv;
            progressed = true;
          }
        }
        if (!progressed && ++spins == (1u << 30)) asm volatile("trap;");
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int q = warp & 3;             // TMEM lane quadrant (rows q*32 .. q*32+31)
    const int half = (warp - 2) >> 2;   // key half (P / S columns) and O column half
    const int rloc = q * 32 + lane;     // row within the tile
    const int row = q0 + rloc;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const uint32_t bar_id = 1 + uint32_t(q);  // named barrier of the two warps of a quadrant
    float m_run = -INFINITY, l_run = 0.f;
    const int r8 = rloc & 7;
    const int prow_off = rloc * 128 + half * Cfg::kHalf;  // my 64-key block of the P row
    auto wait_pv = [&](int k) {
      mbar_wait(&o_done[k & 1], (k >> 1) & 1);
      tc_fence_after();
    };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      float s[64];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_off + uint32_t(sb * 128 + half * 64 + c * 32), v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      // causal / length mask on the diagonal tile only, raw-score max
      const int key0 = j * kAttnN + half * 64;
      const bool diag = key0 + 63 > row || key0 + 64 > a.n;
      if (__any_sync(0xffffffffu, diag)) {  // warp-uniform: only the diagonal / tail tile
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (key0 + i > row || key0 + i >= a.n) s[i] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) mx = fmaxf(mx, s[i]);
      // row max across the two halves (smem, double-buffered by tile parity)
      xmax[(sb * 2 + half) * kAttnM + rloc] = mx;
      pair_sync();
      mx = fmaxf(mx, xmax[(sb * 2 + (half ^ 1)) * kAttnM + rloc]) * a.scale_log2;
      // lazy max: keep m_run unless the tile max exceeds it by > 8 (P <= 2^8)
      const bool rescale = mx > m_run + 8.0f;
      const float m_use = rescale ? mx : m_run;
      uint32_t pk[32];
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        const float p0 = ex2_approx(fmaf(s[i], a.scale_log2, -m_use));
        const float p1 = ex2_approx(fmaf(s[i + 1], a.scale_log2, -m_use));
        sum0 += p0;
        sum1 += p1;
        pk[i >> 1] = pack_bf16x2(p0, p1);
      }
      // P buffer (j & 1) is free once PV_{j-2} is done; an O rescale needs
      // PV_{j-1} done (no PV in flight while O is rewritten)
      if (rescale && j >= 1) wait_pv(j - 1);
      else if (j >= 2) wait_pv(j - 2);
      if (rescale) {
        const float corr = ex2_approx(m_run - m_use);
        l_run *= corr;
        if (j > 0) {
#pragma unroll 1
          for (int c = 0; c < DH / 64; ++c) {
            uint32_t v[32];
            const uint32_t ta = t_o + lane_off + uint32_t(half * (DH / 2) + c * 32);
            tmem_ld_32x32b_x32(ta, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(ta, v);
          }
          tmem_wait_st();
        }
        m_run = m_use;
      }
      l_run += sum0 + sum1;
      uint8_t* prow = sP + (j & 1) * Cfg::kPBytes + prow_off;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(prow + ((ch ^ r8) << 4)) =
            make_uint4(pk[ch * 4], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
      fence_proxy_async_smem();  // generic-proxy P writes -> tensor core (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    wait_pv(n_tiles - 1);  // every PV done: the P buffers are free
    xsum[half * kAttnM + rloc] = l_run;
    pair_sync();
    const float inv = 1.0f / (l_run + xsum[(half ^ 1) * kAttnM + rloc]);
    __nv_bfloat16* dst = a.out + size_t(row) * size_t(a.n_heads * DH) + size_t(h) * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 64; ++c) {
      const int col = half * (DH / 2) + c * 32;
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_o + lane_off + uint32_t(col), v);
      tmem_wait_ld();
      if (row < a.n) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * i + 0]) * inv, __uint_as_float(v[8 * i + 1]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================================
// Two-Q-tile kernel (default): one CTA per (256 queries, head). The two
// 128-row Q tiles A and B share every K/V tile the TMA warp streams in, and
// take turns on the tensor core: while the softmax warps of A turn S_A(j)
// into P_A(j), the tensor core runs P_B(j-1) V and Q_B K(j)^T, and vice versa.
//   TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,256+DH),
//   O_B [384,384+DH). P_t(j) (bf16, two keys per 32-bit column) overwrites
//   the first 64 columns of S_t and is the A operand of O_t += P_t V straight
//   from TMEM -- no smem round trip. QK_t(j+1) is issued after PV_t(j); the
//   tensor pipe executes MMAs in issue order, so it never overwrites P_t(j)
//   before PV_t(j) has read it.
//   warp 0      TMA (Q_A, Q_B once; K(j), V(j-1) into two 2-stage rings)
//   warp 1      TMEM owner + MMA issuer
//   warps 2-9   softmax of tile A, warps 10-17 of tile B (the two overlap on
//               every SM sub-partition): two threads per query row (64 keys
//               each, row max exchanged through smem)
// HC_FA_EMU of every 8 exponential pairs can run as a Cody-Waite + degree-3
// polynomial on the FMA pipe (rel. error 7.5e-5, far below bf16 P's 3.9e-3)
// instead of MUFU. With the SMs 76 % busy (head-major block order) 3 of 8 was
// best; once the launch kept them 94 % busy, all-MUFU won (7B layer 150 ->
// 143 us, 16K x 40 heads 2.44 -> 2.29 ms; scripts/ab_fa_emu.sh), so the
// default is 0. The softmax arithmetic is packed fp32x2 (FFMA2/FADD2) to
// halve its issue slots.
// ============================================================================
constexpr int kFaM = 128;       // rows per Q tile (two per CTA)
constexpr int kFaThreads = 576;  // TMA, MMA, 8 softmax warps per Q tile (two threads per row)
// ROWS variant: TMA, MMA, 4 softmax warps per Q tile, one thread per query row
// holding its 128 scores in registers (one TMEM pass over S, no max exchange)
constexpr int kFaRowsThreads = 320;
template <bool ROWS>
constexpr int fa_threads() { return ROWS ? kFaRowsThreads : kFaThreads; }
#ifndef HC_FA_EMU
#define HC_FA_EMU 0
#endif
#ifndef HC_FA_EXP_NOMAXPASS  // 1: skip the row-max TMEM pass after tile 0 (timing only)
#define HC_FA_EXP_NOMAXPASS 0
#endif
#ifndef HC_FA_SREG  // 1: pass 1 reads both score chunks with one wait and keeps chunk 0 in
                    // registers for pass 2, which reads chunk 1 while chunk 0's exponentials run
#define HC_FA_SREG 1
#endif
#ifndef HC_FA_PCHUNK  // 1: P published per 32-key chunk, 0: once per tile (experiments)
#define HC_FA_PCHUNK 1
#endif
constexpr int kFaEmuPairs = HC_FA_EMU;  // of every 8 exponential pairs, this many on the FMA pipe

template <int DH>
struct FaCfg {
  static constexpr uint32_t kQBytes = kFaM * DH * 2;        // one Q tile
  static constexpr uint32_t kKVBytes = kAttnN * DH * 2;     // one K or V tile
  static constexpr uint32_t kHalf = kFaM * 64 * 2;          // one 64-column block
  // + barriers (256 B) + row max exchange [2 parity][2 tiles][2 halves][128] + row sums [2][2][128]
  static constexpr size_t kSmem = 2 * size_t(kQBytes) + 4 * size_t(kKVBytes) + 256 + 8 * kFaM * 4 + 4 * kFaM * 4;
};

// packed fp32x2 arithmetic (FFMA2 / FADD2: two lanes per instruction)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return uint64_t(__float_as_uint(lo)) | (uint64_t(__float_as_uint(hi)) << 32);
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float(uint32_t(v >> 32)); }
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair, on the FMA pipe: Cody-Waite split x = j + f (j = round(x),
// f in [-0.5, 0.5]) with the 1.5*2^23 trick, degree-3 minimax polynomial for
// 2^f (max rel. error 7.5e-5), j added to the exponent field with one IMAD
// (bits(t) << 23 == j << 23 mod 2^32). x is clamped at -126 so the result
// stays a (possibly subnormal) positive float.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x) {
  x = f2_pack(fmaxf(f2_lo(x), -126.0f), fmaxf(f2_hi(x), -126.0f));
  const uint64_t magic = f2_pack(12582912.0f, 12582912.0f);
  const uint64_t t = f2_add(x, magic);
  const uint64_t f = f2_sub(x, f2_sub(t, magic));
  uint64_t p = f2_fma(f2_pack(0.055170297622680664f, 0.055170297622680664f), f,
                      f2_pack(0.24260802567005157f, 0.24260802567005157f));
  p = f2_fma(p, f, f2_pack(0.693260908126831f, 0.693260908126831f));
  p = f2_fma(p, f, f2_pack(0.9999282956123352f, 0.9999282956123352f));
  uint32_t t_lo, t_hi, p_lo, p_hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(t_lo), "=r"(t_hi) : "l"(t));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(p_lo), "=r"(p_hi) : "l"(p));
  asm("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(t_lo) : "r"(p_lo));  // one IMAD per lane
  asm("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(t_hi) : "r"(p_hi));
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(t_lo), "r"(t_hi));
  return r;
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem], kind::f16 (A K-major in TMEM: lane = row,
// two 16-bit elements per 32-bit column).
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#ifdef HC_FA_TRACE
// per-event SM clocks of one CTA (blockIdx 0,0): [event][tile][j], written to
// host-mapped memory (readable even after the kernel traps)
__device__ unsigned long long* g_fa_trace;
// per CTA (linear block id): globaltimer at entry and exit, SM id, steps
__device__ unsigned long long* g_fa_cta;
#define FA_CTA(slot, v)                                                                         \
  do {                                                                                          \
    if (g_fa_cta && threadIdx.x == 0)                                                           \
      g_fa_cta[(size_t(blockIdx.z) * gridDim.y * gridDim.x + size_t(blockIdx.y) * gridDim.x +   \
                blockIdx.x) * 4 + (slot)] = (v);                                                \
  } while (0)
#define FA_TRACE(ev, t, j)                                                                     \
  do {                                                                                         \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64)                     \
      *reinterpret_cast<volatile unsigned long long*>(g_fa_trace + ((ev) * 2 + (t)) * 64 + (j)) = \
          clock64();                                                                           \
  } while (0)
#else
#define FA_TRACE(ev, t, j) \
  do {                     \
  } while (0)
#define FA_CTA(slot, v) \
  do {                  \
  } while (0)
#endif

template <int DH, bool ROWS>
__global__ void __launch_bounds__(fa_threads<ROWS>(), 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmK2,
                   const __grid_constant__ CUtensorMap tmV2, AttnArgs a) {
  using Cfg = FaCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) asm volatile("trap;");
  pdl_wait();  // (the ragged batch reads cu_seqlens right below)
  pdl_trigger();
  FA_CTA(0, global_ns());
  uint8_t* sQ = smem_raw;                       // Q_A, Q_B
  uint8_t* sK = sQ + 2 * Cfg::kQBytes;          // K ring, 2 stages
  uint8_t* sV = sK + 2 * Cfg::kKVBytes;         // V ring, 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * Cfg::kKVBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;      // [2]
  uint64_t* k_empty = bars + 3;     // [2]
  uint64_t* v_full = bars + 5;      // [2]
  uint64_t* v_empty = bars + 7;     // [2]
  uint64_t* s_full = bars + 9;      // [tile]
  uint64_t* p_full = bars + 11;     // [tile][key chunk]
  uint64_t* o_done = bars + 15;     // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  uint64_t* v_fix = bars + 18;      // the last V tile's stale rows are zeroed
  float* xmax = reinterpret_cast<float*>(bars + 32);  // [j parity][tile][half][row]
  float* xsum = xmax + 8 * kFaM;                      // [tile][half][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ragged batch: this CTA's sequence, its length and its rows / page table
  const int b_head = a.rank_major ? blockIdx.x : blockIdx.y;
  const int b_seq = a.rank_major ? blockIdx.y : blockIdx.z;
  const int b_rank = a.rank_major ? blockIdx.z : blockIdx.x;
  int row0 = 0;  // first query row of the sequence in q / out
  if (a.cu) {
    row0 = __ldg(a.cu + b_seq);
    a.n = __ldg(a.cu + b_seq + 1) - row0;
    if (a.page_table) a.page_table += size_t(b_seq) * size_t(a.table_stride);
  }
  const int n_pairs = (a.n + 2 * kFaM - 1) / (2 * kFaM);
  const int pt = n_pairs - 1 - b_rank;  // heaviest causal tile pairs first
  if (pt < 0) return;  // (ragged batch: a shorter sequence; uniform for the CTA)
  FA_CTA(3, uint64_t(2 * pt + 2));
  const int h = b_head, hk = h / a.group;
  const int q0 = pt * 2 * kFaM;
  const int kv_tiles = (a.n + kAttnN - 1) / kAttnN;
  const int nt_a = min(2 * pt + 1, kv_tiles);
  const int nt_b = min(2 * pt + 2, kv_tiles);  // == nt_a when tile B is past n
  // The KV tile holding key n-1 also holds rows past the sequence: slots of
  // its last page that no token wrote (or, clamped, that page again). Their
  // scores are masked to -inf, so P = 0 there -- but a P x V product over a
  // stale NaN / Inf row is NaN all the same (caller pages are recycled
  // memory). Warp 0 zeroes those V rows in shared memory once the tile has
  // landed, before the PV MMAs of that tile may read it.
  auto fix_tile_of = [&]() { return (a.n % kAttnN) && kv_tiles - 1 < nt_b ? kv_tiles - 1 : -1; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK2);
    tma_prefetch_desc(&tmV2);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      // the tile's softmax warps (8, or 4 in the ROWS variant), per P chunk
      mbar_init(&p_full[2 * s], ROWS ? 4 : 8);
      mbar_init(&p_full[2 * s + 1], ROWS ? 4 : 8);
      mbar_init(&o_done[s], 1);
    }
    mbar_init(v_fix, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * Cfg::kQBytes);
      for (int t = 0; t < 2; ++t)
        for (int hb = 0; hb < DH / 64; ++hb)
          tma_load_2d(sQ + t * Cfg::kQBytes + hb * Cfg::kHalf, &tmQ, q_full, h * DH + hb * 64,
                      row0 + q0 + t * kFaM);
      auto load_tile = [&](int j, bool is_v) {
        const int st = j & 1;
        uint64_t* full = is_v ? &v_full[st] : &k_full[st];
        mbar_wait(is_v ? &v_empty[st] : &k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(full, Cfg::kKVBytes);
        uint8_t* dst = (is_v ? sV : sK) + st * Cfg::kKVBytes;
        const CUtensorMap* map = is_v ? &tmV : &tmK;
        if (a.page_table && a.box_rows < kAttnN) {
          const int last = (a.n - 1) / a.page_size;
          const int pg0 = min(j * kAttnN / a.page_size, last);
          const int per = kAttnN / a.page_size;
          const int base = __ldg(a.page_table + pg0);
          bool contig = pg0 + per - 1 <= last;
          for (int c = 1; c < per && contig; ++c) contig = __ldg(a.page_table + pg0 + c) == base + c;
          if (contig) {
            const CUtensorMap* map2 = is_v ? &tmV2 : &tmK2;
            for (int hb = 0; hb < DH / 64; ++hb)
              tma_load_2d(dst + hb * Cfg::kHalf, map2, full, hk * DH + hb * 64, base * a.page_size);
            return;
          }
        }
        for (int c = 0; c < kAttnN / a.box_rows; ++c) {
          const int key0 = j * kAttnN + c * a.box_rows;
          int row = key0;
          if (a.page_table) {
            const int last = (a.n - 1) / a.page_size;
            const int pg = min(key0 / a.page_size, last);
            row = __ldg(a.page_table + pg) * a.page_size + key0 % a.page_size;
          }
          for (int hb = 0; hb < DH / 64; ++hb)
            tma_load_2d(dst + hb * Cfg::kHalf + c * a.box_rows * 128, map, full,
                        hk * DH + hb * 64, row);
        }
      };
      for (int j = 0; j <= nt_b; ++j) {
        if (j < nt_b) load_tile(j, false);
        if (j >= 1) load_tile(j - 1, true);
      }
    }
    __syncwarp();
    const int fix_tile = fix_tile_of();
    if (fix_tile >= 0) {
      // (the tile's stage is never refilled: it is the last V load)
      const int st = fix_tile & 1;
      mbar_wait(&v_full[st], (fix_tile >> 1) & 1);
      const int r0 = a.n - fix_tile * kAttnN;  // first row past the sequence
      uint8_t* base = sV + st * Cfg::kKVBytes;
      const int nvec = (kAttnN - r0) * 128 / 16;  // 128-byte rows of each 64-column block
      for (int hb = 0; hb < DH / 64; ++hb) {
        uint4* p = reinterpret_cast<uint4*>(base + hb * Cfg::kHalf + r0 * 128);
        for (int i = lane; i < nvec; i += 32) p[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async_smem();  // generic stores -> the tensor core's reads
      __syncwarp();
      if (lane == 0) mbar_arrive(v_fix);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA
    // warp-uniform loop; one elected lane issues (see elect_one)
    const uint32_t id_qk = umma_idesc_f16(kFaM, kAttnN, true);
    const uint32_t id_pv = umma_idesc_f16(kFaM, DH, true) | (1u << 16);  // B (V) MN-major
    const uint64_t dq = umma_desc_sw128(smem_u32(sQ));
    const uint64_t dk = umma_desc_sw128(smem_u32(sK));
    const uint64_t dv = umma_desc_sw128_mn(smem_u32(sV), Cfg::kHalf);
    const int fix_tile = fix_tile_of();
    mbar_wait(q_full, 0);
    tc_fence_after();
    auto issue_qk = [&](int t, int j) {
      const int st = j & 1;
      FA_TRACE(4, t, j);
      mbar_wait(&k_full[st], (j >> 1) & 1);
      tc_fence_after();
      FA_TRACE(0, t, j);
      if (elect_one()) {
        const uint64_t q = dq + uint64_t(t * (Cfg::kQBytes >> 4));
        const uint64_t k = dk + uint64_t(st * (Cfg::kKVBytes >> 4));
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint64_t off = uint64_t(((kk >> 2) * Cfg::kHalf + (kk & 3) * 32) >> 4);
          umma_f16(tmem + uint32_t(t * 128), q + off, k + off, id_qk, kk != 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
        if (t == 1) umma_commit(&k_empty[st]);  // tile B is the last reader of K(j)
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {
      const int st = j & 1;
      FA_TRACE(5, t, j);
      mbar_wait(&v_full[st], (j >> 1) & 1);
      if (j == fix_tile) mbar_wait(v_fix, 0);
      // P arrives in two 32-key chunks per key half; the first chunk's MMAs
      // run while the softmax warps still compute the second
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        mbar_wait(&p_full[2 * t + c], j & 1);
        tc_fence_after();
        if (c == 0) FA_TRACE(1, t, j);
        if (elect_one()) {
          const uint64_t v = dv + uint64_t(st * (Cfg::kKVBytes >> 4));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // P of keys 16kk..: key half kk/4 wrote its 32 columns at the
            // start of its own 64-column S half, chunk c in columns 16c..
            // (ROWS: one thread per row wrote keys 0..127 to columns 0..63,
            // chunk c = keys 64c..64c+63)
            const int kk = ROWS ? c * 4 + u : (u >> 1) * 4 + c * 2 + (u & 1);
            const int pcol = ROWS ? kk * 8 : (kk >> 2) * 64 + (kk & 3) * 8;
            umma_f16_ts(tmem + 256 + uint32_t(t * 128), tmem + uint32_t(t * 128 + pcol),
                        v + uint64_t(kk * (2048 >> 4)), id_pv, (j | kk) != 0 ? 1u : 0u);
          }
          if (c == 1) {
            umma_commit(&o_done[t]);
            if (t == 1) umma_commit(&v_empty[st]);
          }
        }
        __syncwarp();
      }
    };
    issue_qk(0, 0);
    issue_qk(1, 0);
    for (int j = 0; j < nt_b; ++j) {
      if (j < nt_a) {
        issue_pv(0, j);
        if (j + 1 < nt_a) issue_qk(0, j + 1);
      }
      issue_pv(1, j);
      if (j + 1 < nt_b) issue_qk(1, j + 1);
    }
  } else if (ROWS) {
    // ------------------------------------------------------------ softmax (ROWS)
    // warps 2-5 own Q tile A, 6-9 tile B; a thread owns one query row: its
    // 128 scores come out of TMEM once, the row max needs no exchange, and
    // the bf16 P of keys 0..127 goes to columns 0..63 of its S row (the
    // scores are in registers by then). P is published in two 64-key chunks.
    const int t = (warp - 2) >> 2;
    const int qd = warp & 3;  // TMEM lane quadrant (warp % 4)
    const int rloc = qd * 32 + lane;
    const int row = q0 + t * kFaM + rloc;
    const int nt = t == 0 ? nt_a : nt_b;
    const int row_lim = min(row, a.n - 1);
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t t_s = tmem + lane_off + uint32_t(t * 128);
    const uint32_t t_o = tmem + lane_off + 256u + uint32_t(t * 128);
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t sc2 = f2_pack(a.scale_log2, a.scale_log2);
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (rloc == 0) FA_TRACE(2, t, j);
      const int key0 = j * kAttnN;
      const bool diag = __any_sync(0xffffffffu, key0 + kAttnN - 1 > row_lim);
      const int lim = row_lim - key0;
      uint32_t v[128];
      tmem_ld_32x32b_x32(t_s + 0u, *reinterpret_cast<uint32_t(*)[32]>(v + 0));
      tmem_ld_32x32b_x32(t_s + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_ld_32x32b_x32(t_s + 64u, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
      tmem_ld_32x32b_x32(t_s + 96u, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
      tmem_wait_ld();
      if (diag) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i > lim) v[i] = __float_as_uint(-INFINITY);
      }
      if (rloc == 0) FA_TRACE(6, t, j);
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = __uint_as_float(v[u]);
#pragma unroll
      for (int i = 8; i < 128; i += 16)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          m8[u] = fmaxf(m8[u], fmaxf(__uint_as_float(v[i + u]),
                                     __uint_as_float(v[(i + 8 + u) & 127])));
      const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                             fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * a.scale_log2;
      // lazy max: keep m_run unless the tile max exceeds it by > 8 (P <= 2^8)
      const bool resc = mx > m_run + 8.0f;
      const float m_use = resc ? mx : m_run;
      if (rloc == 0) FA_TRACE(7, t, j);
      if (__any_sync(0xffffffffu, resc)) {
        const float corr = resc ? ex2_approx(m_run - m_use) : 1.0f;
        l_run *= corr;
        if (j > 0) {
          mbar_wait(&o_done[t], (j - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + uint32_t(c * 32), o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st_32x32b_x32(t_o + uint32_t(c * 32), o);
          }
        }
        m_run = m_use;
      }
      const uint64_t nm2 = f2_pack(-m_use, -m_use);
      uint64_t sum2 = 0, sum2b = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed columns at a time
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = f2_fma(uint64_t(v[32 * c + 2 * i]) |
                                        (uint64_t(v[32 * c + 2 * i + 1]) << 32),
                                    sc2, nm2);
          const uint64_t pv = f2_pack(ex2_approx(f2_lo(x)), ex2_approx(f2_hi(x)));
          if (i & 1) sum2b = f2_add(sum2b, pv);
          else sum2 = f2_add(sum2, pv);
          pk[i] = pack_bf16x2(f2_lo(pv), f2_hi(pv));
        }
        tmem_st_32x32b_x16(t_s + uint32_t(c * 16), pk);
        if (c & 1) {  // keys 64(c/2)..: publish the chunk
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[2 * t + (c >> 1)]);
        }
      }
      sum2 = f2_add(sum2, sum2b);
      if (rloc == 0) FA_TRACE(3, t, j);
      l_run += f2_lo(sum2) + f2_hi(sum2);
    }
    mbar_wait(&o_done[t], (nt - 1) & 1);
    tc_fence_after();
    const float inv = 1.0f / l_run;
    __nv_bfloat16* dst = a.out + size_t(row0 + row) * size_t(a.n_heads * DH) + size_t(h) * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(t_o + uint32_t(c * 32), o);
      tmem_wait_ld();
      if (row < a.n) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(pack_bf16x2(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv),
                             pack_bf16x2(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv),
                             pack_bf16x2(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv),
                             pack_bf16x2(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv));
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    // warps 2-9 own Q tile A, 10-17 tile B, so the two tiles' softmax
    // overlap on every SM sub-partition. In a tile's group warps w and w+4
    // share a TMEM lane quadrant (32 query rows); `half` selects 64 of the
    // 128 keys (and DH/2 of the O columns). S is read from TMEM in 32-column
    // chunks, twice (row max, then exponentials), to keep registers for
    // instruction-level parallelism; a thread writes the bf16 P of its 64 keys
    // into the first 32 columns of its own S half, so it never overwrites
    // scores its partner has not read.
    const int t = (warp - 2) >> 3;  // Q tile
    const int qd = warp & 3;
    const int half = ((warp - 2) >> 2) & 1;
    const int rloc = qd * 32 + lane;
    const int row = q0 + t * kFaM + rloc;
    const int nt = t == 0 ? nt_a : nt_b;
    const int row_lim = min(row, a.n - 1);  // last visible key of this row
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t t_s = tmem + lane_off + uint32_t(t * 128 + half * 64);  // my S half
    const uint32_t t_o = tmem + lane_off + 256u + uint32_t(t * 128);
    const uint32_t bar_id = 1 + uint32_t(t * 4 + qd);  // named barrier of the row pair
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t sc2 = f2_pack(a.scale_log2, a.scale_log2);
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (rloc == 0 && half == 0) FA_TRACE(2, t, j);
      const int key0 = j * kAttnN + half * 64;
      const bool diag = __any_sync(0xffffffffu, key0 + 63 > row_lim);  // diagonal / tail
      const int lim = row_lim - key0;
      // pass 1: row max of my 64 scores
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = -INFINITY;
#if HC_FA_SREG
      // both 32-column loads in flight at once, one wait; the scores stay in
      // registers for pass 2 (no second TMEM read of S)
      uint32_t sv0[32], sv1[32];
      tmem_ld_32x32b_x32(t_s + 0u, sv0);
      tmem_ld_32x32b_x32(t_s + 32u, sv1);
      tmem_wait_ld();
#endif
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (HC_FA_EXP_NOMAXPASS && j > 0) break;  // timing experiment only (wrong results)
#if HC_FA_SREG
        uint32_t (&v)[32] = c ? sv1 : sv0;
#else
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_s + uint32_t(c * 32), v);
        tmem_wait_ld();
#endif
        if (diag) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i > lim) v[i] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int i = 0; i < 32; i += 16)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            m8[u] = fmaxf(m8[u], fmaxf(__uint_as_float(v[i + u]), __uint_as_float(v[i + 8 + u])));
      }
      if (rloc == 0 && half == 0) FA_TRACE(6, t, j);
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      float* xm = xmax + ((j & 1) * 4 + t * 2) * kFaM;
      xm[half * kFaM + rloc] = mx;
      pair_sync();
      mx = fmaxf(mx, xm[(half ^ 1) * kFaM + rloc]) * a.scale_log2;
      // lazy max: keep m_run unless the tile max exceeds it by > 8 (P <= 2^8)
      const bool resc = mx > m_run + 8.0f;
      const float m_use = resc ? mx : m_run;
      if (rloc == 0 && half == 0) FA_TRACE(7, t, j);
      // O_t rescale (rare with the lazy max), before any P of this step is
      // published: PV_t(j-1) has retired (QK_t(j), whose S we hold, was
      // issued after it), and PV_t(j) waits for p_full below
      if (__any_sync(0xffffffffu, resc)) {
        const float corr = resc ? ex2_approx(m_run - m_use) : 1.0f;
        l_run *= corr;
        if (j > 0) {
          mbar_wait(&o_done[t], (j - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < DH / 64; ++c) {
            uint32_t v[32];
            const uint32_t ta = t_o + uint32_t(half * (DH / 2) + c * 32);
            tmem_ld_32x32b_x32(ta, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(ta, v);
          }
        }
        m_run = m_use;
      }
      // pass 2: P = 2^(s * scale_log2 - m), 32 keys -> 16 columns at a time,
      // each chunk published as soon as it is in TMEM
      const uint64_t nm2 = f2_pack(-m_use, -m_use);
      uint64_t sum2 = 0, sum2b = 0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#if HC_FA_SREG
        if (c == 0) tmem_ld_32x32b_x32(t_s + 32u, sv1);  // in flight during chunk 0
        else tmem_wait_ld();
        uint32_t (&v)[32] = c ? sv1 : sv0;  // chunk 0 masked in pass 1
        if (c == 1 && diag) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 + i > lim) v[i] = __float_as_uint(-INFINITY);
        }
#else
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_s + uint32_t(c * 32), v);
        tmem_wait_ld();
        if (diag) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i > lim) v[i] = __float_as_uint(-INFINITY);
        }
#endif
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = f2_fma(uint64_t(v[2 * i]) | (uint64_t(v[2 * i + 1]) << 32), sc2, nm2);
          uint64_t pv;
          if ((i & 7) < kFaEmuPairs) {
            pv = ex2_poly2(x);
          } else {
            pv = f2_pack(ex2_approx(f2_lo(x)), ex2_approx(f2_hi(x)));
          }
          if (i & 1) sum2b = f2_add(sum2b, pv);
          else sum2 = f2_add(sum2, pv);
          pk[i] = pack_bf16x2(f2_lo(pv), f2_hi(pv));
        }
        // columns c*16.. of my half: scores already read (chunk 0)
        tmem_st_32x32b_x16(t_s + uint32_t(c * 16), pk);
#if HC_FA_PCHUNK
        tmem_wait_st();
        if (c == 1 && rloc == 0 && half == 0) FA_TRACE(9, t, j);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * t + c]);
#else
        if (c == 1) {  // both chunks published together (experiments)
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&p_full[2 * t]);
            mbar_arrive(&p_full[2 * t + 1]);
          }
        }
#endif
      }
      sum2 = f2_add(sum2, sum2b);
      if (rloc == 0 && half == 0) FA_TRACE(8, t, j);
      l_run += f2_lo(sum2) + f2_hi(sum2);
      if (rloc == 0 && half == 0) FA_TRACE(3, t, j);
    }
    xsum[(t * 2 + half) * kFaM + rloc] = l_run;
    mbar_wait(&o_done[t], (nt - 1) & 1);
    tc_fence_after();
    pair_sync();
    const float inv = 1.0f / (l_run + xsum[(t * 2 + (half ^ 1)) * kFaM + rloc]);
    __nv_bfloat16* dst = a.out + size_t(row0 + row) * size_t(a.n_heads * DH) + size_t(h) * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 64; ++c) {
      const int col = half * (DH / 2) + c * 32;
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_o + uint32_t(col), v);
      tmem_wait_ld();
      if (row < a.n) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * i + 0]) * inv, __uint_as_float(v[8 * i + 1]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv),
                             pack_bf16x2(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  FA_CTA(1, global_ns());
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    FA_CTA(2, uint64_t(smid));
  }
}

// ============================================================================
// Persistent variant of the two-Q-tile kernel (one sequence, HC_FA_PERSIST):
// one CTA per SM loops over (head, tile pair) items from a host-computed
// longest-processing-time schedule. Barrier phases run on per-role counters
// across items; the next item's Q load waits for the last QK of the previous
// item (q_empty) and its first PV for the softmax warps to have read O out
// (o_free), so an item's Q load, first QK and first softmax overlap the
// previous item's last PV and O epilogue, and TMEM, barriers and the CTA
// launch are paid once per SM instead of once per item.
template <int DH>
__global__ void __launch_bounds__(kFaThreads, 1)
    attn_fa_persist_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV,
                           const __grid_constant__ CUtensorMap tmK2,
                           const __grid_constant__ CUtensorMap tmV2, AttnArgs a,
                           const int32_t* __restrict__ sched, int sched_stride) {
  using Cfg = FaCfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) asm volatile("trap;");
  pdl_wait();
  pdl_trigger();
  uint8_t* sQ = smem_raw;
  uint8_t* sK = sQ + 2 * Cfg::kQBytes;
  uint8_t* sV = sK + 2 * Cfg::kKVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * Cfg::kKVBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* k_empty = bars + 3;   // [2]
  uint64_t* v_full = bars + 5;    // [2]
  uint64_t* v_empty = bars + 7;   // [2]
  uint64_t* s_full = bars + 9;    // [tile]
  uint64_t* p_full = bars + 11;   // [tile][key chunk]
  uint64_t* o_done = bars + 15;   // [tile]
  uint64_t* v_fix = bars + 17;
  uint64_t* q_empty = bars + 18;  // the item's last QK has read Q
  uint64_t* o_free = bars + 19;   // [tile] the softmax warps have read O out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);
  float* xmax = reinterpret_cast<float*>(bars + 32);  // [step parity][tile][half][row]
  float* xsum = xmax + 8 * kFaM;                      // [tile][half][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* my = sched + size_t(blockIdx.x) * size_t(sched_stride);
  const int n_items = __ldg(my);
  const int n_pairs = (a.n + 2 * kFaM - 1) / (2 * kFaM);
  const int kv_tiles = (a.n + kAttnN - 1) / kAttnN;
  struct Item {
    int h, hk, q0, nt_a, nt_b, fix;
  };
  auto item = [&](int i) {
    const int w = __ldg(my + 1 + i);  // rank-major: head fastest
    Item it;
    it.h = w % a.n_heads;
    const int pt = n_pairs - 1 - w / a.n_heads;
    it.hk = it.h / a.group;
    it.q0 = pt * 2 * kFaM;
    it.nt_a = min(2 * pt + 1, kv_tiles);
    it.nt_b = min(2 * pt + 2, kv_tiles);
    it.fix = (a.n % kAttnN) && kv_tiles - 1 < it.nt_b ? kv_tiles - 1 : -1;
    return it;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK2);
    tma_prefetch_desc(&tmV2);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[2 * s], 8);
      mbar_init(&p_full[2 * s + 1], 8);
      mbar_init(&o_done[s], 1);
      mbar_init(&o_free[s], 8);
    }
    mbar_init(v_fix, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA
    int gk = 0, gv = 0;  // K / V tiles loaded by this CTA so far (ring position)
    for (int i = 0; i < n_items; ++i) {
      const Item it = item(i);
      if (lane == 0) {
        if (i > 0) mbar_wait(q_empty, (i - 1) & 1);
        mbar_arrive_expect_tx(q_full, 2 * Cfg::kQBytes);
        for (int t = 0; t < 2; ++t)
          for (int hb = 0; hb < DH / 64; ++hb)
            tma_load_2d(sQ + t * Cfg::kQBytes + hb * Cfg::kHalf, &tmQ, q_full,
                        it.h * DH + hb * 64, it.q0 + t * kFaM);
        auto load_tile = [&](int g, int j, bool is_v) {
          const int st = g & 1;
          uint64_t* full = is_v ? &v_full[st] : &k_full[st];
          mbar_wait(is_v ? &v_empty[st] : &k_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(full, Cfg::kKVBytes);
          uint8_t* dst = (is_v ? sV : sK) + st * Cfg::kKVBytes;
          const CUtensorMap* map = is_v ? &tmV : &tmK;
          if (a.page_table && a.box_rows < kAttnN) {
            const int last = (a.n - 1) / a.page_size;
            const int pg0 = min(j * kAttnN / a.page_size, last);
            const int per = kAttnN / a.page_size;
            const int base = __ldg(a.page_table + pg0);
            bool contig = pg0 + per - 1 <= last;
            for (int c = 1; c < per && contig; ++c)
              contig = __ldg(a.page_table + pg0 + c) == base + c;
            if (contig) {
              const CUtensorMap* map2 = is_v ? &tmV2 : &tmK2;
              for (int hb = 0; hb < DH / 64; ++hb)
                tma_load_2d(dst + hb * Cfg::kHalf, map2, full, it.hk * DH + hb * 64,
                            base * a.page_size);
              return;
            }
          }
          for (int c = 0; c < kAttnN / a.box_rows; ++c) {
            const int key0 = j * kAttnN + c * a.box_rows;
            int row = key0;
            if (a.page_table) {
              const int last = (a.n - 1) / a.page_size;
              const int pg = min(key0 / a.page_size, last);
              row = __ldg(a.page_table + pg) * a.page_size + key0 % a.page_size;
            }
            for (int hb = 0; hb < DH / 64; ++hb)
              tma_load_2d(dst + hb * Cfg::kHalf + c * a.box_rows * 128, map, full,
                          it.hk * DH + hb * 64, row);
          }
        };
        for (int j = 0; j <= it.nt_b; ++j) {
          if (j < it.nt_b) load_tile(gk + j, j, false);
          if (j >= 1) load_tile(gv + j - 1, j - 1, true);
        }
      }
      __syncwarp();
      if (it.fix >= 0) {  // zero the last V tile's rows past the sequence (attn_fa_kernel)
        const int g = gv + it.fix, st = g & 1;
        mbar_wait(&v_full[st], (g >> 1) & 1);
        const int r0 = a.n - it.fix * kAttnN;
        uint8_t* base = sV + st * Cfg::kKVBytes;
        const int nvec = (kAttnN - r0) * 128 / 16;
        for (int hb = 0; hb < DH / 64; ++hb) {
          uint4* p = reinterpret_cast<uint4*>(base + hb * Cfg::kHalf + r0 * 128);
          for (int e = lane; e < nvec; e += 32) p[e] = make_uint4(0u, 0u, 0u, 0u);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(v_fix);
      }
      gk += it.nt_b;
      gv += it.nt_b;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA
    const uint32_t id_qk = umma_idesc_f16(kFaM, kAttnN, true);
    const uint32_t id_pv = umma_idesc_f16(kFaM, DH, true) | (1u << 16);
    const uint64_t dq = umma_desc_sw128(smem_u32(sQ));
    const uint64_t dk = umma_desc_sw128(smem_u32(sK));
    const uint64_t dv = umma_desc_sw128_mn(smem_u32(sV), Cfg::kHalf);
    int gk = 0, gv = 0, nfix = 0;
    int pvc[2] = {0, 0};  // PV steps issued per tile (= o_done / p_full phases)
    for (int i = 0; i < n_items; ++i) {
      const Item it = item(i);
      mbar_wait(q_full, i & 1);
      tc_fence_after();
      auto issue_qk = [&](int t, int j) {
        const int g = gk + j, st = g & 1;
        mbar_wait(&k_full[st], (g >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t q = dq + uint64_t(t * (Cfg::kQBytes >> 4));
          const uint64_t k = dk + uint64_t(st * (Cfg::kKVBytes >> 4));
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint64_t off = uint64_t(((kk >> 2) * Cfg::kHalf + (kk & 3) * 32) >> 4);
            umma_f16(tmem + uint32_t(t * 128), q + off, k + off, id_qk, kk != 0 ? 1u : 0u);
          }
          umma_commit(&s_full[t]);
          if (t == 1) {
            umma_commit(&k_empty[st]);
            if (j == it.nt_b - 1) umma_commit(q_empty);  // the item's last read of Q
          }
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const int g = gv + j, st = g & 1;
        mbar_wait(&v_full[st], (g >> 1) & 1);
        if (j == it.fix) mbar_wait(v_fix, nfix & 1);
        if (j == 0 && i > 0) mbar_wait(&o_free[t], (i - 1) & 1);  // O of the last item read out
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_wait(&p_full[2 * t + c], (pvc[t] + j) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t v = dv + uint64_t(st * (Cfg::kKVBytes >> 4));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int kk = (u >> 1) * 4 + c * 2 + (u & 1);
              umma_f16_ts(tmem + 256 + uint32_t(t * 128),
                          tmem + uint32_t(t * 128 + (kk >> 2) * 64 + (kk & 3) * 8),
                          v + uint64_t(kk * (2048 >> 4)), id_pv, (j | kk) != 0 ? 1u : 0u);
            }
            if (c == 1) {
              umma_commit(&o_done[t]);
              if (t == 1) umma_commit(&v_empty[st]);
            }
          }
          __syncwarp();
        }
      };
      issue_qk(0, 0);
      issue_qk(1, 0);
      for (int j = 0; j < it.nt_b; ++j) {
        if (j < it.nt_a) {
          issue_pv(0, j);
          if (j + 1 < it.nt_a) issue_qk(0, j + 1);
        }
        issue_pv(1, j);
        if (j + 1 < it.nt_b) issue_qk(1, j + 1);
      }
      gk += it.nt_b;
      gv += it.nt_b;
      pvc[0] += it.nt_a;
      pvc[1] += it.nt_b;
      if (it.fix >= 0) ++nfix;
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int t = (warp - 2) >> 3;
    const int qd = warp & 3;
    const int half = ((warp - 2) >> 2) & 1;
    const int rloc = qd * 32 + lane;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t t_s = tmem + lane_off + uint32_t(t * 128 + half * 64);
    const uint32_t t_o = tmem + lane_off + 256u + uint32_t(t * 128);
    const uint32_t bar_id = 1 + uint32_t(t * 4 + qd);
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    const uint64_t sc2 = f2_pack(a.scale_log2, a.scale_log2);
    int sc = 0;  // steps of my tile so far (s_full / o_done phases, xmax parity)
    for (int i = 0; i < n_items; ++i) {
      const Item it = item(i);
      const int row = it.q0 + t * kFaM + rloc;
      const int nt = t == 0 ? it.nt_a : it.nt_b;
      const int row_lim = min(row, a.n - 1);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nt; ++j) {
        const int g = sc + j;
        mbar_wait(&s_full[t], g & 1);
        tc_fence_after();
        const int key0 = j * kAttnN + half * 64;
        const bool diag = __any_sync(0xffffffffu, key0 + 63 > row_lim);
        const int lim = row_lim - key0;
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = -INFINITY;
#if HC_FA_SREG
        uint32_t sv0[32], sv1[32];
        tmem_ld_32x32b_x32(t_s + 0u, sv0);
        tmem_ld_32x32b_x32(t_s + 32u, sv1);
        tmem_wait_ld();
#endif
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#if HC_FA_SREG
          uint32_t (&v)[32] = c ? sv1 : sv0;
#else
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_s + uint32_t(c * 32), v);
          tmem_wait_ld();
#endif
          if (diag) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e > lim) v[e] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int e = 0; e < 32; e += 16)
#pragma unroll
            for (int u = 0; u < 8; ++u)
              m8[u] = fmaxf(m8[u], fmaxf(__uint_as_float(v[e + u]), __uint_as_float(v[e + 8 + u])));
        }
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        float* xm = xmax + ((g & 1) * 4 + t * 2) * kFaM;
        xm[half * kFaM + rloc] = mx;
        pair_sync();
        mx = fmaxf(mx, xm[(half ^ 1) * kFaM + rloc]) * a.scale_log2;
        const bool resc = mx > m_run + 8.0f;
        const float m_use = resc ? mx : m_run;
        if (__any_sync(0xffffffffu, resc)) {
          const float corr = resc ? ex2_approx(m_run - m_use) : 1.0f;
          l_run *= corr;
          if (j > 0) {
            mbar_wait(&o_done[t], (g - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < DH / 64; ++c) {
              uint32_t v[32];
              const uint32_t ta = t_o + uint32_t(half * (DH / 2) + c * 32);
              tmem_ld_32x32b_x32(ta, v);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * corr);
              tmem_st_32x32b_x32(ta, v);
            }
          }
          m_run = m_use;
        }
        const uint64_t nm2 = f2_pack(-m_use, -m_use);
        uint64_t sum2 = 0, sum2b = 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#if HC_FA_SREG
          if (c == 0) tmem_ld_32x32b_x32(t_s + 32u, sv1);  // in flight during chunk 0
          else tmem_wait_ld();
          uint32_t (&v)[32] = c ? sv1 : sv0;  // chunk 0 masked in pass 1
          if (c == 1 && diag) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (32 + e > lim) v[e] = __float_as_uint(-INFINITY);
          }
#else
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_s + uint32_t(c * 32), v);
          tmem_wait_ld();
          if (diag) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e > lim) v[e] = __float_as_uint(-INFINITY);
          }
#endif
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint64_t x = f2_fma(uint64_t(v[2 * e]) | (uint64_t(v[2 * e + 1]) << 32), sc2, nm2);
            const uint64_t pv = f2_pack(ex2_approx(f2_lo(x)), ex2_approx(f2_hi(x)));
            if (e & 1) sum2b = f2_add(sum2b, pv);
            else sum2 = f2_add(sum2, pv);
            pk[e] = pack_bf16x2(f2_lo(pv), f2_hi(pv));
          }
          tmem_st_32x32b_x16(t_s + uint32_t(c * 16), pk);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[2 * t + c]);
        }
        sum2 = f2_add(sum2, sum2b);
        l_run += f2_lo(sum2) + f2_hi(sum2);
      }
      xsum[(t * 2 + half) * kFaM + rloc] = l_run;
      mbar_wait(&o_done[t], (sc + nt - 1) & 1);
      tc_fence_after();
      pair_sync();
      const float inv = 1.0f / (l_run + xsum[(t * 2 + (half ^ 1)) * kFaM + rloc]);
      __nv_bfloat16* dst = a.out + size_t(row) * size_t(a.n_heads * DH) + size_t(it.h) * DH;
#pragma unroll 1
      for (int c = 0; c < DH / 64; ++c) {
        const int col = half * (DH / 2) + c * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_o + uint32_t(col), v);
        tmem_wait_ld();
        if (row < a.n) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            d4[e] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * e + 0]) * inv, __uint_as_float(v[8 * e + 1]) * inv),
                               pack_bf16x2(__uint_as_float(v[8 * e + 2]) * inv, __uint_as_float(v[8 * e + 3]) * inv),
                               pack_bf16x2(__uint_as_float(v[8 * e + 4]) * inv, __uint_as_float(v[8 * e + 5]) * inv),
                               pack_bf16x2(__uint_as_float(v[8 * e + 6]) * inv, __uint_as_float(v[8 * e + 7]) * inv));
        }
      }
      // O of this item is in registers / global memory: the next item's
      // first PV may overwrite it; the partner's xsum read is behind the
      // pair_sync above, and the next item's xsum write is many syncs later
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      sc += nt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Longest-processing-time schedule of a single sequence's (head, pair) items
// over `grid` CTAs, cached per (device, n, heads, grid): row c = [count,
// item ids...]; items in rank-major order (head fastest), cost ~ fixed + key
// steps of the pair.
const int32_t* fa_persist_schedule(int n, int n_heads, int grid, bool head_major,
                                   cudaStream_t stream, int* stride_out) {
  struct Key {
    int dev, n, heads, grid;
    bool hm;
    bool operator<(const Key& o) const {
      return std::tie(dev, n, heads, grid, hm) < std::tie(o.dev, o.n, o.heads, o.grid, o.hm);
    }
  };
  static std::mutex mu;
  struct Entry {
    int32_t* dev;
    int stride;
    std::vector<int32_t> host;  // the copy's source, alive as long as the entry
    cudaEvent_t ready;          // the upload on the private stream
  };
  static std::map<Key, Entry> cache;
  static std::map<int, cudaStream_t> upload;  // per device, nothing else queued on it
  int dev = 0;
  cudaGetDevice(&dev);
  const Key key{dev, n, n_heads, grid, head_major};
  std::lock_guard<std::mutex> lk(mu);
  auto f = cache.find(key);
  if (f != cache.end()) {
    if (cudaStreamWaitEvent(stream, f->second.ready, 0) != cudaSuccess) return nullptr;
    *stride_out = f->second.stride;
    return f->second.dev;
  }
  // bounded: schedules are kept for the process (a launch may still read
  // one), so past 64 shapes (a serving run's many context lengths) new
  // shapes take the grid kernel instead
  if (cache.size() >= 64) return nullptr;
  const int pairs = (n + 2 * kFaM - 1) / (2 * kFaM), kv_tiles = (n + kAttnN - 1) / kAttnN;
  const int items = pairs * n_heads;
  std::vector<std::vector<int32_t>> lists(static_cast<size_t>(grid));
  std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>,
                      std::greater<std::pair<double, int>>>
      load;
  for (int c = 0; c < grid; ++c) load.push({0.0, c});
  // head_major: the items of one head (heaviest pair first) before the next
  // head's, so the CTAs working at any moment share a few heads' K/V in L2
  for (int o = 0; o < items; ++o) {
    const int w = head_major ? (o % pairs) * n_heads + o / pairs : o;
    const int pt = pairs - 1 - w / n_heads;
    const double cost = 2.5 + 2.24 * (std::min(2 * pt + 1, kv_tiles) + std::min(2 * pt + 2, kv_tiles)) / 2.0;
    auto top = load.top();
    load.pop();
    lists[size_t(top.second)].push_back(w);
    load.push({top.first + cost, top.second});
  }
  size_t mx = 0;
  for (const auto& l : lists) mx = std::max(mx, l.size());
  const int stride = int(mx) + 1;
  std::vector<int32_t> host(size_t(grid) * size_t(stride), 0);
  for (int c = 0; c < grid; ++c) {
    host[size_t(c) * size_t(stride)] = int32_t(lists[size_t(c)].size());
    std::copy(lists[size_t(c)].begin(), lists[size_t(c)].end(),
              host.begin() + std::ptrdiff_t(size_t(c) * size_t(stride) + 1));
  }
  // uploaded on a private stream and ordered before the launch by an event:
  // no device-wide synchronisation when a new shape shows up in the middle
  // of a restore or a serving run, and launches on any stream wait for it;
  // never freed
  cudaStream_t& up = upload[dev];
  if (!up && cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  int32_t* d = nullptr;
  cudaEvent_t ev = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&d), host.size() * sizeof(int32_t), up) !=
          cudaSuccess ||
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  auto& e = cache[key];
  e.dev = d;
  e.stride = stride;
  e.host = std::move(host);
  e.ready = ev;
  if (cudaMemcpyAsync(d, e.host.data(), e.host.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                      up) != cudaSuccess ||
      cudaEventRecord(ev, up) != cudaSuccess || cudaStreamWaitEvent(stream, ev, 0) != cudaSuccess) {
    cache.erase(key);
    return nullptr;
  }
  *stride_out = stride;
  return d;
}

template <int DH>
cudaError_t launch_attn_tc(const void* q, int n, int n_heads, int n_kv_heads, const KvOut& kv,
                           int64_t kv_rows, void* out, cudaStream_t stream,
                           const int32_t* cu = nullptr, int n_seqs = 1, int max_len = 0) {
  const int box_rows = kv.page_table ? (kv.page_size < kAttnN ? kv.page_size : kAttnN) : kAttnN;
  CUtensorMap tq, tk, tv, tk2, tv2;
  const uint64_t ldq = uint64_t(n_heads) * DH;
  if (!make_tmap_kmajor(&tq, q, ldq, uint64_t(n), ldq * 2, kAttnM)) return cudaErrorInvalidValue;
  // K/V maps cover the whole page pool (rows are gathered page by page) or,
  // dense, the n rows (tiles past n are zero-filled by TMA and masked)
  const uint64_t rows = kv.page_table ? uint64_t(kv_rows) : uint64_t(n);
  if (!make_tmap_kmajor(&tk, kv.k_base, uint64_t(kv.d_kv), rows, uint64_t(kv.d_kv) * 2,
                        uint32_t(box_rows)) ||
      !make_tmap_kmajor(&tv, kv.v_base, uint64_t(kv.d_kv), rows, uint64_t(kv.d_kv) * 2,
                        uint32_t(box_rows)) ||
      !make_tmap_kmajor(&tk2, kv.k_base, uint64_t(kv.d_kv), rows, uint64_t(kv.d_kv) * 2, kAttnN) ||
      !make_tmap_kmajor(&tv2, kv.v_base, uint64_t(kv.d_kv), rows, uint64_t(kv.d_kv) * 2, kAttnN))
    return cudaErrorInvalidValue;
  AttnArgs a;
  a.n = n;
  a.n_heads = n_heads;
  a.group = n_heads / n_kv_heads;
  a.page_size = kv.page_table ? kv.page_size : n;
  a.box_rows = box_rows;
  a.page_table = kv.page_table;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.scale_log2 = (1.0f / sqrtf(float(DH))) * 1.4426950408889634f;
  a.cu = cu;
  a.table_stride = kv.table_stride;
  // HC_ATTN_TC=1: the one-Q-tile kernel (kept for A/B measurements)
  static const bool two_tile = [] {
    const char* e = getenv("HC_ATTN_TC");
    return !e || atoi(e) != 1;
  }();
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<DH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(AttnCfg<DH>::kSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_fa_kernel<DH, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(FaCfg<DH>::kSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_fa_kernel<DH, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(FaCfg<DH>::kSmem));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  if (cu || two_tile) {
    // Block order. The scheduler dispatches x fastest. Rank-major (heads,
    // sequences, pair rank) hands out every head's heaviest causal tile pair
    // before any lighter one -- longest-first over the launch; head-major
    // (pair rank, heads, sequences) left the heaviest pairs of the last heads
    // running alone at the end (7B 4K: SMs 76 % busy, 176 us; rank-major 94 %,
    // 145 us). Head-major keeps one head's K/V hot in L2 while its pairs run,
    // which wins once the launch's K/V outgrows L2 (16K x 40 heads: 2.37 vs
    // 2.42 ms), so rank-major is used while K/V fits in 80 MB.
    const int pairs = ((cu ? max_len : n) + 2 * kFaM - 1) / (2 * kFaM);
    const double kv_bytes = double(n) * double(n_kv_heads) * DH * 2 * 2;  // n = total rows
    a.rank_major = kv_bytes <= 80.0 * (1 << 20);
    const dim3 grid = a.rank_major ? dim3(n_heads, n_seqs, pairs) : dim3(pairs, n_heads, n_seqs);
    // One persistent CTA per SM over an LPT schedule for a single sequence
    // whose K/V fit in L2 (7B 4K: 138.8 -> 135.2 us). Past that size the
    // head-major grid's L2 locality wins (16K x 40 heads: 2347 us grid vs
    // 2420 persistent), and a ragged batch's lengths are not on the host.
    // HC_FA_PERSIST=0 / 1 forces it off / on (single sequence).
    static const int persist_env = [] {
      const char* e = getenv("HC_FA_PERSIST");
      return e ? atoi(e) : -1;
    }();
    bool persist = persist_env < 0 ? a.rank_major : persist_env != 0;
    if (persist) {  // (the schedule upload is not capturable: graphs keep the grid kernel)
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(stream, &cap);
      persist = cap == cudaStreamCaptureStatusNone;
    }
    // (HC_FA_PERSIST=2: persistent with the head-major item order as well)
    if (persist && !cu) {
      static thread_local int pattr_dev = -1;
      if (pattr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(attn_fa_persist_kernel<DH>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(FaCfg<DH>::kSmem));
        if (e != cudaSuccess) return e;
        pattr_dev = dev;
      }
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int items = pairs * n_heads;
      const int pgrid = std::min(sms, items);
      int stride = 0;
      const int32_t* sched = fa_persist_schedule(n, n_heads, pgrid,
                                                 !a.rank_major && persist_env == 2, stream,
                                                 &stride);
      if (sched)
        return launch_pdl(attn_fa_persist_kernel<DH>, dim3(pgrid), dim3(kFaThreads),
                          FaCfg<DH>::kSmem, stream, tq, tk, tv, tk2, tv2, a, sched, stride);
    }
    // HC_FA_ROWS=1: one softmax thread per query row (ROWS variant)
    static const bool rows = [] {
      const char* e = getenv("HC_FA_ROWS");
      return e && atoi(e) != 0;
    }();
    if (rows)
      return launch_pdl(attn_fa_kernel<DH, true>, grid, dim3(kFaRowsThreads), FaCfg<DH>::kSmem,
                        stream, tq, tk, tv, tk2, tv2, a);
    return launch_pdl(attn_fa_kernel<DH, false>, grid, dim3(kFaThreads), FaCfg<DH>::kSmem, stream,
                      tq, tk, tv, tk2, tv2, a);
  } else {
    const dim3 grid((n + kAttnM - 1) / kAttnM, n_heads);
    attn_tc_kernel<DH><<<grid, kAttnThreads, AttnCfg<DH>::kSmem, stream>>>(tq, tk, tv, tk2, tv2, a);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_tc(const void* q, int n, int n_heads, int n_kv_heads, int dh,
                                const KvOut& kv, int64_t kv_rows, void* out,
                                cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (kv.page_table && (kv.page_size & (kv.page_size - 1)) != 0) return cudaErrorInvalidValue;
  if (kv.page_table && kv.page_size < 8) return cudaErrorInvalidValue;
  if (dh == 128) return launch_attn_tc<128>(q, n, n_heads, n_kv_heads, kv, kv_rows, out, stream);
  if (dh == 64) return launch_attn_tc<64>(q, n, n_heads, n_kv_heads, kv, kv_rows, out, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attention_tc_varlen(const void* q, int64_t total, int n_seqs, int max_len,
                                       const int32_t* cu, int n_heads, int n_kv_heads, int dh,
                                       const KvOut& kv, int64_t kv_rows, void* out,
                                       cudaStream_t stream) {
  if (total <= 0 || n_seqs <= 0 || max_len <= 0) return cudaSuccess;
  if (!cu || !kv.page_table || kv.page_size < 8 || (kv.page_size & (kv.page_size - 1)) != 0)
    return cudaErrorInvalidValue;
  if (dh == 128)
    return launch_attn_tc<128>(q, int(total), n_heads, n_kv_heads, kv, kv_rows, out, stream, cu,
                               n_seqs, max_len);
  if (dh == 64)
    return launch_attn_tc<64>(q, int(total), n_heads, n_kv_heads, kv, kv_rows, out, stream, cu,
                              n_seqs, max_len);
  return cudaErrorInvalidValue;
}

}  // namespace hc
