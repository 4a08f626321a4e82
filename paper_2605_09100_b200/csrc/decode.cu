// decode.cu -- hybrid paged decode attention for sm_100a (SURVEY §8(a) a4 + a5).
//
// What it computes (§3 HPA; reading A1/A8):
// for each request b and kv-head h, the G = Hq/H_kv query heads of its LAST
// logical row attend every stored row of the block table (latent and token
// pages alike -- the kernel is kind-agnostic):
//   o[b][hq] = sum_j softmax_j(scale * q.K_log[h][j]) V_log[h][j],  h = hq / G.
//
// Design (B200-first, HBM-bound; roofline in DESIGN.md "Kernels"):
//  * grid (split, kv-head, request); one CTA = 1 TMA producer warp + NCONS
//    consumer warps. The producer walks the split's block-table entries and
//    streams 16-row page chunks of K and V (2 x 4 KB at d=128) into an
//    NST-deep shared-memory ring with 2-D TMA (128-B swizzle), completion on
//    per-slot mbarriers. Chunk i goes to consumer warp i % NCONS.
//  * each consumer runs mma.sync m16n8k16 (bf16 -> fp32) with the GQA group
//    packed into the M dimension (rows 0..G-1 valid), an online softmax in the
//    log2 domain (ex2.approx), and P rounded to bf16 for the PV product.
//  * consumers merge their (m, l, O) through shared memory; with one split the
//    CTA writes bf16 output directly, otherwise fp32 partials + LSE, and the
//    last split CTA of each (request, kv-head) to finish (atomic counter)
//    performs the LSE-weighted combine (a5) in the same launch.
//  * rows >= valid_rows of a partial page are masked to -inf; the pool is
//    zero-initialised so those rows are always finite (0 * finite = 0).
#include "hpa_kernels.h"
#include "ptx.cuh"
#include <cuda_bf16.h>
#include <math_constants.h>
#include <algorithm>

namespace hpa {
namespace {

constexpr int kChunk = 16;  // rows per pipeline chunk (one m16n8k16 K-step of keys)
#ifndef HPA_DEC_NCONS
#define HPA_DEC_NCONS 4
#endif
constexpr int kNCons = HPA_DEC_NCONS;  // consumer warps per CTA
#ifndef HPA_DEC_MAP3
#define HPA_DEC_MAP3 1  // must match runtime.cpp: decode tensor maps are 3-D (one TMA per tile)
#endif
#ifndef HPA_DEC_EVICT_FIRST
#define HPA_DEC_EVICT_FIRST 1  // L2 evict-first hint on the streamed K/V tiles (+4 %)
#endif
#ifndef HPA_DEC_DEBUG_RING
#define HPA_DEC_DEBUG_RING 0  // debug builds: stage tags checked by the consumers (printf + trap)
#endif
#ifndef HPA_DEC_ALLOW_ANY_DEPTH
#define HPA_DEC_ALLOW_ANY_DEPTH 0
#endif
#ifndef HPA_DEC_STAGES
#define HPA_DEC_STAGES 12  // ring depth of the grid-per-split decode_split_kernel (HPA_DECODE_PERSISTENT=0); the persistent kernel uses HPA_DEC_PSTAGES
#endif
#ifndef HPA_DEC_DYNAMIC
#define HPA_DEC_DYNAMIC 1  // 1: units fetched from a ticket counter; 0: static striding over the list
#endif
#ifndef HPA_FP8_CVT_INT
#define HPA_FP8_CVT_INT 0  // 1: integer placement + bf16x2 multiply instead of F2FP (exact; measured slower)
#endif
#ifndef HPA_COMBINE_WARP
#define HPA_COMBINE_WARP 1  // a5: one warp per (request, q-head) instead of one CTA of D threads
#endif
#ifndef HPA_FP8_F16
#define HPA_FP8_F16 0  // 1: fp8 chunks converted to f16 and run as f16 MMAs (measured slower: 197 vs 187 us)
#endif
#ifndef HPA_DEC_SWAP
#define HPA_DEC_SWAP 1  // G <= 8: swapped-operand consumers (keys in M, heads in N)
#endif
#ifndef HPA_DEC_PAIR
#define HPA_DEC_PAIR 0  // 1: swapped consumers take two chunks per softmax step (needs KSWZ, VPAIR, !F16; measured slower: 178.5 vs 166.1 us fp8, 208 vs 202 us bf16)
#endif
#ifndef HPA_DEC_VOTE_MAX
#define HPA_DEC_VOTE_MAX 1  // swapped consumers: vote before the chunk-max reduction (skipped unless the max grows)
#endif
#ifndef HPA_DEC_F32
#define HPA_DEC_F32 1  // fp8 token pages (G <= 8): 32-row fp8 chunks, two 16-row blocks per ring stage
#endif
#ifndef HPA_DEC_PSTAGES
// ring depth of the persistent decode kernel (bf16): 10 stages ran the configs[1] step ~1.2 %
// faster than 12, 11 or 8 (profiles/r2_decode_ring_depth_ab.log; depths that are not a multiple
// of the consumer count use stage tags)
#define HPA_DEC_PSTAGES 10
#endif
#ifndef HPA_CS_PAIR
#define HPA_CS_PAIR 1  // cascade group units: consumers take HPA_CS_STEP chunks per softmax step
#endif
#ifndef HPA_CS_STEP
#define HPA_CS_STEP 2
#endif
#ifndef HPA_DEC_CS_STAGES
#define HPA_DEC_CS_STAGES 10  // ring depth of the cascade variant (its Q buffers hold 32 rows)
#endif
#ifndef HPA_WHATIF_EARLY_REL
#define HPA_WHATIF_EARLY_REL 0  // timing what-if only (wrong results): 32-row chunks release their stage
                                // 1: on arrival, 2: after QK^T (the bound for holding V in registers), 3: on arrival, no math
#endif
#ifndef HPA_DEC_F32_STAGES
#define HPA_DEC_F32_STAGES 10  // ring depth of the 32-row fp8 variant (d = 128): 10 x 9 KB, two CTAs per SM (147.0 vs 148.2 us with 8, profiles/r2_fp8_ring10_ab.log)
#endif
#ifndef HPA_DEC_LAZY
#define HPA_DEC_LAZY 1  // decode consumers: lazy running-max rescale (threshold 2^8)
#endif
constexpr int kNSt = HPA_DEC_STAGES;  // ring depth
// Ring depth must be a multiple of the consumer count, so that every slot is consumed by one
// consumer, which then waits the slot's mbarrier phases in order. Otherwise (e.g. 10 stages,
// 4 consumers) consumer 3 takes items 3 and 23 of slot 3 while consumer 1 takes item 13; TMA
// completions land out of order, so consumer 3 can wait for item 23 (phase 2) while phase 1
// is still open, and try_wait.parity(phase 2) matches the completed phase 0 (same parity):
// an ABA that reads a stale stage (found with HPA_DEC_DEBUG_RING stage tags).
static_assert(HPA_DEC_STAGES % kNCons == 0 || HPA_DEC_ALLOW_ANY_DEPTH, "decode ring depth must be a multiple of the consumer count");
#ifndef HPA_FENCE_MODE
#define HPA_FENCE_MODE 2  // 0: fence.sc (threadfence), 1: fence.acq_rel, 2: atom.acq_rel
#endif
#ifndef HPA_DECODE_PERSISTENT
#define HPA_DECODE_PERSISTENT 1  // persistent CTAs streaming consecutive work units through one ring
#endif
#ifndef HPA_DECODE_CTAS_PER_SM
#define HPA_DECODE_CTAS_PER_SM 2
#endif
#ifndef HPA_FUSED_COMBINE
#define HPA_FUSED_COMBINE 0  // 1: a5 by the last split CTA (atomic + GPU fence: measured slower)
#endif

template <int D>
struct DecodeSmem {
  static constexpr int kHalves = D / 64;
  static constexpr int kTileBytes = kChunk * D * 2;   // one 16-row K or V chunk
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kQBytes = 16 * D * 2;
  static constexpr int kBytes = 1024 + kNSt * kStageBytes + kQBytes + 2 * kNSt * 8 + kNSt * 4;
};

template <int D>
__global__ void __launch_bounds__((kNCons + 1) * 32, 3)
decode_split_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const DecodeArgs a) {
  using L = DecodeSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint8_t* qs = smem + kNSt * L::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(qs + L::kQBytes);
  uint64_t* empty = full + kNSt;
  volatile int32_t* cmeta = reinterpret_cast<int32_t*>(empty + kNSt);

  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNSt; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  grid_dependency_wait();  // PDL: everything above overlapped the previous kernel
  grid_launch_dependents();
  const int seq = a.seq_rows[b];
  // q rows of this kv-head's group -> swizzled smem tile [16][D]; rows >= G are 0.
  {
    const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(a.q) + (int64_t(b) * a.Hq + int64_t(h) * G) * D;
    for (int i = threadIdx.x; i < 16 * (D / 8); i += blockDim.x) {
      const int row = i / (D / 8), c = i % (D / 8);
      int4 val = make_int4(0, 0, 0, 0);
      if (row < G) val = *reinterpret_cast<const int4*>(qg + row * D + c * 8);
      *reinterpret_cast<int4*>(qs + (c >> 3) * 2048 + sw128(row, c & 7)) = val;
    }
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const int ne = a.t.n_entries[seq];
      const int e0 = int(int64_t(split) * ne / a.splits);
      const int e1 = int(int64_t(split + 1) * ne / a.splits);
      const int32_t* bt = a.t.block_table + int64_t(seq) * a.t.max_pages;
      const int32_t* mt = a.t.meta + int64_t(seq) * a.t.max_pages;
      uint32_t i = 0;
      for (int e = e0; e < e1; ++e) {
        const int page = bt[e];
        const int valid = mt[e] & kMetaRowsMask;
        const int rowbase = ((a.layer * a.NP + page) * a.Hkv + h) * a.P;
        for (int sub = 0; sub * kChunk < valid; ++sub, ++i) {
          const int slot = i % kNSt;
          if (i >= kNSt) mbar_wait(&empty[slot], ((i / kNSt) - 1) & 1);
          cmeta[slot] = min(kChunk, valid - sub * kChunk);
          mbar_arrive_expect_tx(&full[slot], 2 * L::kTileBytes);
          uint8_t* kd = stages + slot * L::kStageBytes;
          uint8_t* vd = kd + L::kTileBytes;
          if (HPA_DEC_MAP3) {
            tma_load_3d(kd, &tm_k, &full[slot], 0, rowbase + sub * kChunk, 0);
            tma_load_3d(vd, &tm_v, &full[slot], 0, rowbase + sub * kChunk, 0);
          } else {
#pragma unroll
            for (int hf = 0; hf < L::kHalves; ++hf) {
              tma_load_2d(kd + hf * 2048, &tm_k, &full[slot], hf * 64, rowbase + sub * kChunk);
              tma_load_2d(vd + hf * 2048, &tm_v, &full[slot], hf * 64, rowbase + sub * kChunk);
            }
          }
        }
      }
      for (int c = 0; c < kNCons; ++c, ++i) {  // one end-of-work sentinel per consumer
        const int slot = i % kNSt;
        if (i >= kNSt) mbar_wait(&empty[slot], ((i / kNSt) - 1) & 1);
        cmeta[slot] = -1;
        mbar_arrive(&full[slot]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;
  uint32_t qa[D / 16][4];
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int mi = lane >> 3;
    const int row = (lane & 7) + (mi & 1) * 8;
    const int kc = ks * 2 + (mi >> 1);
    ldsm_x4(smem_u32(qs + (kc >> 3) * 2048 + sw128(row, kc & 7)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
  }
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_r[2] = {-CUDART_INF_F, -CUDART_INF_F};
  float l_r[2] = {0.f, 0.f};
  const float sl2 = a.scale_log2;

  for (uint32_t i = cw;; i += kNCons) {
    const int slot = i % kNSt;
    mbar_wait(&full[slot], (i / kNSt) & 1);
    const int nvalid = cmeta[slot];
    if (nvalid < 0) break;
    const uint8_t* kt = stages + slot * L::kStageBytes;
    const uint8_t* vt = kt + L::kTileBytes;

    // S = Q K^T : 16 x 16
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int mi = lane >> 3;
      const int n = (mi >> 1) * 8 + (lane & 7);
      const int kc = ks * 2 + (mi & 1);
      uint32_t b00, b01, b10, b11;
      ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(n, kc & 7)), b00, b01, b10, b11);
      mma_bf16_16816(s[0], qa[ks], b00, b01);
      mma_bf16_16816(s[1], qa[ks], b10, b11);
    }
    // online softmax (log2 domain)
    float x[2][4];
    float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = j * 8 + 2 * (lane & 3) + (e & 1);
        x[j][e] = col < nvalid ? s[j][e] * sl2 : -CUDART_INF_F;
      }
      mx0 = fmaxf(mx0, fmaxf(x[j][0], x[j][1]));
      mx1 = fmaxf(mx1, fmaxf(x[j][2], x[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m_r[0], mx0), mn1 = fmaxf(m_r[1], mx1);
    const float al0 = fast_exp2(m_r[0] - mn0), al1 = fast_exp2(m_r[1] - mn1);
    m_r[0] = mn0;
    m_r[1] = mn1;
    float p[2][4];
    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      p[j][0] = fast_exp2(x[j][0] - mn0);
      p[j][1] = fast_exp2(x[j][1] - mn0);
      p[j][2] = fast_exp2(x[j][2] - mn1);
      p[j][3] = fast_exp2(x[j][3] - mn1);
      ps0 += p[j][0] + p[j][1];
      ps1 += p[j][2] + p[j][3];
    }
    l_r[0] = l_r[0] * al0 + ps0;
    l_r[1] = l_r[1] * al1 + ps1;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= al0;
      o[n][1] *= al0;
      o[n][2] *= al1;
      o[n][3] *= al1;
    }
    uint32_t pa[4];
    pa[0] = pack_bf16(p[0][0], p[0][1]);
    pa[1] = pack_bf16(p[0][2], p[0][3]);
    pa[2] = pack_bf16(p[1][0], p[1][1]);
    pa[3] = pack_bf16(p[1][2], p[1][3]);
    // O += P V : 16 x D
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      const int mi = lane >> 3;
      const int key = (mi & 1) * 8 + (lane & 7);
      const int dc = dp * 2 + (mi >> 1);
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), v0, v1, v2, v3);
      mma_bf16_16816(o[2 * dp], pa, v0, v1);
      mma_bf16_16816(o[2 * dp + 1], pa, v2, v3);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  l_r[0] += __shfl_xor_sync(0xffffffffu, l_r[0], 1);
  l_r[0] += __shfl_xor_sync(0xffffffffu, l_r[0], 2);
  l_r[1] += __shfl_xor_sync(0xffffffffu, l_r[1], 1);
  l_r[1] += __shfl_xor_sync(0xffffffffu, l_r[1], 2);

  // ---------------------------------------------- merge the consumers' states
  constexpr int kNT = kNCons * 32;
  named_bar_sync(1, kNT);  // every consumer is done with the ring
  float* mo = reinterpret_cast<float*>(stages);        // [NCONS][G][D]
  float* mm = mo + kNCons * G * D;                       // [NCONS][G]
  float* ml = mm + kNCons * G;                           // [NCONS][G]
  {
    const int g0 = lane >> 2, g1 = g0 + 8;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int dcol = n * 8 + 2 * (lane & 3);
      if (g0 < G) {
        mo[(cw * G + g0) * D + dcol] = o[n][0];
        mo[(cw * G + g0) * D + dcol + 1] = o[n][1];
      }
      if (g1 < G) {
        mo[(cw * G + g1) * D + dcol] = o[n][2];
        mo[(cw * G + g1) * D + dcol + 1] = o[n][3];
      }
    }
    if ((lane & 3) == 0) {
      if (g0 < G) { mm[cw * G + g0] = m_r[0]; ml[cw * G + g0] = l_r[0]; }
      if (g1 < G) { mm[cw * G + g1] = m_r[1]; ml[cw * G + g1] = l_r[1]; }
    }
  }
  named_bar_sync(1, kNT);
  const int tid = threadIdx.x - 32;
  for (int idx = tid; idx < G * D; idx += kNT) {
    const int g = idx / D, dcol = idx % D;
    float M = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < kNCons; ++c) M = fmaxf(M, mm[c * G + g]);
    float Ls = 0.f, Os = 0.f;
    if (M != -CUDART_INF_F) {
#pragma unroll
      for (int c = 0; c < kNCons; ++c) {
        const float w = fast_exp2(mm[c * G + g] - M);
        Ls += w * ml[c * G + g];
        Os += w * mo[(c * G + g) * D + dcol];
      }
    }
    const int hq = h * G + g;
    if (a.splits == 1 && !a.part_o) {
      static_cast<__nv_bfloat16*>(a.out)[(int64_t(b) * a.Hq + hq) * D + dcol] = __float2bfloat16_rn(Os / Ls);
    } else {
      const int64_t pi = (int64_t(b) * a.Hq + hq) * a.splits + split;
      a.o_part[pi * D + dcol] = Ls > 0.f ? Os / Ls : 0.f;
      if (dcol == 0) a.lse_part[pi] = Ls > 0.f ? M + __log2f(Ls) : -CUDART_INF_F;
    }
  }
  if (a.splits == 1 || !HPA_FUSED_COMBINE || a.part_o) return;
  // ------------------------------------------------ a5: the last split of (b, h) combines
  //   O = sum_s 2^(lse_s - LSE) O_s / sum_s 2^(lse_s - LSE)   (fp32, log2 domain)
  named_bar_sync(1, kNT);  // every consumer's partial writes precede thread 0's release
  if (tid == 0) {
    // release our partials / acquire everyone else's (the last arrival reads them)
    int prev;
#if HPA_FENCE_MODE == 0
    __threadfence();
    prev = atomicAdd(&a.counters[b * a.Hkv + h], 1);
    __threadfence();
#elif HPA_FENCE_MODE == 1
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    prev = atomicAdd(&a.counters[b * a.Hkv + h], 1);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(&a.counters[b * a.Hkv + h]) : "memory");
#endif
    cmeta[0] = prev == a.splits - 1 ? 1 : 0;
  }
  named_bar_sync(1, kNT);
  if (cmeta[0] == 0) return;
  const int S = a.splits;
  float* wts = mo;  // [G][S] normalised split weights (ring memory is free now)
  const int64_t pbase = (int64_t(b) * a.Hq + h * G) * S;
  for (int i = tid; i < G * S; i += kNT) wts[i] = __ldcg(a.lse_part + pbase + i);
  named_bar_sync(1, kNT);
  if (tid < G) {
    float M = -CUDART_INF_F, W = 0.f;
    for (int sp = 0; sp < S; ++sp) M = fmaxf(M, wts[tid * S + sp]);
    for (int sp = 0; sp < S; ++sp) {
      const float ls = wts[tid * S + sp];
      const float w = ls == -CUDART_INF_F ? 0.f : fast_exp2(ls - M);
      wts[tid * S + sp] = w;
      W += w;
    }
    const float inv = 1.f / W;
    for (int sp = 0; sp < S; ++sp) wts[tid * S + sp] *= inv;
  }
  named_bar_sync(1, kNT);
  for (int idx = tid; idx < G * (D / 4); idx += kNT) {
    const int g = idx / (D / 4), d4 = idx % (D / 4);
    const float4* src = reinterpret_cast<const float4*>(a.o_part + (pbase + int64_t(g) * S) * D) + d4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int sp = 0; sp < S; ++sp) {
      const float w = wts[g * S + sp];
      const float4 o = __ldcg(src + int64_t(sp) * (D / 4));
      acc.x += w * o.x;
      acc.y += w * o.y;
      acc.z += w * o.z;
      acc.w += w * o.w;
    }
    uint2 pk;
    pk.x = pack_bf16(acc.x, acc.y);
    pk.y = pack_bf16(acc.z, acc.w);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (int64_t(b) * a.Hq + h * G + g) * D + d4 * 4) = pk;
  }
  if (tid == 0) a.counters[b * a.Hkv + h] = 0;  // ready for the next call (stream order)
}


// ---------------------------------------------------------------------------
// Persistent variant: grid = (#SMs x CTAs/SM); CTA c processes work units
// u = c, c + grid, ... (unit = (request, kv-head, split)). The producer streams
// the chunks of consecutive units through the same ring, so the pipeline never
// drains between units: while the consumers merge unit u the next unit's pages
// are already in flight. Per unit: a 1-D bulk copy of the G q rows into a
// 2-deep Q buffer, the unit's chunks, then one end-of-unit sentinel per consumer
// (cmeta 0); after the last unit one end-of-kernel sentinel per consumer (-1).
// NEXT-4c: one 16-row fp8 tile (codes, row stride D bytes) -> the bf16 [D/64][16][128 B]
// 128-B-swizzled layout the ldmatrix code reads; raw code values (exact in bf16), the
// per-row scales are applied to S and P. Warp-wide: lane -> row lane/2, half the columns.
// All lanes read before any lane writes, so src may overlap dst (the V tile converts in place).
template <int D, bool KSW = false>
__device__ __forceinline__ void fp8_tile_to_bf16(const uint8_t* src, uint8_t* dst, int lane) {
  constexpr int kG = D / 16;  // 8-byte groups per lane (16 x D bytes / 32 lanes / 8)
  // lane reads bytes [(32 g + lane) * 8, +8): each LDS.64 covers 256 contiguous bytes
  // (conflict-free; a row-per-lane-pair mapping was a 16-way bank conflict)
  uint2 c[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) c[g] = reinterpret_cast<const uint2*>(src)[32 * g + lane];
  __syncwarp();
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    const int byte = (32 * g + lane) * 8;
    const int r = byte / D;
    int cc = (byte % D) >> 3;  // 8-code group = 16-B bf16 chunk index in the row
    if (KSW) cc = fp8_kswz(cc * 8, r, D) >> 3;  // swizzled K codes: physical -> logical (an involution)
    int4 out;
    if (HPA_FP8_CVT_INT) {
      // e4m3 -> bf16 without the conversion unit: a code's 7 magnitude bits placed at bf16
      // bits 4..10 (sign at 15) read as bf16 are the value times 2^-120 for every code,
      // subnormals included (e4m3 bias 7 vs bf16 bias 127); one bf16x2 multiply by 2^120
      // restores it exactly
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t bytes = q == 0 ? c[g].x : c[g].y;
        const uint32_t t0 = __byte_perm(bytes, 0u, 0x1404), t1 = __byte_perm(bytes, 0u, 0x3424);
        const uint32_t u0 = ((t0 >> 4) & 0x07f007f0u) | (t0 & 0x80008000u);
        const uint32_t u1 = ((t1 >> 4) & 0x07f007f0u) | (t1 & 0x80008000u);
        asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(w[2 * q]) : "r"(u0), "r"(0x7b807b80u));
        asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(w[2 * q + 1]) : "r"(u1), "r"(0x7b807b80u));
      }
      out = make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
    } else {
      out = bf16x8_from_e4m3(c[g], 1.f);
    }
    *reinterpret_cast<int4*>(dst + (cc >> 3) * 2048 + sw128(r, cc & 7)) = out;
  }
}
// The V tile of an fp8 chunk in the HPA_FP8_VPAIR layout (pair rows of interleaved key codes,
// swizzled 16-byte chunks; ptx.cuh fp8_voff) -> the bf16 [D/64][16][128 B] layout: the two chunks
// of a (pair row, 16-dim group) hold 8-dim groups 2m and 2m + 1 of both keys; all lanes read
// before any lane writes (src overlaps dst).
template <int D>
__device__ __forceinline__ void fp8_vtile_to_bf16(const uint8_t* src, uint8_t* dst, int lane) {
  constexpr int kGroups = D / 16;           // 16-dim groups per pair row
  constexpr int kPer = 8 * kGroups / 32;    // (pair row, group) items per lane
  uint4 ca[kPer], cb[kPer];                 // the group's two chunks: dims g and g + 8, g < 4 / g >= 4
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int q = 32 * i + lane, pr = q / kGroups, m = q % kGroups;
    ca[i] = *reinterpret_cast<const uint4*>(src + fp8_voff(2 * pr, 16 * m, D));
    cb[i] = *reinterpret_cast<const uint4*>(src + fp8_voff(2 * pr, 16 * m + 4, D));
  }
  __syncwarp();  // the source overlaps the destination tile
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int q = 32 * i + lane, pr = q / kGroups, m = q % kGroups;
#pragma unroll
    for (int b = 0; b < 4; ++b) {  // byte b = 2 h + key parity of every word
      const uint32_t sel = uint32_t(b) | (uint32_t(b + 4) << 4);
      const uint2 codes = make_uint2(
          __byte_perm(__byte_perm(ca[i].x, ca[i].y, sel), __byte_perm(ca[i].z, ca[i].w, sel), 0x5410),
          __byte_perm(__byte_perm(cb[i].x, cb[i].y, sel), __byte_perm(cb[i].z, cb[i].w, sel), 0x5410));
      const int r = 2 * pr + (b & 1), dg = 2 * m + (b >> 1);  // row, 8-dim group
      *reinterpret_cast<int4*>(dst + (dg >> 3) * 2048 + sw128(r, dg & 7)) = bf16x8_from_e4m3(codes, 1.f);
    }
  }
}
// fp8 V path of the swapped consumers (HPA_FP8_VPAIR): P^T goes to f16 as p * s_V * vpre with
// p <= 2^8 (lazy rescale). svmax = this lane's largest valid V scale of the chunk(s) about to be
// packed. If some lane would reach p * s_V * vpre > 2^15 (f16 overflows at 65504), or every lane
// stays below 2^0 (weights drifting toward f16 subnormals), vpre moves to the power of two that
// puts the warp's largest scale times vpre in [2^6, 2^7), and O -- accumulated in units of
// 1 / vpre -- is multiplied by the same exact factor. Rare: never for V rows of similar size.
template <int D>
__device__ __forceinline__ void fp8_vpre_adjust(float svmax, float& vpre, float (&o)[D / 16][4]) {
  const float sv = svmax * vpre;
  const bool hi = __any_sync(0xffffffffu, sv > 128.f);
  const bool lo = __all_sync(0xffffffffu, sv < 1.f / 256.f);
  if (!(hi || lo)) return;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) svmax = fmaxf(svmax, __shfl_xor_sync(0xffffffffu, svmax, off));
  if (!(svmax > 0.f) || !(svmax < CUDART_INF_F)) return;
  const int e = int((__float_as_uint(svmax) >> 23) & 0xffu) - 127;  // floor(log2 svmax) (normal scales)
  const int k = min(max(6 - e, -100), 100);                         // new vpre = 2^k
  const float nv = __uint_as_float(uint32_t(127 + k) << 23);
  const float r = nv / vpre;  // a power of two: exact
#pragma unroll
  for (int n = 0; n < D / 16; ++n) {
    o[n][0] *= r;
    o[n][1] *= r;
    o[n][2] *= r;
    o[n][3] *= r;
  }
  vpre = nv;
}

// Same as fp8_tile_to_bf16 but to f16 (one cvt per code pair; e4m3 values are exact in f16):
// the swapped-operand consumers run fp8 chunks as f16 MMAs.
template <int D, bool KSW = false>
__device__ __forceinline__ void fp8_tile_to_f16(const uint8_t* src, uint8_t* dst, int lane) {
  constexpr int kG = D / 16;
  uint2 c[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) c[g] = reinterpret_cast<const uint2*>(src)[32 * g + lane];
  __syncwarp();
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    const int byte = (32 * g + lane) * 8;
    const int r = byte / D;
    int cc = (byte % D) >> 3;
    if (KSW) cc = fp8_kswz(cc * 8, r, D) >> 3;
    const uint32_t in[4] = {c[g].x & 0xffffu, c[g].x >> 16, c[g].y & 0xffffu, c[g].y >> 16};
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(w[q]) : "h"(uint16_t(in[q])));
    *reinterpret_cast<int4*>(dst + (cc >> 3) * 2048 + sw128(r, cc & 7)) =
        make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// the same with an L2 cache-policy hint (evict-first for streamed K/V blocks)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
#ifndef HPA_FP8_EVICT_FIRST
#define HPA_FP8_EVICT_FIRST 1  // fp8 K/V blocks streamed with the evict-first L2 policy, like the bf16 tiles
#endif

constexpr int kWB = 8;  // table-walker ring: pieces of one header + up to 31 page entries

// F32 (fp8 token pages, swapped consumers): a ring stage holds either one 16-row bf16 chunk
// (K tile, V tile) or a 32-row fp8 chunk = two 16-row blocks [16 x D codes | 16 scales] of K
// (A at 0, B at kBlk8) and of V (A at 2 kBlk8, B at 3 kBlk8): twice the keys per hand-off and per
// softmax step, and twice the fp8 bytes in flight per stage. The stage stride stays 1024-B
// aligned (128-B swizzled TMA tiles), so the ring is 8 stages deep instead of 12 (two CTAs per SM).
// CS (cascade decode, NEXT-2): the kernel also runs group units -- one shared run of entries
// read once for up to 32 query rows of several requests (4 consumers x 8 columns): the Q buffers
// hold 32 rows and the ring is 8 stages deep so two CTAs still fit on an SM.
template <int D, bool F32 = false, bool CS = false>
struct PDecodeSmem {
  static constexpr int kHalves = D / 64;
  static constexpr int kTileBytes = kChunk * D * 2;
  static constexpr int kBlk8 = 16 * D + 64;
  static constexpr int kStageBytes =
      F32 ? (((2 * kTileBytes > 4 * kBlk8 ? 2 * kTileBytes : 4 * kBlk8) + 1023) & ~1023) : 2 * kTileBytes;
  static constexpr int kStages =
      F32 ? (CS ? 8 : (D == 128 ? HPA_DEC_F32_STAGES : 12)) : (CS ? HPA_DEC_CS_STAGES : HPA_DEC_PSTAGES);
  // a depth that is not a multiple of the consumer count puts successive items of one slot on
  // different consumers, and a consumer could then take the slot's previous phase of the same
  // parity for its item (mbarrier-parity ABA): every stage then carries its item index (ctag),
  // which the consumer waits for before its parity wait
  static constexpr bool kTags = kStages % kNCons != 0;
  static constexpr int oRing = 0;
  // full[NST], empty[NST], q_full[2], q_empty[2], w_full[WB], w_empty[WB]
  static constexpr int oBar = kStages * kStageBytes;
  static constexpr int oMeta = oBar + (2 * kStages + 4 + 2 * kWB) * 8;
  static constexpr int oTag = oMeta + kStages * 4;               // [kStages] item index per stage (kTags)
  static constexpr int oQMeta = (oTag + kStages * 4 + 15) & ~15;  // 2 x int4 {b, h, split, -}: unit of Q buffer
  static constexpr int oWalk = oQMeta + 32;                      // [WB][32] int2 pieces
  static constexpr int oZero = oWalk + kWB * 32 * 8;             // 16 zero bytes: A-operand rows >= G
  // fp8 chunk (NEXT-4c): the K and V blocks [16 x D codes | 16 scales] sit at the top of the
  // stage; the consumer reads the scales, then converts K to [0, kTile), V to [kTile, 2 kTile)
  // (F32: blocks at the bottom, see above; read in place, never converted)
  static constexpr int oK8 = F32 ? 0 : kStageBytes - 2 * kBlk8;
  static constexpr int oV8 = F32 ? 2 * kBlk8 : kStageBytes - kBlk8;
  static constexpr int oQ = oZero + 16;                          // 2 x [G][D] q rows (unswizzled)
  static constexpr int kQRows = 32;  // CS: query rows of a group unit
  static __host__ __device__ int qbuf(int G) { return (CS && G < kQRows ? kQRows : G) * D * 2; }
  static __host__ __device__ int oMerge(int G) { return oQ + 2 * qbuf(G); }
  // no alignment slack: the dynamic smem base is 1024-B aligned (checked in the kernel)
  static int bytes(int G) { return oMerge(G) + kNCons * G * (D + 2) * 4; }
};

// Fused-append kernel parameters (AppendRows with the tail records by value); NA = 1 is the
// plain decode (n = 0).
template <int NA>
struct AppendParams {
  const __nv_bfloat16* k;  // new rows, bf16 [L][n][H_kv][d]
  const __nv_bfloat16* v;
  __nv_bfloat16* k_pool;   // bf16 [L][NP][H_kv][P][d]
  __nv_bfloat16* v_pool;
  int64_t stride_l;
  int32_t n, L;
  int4 tail[NA];           // {n_entries, page, meta, pos0} of each request's last entry
};

// One warp copies the new row of (request b, head h) into row (valid - 1) of the tail page,
// in every layer: lanes [0, D/8) move K, [D/8, D/4) move V, 16 B each. Then the proxy fence:
// the tile holding the row is read next by TMA (async proxy) after an mbarrier hand-off.
template <int D, int NA>
__device__ __forceinline__ void append_tail_row(const AppendParams<NA>& ap, const DecodeArgs& a, int b, int h,
                                                int4 tl, int lane) {
  constexpr int NV = D / 8;
  if (lane < 2 * NV) {
    const int vi = lane % NV;
    const bool is_v = lane >= NV;
    const int r = (tl.z & kMetaRowsMask) - 1;
    const __nv_bfloat16* src = (is_v ? ap.v : ap.k) + (int64_t(b) * a.Hkv + h) * D + vi * 8;
    __nv_bfloat16* dst = (is_v ? ap.v_pool : ap.k_pool) + (int64_t(tl.y) * a.Hkv + h) * a.P * D +
                         int64_t(r) * D + vi * 8;
    const int64_t lstride = int64_t(a.NP) * a.Hkv * a.P * D;
    for (int l = 0; l < ap.L; ++l)
      *reinterpret_cast<int4*>(dst + l * lstride) = *reinterpret_cast<const int4*>(src + l * ap.stride_l);
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
}

template <int D, bool SW, int NA, bool F32 = false, bool CS = false>
__global__ void __launch_bounds__((kNCons + 2) * 32, HPA_DECODE_CTAS_PER_SM)
decode_persistent_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                         const DecodeArgs a, const __grid_constant__ AppendParams<NA> ap) {
  static_assert(!F32 || (SW && NA == 1 && HPA_FP8_KSWZ && HPA_FP8_VPAIR && !HPA_FP8_F16 && !HPA_DEC_PAIR),
                "32-row fp8 chunks: swapped consumers with the register-direct fp8 operands only");
  static_assert(!CS || (SW && !HPA_DEC_PAIR), "cascade units: swapped consumers only");
  using L = PDecodeSmem<D, F32, CS>;
  constexpr int kNSt = L::kStages;  // ring depth of this variant
  extern __shared__ __align__(1024) uint8_t smem_pd[];
  uint8_t* smem = smem_pd;
  if (smem_u32(smem) & 1023) {  // TMA 128-B swizzle needs 1024-B aligned stage buffers
    if (threadIdx.x == 0) printf("hpa decode: dynamic smem base 0x%x not 1024-B aligned\n", smem_u32(smem));
    __trap();
  }
#ifdef HPA_TRACE
  long long t_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
  if (a.trace && threadIdx.x == 0) a.trace[4 * blockIdx.x] = t_entry;
#endif
  const int G = a.G;
  uint8_t* stages = smem + L::oRing;
  uint8_t* qbuf = smem + L::oQ;
  const int qbytes = L::qbuf(G);
  uint8_t* zero = smem + L::oZero;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* empty = full + kNSt;
  uint64_t* q_full = empty + kNSt;
  uint64_t* q_empty = q_full + 2;
  uint64_t* w_full = q_empty + 2;
  uint64_t* w_empty = w_full + kWB;
  volatile int32_t* cmeta = reinterpret_cast<int32_t*>(smem + L::oMeta);
  volatile int32_t* ctag = reinterpret_cast<int32_t*>(smem + L::oTag);
  int4* qmeta = reinterpret_cast<int4*>(smem + L::oQMeta);
  int2* walk = reinterpret_cast<int2*>(smem + L::oWalk);
#if HPA_DEC_DEBUG_RING
  __shared__ volatile uint32_t dbg_tag[kNSt];
#endif
  float* mo = reinterpret_cast<float*>(smem + L::oMerge(G));  // [NCONS][G][D]
  float* mm = mo + kNCons * G * D;                          // [NCONS][G]
  float* ml = mm + kNCons * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNSt; ++i) {
      mbar_init(&full[i], 1);
      // CS: a group unit's stage is released by every consumer, a normal one by its consumer
      // with an arrival count of kNCons
      mbar_init(&empty[i], CS ? kNCons : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], kNCons);
    }
    for (int i = 0; i < kWB; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(zero)[threadIdx.x] = 0u;
  if (L::kTags && threadIdx.x < kNSt) ctag[threadIdx.x] = -1;
  __syncthreads();
  grid_dependency_wait();  // PDL: everything above overlapped the previous kernel
  grid_launch_dependents();

  if (warp == kNCons + 1) {
    // --------------------------------------------------------- table walker
    // Resolves work units (ticket -> record -> entry count) and their block-table entries
    // (coalesced, one lane per entry) into pieces of {header, <= 31 x (rowbase, valid)} up to
    // kWB pieces ahead, so no global-load latency ever sits on the TMA producer's path.
    const int U = a.n_units;
    uint32_t pc = 0;
    int t = 0;
    if (lane == 0) t = HPA_DEC_DYNAMIC ? atomicAdd(a.sched, 1) : int(blockIdx.x);
    t = __shfl_sync(0xffffffffu, t, 0);
    for (;;) {
      if (t >= U) {
        const int ws = pc % kWB;
        if (lane == 0) {
          if (pc >= kWB) mbar_wait(&w_empty[ws], ((pc / kWB) - 1) & 1);
          walk[ws * 32] = make_int2(-1, 0);
          mbar_arrive(&w_full[ws]);
        }
        break;
      }
      int tn = 0;
      if (lane == 0) tn = HPA_DEC_DYNAMIC ? atomicAdd(a.sched, 1) : t + int(gridDim.x);
      const int4 ur = a.units[t];
      const int seq = ur.y, h = ur.z & 0xff, split = (ur.z >> 8) & 0xff, sb = ur.z >> 16;
      // fused append (NA > 1): the request's last entry and entry count come from the tail
      // record; the device table still holds the values from before this step's append
      int4 tl = make_int4(0, 0, 0, 0);
      const bool gunit = CS && ur.x <= -2;  // cascade group unit: no tail record (its run is shared)
      if constexpr (NA > 1) {
        if (!gunit) tl = ap.tail[ur.x];
      }
      const int ne = NA > 1 && !gunit ? tl.x : a.t.n_entries[seq];
      int e0, e1;
      if (CS && ur.x <= -2) {  // cascade group piece: a fixed entry range of the shared run
        const int32_t* gr = a.groups + int64_t(-2 - ur.x) * kGroupRec;
        e0 = gr[0];
        e1 = gr[1];
      } else {  // the request's own entries [r, ne) (r = ur.w: its cascaded shared run), split sb ways
        const int r = ur.w;
        e0 = r + int(int64_t(split) * (ne - r) / sb);
        e1 = r + int(int64_t(split + 1) * (ne - r) / sb);
      }
      const int32_t* bt = a.t.block_table + int64_t(seq) * a.t.max_pages;
      const int32_t* mt = a.t.meta + int64_t(seq) * a.t.max_pages;
      for (int e = e0, first = 1;; e += 31, first = 0) {
        const int cnt = min(31, e1 - e);
        const int last = e + cnt >= e1;
        if constexpr (NA > 1) {
          if (last && e1 == ne && !gunit) {
            // this unit holds the new row of (request, head h): write it into its pool slot
            // (every layer) before the piece that loads its tile is published; the proxy
            // fence orders these generic stores before the producer's TMA reads of the tile
            append_tail_row<D>(ap, a, ur.x, h, tl, lane);
            if (h == 0 && lane == 0) {  // write the entry back for later calls
              const int64_t x = int64_t(seq) * a.t.max_pages + ne - 1;
              a.t.block_table[x] = tl.y;
              a.t.pos0[x] = tl.w;
              a.t.meta[x] = tl.z;
              a.t.seq_len[seq] = tl.w + (tl.z & kMetaRowsMask);
              a.t.n_entries[seq] = ne;
            }
          }
        }
        int2 item;
        if (lane == 0) {
          item = make_int2(ur.x, h | (split << 8) | (cnt << 16) | (first << 24) | (last << 25));
        } else if (lane <= cnt) {
          const bool tail_entry = NA > 1 && !gunit && e + lane == ne;  // (a group unit has no tail record)
          const int page = tail_entry ? tl.y : bt[e + lane - 1];
          const int mv = tail_entry ? tl.z : mt[e + lane - 1];
          const int f8 = a.fp8 && !(mv & kMetaLatent);  // fp8 token page (NEXT-4c)
          item = make_int2(((a.layer * (f8 ? a.NPt : a.NP) + page) * a.Hkv + h) * a.P,
                           (mv & kMetaRowsMask) | (f8 << 16));
        }
        const int ws = pc % kWB;
        if (pc >= kWB) mbar_wait(&w_empty[ws], ((pc / kWB) - 1) & 1);
        if (lane <= cnt) walk[ws * 32 + lane] = item;
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_full[ws]);
        ++pc;
        if (last) break;
      }
      t = __shfl_sync(0xffffffffu, tn, 0);
    }
    // every ticket fetch of every CTA is done once all CTAs got here: the last one resets
    if (lane == 0 && HPA_DEC_DYNAMIC && atomicAdd(a.sched + 1, 1) == int(gridDim.x) - 1) {
      atomicExch(a.sched, 0);
      atomicExch(a.sched + 1, 0);
    }
    return;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Consumes the walker's pieces: a unit's first piece starts its Q copy, every entry
    // becomes TMA chunks, the unit's last piece ends with one sentinel per consumer.
    if (lane == 0) {
      uint32_t i = 0, pc = 0;
      int ul = 0;
      const uint64_t pol = HPA_DEC_EVICT_FIRST ? l2_policy_evict_first() : 0;
      // F32: one 32-row fp8 stage = blocks A (+ B): [K A | K B | V A | V B]
      int64_t pend_blk = 0;
      int pend_n = 0;  // rows of a held fp8 block A (0: none)
      auto issue_f8 = [&](int64_t blk_a, int na, int64_t blk_b, int nb) {
        const int slot = i % kNSt;
        if (i >= kNSt) mbar_wait(&empty[slot], ((i / kNSt) - 1) & 1);
#if HPA_DEC_DEBUG_RING
        dbg_tag[slot] = i;
#endif
        cmeta[slot] = na | (nb << 8) | (1 << 16);
        if (L::kTags) ctag[slot] = int(i);
        uint8_t* kd = stages + slot * L::kStageBytes;
        mbar_arrive_expect_tx(&full[slot], uint32_t((nb ? 4 : 2) * L::kBlk8));
        if (HPA_FP8_EVICT_FIRST) {  // 148 vs 152 us at configs[1] (profiles/r2_fp8_evict_first_ab.log)
          bulk_g2s_hint(kd, a.k8 + blk_a * L::kBlk8, L::kBlk8, &full[slot], pol);
          bulk_g2s_hint(kd + 2 * L::kBlk8, a.v8 + blk_a * L::kBlk8, L::kBlk8, &full[slot], pol);
          if (nb) {
            bulk_g2s_hint(kd + L::kBlk8, a.k8 + blk_b * L::kBlk8, L::kBlk8, &full[slot], pol);
            bulk_g2s_hint(kd + 3 * L::kBlk8, a.v8 + blk_b * L::kBlk8, L::kBlk8, &full[slot], pol);
          }
        } else {
          bulk_g2s(kd, a.k8 + blk_a * L::kBlk8, L::kBlk8, &full[slot]);
          bulk_g2s(kd + 2 * L::kBlk8, a.v8 + blk_a * L::kBlk8, L::kBlk8, &full[slot]);
          if (nb) {
            bulk_g2s(kd + L::kBlk8, a.k8 + blk_b * L::kBlk8, L::kBlk8, &full[slot]);
            bulk_g2s(kd + 3 * L::kBlk8, a.v8 + blk_b * L::kBlk8, L::kBlk8, &full[slot]);
          }
        }
        ++i;
      };
      auto flush_pend = [&]() {
        if (pend_n) {
          issue_f8(pend_blk, pend_n, 0, 0);
          pend_n = 0;
        }
      };
      for (;;) {
        const int ws = pc % kWB;
        mbar_wait(&w_full[ws], (pc / kWB) & 1);
        const int2* it = walk + ws * 32;
        const int2 hd = it[0];
        if (hd.x == -1) {  // end of work: tell the consumers through the Q slot
          const int qb = ul & 1;
          if (ul >= 2) mbar_wait(&q_empty[qb], ((ul >> 1) - 1) & 1);
          qmeta[qb] = make_int4(-1, 0, 0, 0);
          mbar_arrive(&q_full[qb]);
          break;
        }
        const int b = hd.x, h = hd.y & 0xff, split = (hd.y >> 8) & 0xff, cnt = (hd.y >> 16) & 0xff;
        const bool grp = CS && b <= -2;  // cascade group unit (b = -2 - group piece)
        if ((hd.y >> 24) & 1) {  // first piece of a unit: its Q rows
          const int qb = ul & 1;
          if (ul >= 2) mbar_wait(&q_empty[qb], ((ul >> 1) - 1) & 1);
          if (grp) {  // the G rows of every member request, stacked
            const int32_t* gr = a.groups + int64_t(-2 - b) * kGroupRec;
            const int nm = gr[2];
            qmeta[qb] = make_int4(b, h, nm, int(i));
            mbar_arrive_expect_tx(&q_full[qb], uint32_t(nm * G * D * 2));
            for (int m = 0; m < nm; ++m)
              bulk_g2s(qbuf + qb * qbytes + m * G * D * 2,
                       static_cast<const __nv_bfloat16*>(a.q) + (int64_t(gr[4 + m]) * a.Hq + int64_t(h) * G) * D,
                       uint32_t(G * D * 2), &q_full[qb]);
          } else {
            qmeta[qb] = make_int4(b, h, split, int(i));  // ring position of the unit's first chunk
            mbar_arrive_expect_tx(&q_full[qb], uint32_t(G * D * 2));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(qbuf + qb * qbytes)),
                "l"(static_cast<const __nv_bfloat16*>(a.q) + (int64_t(b) * a.Hq + int64_t(h) * G) * D),
                "r"(uint32_t(G * D * 2)), "r"(smem_u32(&q_full[qb]))
                : "memory");
          }
        }
        const int last = (hd.y >> 25) & 1;
        for (int j = 1; j <= cnt; ++j) {
          const int2 en = it[j];
          const int rowbase = en.x, valid = en.y & 0xffff, f8 = en.y >> 16;
          if constexpr (F32) {
            if (f8) {
              // fp8 token rows: 16-row blocks paired two per stage; a lone block is published
              // alone when a bf16 chunk or the unit's end follows (flush_pend)
              for (int sub = 0; sub * kChunk < valid; ++sub) {
                const int nrows = min(kChunk, valid - sub * kChunk);
                const int64_t blk = (int64_t(rowbase) + sub * kChunk) >> 4;
                if (pend_n == 0) {
                  pend_blk = blk;
                  pend_n = nrows;
                } else {
                  issue_f8(pend_blk, pend_n, blk, nrows);
                  pend_n = 0;
                }
              }
              continue;
            }
            flush_pend();
          }
          for (int sub = 0; sub * kChunk < valid; ++sub, ++i) {
            const int slot = i % kNSt;
            if (i >= kNSt) mbar_wait(&empty[slot], ((i / kNSt) - 1) & 1);
            cmeta[slot] = min(kChunk, valid - sub * kChunk) | (f8 << 16);
            if (L::kTags) ctag[slot] = int(i);
#if HPA_DEC_DEBUG_RING
            dbg_tag[slot] = i;
#endif
            uint8_t* kd = stages + slot * L::kStageBytes;
            uint8_t* vd = kd + L::kTileBytes;
            if (f8) {
              // fp8 chunk (NEXT-4c): one bulk copy per K / V block (codes + row scales) into the
              // top of the stage; the consumer converts them to the bf16 layout in place
              const int64_t blk = (int64_t(rowbase) + sub * kChunk) >> 4;
              mbar_arrive_expect_tx(&full[slot], uint32_t(2 * L::kBlk8));
              bulk_g2s(kd + L::oK8, a.k8 + blk * L::kBlk8, L::kBlk8, &full[slot]);
              bulk_g2s(kd + L::oV8, a.v8 + blk * L::kBlk8, L::kBlk8, &full[slot]);
              continue;
            }
            mbar_arrive_expect_tx(&full[slot], 2 * L::kTileBytes);  // K and V tiles (F32 stages are larger)
            if (HPA_DEC_MAP3 && HPA_DEC_EVICT_FIRST) {
              tma_load_3d_hint(kd, &tm_k, &full[slot], 0, rowbase + sub * kChunk, 0, pol);
              tma_load_3d_hint(vd, &tm_v, &full[slot], 0, rowbase + sub * kChunk, 0, pol);
            } else if (HPA_DEC_MAP3) {
              tma_load_3d(kd, &tm_k, &full[slot], 0, rowbase + sub * kChunk, 0);
              tma_load_3d(vd, &tm_v, &full[slot], 0, rowbase + sub * kChunk, 0);
            } else {
#pragma unroll
              for (int hf = 0; hf < L::kHalves; ++hf) {
                tma_load_2d(kd + hf * 2048, &tm_k, &full[slot], hf * 64, rowbase + sub * kChunk);
                tma_load_2d(vd + hf * 2048, &tm_v, &full[slot], hf * 64, rowbase + sub * kChunk);
              }
            }
          }
        }
        mbar_arrive(&w_empty[ws]);
        ++pc;
        if (last) {
          if constexpr (F32) flush_pend();
          // end of unit: one sentinel per consumer (a group unit's consumers all read one)
          for (int c = 0; c < (grp ? 1 : kNCons); ++c, ++i) {
            const int slot = i % kNSt;
            if (i >= kNSt) mbar_wait(&empty[slot], ((i / kNSt) - 1) & 1);
            cmeta[slot] = 0;
            if (L::kTags) ctag[slot] = int(i);
#if HPA_DEC_DEBUG_RING
            dbg_tag[slot] = i;
#endif
            mbar_arrive(&full[slot]);
          }
          ++ul;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;
  const int tid = threadIdx.x - 32;
  constexpr int kNT = kNCons * 32;
  const float sl2 = a.scale_log2;
  uint32_t i = cw;
  for (int ul = 0;; ++ul) {
    const int qb = ul & 1;
    mbar_wait(&q_full[qb], (ul >> 1) & 1);
    const int4 um = qmeta[qb];
    if (um.x == -1) {  // end of work (x <= -2: a cascade group unit)
#ifdef HPA_TRACE
      if (a.trace && lane == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 4 * blockIdx.x + 1), (unsigned long long)t);
        if (cw == 0) a.trace[4 * blockIdx.x + 2] = ul;
      }
#endif
      break;
    }
    const int b = um.x, h = um.y, split = um.z;
    // merge slot = this consumer's chunk group within the unit (chunks j = cg mod kNCons):
    // the unit's result then does not depend on where in the ring it started, i.e. on the
    // dynamic unit schedule (run-to-run deterministic decode)
    const int cg = (cw - int(uint32_t(um.w) % kNCons) + kNCons) % kNCons;
    // CS group unit: every consumer reads every chunk of the unit for its own 8 query columns
    // (rows 8 cw .. 8 cw + 7 of the stacked member rows) and finishes them itself
    const bool grp = CS && b <= -2;
    if (grp) i = uint32_t(um.w);
    const uint32_t istep = grp ? 1u : uint32_t(kNCons);
    auto release = [&](int slot) {
      if (lane == 0) {
        if (CS && !grp) mbar_arrive_cnt(&empty[slot], kNCons);
        else mbar_arrive(&empty[slot]);
      }
    };
    auto after_sentinel = [&]() {  // the consumer's next item: its own residue class again
      if (grp) {
        const uint32_t nx = i + 1;
        i = nx + uint32_t((cw - int(nx % kNCons) + kNCons) % kNCons);
      } else {
        i += kNCons;
      }
    };
    if constexpr (SW) {
    // ---- swapped operands (G <= 8): S^T = K Q^T with the chunk's 16 keys in M and the
    // G heads in N = 8; O^T = V^T P^T with 16 head dims per M tile. Half the MMAs of the
    // Q-in-M form (whose 16-row M tile is 3/4 padding at G = 4) and half the O registers.
    // Fragment owner: g = lane / 4 (key row / dim row), t = lane % 4 (heads 2t, 2t+1).
    const int gq = lane >> 2, tq = lane & 3;
    uint32_t qbf[D / 16][2];  // B operand Q^T: (dims 16 ks + 2t.., head g), (dims + 8.., head g)
    // HPA_FP8_KSWZ: f16 B operand over the dims in the register-direct order of the fp8 K
    // path: k (2t, 2t+1) <-> dims 16 ks + 4t, +1 and k (2t+8, 2t+9) <-> dims 16 ks + 4t + 2, +3
    uint32_t qbk[D / 16][2];
    // fp8 units: the f16 copies of Q (qbk, qbh) hold q * 2^-qs, with qs chosen per unit so that
    // max |q| stays inside f16's range (bf16 -> f16 would overflow above 65504); the fp8 K
    // chunks' score multiplier carries 2^qs back. qs = 0 unless max |q| >= 2^15 or < 2^-10.
    float qmul = 1.f, sl2k = sl2;
    {
      const int qr = grp ? 8 * cw + gq : gq;               // this lane's query row in the Q buffer
      const bool qv = qr < (grp ? split * G : G);          // (group unit: split = member count)
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(qbuf + qb * qbytes + qr * D * 2);
      if (a.fp8) {
        float qmax = 0.f;
#pragma unroll
        for (int w = 0; w < D / 2; w += 4) {
          const uint32_t v = qv ? qrow[w + tq] : 0u;
          qmax = fmaxf(qmax, fmaxf(fabsf(__uint_as_float(v << 16)), fabsf(__uint_as_float(v & 0xffff0000u))));
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) qmax = fmaxf(qmax, __shfl_xor_sync(0xffffffffu, qmax, off));
        const int e = qmax > 0.f ? int((__float_as_uint(qmax) >> 23) & 0xffu) - 127 : 0;  // floor(log2), normals
        const int qs = (e >= 15 || e < -10) ? min(max(e - 14, -100), 100) : 0;
        qmul = __uint_as_float(uint32_t(127 - qs) << 23);
        sl2k = sl2 * __uint_as_float(uint32_t(127 + qs) << 23);
      }
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        qbf[ks][0] = qv ? qrow[8 * ks + tq] : 0u;
        qbf[ks][1] = qv ? qrow[8 * ks + 4 + tq] : 0u;
        if (HPA_FP8_KSWZ && a.fp8) {
          qbk[ks][0] = qv ? bf16x2_to_f16x2_scaled(qrow[8 * ks + 2 * tq], qmul) : 0u;
          qbk[ks][1] = qv ? bf16x2_to_f16x2_scaled(qrow[8 * ks + 2 * tq + 1], qmul) : 0u;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&q_empty[qb]);
    uint32_t qbh[D / 16][2];  // the same B operand in f16, for fp8 chunks (f16 MMAs)
    if (a.fp8) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        qbh[ks][0] = bf16x2_to_f16x2_scaled(qbf[ks][0], qmul);
        qbh[ks][1] = bf16x2_to_f16x2_scaled(qbf[ks][1], qmul);
      }
    }
    // score multiplier of an fp8 chunk's keys: those run on the f16 copies of Q
    const float slk = (HPA_FP8_KSWZ || HPA_FP8_F16) ? sl2k : sl2;

    // HPA_FP8_VPAIR: every P^T fragment is pre-scaled by vpre, a power of two (f16 range for
    // the fp8 chunks; latent bf16 chunks carry the same factor so O stays consistent); undone
    // at the merge. It starts at 2^8 and moves (fp8_vpre_adjust, O rescaled by the same exact
    // power of two) whenever a chunk's V scales would push p * s_V * vpre (p <= 2^8 under the
    // lazy rescale) past 2^15, or leave all of it below 2^0: f16 never overflows and keeps its
    // normal range for the weights whatever the V row magnitudes.
    float vpre = (HPA_FP8_VPAIR && a.fp8) ? 256.f : 1.f;
    float o[D / 16][4];  // O^T tile mt: (dim 16mt+g, head 2t), (.., 2t+1), (dim +8, 2t), (dim +8, 2t+1)
#pragma unroll
    for (int n = 0; n < D / 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_h[2] = {-CUDART_INF_F, -CUDART_INF_F};  // running max of heads 2t, 2t+1 (log2 domain)
    float l_h[2] = {0.f, 0.f};                       // partial sums over this lane's keys
    if constexpr (F32) {
      // 32-row fp8 chunks: blocks A and B of a stage give two independent QK^T chains, one
      // softmax step over 32 keys and two PV k-steps; a 16-row bf16 (latent) chunk is block A only
      for (;; i += istep) {
        const int slot = i % kNSt;
        if (L::kTags) while (ctag[slot] != int(i)) {}  // this stage holds item i (depth % consumers != 0)
      mbar_wait(&full[slot], (i / kNSt) & 1);
#if HPA_DEC_DEBUG_RING
        if (dbg_tag[slot] != i) {
          if (lane == 0)
            printf("hpa decode ring: block %d consumer %d slot %d expected item %u, stage holds %u\n", blockIdx.x, cw,
                   slot, i, dbg_tag[slot]);
          __trap();
        }
#endif
        const int meta = cmeta[slot];
        if (meta <= 0) {  // sentinel: release the slot and finish the unit
          __syncwarp();
          release(slot);
          after_sentinel();
          break;
        }
        const uint8_t* kt = stages + slot * L::kStageBytes;
        const bool c8 = meta >= 0x10000;
        const int nb0 = meta & 0xff, nb1 = (meta >> 8) & 0xff;
        const bool two = c8 && nb1 > 0;
#if HPA_WHATIF_EARLY_REL == 1 || HPA_WHATIF_EARLY_REL == 3
        __syncwarp();
        release(slot);
        if (HPA_WHATIF_EARLY_REL == 3) continue;  // 3: no math at all (the data-movement bound)
#endif
        float x[2][4], vm[2][2];
        float svmax = 0.f;  // this lane's largest valid V scale
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          x[c][0] = x[c][1] = x[c][2] = x[c][3] = -CUDART_INF_F;
          vm[c][0] = vm[c][1] = 0.f;
          if (c == 1 && !two) continue;
          const int nv = c ? nb1 : nb0;
          float sacc[4] = {0.f, 0.f, 0.f, 0.f};
          float kmul0 = sl2, kmul1 = sl2;
          if (c8) {
            const uint8_t* kb = kt + c * L::kBlk8;
            const float* ksc = reinterpret_cast<const float*>(kb + 16 * D);
            const float* vsc = reinterpret_cast<const float*>(kt + (2 + c) * L::kBlk8 + 16 * D);
            kmul0 = ksc[gq] * slk;
            kmul1 = ksc[gq + 8] * slk;
            vm[c][0] = vsc[gq];
            vm[c][1] = vsc[gq + 8];
            svmax = fmaxf(svmax, fmaxf(gq < nv ? vm[c][0] : 0.f, gq + 8 < nv ? vm[c][1] : 0.f));
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {  // K fragments straight from the swizzled codes
              const uint32_t w0 = *reinterpret_cast<const uint32_t*>(kb + gq * D + fp8_kswz(ks * 16 + 4 * tq, gq, D));
              const uint32_t w1 =
                  *reinterpret_cast<const uint32_t*>(kb + (gq + 8) * D + fp8_kswz(ks * 16 + 4 * tq, gq + 8, D));
              uint32_t ka[4];
              ka[0] = f16x2_from_e4m3x2(w0);
              ka[1] = f16x2_from_e4m3x2(w1);
              ka[2] = f16x2_from_e4m3x2(w0 >> 16);
              ka[3] = f16x2_from_e4m3x2(w1 >> 16);
              mma_f16_16816(sacc, ka, qbk[ks][0], qbk[ks][1]);
            }
          } else {
            vm[c][0] = vm[c][1] = 1.f;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {  // A = K (16 keys x 16 dims), bf16 tile
              const int mi = lane >> 3;
              const int row = (lane & 7) + (mi & 1) * 8;
              const int kc = ks * 2 + (mi >> 1);
              uint32_t ka[4];
              ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(row, kc & 7)), ka[0], ka[1], ka[2], ka[3]);
              mma_bf16_16816(sacc, ka, qbf[ks][0], qbf[ks][1]);
            }
          }
          x[c][0] = gq < nv ? sacc[0] * kmul0 : -CUDART_INF_F;      // key g,   head 2t
          x[c][1] = gq < nv ? sacc[1] * kmul0 : -CUDART_INF_F;      // key g,   head 2t+1
          x[c][2] = gq + 8 < nv ? sacc[2] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t
          x[c][3] = gq + 8 < nv ? sacc[3] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t+1
        }
#if HPA_WHATIF_EARLY_REL == 2
        __syncwarp();
        release(slot);
#endif
        if (c8) fp8_vpre_adjust<D>(svmax, vpre, o);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          vm[c][0] *= vpre;
          vm[c][1] *= vpre;
        }
        float mx0 = fmaxf(fmaxf(x[0][0], x[0][2]), fmaxf(x[1][0], x[1][2]));
        float mx1 = fmaxf(fmaxf(x[0][1], x[0][3]), fmaxf(x[1][1], x[1][3]));
        const bool any_grow = __any_sync(0xffffffffu, mx0 > m_h[0] + 8.f || mx1 > m_h[1] + 8.f);
        if (any_grow) {
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {  // over the 8 key-row lanes
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
          }
        }
        const bool g0 = any_grow && mx0 > m_h[0] + 8.f, g1 = any_grow && mx1 > m_h[1] + 8.f;
        const float mn0 = g0 ? mx0 : m_h[0], mn1 = g1 ? mx1 : m_h[1];
        float pp[2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          pp[c][0] = fast_exp2(x[c][0] - mn0);
          pp[c][1] = fast_exp2(x[c][1] - mn1);
          pp[c][2] = fast_exp2(x[c][2] - mn0);
          pp[c][3] = fast_exp2(x[c][3] - mn1);
        }
        const float s0 = (pp[0][0] + pp[0][2]) + (pp[1][0] + pp[1][2]);
        const float s1 = (pp[0][1] + pp[0][3]) + (pp[1][1] + pp[1][3]);
        if (!any_grow) {  // max unchanged: the factors are 1
          l_h[0] += s0;
          l_h[1] += s1;
        } else {
          const float al0 = fast_exp2(m_h[0] - mn0), al1 = fast_exp2(m_h[1] - mn1);
          m_h[0] = mn0;
          m_h[1] = mn1;
          l_h[0] = l_h[0] * al0 + s0;
          l_h[1] = l_h[1] * al1 + s1;
#pragma unroll
          for (int n = 0; n < D / 16; ++n) {
            o[n][0] *= al0;
            o[n][1] *= al1;
            o[n][2] *= al0;
            o[n][3] *= al1;
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c == 1 && !two) continue;
          if (c8) {  // V^T fragments straight from the pair-row codes, P^T in f16 (x vpre)
            const uint32_t pb0 = movmatrix_t(pack_f16(pp[c][0] * vm[c][0], pp[c][1] * vm[c][0]));
            const uint32_t pb1 = movmatrix_t(pack_f16(pp[c][2] * vm[c][1], pp[c][3] * vm[c][1]));
            const uint8_t* vb = kt + (2 + c) * L::kBlk8;
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
              const int d = 16 * mt + gq;
              const uint32_t w0 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq, d, D));
              const uint32_t w1 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq + 8, d, D));
              uint32_t va[4];
              va[0] = f16x2_from_e4m3x2(w0);
              va[1] = f16x2_from_e4m3x2(w0 >> 16);
              va[2] = f16x2_from_e4m3x2(w1);
              va[3] = f16x2_from_e4m3x2(w1 >> 16);
              mma_f16_16816(o[mt], va, pb0, pb1);
            }
          } else {
            const uint32_t pb0 = movmatrix_t(pack_bf16(pp[c][0] * vm[c][0], pp[c][1] * vm[c][0]));
            const uint32_t pb1 = movmatrix_t(pack_bf16(pp[c][2] * vm[c][1], pp[c][3] * vm[c][1]));
            const uint8_t* vt = kt + L::kTileBytes;
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {  // A = V^T (16 dims x 16 keys)
              const int mi = lane >> 3;
              const int key = (lane & 7) + (mi >> 1) * 8;
              const int dc = 2 * mt + (mi & 1);
              uint32_t va[4];
              ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), va[0], va[1], va[2], va[3]);
              mma_bf16_16816(o[mt], va, pb0, pb1);
            }
          }
        }
#if !HPA_WHATIF_EARLY_REL
        __syncwarp();
        release(slot);
#endif
      }
    } else {
#if HPA_DEC_PAIR
    static_assert(HPA_FP8_KSWZ && HPA_FP8_VPAIR && !HPA_FP8_F16, "HPA_DEC_PAIR needs the register-direct fp8 paths");
    // HPA_DEC_PAIR: a consumer takes its next two chunks (items i, i + kNCons) together: two
    // independent QK^T MMA chains, one softmax step over 32 keys, then both PV halves. The
    // stages are released together. No deadlock with kNSt >= 3 kNCons: the producer waiting for
    // item n - kNSt finds its holder waiting at most for item n - kNSt + kNCons < n.
    static_assert(kNSt >= 3 * kNCons, "paired decode consumers need a ring of >= 3 items per consumer");
    for (;;) {
      const int sA = i % kNSt;
      mbar_wait(&full[sA], (i / kNSt) & 1);
      int nv[2];
      nv[0] = cmeta[sA];
      if (nv[0] <= 0) {  // sentinel: release the slot and finish the unit
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sA]);
        i += kNCons;
        break;
      }
      const uint32_t iB = i + kNCons;
      const int sB = iB % kNSt;
      mbar_wait(&full[sB], (iB / kNSt) & 1);
      nv[1] = cmeta[sB];
      const bool haveB = nv[1] > 0;  // else item iB is the unit's sentinel
      const int sl[2] = {sA, sB};
      float x[2][4], vm[2][2];
      bool c8[2] = {false, false};
      float svmax = 0.f;  // this lane's largest valid V scale over both chunks
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        x[c][0] = x[c][1] = x[c][2] = x[c][3] = -CUDART_INF_F;
        vm[c][0] = vm[c][1] = 0.f;
        if (c == 1 && !haveB) continue;
        c8[c] = nv[c] >= 0x10000;
        const int nvalid = nv[c] & 0xffff;
        const uint8_t* kt = stages + sl[c] * L::kStageBytes;
        float kmul0 = sl2, kmul1 = sl2;
        vm[c][0] = vm[c][1] = 1.f;  // raw V scales here; times vpre after the adjustment below
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        if (c8[c]) {
          const float* ksc = reinterpret_cast<const float*>(kt + L::oK8 + 16 * D);
          const float* vsc = reinterpret_cast<const float*>(kt + L::oV8 + 16 * D);
          kmul0 = ksc[gq] * slk;
          kmul1 = ksc[gq + 8] * slk;
          vm[c][0] = vsc[gq];
          vm[c][1] = vsc[gq + 8];
          svmax = fmaxf(svmax, fmaxf(gq < nvalid ? vm[c][0] : 0.f, gq + 8 < nvalid ? vm[c][1] : 0.f));
          const uint8_t* kb = kt + L::oK8;
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(kb + gq * D + fp8_kswz(ks * 16 + 4 * tq, gq, D));
            const uint32_t w1 =
                *reinterpret_cast<const uint32_t*>(kb + (gq + 8) * D + fp8_kswz(ks * 16 + 4 * tq, gq + 8, D));
            uint32_t ka[4];
            ka[0] = f16x2_from_e4m3x2(w0);
            ka[1] = f16x2_from_e4m3x2(w1);
            ka[2] = f16x2_from_e4m3x2(w0 >> 16);
            ka[3] = f16x2_from_e4m3x2(w1 >> 16);
            mma_f16_16816(sacc, ka, qbk[ks][0], qbk[ks][1]);
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {  // A = K (16 keys x 16 dims)
            const int mi = lane >> 3;
            const int row = (lane & 7) + (mi & 1) * 8;
            const int kc = ks * 2 + (mi >> 1);
            uint32_t ka[4];
            ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(row, kc & 7)), ka[0], ka[1], ka[2], ka[3]);
            mma_bf16_16816(sacc, ka, qbf[ks][0], qbf[ks][1]);
          }
        }
        x[c][0] = gq < nvalid ? sacc[0] * kmul0 : -CUDART_INF_F;      // key g,   head 2t
        x[c][1] = gq < nvalid ? sacc[1] * kmul0 : -CUDART_INF_F;      // key g,   head 2t+1
        x[c][2] = gq + 8 < nvalid ? sacc[2] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t
        x[c][3] = gq + 8 < nvalid ? sacc[3] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t+1
      }
      if (HPA_FP8_VPAIR && a.fp8 && (c8[0] || c8[1])) fp8_vpre_adjust<D>(svmax, vpre, o);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        vm[c][0] *= vpre;
        vm[c][1] *= vpre;
      }
      float mx0 = fmaxf(fmaxf(x[0][0], x[0][2]), fmaxf(x[1][0], x[1][2]));
      float mx1 = fmaxf(fmaxf(x[0][1], x[0][3]), fmaxf(x[1][1], x[1][3]));
      const bool any_grow = __any_sync(0xffffffffu, mx0 > m_h[0] + 8.f || mx1 > m_h[1] + 8.f);
      if (any_grow) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {  // over the 8 key-row lanes
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
      }
      const bool g0 = any_grow && mx0 > m_h[0] + 8.f, g1 = any_grow && mx1 > m_h[1] + 8.f;
      const float mn0 = g0 ? mx0 : m_h[0], mn1 = g1 ? mx1 : m_h[1];
      float pp[2][4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        pp[c][0] = fast_exp2(x[c][0] - mn0);
        pp[c][1] = fast_exp2(x[c][1] - mn1);
        pp[c][2] = fast_exp2(x[c][2] - mn0);
        pp[c][3] = fast_exp2(x[c][3] - mn1);
      }
      const float s0 = (pp[0][0] + pp[0][2]) + (pp[1][0] + pp[1][2]);
      const float s1 = (pp[0][1] + pp[0][3]) + (pp[1][1] + pp[1][3]);
      if (!any_grow) {
        l_h[0] += s0;
        l_h[1] += s1;
      } else {
        const float al0 = fast_exp2(m_h[0] - mn0), al1 = fast_exp2(m_h[1] - mn1);
        m_h[0] = mn0;
        m_h[1] = mn1;
        l_h[0] = l_h[0] * al0 + s0;
        l_h[1] = l_h[1] * al1 + s1;
#pragma unroll
        for (int n = 0; n < D / 16; ++n) {
          o[n][0] *= al0;
          o[n][1] *= al1;
          o[n][2] *= al0;
          o[n][3] *= al1;
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c == 1 && !haveB) continue;
        const uint8_t* kt = stages + sl[c] * L::kStageBytes;
        if (c8[c]) {  // fp8 V^T fragments straight from the pair-row codes (see the unpaired loop)
          const uint32_t pb0 = movmatrix_t(pack_f16(pp[c][0] * vm[c][0], pp[c][1] * vm[c][0]));
          const uint32_t pb1 = movmatrix_t(pack_f16(pp[c][2] * vm[c][1], pp[c][3] * vm[c][1]));
          const uint8_t* vb = kt + L::oV8;
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            const int d = 16 * mt + gq;
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq, d, D));
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq + 8, d, D));
            uint32_t va[4];
            va[0] = f16x2_from_e4m3x2(w0);
            va[1] = f16x2_from_e4m3x2(w0 >> 16);
            va[2] = f16x2_from_e4m3x2(w1);
            va[3] = f16x2_from_e4m3x2(w1 >> 16);
            mma_f16_16816(o[mt], va, pb0, pb1);
          }
        } else {
          const uint32_t pb0 = movmatrix_t(pack_bf16(pp[c][0] * vm[c][0], pp[c][1] * vm[c][0]));
          const uint32_t pb1 = movmatrix_t(pack_bf16(pp[c][2] * vm[c][1], pp[c][3] * vm[c][1]));
          const uint8_t* vt = kt + L::kTileBytes;
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {  // A = V^T (16 dims x 16 keys)
            const int mi = lane >> 3;
            const int key = (lane & 7) + (mi >> 1) * 8;
            const int dc = 2 * mt + (mi & 1);
            uint32_t va[4];
            ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), va[0], va[1], va[2], va[3]);
            mma_bf16_16816(o[mt], va, pb0, pb1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[sA]);
        mbar_arrive(&empty[sB]);
      }
      i = iB + kNCons;
      if (!haveB) break;
    }
#else
    if (CS && grp && HPA_CS_PAIR) {
      // Group unit (cascade): every consumer works through every chunk, so kCsStep chunks per
      // step -- items i .. i + kCsStep - 1, independent QK^T chains, one softmax step over all
      // their keys, then the PV k-steps -- cut the chain latency per chunk. Any item after the
      // first may be the unit's sentinel.
      constexpr int kCsStep = HPA_CS_STEP;
      for (;;) {
        int sl[kCsStep], nv[kCsStep];
        int nit = 0;  // chunks in this step (items before a sentinel)
        bool ends = false;
#pragma unroll
        for (int c = 0; c < kCsStep; ++c) {
          sl[c] = int((i + c) % kNSt);
          nv[c] = 0;
          if (ends) continue;
          if (L::kTags) while (ctag[sl[c]] != int(i + c)) {}
          mbar_wait(&full[sl[c]], ((i + c) / kNSt) & 1);
          nv[c] = cmeta[sl[c]];
          if (nv[c] <= 0) ends = true;
          else nit = c + 1;
        }
        float x[kCsStep][4];
#pragma unroll
        for (int c = 0; c < kCsStep; ++c) {
          x[c][0] = x[c][1] = x[c][2] = x[c][3] = -CUDART_INF_F;
          if (c >= nit) continue;
          const uint8_t* kt = stages + sl[c] * L::kStageBytes;
          float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {  // A = K (16 keys x 16 dims)
            const int mi = lane >> 3;
            const int row = (lane & 7) + (mi & 1) * 8;
            const int kc = ks * 2 + (mi >> 1);
            uint32_t ka[4];
            ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(row, kc & 7)), ka[0], ka[1], ka[2], ka[3]);
            mma_bf16_16816(sacc, ka, qbf[ks][0], qbf[ks][1]);
          }
          x[c][0] = gq < nv[c] ? sacc[0] * sl2 : -CUDART_INF_F;
          x[c][1] = gq < nv[c] ? sacc[1] * sl2 : -CUDART_INF_F;
          x[c][2] = gq + 8 < nv[c] ? sacc[2] * sl2 : -CUDART_INF_F;
          x[c][3] = gq + 8 < nv[c] ? sacc[3] * sl2 : -CUDART_INF_F;
        }
        if (nit > 0) {
          float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
          for (int c = 0; c < kCsStep; ++c) {
            mx0 = fmaxf(mx0, fmaxf(x[c][0], x[c][2]));
            mx1 = fmaxf(mx1, fmaxf(x[c][1], x[c][3]));
          }
          const bool any_grow = __any_sync(0xffffffffu, mx0 > m_h[0] + 8.f || mx1 > m_h[1] + 8.f);
          if (any_grow) {
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
              mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
              mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
            }
          }
          const bool g0 = any_grow && mx0 > m_h[0] + 8.f, g1 = any_grow && mx1 > m_h[1] + 8.f;
          const float mn0 = g0 ? mx0 : m_h[0], mn1 = g1 ? mx1 : m_h[1];
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int c = 0; c < kCsStep; ++c) {  // x becomes p (exp2 against the running max)
            x[c][0] = fast_exp2(x[c][0] - mn0);
            x[c][1] = fast_exp2(x[c][1] - mn1);
            x[c][2] = fast_exp2(x[c][2] - mn0);
            x[c][3] = fast_exp2(x[c][3] - mn1);
            s0 += x[c][0] + x[c][2];
            s1 += x[c][1] + x[c][3];
          }
          if (!any_grow) {
            l_h[0] += s0;
            l_h[1] += s1;
          } else {
            const float al0 = fast_exp2(m_h[0] - mn0), al1 = fast_exp2(m_h[1] - mn1);
            m_h[0] = mn0;
            m_h[1] = mn1;
            l_h[0] = l_h[0] * al0 + s0;
            l_h[1] = l_h[1] * al1 + s1;
#pragma unroll
            for (int n = 0; n < D / 16; ++n) {
              o[n][0] *= al0;
              o[n][1] *= al1;
              o[n][2] *= al0;
              o[n][3] *= al1;
            }
          }
#pragma unroll
          for (int c = 0; c < kCsStep; ++c) {
            if (c >= nit) continue;
            const uint32_t pb0 = movmatrix_t(pack_bf16(x[c][0] * vpre, x[c][1] * vpre));
            const uint32_t pb1 = movmatrix_t(pack_bf16(x[c][2] * vpre, x[c][3] * vpre));
            const uint8_t* vt = stages + sl[c] * L::kStageBytes + L::kTileBytes;
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {  // A = V^T (16 dims x 16 keys)
              const int mi = lane >> 3;
              const int key = (lane & 7) + (mi >> 1) * 8;
              const int dc = 2 * mt + (mi & 1);
              uint32_t va[4];
              ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), va[0], va[1], va[2], va[3]);
              mma_bf16_16816(o[mt], va, pb0, pb1);
            }
          }
        }
        __syncwarp();
        const int waited = ends ? nit + 1 : kCsStep;  // (the sentinel's stage too)
#pragma unroll
        for (int c = 0; c < kCsStep; ++c)
          if (c < waited) release(sl[c]);
        if (ends) {
          i += nit;  // the sentinel's item
          after_sentinel();
          break;
        }
        i += kCsStep;
      }
    } else
    for (;; i += istep) {
      const int slot = i % kNSt;
      if (L::kTags) while (ctag[slot] != int(i)) {}  // this stage holds item i (depth % consumers != 0)
      mbar_wait(&full[slot], (i / kNSt) & 1);
#if HPA_DEC_DEBUG_RING
      if (dbg_tag[slot] != i) {
        if (lane == 0)
          printf("hpa decode ring: block %d consumer %d slot %d expected item %u, stage holds %u\n", blockIdx.x, cw,
                 slot, i, dbg_tag[slot]);
        __trap();
      }
#endif
      int nvalid = cmeta[slot];
      if (nvalid <= 0) {  // sentinel: release the slot and finish the unit
        __syncwarp();
        release(slot);
        after_sentinel();
        break;
      }
      const bool c8 = nvalid >= 0x10000;  // fp8 chunk (NEXT-4c)
      nvalid &= 0xffff;
      uint8_t* kt = stages + slot * L::kStageBytes;
      uint8_t* vt = kt + L::kTileBytes;
      float kmul0 = sl2, kmul1 = sl2, vmul0 = vpre, vmul1 = vpre;  // keys g and g + 8
      if (c8) {
        const float* ksc = reinterpret_cast<const float*>(kt + L::oK8 + 16 * D);
        const float* vsc = reinterpret_cast<const float*>(kt + L::oV8 + 16 * D);
        kmul0 = ksc[gq] * slk;  // scales first: the conversion overwrites them
        kmul1 = ksc[gq + 8] * slk;
        const float sv0 = vsc[gq], sv1 = vsc[gq + 8];
        if (HPA_FP8_VPAIR)
          fp8_vpre_adjust<D>(fmaxf(gq < nvalid ? sv0 : 0.f, gq + 8 < nvalid ? sv1 : 0.f), vpre, o);
        vmul0 = sv0 * vpre;
        vmul1 = sv1 * vpre;
      }
      float sacc[4] = {0.f, 0.f, 0.f, 0.f};
      const bool kreg = HPA_FP8_KSWZ && !HPA_FP8_F16 && c8;
      if (kreg) {
        // fp8 K straight into registers (no shared-memory conversion): lane (g, t) reads codes
        // 4t..4t+3 of each 16-column group of keys g and g + 8 (chunk-swizzled rows: no bank
        // conflict) and converts them to f16 pairs for f16 MMAs against qbk. K is consumed
        // before the V tile conversion below overwrites the upper part of the K code block.
        const uint8_t* kb = kt + L::oK8;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t w0 = *reinterpret_cast<const uint32_t*>(kb + gq * D + fp8_kswz(ks * 16 + 4 * tq, gq, D));
          const uint32_t w1 =
              *reinterpret_cast<const uint32_t*>(kb + (gq + 8) * D + fp8_kswz(ks * 16 + 4 * tq, gq + 8, D));
          uint32_t ka[4];
          ka[0] = f16x2_from_e4m3x2(w0);
          ka[1] = f16x2_from_e4m3x2(w1);
          ka[2] = f16x2_from_e4m3x2(w0 >> 16);
          ka[3] = f16x2_from_e4m3x2(w1 >> 16);
          mma_f16_16816(sacc, ka, qbk[ks][0], qbk[ks][1]);
        }
      }
      // shared-memory conversions only for the variant builds (both operands are read from the
      // codes directly by default)
      if (c8 && (HPA_FP8_F16 || !kreg || !HPA_FP8_VPAIR)) {
        __syncwarp();
        if (HPA_FP8_F16) {
          fp8_tile_to_f16<D, true>(kt + L::oK8, kt, lane);
          fp8_tile_to_f16<D>(kt + L::oV8, vt, lane);
        } else {
          if (!kreg) fp8_tile_to_bf16<D, true>(kt + L::oK8, kt, lane);
          if (!HPA_FP8_VPAIR) fp8_tile_to_bf16<D>(kt + L::oV8, vt, lane);  // (VPAIR: V read below)
        }
        __syncwarp();
      }
      const bool h16 = HPA_FP8_F16 && c8;  // this chunk runs as f16 MMAs
      if (!kreg) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {  // A = K (16 keys x 16 dims)
        const int mi = lane >> 3;
        const int row = (lane & 7) + (mi & 1) * 8;
        const int kc = ks * 2 + (mi >> 1);
        uint32_t ka[4];
        ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(row, kc & 7)), ka[0], ka[1], ka[2], ka[3]);
        if (h16) mma_f16_16816(sacc, ka, qbh[ks][0], qbh[ks][1]);
        else mma_bf16_16816(sacc, ka, qbf[ks][0], qbf[ks][1]);
      }
      }
      const float x0 = gq < nvalid ? sacc[0] * kmul0 : -CUDART_INF_F;      // key g,   head 2t
      const float x1 = gq < nvalid ? sacc[1] * kmul0 : -CUDART_INF_F;      // key g,   head 2t+1
      const float x2 = gq + 8 < nvalid ? sacc[2] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t
      const float x3 = gq + 8 < nvalid ? sacc[3] * kmul1 : -CUDART_INF_F;  // key g+8, head 2t+1
      float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
      // lazy rescale: the running max moves only when the chunk max exceeds it by > 2^8.
      // HPA_DEC_VOTE_MAX: one vote on the lanes' own keys first; the 8-lane max reduction
      // runs only when some key grows the max (same result: no lane grows <=> the max doesn't)
      bool any_grow = true;
      if (HPA_DEC_VOTE_MAX) any_grow = __any_sync(0xffffffffu, mx0 > m_h[0] + 8.f || mx1 > m_h[1] + 8.f);
      if (any_grow) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {  // over the 8 key-row lanes
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
      }
      const bool g0 = any_grow && mx0 > m_h[0] + 8.f, g1 = any_grow && mx1 > m_h[1] + 8.f;
      const float mn0 = g0 ? mx0 : m_h[0], mn1 = g1 ? mx1 : m_h[1];
      if (!HPA_DEC_VOTE_MAX) any_grow = __any_sync(0xffffffffu, g0 || g1);
      const float p0 = fast_exp2(x0 - mn0), p1 = fast_exp2(x1 - mn1);
      const float p2 = fast_exp2(x2 - mn0), p3 = fast_exp2(x3 - mn1);
      if (HPA_DEC_VOTE_MAX && !any_grow) {  // max unchanged: the factors are 1 (l * 1 + s == l + s)
        l_h[0] += p0 + p2;
        l_h[1] += p1 + p3;
      } else {
        const float al0 = fast_exp2(m_h[0] - mn0), al1 = fast_exp2(m_h[1] - mn1);
        m_h[0] = mn0;
        m_h[1] = mn1;
        l_h[0] = l_h[0] * al0 + (p0 + p2);
        l_h[1] = l_h[1] * al1 + (p1 + p3);
        if (any_grow) {
#pragma unroll
          for (int n = 0; n < D / 16; ++n) {
            o[n][0] *= al0;
            o[n][1] *= al1;
            o[n][2] *= al0;
            o[n][3] *= al1;
          }
        }
      }
      // B operand P^T: (key g: heads 2t, 2t+1) pairs transposed in registers to (head g: keys
      // 2t, 2t+1); the V scales (fp8 chunks) fold into P per key
      if (HPA_FP8_VPAIR && c8) {
        // fp8 V^T fragments straight from the pair-row codes: one 16-bit load = the (key 2t,
        // key 2t+1) code pair of one dim = one f16x2 register; P^T in f16 (pre-scaled by vpre
        // so tiny V scales stay normal in f16; O is divided by vpre at the unit's merge)
        const uint32_t pb0 = movmatrix_t(pack_f16(p0 * vmul0, p1 * vmul0));
        const uint32_t pb1 = movmatrix_t(pack_f16(p2 * vmul1, p3 * vmul1));
        const uint8_t* vb = kt + L::oV8;
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
          const int d = 16 * mt + gq;
          // one 32-bit load = dims d and d + 8 of keys (2t, 2t+1) (resp. 2t+8, 2t+9)
          const uint32_t w0 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq, d, D));
          const uint32_t w1 = *reinterpret_cast<const uint32_t*>(vb + fp8_voff(2 * tq + 8, d, D));
          uint32_t va[4];
          va[0] = f16x2_from_e4m3x2(w0);
          va[1] = f16x2_from_e4m3x2(w0 >> 16);
          va[2] = f16x2_from_e4m3x2(w1);
          va[3] = f16x2_from_e4m3x2(w1 >> 16);
          mma_f16_16816(o[mt], va, pb0, pb1);
        }
      } else {
      const uint32_t pb0 = movmatrix_t(h16 ? pack_f16(p0 * vmul0, p1 * vmul0) : pack_bf16(p0 * vmul0, p1 * vmul0));
      const uint32_t pb1 = movmatrix_t(h16 ? pack_f16(p2 * vmul1, p3 * vmul1) : pack_bf16(p2 * vmul1, p3 * vmul1));
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt) {  // A = V^T (16 dims x 16 keys)
        const int mi = lane >> 3;
        const int key = (lane & 7) + (mi >> 1) * 8;
        const int dc = 2 * mt + (mi & 1);
        uint32_t va[4];
        ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), va[0], va[1], va[2], va[3]);
        if (h16) mma_f16_16816(o[mt], va, pb0, pb1);
        else mma_bf16_16816(o[mt], va, pb0, pb1);
      }
      }
      __syncwarp();
      release(slot);
    }
#endif  // HPA_DEC_PAIR
    }  // F32
    // ---------------------------------------------- merge the consumers' states
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l_h[0] += __shfl_xor_sync(0xffffffffu, l_h[0], off);
      l_h[1] += __shfl_xor_sync(0xffffffffu, l_h[1], off);
    }
    if (CS && grp) {
      // group unit: this consumer saw every key of the piece for its columns 2t, 2t+1, i.e.
      // rows 8 cw + 2t (+1) = (member m, head) -> that member's partial slot of this piece
      const int32_t* gr = a.groups + int64_t(-2 - b) * kGroupRec;
      const int nrows = split * G;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        const int row = 8 * cw + 2 * tq + c2;
        if (row < nrows) {
          const int m = row / G, hq = h * G + row % G;
          const int64_t pi = (int64_t(gr[4 + m]) * a.Hq + hq) * a.splits + gr[4 + kGroupMax + m];
          const float inv = l_h[c2] > 0.f ? 1.f / (l_h[c2] * vpre) : 0.f;
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            a.o_part[pi * D + 16 * mt + gq] = o[mt][c2] * inv;
            a.o_part[pi * D + 16 * mt + gq + 8] = o[mt][2 + c2] * inv;
          }
          if (gq == 0) a.lse_part[pi] = l_h[c2] > 0.f ? m_h[c2] + __log2f(l_h[c2]) : -CUDART_INF_F;
        }
      }
      continue;
    }
    {
      const int h0 = 2 * tq, h1 = 2 * tq + 1;
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt) {
        const int d0 = 16 * mt + gq;
        const float ivp = 1.f / vpre;
        if (h0 < G) {
          mo[(cg * G + h0) * D + d0] = o[mt][0] * ivp;
          mo[(cg * G + h0) * D + d0 + 8] = o[mt][2] * ivp;
        }
        if (h1 < G) {
          mo[(cg * G + h1) * D + d0] = o[mt][1] * ivp;
          mo[(cg * G + h1) * D + d0 + 8] = o[mt][3] * ivp;
        }
      }
      if (gq == 0) {
        if (h0 < G) { mm[cg * G + h0] = m_h[0]; ml[cg * G + h0] = l_h[0]; }
        if (h1 < G) { mm[cg * G + h1] = m_h[1]; ml[cg * G + h1] = l_h[1]; }
      }
    }
    } else {
    // Q fragments of this unit (rows >= G read the zero chunk)
    uint32_t qa[D / 16][4];
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int mi = lane >> 3;
      const int row = (lane & 7) + (mi & 1) * 8;
      const int kc = ks * 2 + (mi >> 1);
      const uint8_t* src = row < G ? qbuf + qb * qbytes + row * D * 2 + kc * 16 : zero;
      ldsm_x4(smem_u32(src), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&q_empty[qb]);
    float o[D / 8][4];
#pragma unroll
    for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_r[2] = {-CUDART_INF_F, -CUDART_INF_F};
    float l_r[2] = {0.f, 0.f};
    for (;; i += istep) {
      const int slot = i % kNSt;
      if (L::kTags) while (ctag[slot] != int(i)) {}  // this stage holds item i (depth % consumers != 0)
      mbar_wait(&full[slot], (i / kNSt) & 1);
#if HPA_DEC_DEBUG_RING
      if (dbg_tag[slot] != i) {
        if (lane == 0)
          printf("hpa decode ring: block %d consumer %d slot %d expected item %u, stage holds %u\n", blockIdx.x, cw,
                 slot, i, dbg_tag[slot]);
        __trap();
      }
#endif
      int nvalid = cmeta[slot];
      if (nvalid <= 0) {  // sentinel: release the slot and finish the unit
        __syncwarp();
        release(slot);
        after_sentinel();
        break;
      }
      const bool c8 = nvalid >= 0x10000;  // fp8 chunk (NEXT-4c)
      nvalid &= 0xffff;
      uint8_t* kt = stages + slot * L::kStageBytes;
      uint8_t* vt = kt + L::kTileBytes;
      // per owned key column (2t, 2t+1, 8+2t, 9+2t): K scale (x softmax scale) and V scale
      float kmul[4] = {sl2, sl2, sl2, sl2}, vmul[4] = {1.f, 1.f, 1.f, 1.f};
      if (c8) {
        const float* ksc = reinterpret_cast<const float*>(kt + L::oK8 + 16 * D);
        const float* vsc = reinterpret_cast<const float*>(kt + L::oV8 + 16 * D);
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // scales first: the conversion overwrites them
          const int col = (q >> 1) * 8 + 2 * (lane & 3) + (q & 1);
          kmul[q] = ksc[col] * sl2;
          vmul[q] = vsc[col];
        }
        __syncwarp();
        fp8_tile_to_bf16<D, true>(kt + L::oK8, kt, lane);
        if (HPA_FP8_VPAIR) fp8_vtile_to_bf16<D>(kt + L::oV8, vt, lane);
        else fp8_tile_to_bf16<D>(kt + L::oV8, vt, lane);
        __syncwarp();
      }
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int mi = lane >> 3;
        const int n = (mi >> 1) * 8 + (lane & 7);
        const int kc = ks * 2 + (mi & 1);
        uint32_t b00, b01, b10, b11;
        ldsm_x4(smem_u32(kt + (kc >> 3) * 2048 + sw128(n, kc & 7)), b00, b01, b10, b11);
        mma_bf16_16816(s[0], qa[ks], b00, b01);
        mma_bf16_16816(s[1], qa[ks], b10, b11);
      }
      float x[2][4];
      float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = j * 8 + 2 * (lane & 3) + (e & 1);
          x[j][e] = col < nvalid ? s[j][e] * kmul[j * 2 + (e & 1)] : -CUDART_INF_F;
        }
        mx0 = fmaxf(mx0, fmaxf(x[j][0], x[j][1]));
        mx1 = fmaxf(mx1, fmaxf(x[j][2], x[j][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
#if HPA_DEC_LAZY
      // lazy rescale (as in prefill): the running max moves only when a row's chunk max exceeds
      // it by > 2^8, so p <= 2^8 (exact enough in bf16, far from fp32 limits) and the O rescale
      // below is skipped for most chunks
      const bool g0 = mx0 > m_r[0] + 8.f, g1 = mx1 > m_r[1] + 8.f;
      const float mn0 = g0 ? mx0 : m_r[0], mn1 = g1 ? mx1 : m_r[1];
      const bool any_grow = __any_sync(0xffffffffu, g0 || g1);
#else
      const float mn0 = fmaxf(m_r[0], mx0), mn1 = fmaxf(m_r[1], mx1);
      const bool any_grow = true;
#endif
      const float al0 = fast_exp2(m_r[0] - mn0), al1 = fast_exp2(m_r[1] - mn1);
      m_r[0] = mn0;
      m_r[1] = mn1;
      float p[2][4];
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        p[j][0] = fast_exp2(x[j][0] - mn0);
        p[j][1] = fast_exp2(x[j][1] - mn0);
        p[j][2] = fast_exp2(x[j][2] - mn1);
        p[j][3] = fast_exp2(x[j][3] - mn1);
        ps0 += p[j][0] + p[j][1];
        ps1 += p[j][2] + p[j][3];
      }
      l_r[0] = l_r[0] * al0 + ps0;
      l_r[1] = l_r[1] * al1 + ps1;
      if (any_grow) {
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          o[n][0] *= al0;
          o[n][1] *= al0;
          o[n][2] *= al1;
          o[n][3] *= al1;
        }
      }
      uint32_t pa[4];
      pa[0] = pack_bf16(p[0][0] * vmul[0], p[0][1] * vmul[1]);  // V scales fold into P (fp8 chunks)
      pa[1] = pack_bf16(p[0][2] * vmul[0], p[0][3] * vmul[1]);
      pa[2] = pack_bf16(p[1][0] * vmul[2], p[1][1] * vmul[3]);
      pa[3] = pack_bf16(p[1][2] * vmul[2], p[1][3] * vmul[3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int mi = lane >> 3;
        const int key = (mi & 1) * 8 + (lane & 7);
        const int dc = dp * 2 + (mi >> 1);
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(smem_u32(vt + (dc >> 3) * 2048 + sw128(key, dc & 7)), v0, v1, v2, v3);
        mma_bf16_16816(o[2 * dp], pa, v0, v1);
        mma_bf16_16816(o[2 * dp + 1], pa, v2, v3);
      }
      __syncwarp();
      release(slot);
    }
    // ---------------------------------------------- merge the consumers' states
    l_r[0] += __shfl_xor_sync(0xffffffffu, l_r[0], 1);
    l_r[0] += __shfl_xor_sync(0xffffffffu, l_r[0], 2);
    l_r[1] += __shfl_xor_sync(0xffffffffu, l_r[1], 1);
    l_r[1] += __shfl_xor_sync(0xffffffffu, l_r[1], 2);
    {
      const int g0 = lane >> 2, g1 = g0 + 8;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int dcol = n * 8 + 2 * (lane & 3);
        if (g0 < G) {
          mo[(cg * G + g0) * D + dcol] = o[n][0];
          mo[(cg * G + g0) * D + dcol + 1] = o[n][1];
        }
        if (g1 < G) {
          mo[(cg * G + g1) * D + dcol] = o[n][2];
          mo[(cg * G + g1) * D + dcol + 1] = o[n][3];
        }
      }
      if ((lane & 3) == 0) {
        if (g0 < G) { mm[cg * G + g0] = m_r[0]; ml[cg * G + g0] = l_r[0]; }
        if (g1 < G) { mm[cg * G + g1] = m_r[1]; ml[cg * G + g1] = l_r[1]; }
      }
    }
    }
    named_bar_sync(1, kNT);
    for (int idx = tid; idx < G * D; idx += kNT) {
      const int g = idx / D, dcol = idx % D;
      float M = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < kNCons; ++c) M = fmaxf(M, mm[c * G + g]);
      float Ls = 0.f, Os = 0.f;
      if (M != -CUDART_INF_F) {
#pragma unroll
        for (int c = 0; c < kNCons; ++c) {
          const float w = fast_exp2(mm[c * G + g] - M);
          Ls += w * ml[c * G + g];
          Os += w * mo[(c * G + g) * D + dcol];
        }
      }
      const int hq = h * G + g;
      if (a.splits == 1 && !a.part_o) {
        static_cast<__nv_bfloat16*>(a.out)[(int64_t(b) * a.Hq + hq) * D + dcol] = __float2bfloat16_rn(Os / Ls);
      } else {
        const int64_t pi = (int64_t(b) * a.Hq + hq) * a.splits + split;
        a.o_part[pi * D + dcol] = Ls > 0.f ? Os / Ls : 0.f;
        if (dcol == 0) a.lse_part[pi] = Ls > 0.f ? M + __log2f(Ls) : -CUDART_INF_F;
      }
    }
    named_bar_sync(1, kNT);  // merge area free for the next unit
  }
}

// a5 as a separate kernel (HPA_FUSED_COMBINE=0): one CTA per (request, q-head).
// With part_o set (context-parallel shard) it writes fp32 O and the merged LSE instead.
// The same kernel merges context-parallel shards (lse/o_part laid out [rows][S]).
template <int D>
__global__ void __launch_bounds__(D) combine_kernel(const float* __restrict__ o_part,
                                                    const float* __restrict__ lse, __nv_bfloat16* out,
                                                    int S_max, const int32_t* __restrict__ nsplit, int Hq,
                                                    float* part_o, float* part_lse) {
  grid_dependency_wait();
  grid_launch_dependents();
  const int64_t bh = blockIdx.x;
  const int S = nsplit ? nsplit[bh / Hq] : S_max;  // this request's split count
  const float* ls = lse + bh * S_max;
  float M = -CUDART_INF_F;
  for (int s = 0; s < S; ++s) M = fmaxf(M, ls[s]);
  float W = 0.f, acc = 0.f;
  for (int s = 0; s < S; ++s) {
    const float w = ls[s] == -CUDART_INF_F ? 0.f : fast_exp2(ls[s] - M);
    W += w;
    acc += w * o_part[(bh * S_max + s) * D + threadIdx.x];
  }
  if (part_o) {
    part_o[bh * D + threadIdx.x] = acc / W;
    if (threadIdx.x == 0) part_lse[bh] = M + __log2f(W);
  } else {
    out[bh * D + threadIdx.x] = __float2bfloat16_rn(acc / W);
  }
}

// a5 with one warp per (request, q-head): the lanes read the S_b split LSEs at once (S <= 64),
// reduce max and weight sum with shuffles, then each lane accumulates D/32 contiguous dims
// over the splits (independent float4 / float2 loads). 4 rows per 128-thread CTA.
template <int D>
__global__ void __launch_bounds__(128) combine_warp_kernel(const float* __restrict__ o_part,
                                                           const float* __restrict__ lse, __nv_bfloat16* out,
                                                           int S_max, const int32_t* __restrict__ nsplit, int Hq,
                                                           int64_t rows, float* part_o, float* part_lse) {
  grid_dependency_wait();
  grid_launch_dependents();
  constexpr int kV = D / 32;  // dims per lane
  const int lane = threadIdx.x & 31;
  const int64_t bh = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (bh >= rows) return;
  const int S = nsplit ? nsplit[bh / Hq] : S_max;
  const float* ls = lse + bh * S_max;
  const float l0 = lane < S ? ls[lane] : -CUDART_INF_F;
  const float l1 = lane + 32 < S ? ls[lane + 32] : -CUDART_INF_F;
  float M = fmaxf(l0, l1);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w0 = l0 == -CUDART_INF_F ? 0.f : fast_exp2(l0 - M);
  const float w1 = l1 == -CUDART_INF_F ? 0.f : fast_exp2(l1 - M);
  float W = w0 + w1;
#pragma unroll
  for (int o = 16; o; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
  float acc[kV];
#pragma unroll
  for (int v = 0; v < kV; ++v) acc[v] = 0.f;
  const float* op = o_part + bh * S_max * D + lane * kV;
  for (int s0 = 0; s0 < S; s0 += 4) {
    float vals[4][kV];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // up to 4 splits' loads in flight
      if (s0 + u < S) {
        if (kV == 4) {
          const float4 t = *reinterpret_cast<const float4*>(op + (s0 + u) * D);
          vals[u][0] = t.x; vals[u][1] = t.y; vals[u][2 % kV] = t.z; vals[u][3 % kV] = t.w;
        } else {
          const float2 t = *reinterpret_cast<const float2*>(op + (s0 + u) * D);
          vals[u][0] = t.x; vals[u][1 % kV] = t.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int sidx = s0 + u;
      const float w = __shfl_sync(0xffffffffu, sidx < 32 ? w0 : w1, sidx & 31);
      if (sidx < S) {
#pragma unroll
        for (int v = 0; v < kV; ++v) acc[v] += w * vals[u][v];
      }
    }
  }
  const float inv = 1.f / W;
  if (part_o) {
#pragma unroll
    for (int v = 0; v < kV; ++v) part_o[bh * D + lane * kV + v] = acc[v] * inv;
    if (lane == 0) part_lse[bh] = M + __log2f(W);
  } else {
    __nv_bfloat16* orow = out + bh * D + lane * kV;
    if (kV == 4) {
      uint2 w;
      w.x = pack_bf16(acc[0] * inv, acc[1] * inv);
      w.y = pack_bf16(acc[2 % kV] * inv, acc[3 % kV] * inv);
      *reinterpret_cast<uint2*>(orow) = w;
    } else {
      *reinterpret_cast<uint32_t*>(orow) = pack_bf16(acc[0] * inv, acc[1 % kV] * inv);
    }
  }
}

// Context-parallel merge: parts laid out [P][rows] (as all-gathered); one CTA per row.
template <int D>
__global__ void __launch_bounds__(D) merge_kernel(const float* __restrict__ o_parts,
                                                  const float* __restrict__ lse_parts, __nv_bfloat16* out,
                                                  int n_parts, int64_t n_rows) {
  grid_dependency_wait();
  grid_launch_dependents();
  const int64_t r = blockIdx.x;
  float M = -CUDART_INF_F;
  for (int p = 0; p < n_parts; ++p) M = fmaxf(M, lse_parts[p * n_rows + r]);
  float W = 0.f, acc = 0.f;
  for (int p = 0; p < n_parts; ++p) {
    const float l = lse_parts[p * n_rows + r];
    const float w = l == -CUDART_INF_F ? 0.f : fast_exp2(l - M);
    W += w;
    acc += w * o_parts[(p * n_rows + r) * D + threadIdx.x];
  }
  out[r * D + threadIdx.x] = __float2bfloat16_rn(acc / W);
}

template <int D, int NA>
cudaError_t launch_persistent(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const DecodeArgs& a,
                              const AppendRows* ap, cudaStream_t s) {
  AppendParams<NA> p{};
  if (ap) {
    p.k = static_cast<const __nv_bfloat16*>(ap->k);
    p.v = static_cast<const __nv_bfloat16*>(ap->v);
    p.k_pool = static_cast<__nv_bfloat16*>(ap->k_pool);
    p.v_pool = static_cast<__nv_bfloat16*>(ap->v_pool);
    p.stride_l = ap->stride_l;
    p.n = ap->n;
    p.L = ap->L;
    for (int i = 0; i < ap->n; ++i) p.tail[i] = ap->tail[i];
  }
  const int smem = PDecodeSmem<D>::bytes(a.G);
  const int grid = std::max(1, std::min(a.n_units, decode_slots(D, a.G)));
  if constexpr (NA == 1) {
    if (HPA_DEC_F32 && a.fp8 && a.G <= 8 && HPA_DEC_SWAP) {  // fp8 token pages: 32-row fp8 chunks
      if (a.groups)  // with cascade group units
        return launch_pdl(decode_persistent_kernel<D, true, 1, true, true>, dim3(grid), dim3((kNCons + 2) * 32),
                          PDecodeSmem<D, true, true>::bytes(a.G), s, tm_k, tm_v, a, p);
      return launch_pdl(decode_persistent_kernel<D, true, 1, true>, dim3(grid), dim3((kNCons + 2) * 32),
                        PDecodeSmem<D, true>::bytes(a.G), s, tm_k, tm_v, a, p);
    }
    if (a.groups) {  // cascade group units in the plan (bf16 token pages here, G <= 8)
      if (a.fp8 || a.G > 8 || !HPA_DEC_SWAP || HPA_DEC_PAIR) return cudaErrorInvalidValue;
      return launch_pdl(decode_persistent_kernel<D, true, 1, false, true>, dim3(grid), dim3((kNCons + 2) * 32),
                        PDecodeSmem<D, false, true>::bytes(a.G), s, tm_k, tm_v, a, p);
    }
  } else {
    if (a.groups) {  // fused append with cascade group units (bf16 token pages)
      if (a.fp8 || a.G > 8 || !HPA_DEC_SWAP || HPA_DEC_PAIR) return cudaErrorInvalidValue;
      return launch_pdl(decode_persistent_kernel<D, true, NA, false, true>, dim3(grid), dim3((kNCons + 2) * 32),
                        PDecodeSmem<D, false, true>::bytes(a.G), s, tm_k, tm_v, a, p);
    }
  }
  if (a.G <= 8 && HPA_DEC_SWAP)
    return launch_pdl(decode_persistent_kernel<D, true, NA>, dim3(grid), dim3((kNCons + 2) * 32), smem, s, tm_k,
                      tm_v, a, p);
  return launch_pdl(decode_persistent_kernel<D, false, NA>, dim3(grid), dim3((kNCons + 2) * 32), smem, s, tm_k,
                    tm_v, a, p);
}

template <int D>
cudaError_t launch_decode_d(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const DecodeArgs& a,
                            cudaStream_t s, int* launches, const AppendRows* ap) {
  cudaError_t e;
  if (HPA_DECODE_PERSISTENT) {
    if (!ap || ap->n == 0) e = launch_persistent<D, 1>(tm_k, tm_v, a, nullptr, s);
    else if (ap->n != a.n_seqs || ap->n > kAppendFuseMax) return cudaErrorInvalidValue;
    else if (ap->n <= kAppendFuseSmall) e = launch_persistent<D, kAppendFuseSmall>(tm_k, tm_v, a, ap, s);
    else e = launch_persistent<D, kAppendFuseMax>(tm_k, tm_v, a, ap, s);
  } else {
    if (ap && ap->n) return cudaErrorInvalidValue;
    const int smem = DecodeSmem<D>::kBytes;
    e = launch_pdl(decode_split_kernel<D>, dim3(a.splits, a.Hkv, a.n_seqs), dim3((kNCons + 1) * 32), smem, s,
                   tm_k, tm_v, a);
  }
  if (e != cudaSuccess) return e;
  ++*launches;
  if ((a.splits > 1 && !HPA_FUSED_COMBINE) || a.part_o) {
    const int64_t rows = int64_t(a.n_seqs) * a.Hq;
    if (HPA_COMBINE_WARP && a.splits <= 64)
      e = launch_pdl(combine_warp_kernel<D>, dim3(unsigned((rows + 3) / 4)), dim3(128), 0, s,
                     static_cast<const float*>(a.o_part), static_cast<const float*>(a.lse_part),
                     static_cast<__nv_bfloat16*>(a.out), a.splits, HPA_DECODE_PERSISTENT ? a.nsplit : nullptr,
                     a.Hq, rows, a.part_o, a.part_lse);
    else
      e = launch_pdl(combine_kernel<D>, dim3(unsigned(rows)), dim3(D), 0, s,
                     static_cast<const float*>(a.o_part), static_cast<const float*>(a.lse_part),
                     static_cast<__nv_bfloat16*>(a.out), a.splits, HPA_DECODE_PERSISTENT ? a.nsplit : nullptr,
                     a.Hq, a.part_o, a.part_lse);
    ++*launches;
  }
  return e;
}

}  // namespace

cudaError_t launch_merge(int32_t n_parts, int32_t n_rows, int32_t D, const float* o_parts,
                         const float* lse_parts, void* out, cudaStream_t s) {
  if (n_rows == 0) return cudaSuccess;
  if (D == 128)
    return launch_pdl(merge_kernel<128>, dim3(n_rows), dim3(128), 0, s, o_parts, lse_parts,
                      static_cast<__nv_bfloat16*>(out), n_parts, int64_t(n_rows));
  if (D == 64)
    return launch_pdl(merge_kernel<64>, dim3(n_rows), dim3(64), 0, s, o_parts, lse_parts,
                      static_cast<__nv_bfloat16*>(out), n_parts, int64_t(n_rows));
  return cudaErrorInvalidValue;
}

template <int NA>
cudaError_t set_persistent_attrs() {
  auto cap = [](int bytes) { return std::min(bytes, 227 * 1024); };
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(decode_persistent_kernel<128, false, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<128>::bytes(16)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<64, false, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<64>::bytes(16)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<128, true, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<128>::bytes(8)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<64, true, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<64>::bytes(8)))) != cudaSuccess)
    return e;
  if constexpr (NA > 1) {  // fused append with cascade group units
    if ((e = cudaFuncSetAttribute(decode_persistent_kernel<128, true, NA, false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  cap(PDecodeSmem<128, false, true>::bytes(8)))) != cudaSuccess ||
        (e = cudaFuncSetAttribute(decode_persistent_kernel<64, true, NA, false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  cap(PDecodeSmem<64, false, true>::bytes(8)))) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

cudaError_t set_f32_attrs() {
  auto cap = [](int bytes) { return std::min(bytes, 227 * 1024); };
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(decode_persistent_kernel<128, true, 1, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<128, true>::bytes(8)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<64, true, 1, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<64, true>::bytes(8)))) != cudaSuccess)
    return e;
  return cudaSuccess;
}

cudaError_t set_cascade_attrs() {
  auto cap = [](int bytes) { return std::min(bytes, 227 * 1024); };
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(decode_persistent_kernel<128, true, 1, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<128, false, true>::bytes(8)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<64, true, 1, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<64, false, true>::bytes(8)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<128, true, 1, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<128, true, true>::bytes(8)))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_persistent_kernel<64, true, 1, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(PDecodeSmem<64, true, true>::bytes(8)))) != cudaSuccess)
    return e;
  return cudaSuccess;
}

cudaError_t decode_init_attributes() {
  // the opt-in maximum is 227 KB; configurations that need more fail at launch instead
  auto cap = [](int bytes) { return std::min(bytes, 227 * 1024); };
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(decode_split_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(DecodeSmem<128>::kBytes))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(decode_split_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cap(DecodeSmem<64>::kBytes))) != cudaSuccess ||
      (e = set_persistent_attrs<1>()) != cudaSuccess || (e = set_persistent_attrs<kAppendFuseSmall>()) != cudaSuccess ||
      (e = set_persistent_attrs<kAppendFuseMax>()) != cudaSuccess || (e = set_f32_attrs()) != cudaSuccess ||
      (e = set_cascade_attrs()) != cudaSuccess)
    return e;
  return cudaSuccess;
}

bool decode_persistent() { return HPA_DECODE_PERSISTENT != 0; }

int decode_slots(int32_t D, int32_t G) {
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int smem = D == 64 ? PDecodeSmem<64>::bytes(G) : PDecodeSmem<128>::bytes(G);
  const int per_sm = std::max(1, std::min(HPA_DECODE_CTAS_PER_SM, (227 * 1024) / (smem + 1024)));
  return num_sms * per_sm;
}

int decode_ctas_per_sm(int32_t D, int32_t /*G*/) {
  const int smem = (D == 64 ? DecodeSmem<64>::kBytes : DecodeSmem<128>::kBytes) + 1024;
  int by_smem = (228 * 1024) / smem;
  return by_smem < 3 ? by_smem : 3;
}

cudaError_t launch_decode(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const DecodeArgs& a,
                          int32_t D, cudaStream_t s, int* launches, const AppendRows* ap) {
  if (a.n_seqs == 0) return cudaSuccess;
  if (D == 128) return launch_decode_d<128>(tm_k, tm_v, a, s, launches, ap);
  if (D == 64) return launch_decode_d<64>(tm_k, tm_v, a, s, launches, ap);
  return cudaErrorInvalidValue;
}

}  // namespace hpa
