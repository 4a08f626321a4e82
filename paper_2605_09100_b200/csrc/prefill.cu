// prefill.cu -- hybrid paged chunked-prefill attention on tcgen05/TMEM/TMA
// (SURVEY §8(a) a6).
//
// What it computes (§3 HPA P:L248-251; readings A1, A9):
// for each sequence the queries are its LAST q_len logical rows; query row t
// (logical index i = seq_len - q_len + t) attends the keys j <= i of the
// logical KV sequence in block-table order (latent and token pages alike):
//   o = softmax(scale * q K^T, causal bottom-right) V, fp32 accumulation,
//   P rounded to bf16 before the PV product, bf16 output.
//
// Design (sm_100a; roofline: bf16 tensor pipe):
//  * CTA = one 128-row query tile of one q-head (grid: M tiles x Hq x seqs),
//    192 threads: warp 0 = TMA producer, warp 1 = tcgen05 MMA issuer (+ TMEM
//    owner), warps 2..5 = softmax / correction / epilogue (one TMEM lane = one
//    query row per thread).
//  * Key tiles are 128 page *slots*: 128/P whole pages (P <= 128) or a
//    128-row slice of a page (P = 256), each page box loaded by 2-D TMA with
//    128-B swizzle straight from the pool; slots past the table are TMA
//    out-of-bounds (zero-filled). The producer also publishes each slot's
//    logical index (INT_MAX for rows >= valid_rows) for the mask.
//  * S = Q K^T: tcgen05.mma kind::f16, M=128, N=128, K=16 steps, SS operands
//    (K-major SW128 descriptors), fp32 accumulator in TMEM (double-buffered:
//    S_{j+1} is computed while softmax j runs).
//  * softmax: tcgen05.ld of the row, log2-domain online softmax with lazy
//    rescaling (O in TMEM is corrected only when the row max grows by > 2^8),
//    P -> bf16 -> shared memory (K-major SW128) for O += P V (V is the
//    MN-major B operand), O accumulated in TMEM.
#include "hpa_kernels.h"
#include "ptx.cuh"
#include <cuda_bf16.h>
#include <math_constants.h>
#include <climits>

namespace hpa {
namespace {

constexpr int kBM = 128;      // query rows per CTA
constexpr int kBN = 128;      // key slots per tile
constexpr int kNK = 2;        // K ring depth
constexpr int kNV = 2;        // V ring depth
constexpr int kNC = 4;        // column-index ring depth
constexpr float kRescaleThreshold = 8.0f;  // log2 units (factor 256)

template <int D>
struct PSmem {
  static constexpr int kQ = kBM * D * 2;
  static constexpr int kKV = kBN * D * 2;
  static constexpr int kP = kBM * kBN * 2;
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + kQ;
  static constexpr int oV = oK + kNK * kKV;
  static constexpr int oP = oV + kNV * kKV;
  static constexpr int oC = oP + kP;                     // int32 [kNC][kBN + 1] (last = flags)
  static constexpr int oBar = oC + kNC * (kBN + 4) * 4;  // mbarriers
  // barriers: q_full, k_full[NK], k_empty[NK], v_full[NV], v_empty[NV], s_full[2], s_empty[2],
  //           p_full, p_empty, o_full, c_full[NC], c_empty[NC]
  static constexpr int kNBar = 1 + 2 * kNK + 2 * kNV + 4 + 3 + 2 * kNC;
  static constexpr int oTmem = oBar + kNBar * 8;
  // >= 116 KB so that exactly one CTA is resident per SM (it owns all 512 TMEM columns)
  static constexpr int kRaw = oTmem + 16 + 1024;
  static constexpr int kBytes = kRaw > 116 * 1024 ? kRaw : 116 * 1024;
};

// ---- tcgen05 helpers
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "smem descriptor"): start >> 4 in
// bits 0-13, LBO >> 4 in 16-29, SBO >> 4 in 32-45, version 1 in 46-47,
// layout SWIZZLE_128B (2) in 61-63.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
// Instruction descriptor kind::f16: bf16 A/B, fp32 D, M, N, A/B major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int D>
__global__ void __launch_bounds__(192, 1)
prefill_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const PrefillArgs a) {
  using L = PSmem<D>;
  constexpr int kHalves = D / 64;
  const int mt = blockIdx.x, hq = blockIdx.y, b = blockIdx.z;
  const int q_len = a.q_len[b];
  if (mt * kBM >= q_len) return;  // ragged: this sequence has fewer query tiles

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + L::oQ;
  uint8_t* sK = sm + L::oK;
  uint8_t* sV = sm + L::oV;
  uint8_t* sP = sm + L::oP;
  int32_t* sC = reinterpret_cast<int32_t*>(sm + L::oC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kNK;
  uint64_t* v_full = k_empty + kNK;
  uint64_t* v_empty = v_full + kNV;
  uint64_t* s_full = v_empty + kNV;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 1;
  uint64_t* o_full = p_empty + 1;
  uint64_t* c_full = o_full + 1;
  uint64_t* c_empty = c_full + kNC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oTmem);
  int32_t* ntiles_slot = reinterpret_cast<int32_t*>(sm + L::oTmem + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = a.seq_rows[b];
  const int h = hq / a.G;
  const int seq_len = a.t.seq_len[seq];
  const int n_ent = a.t.n_entries[seq];
  const int32_t* bt = a.t.block_table + int64_t(seq) * a.t.max_pages;
  const int32_t* p0 = a.t.pos0 + int64_t(seq) * a.t.max_pages;
  const int32_t* mt_ = a.t.meta + int64_t(seq) * a.t.max_pages;
  const int P = a.P;
  const int i_min = seq_len - q_len + mt * kBM;                       // logical index of row 0
  const int i_max = seq_len - q_len + min(q_len, (mt + 1) * kBM) - 1;  // of the last real row

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < kNK; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < kNV; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 128); }
    mbar_init(p_full, 128);
    mbar_init(p_empty, 1);
    mbar_init(o_full, 1);
    for (int i = 0; i < kNC; ++i) { mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], 128); }
    fence_barrier_init();
    // number of key tiles: the tile holding the slot of logical index i_max
    int lo = 0, hi = n_ent - 1;  // last entry with pos0 <= i_max
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p0[mid] <= i_max) lo = mid; else hi = mid - 1;
    }
    const int64_t slot = int64_t(lo) * P + (i_max - p0[lo]);
    *ntiles_slot = int(slot / kBN) + 1;
  }
  if (warp == 1) {  // TMEM: S0 [0,128), S1 [128,256), O [256, 256+D)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_tiles = *ntiles_slot;

  if (warp == 0) {
    // ================================================================ producer
    // lane 0 issues every TMA; all 32 lanes build the tile's mask indices.
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const int q_tok = a.q_off[b] + mt * kBM;
      mbar_arrive_expect_tx(q_full, L::kQ);
#pragma unroll
      for (int hf = 0; hf < kHalves; ++hf) tma_load_3d(sQ + hf * kBM * 128, &tm_q, q_full, hf * 64, hq, q_tok);
    }
    const int pbox = P < kBN ? P : kBN;
    const int nbox = kBN / pbox;
    constexpr int kOobRow = INT_MAX / 2;  // fully out-of-bounds box -> TMA zero fill
    for (int j = 0; j < n_tiles; ++j) {
      // logical index of every key slot (INT_MAX: row >= valid_rows or past the table)
      const int cs = j % kNC;
      if (j >= kNC) mbar_wait(&c_empty[cs], ((j / kNC) - 1) & 1);
      int32_t* col = sC + cs * (kBN + 4);
      bool vis = true;
#pragma unroll
      for (int x = 0; x < kBN / 32; ++x) {
        const int c = x * 32 + lane;
        const int64_t slot = int64_t(j) * kBN + c;
        const int e = int(slot / P), r = int(slot % P);
        int v = INT_MAX;
        if (e < n_ent && r < (mt_[e] & kMetaRowsMask)) v = p0[e] + r;
        col[c] = v;
        vis &= (v <= i_min);
      }
      vis = __all_sync(0xffffffffu, vis);
      if (lane == 0) col[kBN] = vis ? 1 : 0;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&c_full[cs]);
        const int ks = j % kNK;
        if (j >= kNK) mbar_wait(&k_empty[ks], ((j / kNK) - 1) & 1);
        mbar_arrive_expect_tx(&k_full[ks], L::kKV);
        for (int bx = 0; bx < nbox; ++bx) {
          const int64_t slot = int64_t(j) * kBN + bx * pbox;
          const int e = int(slot / P), r = int(slot % P);
          const int row = e < n_ent ? ((a.layer * a.NP + bt[e]) * a.Hkv + h) * P + r : kOobRow;
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tma_load_2d(sK + ks * L::kKV + hf * kBN * 128 + bx * pbox * 128, &tm_k, &k_full[ks], hf * 64, row);
        }
        const int vs = j % kNV;
        if (j >= kNV) mbar_wait(&v_empty[vs], ((j / kNV) - 1) & 1);
        mbar_arrive_expect_tx(&v_full[vs], L::kKV);
        for (int bx = 0; bx < nbox; ++bx) {
          const int64_t slot = int64_t(j) * kBN + bx * pbox;
          const int e = int(slot / P), r = int(slot % P);
          const int row = e < n_ent ? ((a.layer * a.NP + bt[e]) * a.Hkv + h) * P + r : kOobRow;
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tma_load_2d(sV + vs * L::kKV + hf * kBN * 128 + bx * pbox * 128, &tm_v, &v_full[vs], hf * 64, row);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
      constexpr uint32_t idO = idesc_bf16(kBM, D, 0, 1);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP);
      const uint32_t tO = tmem + 256;
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        mbar_wait(p_full, jj & 1);
        const int vs = jj % kNV;
        mbar_wait(&v_full[vs], (jj / kNV) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBN / 16; ++k) {
          // A = P [128 x 128 keys], K-major, 64-key blocks of 16 KB; B = V [keys x D], MN-major
          const uint64_t ad = sdesc(aP + (k >> 2) * (kBM * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(aV + vs * L::kKV + k * 2048, kBN * 128, 1024);
          tc_mma(tO, ad, bd, idO, (jj > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(&v_empty[vs]);
        tc_commit(p_empty);
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int ks = j % kNK, sb = j & 1;
        mbar_wait(&k_full[ks], (j / kNK) & 1);
        if (j >= 2) mbar_wait(&s_empty[sb], ((j >> 1) - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t ad = sdesc(aQ + (k >> 2) * (kBM * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(aK + ks * L::kKV + (k >> 2) * (kBN * 128) + (k & 3) * 32, 16, 1024);
          tc_mma(tmem + sb * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        tc_commit(&k_empty[ks]);
        tc_commit(&s_full[sb]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
      tc_commit(o_full);
    }
  } else {
    // ================================================================ softmax
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;          // query row within the tile == TMEM lane
    const int t = mt * kBM + row;
    const int my_i = seq_len - q_len + t;         // logical index of this query row
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    const float sl2 = a.scale_log2;
    float m_run = -CUDART_INF_F, l_run = 0.f;
    float s[kBN];
    for (int j = 0; j < n_tiles; ++j) {
      const int sb = j & 1, cs = j % kNC;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c) tc_ld32(tmem + lane_base + sb * 128 + c * 32, s + c * 32);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[sb]);
      mbar_wait(&c_full[cs], (j / kNC) & 1);
      const int32_t* col = sC + cs * (kBN + 4);
      float mx = -CUDART_INF_F;
      if (col[kBN]) {
#pragma unroll
        for (int c = 0; c < kBN; ++c) {
          s[c] *= sl2;
          mx = fmaxf(mx, s[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < kBN; c += 4) {
          const int4 ci = *reinterpret_cast<const int4*>(col + c);
          s[c + 0] = ci.x <= my_i ? s[c + 0] * sl2 : -CUDART_INF_F;
          s[c + 1] = ci.y <= my_i ? s[c + 1] * sl2 : -CUDART_INF_F;
          s[c + 2] = ci.z <= my_i ? s[c + 2] * sl2 : -CUDART_INF_F;
          s[c + 3] = ci.w <= my_i ? s[c + 3] * sl2 : -CUDART_INF_F;
          mx = fmaxf(mx, fmaxf(fmaxf(s[c], s[c + 1]), fmaxf(s[c + 2], s[c + 3])));
        }
      }
      mbar_arrive(&c_empty[cs]);
      // lazy rescale: move the running max only when it grows by > 2^8
      const bool grow = mx > m_run + kRescaleThreshold;
      const float m_new = grow ? mx : m_run;
      const float alpha = grow ? fast_exp2(m_run - m_new) : 1.f;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < kBN; ++c) {
        s[c] = fast_exp2(s[c] - m_new);
        rs += s[c];
      }
      l_run = l_run * alpha + rs;
      m_run = m_new;
      // wait until PV_{j-1} has finished with P and O
      if (j >= 1) mbar_wait(p_empty, (j - 1) & 1);
      tc_fence_after();
      if (j >= 1 && __any_sync(0xffffffffu, grow)) {
        float o[32];
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          tc_ld32(tmem + lane_base + 256 + c * 32, o);
          tc_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) o[x] *= alpha;
          tc_st32(tmem + lane_base + 256 + c * 32, o);
        }
        tc_wait_st();
      }
      // P (bf16) -> smem, K-major SW128: 64-key blocks, row = query row
#pragma unroll
      for (int c8 = 0; c8 < kBN / 8; ++c8) {
        uint4 pk;
        pk.x = pack_bf16(s[c8 * 8 + 0], s[c8 * 8 + 1]);
        pk.y = pack_bf16(s[c8 * 8 + 2], s[c8 * 8 + 3]);
        pk.z = pack_bf16(s[c8 * 8 + 4], s[c8 * 8 + 5]);
        pk.w = pack_bf16(s[c8 * 8 + 6], s[c8 * 8 + 7]);
        *reinterpret_cast<uint4*>(sP + (c8 >> 3) * (kBM * 128) + sw128(row, c8 & 7)) = pk;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 -> global
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv = 1.f / l_run;
    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + (int64_t(a.q_off[b] + t) * a.Hq + hq) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      tc_ld32(tmem + lane_base + 256 + c * 32, o);
      tc_wait_ld();
      if (t < q_len) {
#pragma unroll
        for (int x = 0; x < 32; x += 8) {
          uint4 pk;
          pk.x = pack_bf16(o[x + 0] * inv, o[x + 1] * inv);
          pk.y = pack_bf16(o[x + 2] * inv, o[x + 3] * inv);
          pk.z = pack_bf16(o[x + 4] * inv, o[x + 5] * inv);
          pk.w = pack_bf16(o[x + 6] * inv, o[x + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + x) = pk;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int D>
cudaError_t launch_prefill_d(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                             const PrefillArgs& a, cudaStream_t s, int* launches) {
  dim3 grid((a.max_q_len + kBM - 1) / kBM, a.Hq, a.n_seqs);
  prefill_kernel<D><<<grid, 192, PSmem<D>::kBytes, s>>>(tm_q, tm_k, tm_v, a);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t prefill_init_attributes() {
  cudaError_t e = cudaFuncSetAttribute(prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PSmem<128>::kBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, PSmem<64>::kBytes);
}

cudaError_t launch_prefill(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                           const PrefillArgs& a, int32_t D, cudaStream_t s, int* launches) {
  if (a.n_seqs == 0) return cudaSuccess;
  if (D == 128) return launch_prefill_d<128>(tm_q, tm_k, tm_v, a, s, launches);
  if (D == 64) return launch_prefill_d<64>(tm_q, tm_k, tm_v, a, s, launches);
  return cudaErrorInvalidValue;
}

}  // namespace hpa
