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
//  * CTA = two 128-row query tiles ("slots") that share every K/V tile: two
//    q-heads of the same GQA group over the same token rows (G even), or two
//    consecutive row tiles of one head (G odd). 384 threads = 3 warpgroups:
//      warps 0-3  softmax warpgroup for slot 0 (one TMEM lane = one row)
//      warps 4-7  softmax warpgroup for slot 1
//      warp  8    TMA producer (all lanes build the mask indices; the page
//                 boxes are issued in parallel by several lanes)
//      warp  9    tcgen05 MMA issuer; owns the 512 TMEM columns
//      warp  10   V producer (decoupled from K); warp 11 spare. setmaxnreg moves registers
//                 from warpgroup 2 (72) to the softmax warpgroups (216).
//  * TMEM: S_s / P_s at columns [128 s, 128 s + 128), O_s at [256 + 128 s, ...).
//    S = Q K^T (SS: Q and K K-major, 128-B swizzle); the softmax writes P as
//    packed bf16 over S and O += P V runs in TS form (A = P from TMEM, B = V
//    MN-major from shared memory). The two slots ping-pong so the tensor pipe
//    computes one slot's QK^T / PV while the other slot's softmax runs.
//  * Key tiles are 128 page *slots*: 128/P whole pages (P <= 128) or a 128-row
//    slice of one page (P = 256); each page box is a 2-D TMA load straight from
//    the pool; slots past the table are out-of-bounds boxes (zero fill). The
//    producer publishes each key slot's logical index (INT_MAX when the row is
//    >= valid_rows) for the causal / partial-page mask.
//  * Online softmax in the log2 domain with lazy rescaling: O_s in TMEM is
//    corrected only when a row max grows by more than 2^8.
//  * Work: a host-planned list (plan_prefill in runtime.cpp) gives each CTA its unit and
//    key-tile range; units of an under-filled last wave are split into key ranges whose
//    fp32 O / l + LSE partials prefill_combine_kernel merges. The epilogue stages O in the
//    idle K/V rings and writes it with TMA stores. prefill_persistent_kernel runs one CTA per
//    SM over a host-assigned item list instead (the default below 4 waves of units, with
//    stream-K shares: plan_prefill_streamk in runtime.cpp).
#include "hpa_kernels.h"
#include "ptx.cuh"
#include <cuda_bf16.h>
#include <math_constants.h>
#include <climits>

namespace hpa {
namespace {

// HPA_SM16 = 1: 16 softmax warps -- two per SMSP per slot, each owning 64 of a row's 128
// key columns (and half of O's columns); the row max is exchanged through shared memory.
// A slot's exps are then spread over twice the warps, shortening the QK -> softmax -> PV
// chain. HPA_SM16 = 0: 8 softmax warps, one per row.
// HPA_PF1 = 1: one 128-row query tile per CTA with TWO S buffers in TMEM, so Q K^T of tile
// j+2 runs while the softmax of tile j+1 runs (the QK -> softmax -> PV chain of one tile no
// longer serialises the tensor pipe); the 8 softmax warps split each row's 128 key columns
// in two halves (row max exchanged through shared memory).
#ifndef HPA_PF1
#define HPA_PF1 0
#endif
#ifndef HPA_PF1_CLUSTER
#define HPA_PF1_CLUSTER 1  // HPA_PF1, G even: 2-CTA clusters share K/V boxes by TMA multicast
#endif
#ifndef HPA_SM16
#define HPA_SM16 0  // 1 measured slower (1101 vs 1236 TFLOP/s): a slot's exps share the same SMSP MUFUs
#endif
constexpr int kBM = 128;   // query rows per slot
constexpr int kBN = 128;   // key slots per tile
#ifndef HPA_PF_MC2
#define HPA_PF_MC2 1  // default kernel as 2-CTA clusters (the 4 q-heads of a KV head) sharing K/V by TMA multicast
#endif
#if HPA_PF1
#undef HPA_PF_MC2
#define HPA_PF_MC2 0
#endif
#ifndef HPA_PF_NK
#define HPA_PF_NK (HPA_SM16 ? 2 : 3)  // K ring depth (2 leaves room for the SM16 max exchange)
#endif
#ifndef HPA_PF_NV
#define HPA_PF_NV 2  // V ring depth (NK 2 / NV 3 measured the same)
#endif
constexpr int kNK = HPA_PF_NK;
constexpr int kNV = HPA_PF_NV;
constexpr int kNC = 3;     // mask-index ring depth
constexpr int kSoftWarps = HPA_SM16 ? 16 : 8;
constexpr int kThreads = (kSoftWarps + 4) * 32;  // softmax warpgroups + producer / MMA / V producer / spare
constexpr int kProducerWarp = kSoftWarps;
constexpr int kMmaWarp = kSoftWarps + 1;
constexpr int kVProducerWarp = kSoftWarps + 2;
#ifndef HPA_SOFTMAX_REGS
#define HPA_SOFTMAX_REGS (HPA_SM16 ? 104 : 216)
#endif
#ifndef HPA_OTHER_REGS
#define HPA_OTHER_REGS (HPA_SM16 ? 64 : 72)
#endif
// setmaxnreg: the launch allocates R0 = floor(65536 / kThreads / 8) * 8 regs per thread;
// the softmax warpgroups may grow only by what the role warpgroup gives up.
constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 168 ? 168 : (65536 / kThreads) / 8 * 8;
constexpr int kSoftmaxRegs = HPA_SOFTMAX_REGS;
constexpr int kOtherRegs = HPA_OTHER_REGS;
static_assert((kSoftWarps / 4) * kSoftmaxRegs + kOtherRegs <= (kSoftWarps / 4 + 1) * kLaunchRegs,
              "setmaxnreg budget");
constexpr float kRescaleThreshold = 8.0f;  // log2 units (factor 256)
constexpr int kSpanBit = 1 << 30;          // tags span columns in the mask indices (seq_len < 2^30)
#ifndef HPA_POLY_EVERY
#define HPA_POLY_EVERY 0  // 1 of every N exp2 pairs on the FMA pipe (0 = all on MUFU; measured best)
#endif
// Phase trace (HPA_TRACE builds): stamp[event][tile] for CTA (0,0,0), tiles < 64.
#ifdef HPA_TRACE
#define TRACE(ev, j)                                                                         \
  do {                                                                                       \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64)        \
      a.trace[(ev) * 64 + (j)] = clock64();                                                  \
  } while (0)
// CTA timeline (HPA_TRACE builds): trace[4096 + 8 i ...] = {entry ns, setup done, first S,
// o_full passed, exit ns, smid, n_tiles, 1} of CTA i (globaltimer).
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CTA_STAMP(k, v)                                                                      \
  do {                                                                                       \
    if (a.trace) a.trace[4096 + 8 * int64_t(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) + (k)] = (v); \
  } while (0)
#else
#define TRACE(ev, j) do { } while (0)
#define CTA_STAMP(k, v) do { } while (0)
#endif
#ifndef HPA_P_PACK_ALU
#define HPA_P_PACK_ALU 0  // 1: P -> bf16 on the ALU pipe instead of F2FP (measured slower)
#endif
#ifndef HPA_EXP_INPLACE
#define HPA_EXP_INPLACE 0  // 1: all ex2 of a half first (in place), then sums and packs (measured no faster)
#endif
#ifndef HPA_OPT_EXP  // softmax: first-half exps against the running max with the tile max reduced
#define HPA_OPT_EXP (!HPA_EXP_INPLACE)  // alongside (needs the raw scores, so not with in-place exps)
#endif
#ifndef HPA_SPLIT_LD
#define HPA_SPLIT_LD 0  // 1: S loaded in two halves, P half 0 stored before the max check (measured 1 % slower)
#endif
#ifndef HPA_PV_SPLIT
#define HPA_PV_SPLIT 1    // publish P in two 64-key halves (PV starts on the first half)
#endif
#ifndef HPA_SM_SEQ
#define HPA_SM_SEQ 0  // 1: the two slots' exp phases alternate per SMSP (MUFU hand-off barriers); measured slower (B=4 1253 vs 1266 TFLOP/s, profiles/r2_prefill_ab.log)
#endif
// MUFU hand-off (HPA_SM_SEQ): softmax warp q of slot 0 and warp q of slot 1 share SMSP q and its
// MUFU. Their exp phases take turns -- slot 0 tile j, slot 1 tile j, slot 0 tile j+1, ... -- so
// each runs at the full MUFU rate instead of both at half rate for longer: named barrier
// kSeqBar0 + q (slot 1 -> slot 0) and kSeqBar1 + q (slot 0 -> slot 1), 64 threads each.
constexpr uint32_t kSeqBar0 = 3, kSeqBar1 = 7;

template <int D>
struct PSmem {
  static constexpr int kQ = kBM * D * 2;   // one slot's Q tile
  static constexpr int kKV = kBN * D * 2;
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + (HPA_PF1 ? 1 : 2) * kQ;
  static constexpr int oV = oK + kNK * kKV;
  static constexpr int oC = oV + kNV * kKV;              // int32 [kNC][kBN + 4] (kBN = all-visible flag)
  static constexpr int oBar = oC + kNC * (kBN + 4) * 4;
  // q_full, k_full[NK], k_empty[NK], v_full[NV], v_empty[NV], s_full[2], p_full[2 slots][2 halves],
  // o_full, c_full[NC], c_empty[NC]
  static constexpr int kNBar = 1 + 2 * kNK + 2 * kNV + 2 + 4 + 1 + 2 * kNC + 2;  // + o_ready (HPA_PF1) / q_empty, o_full1 (persistent)
  static constexpr int oX = oBar + kNBar * 8;      // HPA_SM16: row max [2 buf][2 slot][2 half][128], row sum [2][2][128]
  static constexpr int kXBytes = (HPA_SM16 || HPA_PF1) ? (8 + 4) * kBM * 4 : 0;
  static constexpr int oMisc = oX + kXBytes;
  static constexpr int kRaw = oMisc + 16 + 1024;  // tmem addr + 3 tile words
  // >= 116 KB so exactly one CTA is resident per SM (it owns all 512 TMEM columns)
  static constexpr int kBytes = kRaw > 116 * 1024 ? kRaw : 116 * 1024;
};

static_assert(PSmem<128>::kBytes <= 227 * 1024 && PSmem<64>::kBytes <= 227 * 1024, "prefill shared memory");

// ---- tcgen05 helpers
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// One lane of a converged warp (the lowest): the MMA issuer runs its loop warp-uniformly so the
// descriptor arithmetic stays in uniform registers, and only the elected lane issues.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
// D[tmem] (+)= A[smem desc] * B[smem desc]
__device__ __forceinline__ void tc_mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
#define HPA_R32(r)                                                                                       \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),        \
      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),        \
      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define HPA_W32(r)                                                                                       \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),    \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),    \
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),   \
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : HPA_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      HPA_W32(r)
      : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2) and a polynomial exp2
__device__ __forceinline__ uint64_t f2_as_u64(float2 v) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 u64_as_f2(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_as_u64(a)), "l"(f2_as_u64(b)), "l"(f2_as_u64(c)));
  return u64_as_f2(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_as_u64(a)), "l"(f2_as_u64(b)));
  return u64_as_f2(d);
}
// 2^x for x <= 0 on the FMA pipe: x = j + f, j = round(x), f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. error 1.0e-4 < bf16's 2^-9),
// 2^j by adding j to the exponent field. x < -126 flushes towards 0.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float2 lo = make_float2(-126.f, -126.f);
  x.x = fmaxf(x.x, lo.x);
  x.y = fmaxf(x.y, lo.y);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23: round to integer
  const float2 t = fadd2(x, magic);
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = fadd2(x, make_float2(-j.x, -j.y));
  float2 p = ffma2(f, make_float2(0.05499337f, 0.05499337f), make_float2(0.242211f, 0.242211f));
  p = ffma2(f, p, make_float2(0.6932861f, 0.6932861f));
  p = ffma2(f, p, make_float2(1.f, 1.f));
  float2 r;
  r.x = __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23));
  r.y = __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23));
  return r;
}

// ---- HPA_PF1 clusters: TMA multicast to both CTAs of a pair, multicast MMA commit, cluster barrier
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Shared-memory matrix descriptor: start >> 4 (bits 0-13), LBO >> 4 (16-29),
// SBO >> 4 (32-45), version 1 (46-47), layout SWIZZLE_128B = 2 (61-63).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
// Instruction descriptor kind::f16: bf16 A/B, fp32 D, M, N, A/B major (0 = K, 1 = MN).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// Unit (y, x) -> the two slots' (q-head, row tile): G even pairs two q-heads of one GQA group
// over row tile x (y = kv-head * G/2 + pair); G odd pairs row tiles 2x, 2x+1 of q-head y.
__device__ __forceinline__ void unit_slots(int G, int y, int x, int* hq_s, int* mt_s) {
  if ((G & 1) == 0) {
    const int h = y / (G >> 1), pair = y % (G >> 1);
    hq_s[0] = h * G + 2 * pair;
    hq_s[1] = hq_s[0] + 1;
    mt_s[0] = mt_s[1] = x;
  } else {
    hq_s[0] = hq_s[1] = y;
    mt_s[0] = 2 * x;
    mt_s[1] = 2 * x + 1;
  }
}

// One 128-key tile of a slot's online softmax (default kernel configuration): S_s from TMEM,
// the causal / span / partial-page mask from the producer's key indices `col` (ring stage
// released on `cempty`), lazy-rescaled running max, exps (optimistic first half), P as bf16
// pairs over S_s in two published halves (pf[0], pf[1]), running row sum. The caller has
// waited for S_s(j). `j` = the tile's index within its unit (O_s is rescaled only for j > 0).
template <int D>
__device__ __forceinline__ void softmax_tile(const PrefillArgs& a, int s, int quarter, int row, int lane, int j,
                                             uint32_t tS, uint32_t tO, const int32_t* col, uint64_t* cfull,
                                             uint32_t cpar, uint64_t* cempty, uint64_t* pf, int my_i,
                                             int span_from, float sl2, float& m_run, float& l_run,
                                             bool seq = false, bool seq_last = false) {
  float x[kBN];
  constexpr int kLd0 = HPA_SPLIT_LD ? kBN / 2 : kBN;  // columns loaded before the first wait
#pragma unroll
  for (int c = 0; c < kLd0 / 32; ++c) tc_ld32(tS + c * 32, x + c * 32);
  mbar_wait(cfull, cpar);
  const bool all_vis = col[kBN] != 0;
  const int cmask = my_i >= span_from ? -1 : ~kSpanBit;  // span tag visible only to span rows
  auto mask_cols = [&](int c0, int c1) {
#pragma unroll
    for (int c = c0; c < c1; c += 4) {
      const int4 ci = *reinterpret_cast<const int4*>(col + c);
      x[c + 0] = (ci.x & cmask) <= my_i ? x[c + 0] : -CUDART_INF_F;
      x[c + 1] = (ci.y & cmask) <= my_i ? x[c + 1] : -CUDART_INF_F;
      x[c + 2] = (ci.z & cmask) <= my_i ? x[c + 2] : -CUDART_INF_F;
      x[c + 3] = (ci.w & cmask) <= my_i ? x[c + 3] : -CUDART_INF_F;
    }
  };
  tc_wait_ld();
  if (HPA_SPLIT_LD) {  // second half in flight while the first is masked (and exp'd, below)
#pragma unroll
    for (int c = kLd0 / 32; c < kBN / 32; ++c) tc_ld32(tS + c * 32, x + c * 32);
  }
  if (row == 0) TRACE(9 + s, j);
  if (!all_vis) mask_cols(0, kLd0);
  if (!HPA_SPLIT_LD) {
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty);  // col[] consumed (masking done)
  }
  // p = 2^(x*sl2 - m): f32x2 FFMA for the argument, MUFU ex2 (optionally 1 pair in
  // HPA_POLY_EVERY on the FMA pipe); 4 independent partial row sums
  const float2 sl2x2 = make_float2(sl2, sl2);
  float2 rs4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  auto exps_half = [&](int half, float m_use, uint32_t* pk) {
    const float2 negm = make_float2(-m_use, -m_use);
    if (HPA_EXP_INPLACE) {
      // all ex2 first (in place: x of this half is dead once its max is known), then the sums
      // and bf16 packs, so no MUFU result is consumed right behind its producer
#pragma unroll
      for (int c = half * 64; c < half * 64 + 64; c += 2) {
        const float2 arg = ffma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
        x[c] = fast_exp2(arg.x);
        x[c + 1] = fast_exp2(arg.y);
      }
#pragma unroll
      for (int c = half * 64; c < half * 64 + 64; c += 2) {
        const float2 e = make_float2(x[c], x[c + 1]);
        rs4[(c >> 1) & 3] = fadd2(rs4[(c >> 1) & 3], e);
        pk[(c - half * 64) >> 1] = HPA_P_PACK_ALU ? pack_bf16_alu(e.x, e.y) : pack_bf16(e.x, e.y);
      }
      return;
    }
#pragma unroll
    for (int c = half * 64; c < half * 64 + 64; c += 2) {
      const float2 arg = ffma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
      float2 e;
      if (HPA_POLY_EVERY > 0 && ((c >> 1) % (HPA_POLY_EVERY > 0 ? HPA_POLY_EVERY : 1)) == HPA_POLY_EVERY - 1) {
        e = exp2_poly2(arg);
      } else {
        e.x = fast_exp2(arg.x);
        e.y = fast_exp2(arg.y);
      }
      rs4[(c >> 1) & 3] = fadd2(rs4[(c >> 1) & 3], e);
      pk[(c - half * 64) >> 1] = HPA_P_PACK_ALU ? pack_bf16_alu(e.x, e.y) : pack_bf16(e.x, e.y);
    }
  };
  // Optimistic first half: once every row of the warp has a finite running max, the
  // first half's exps are computed against it while the tile max is reduced alongside
  // (ALU work next to MUFU work). Lazy rescaling keeps the running max unless the tile max
  // exceeds it by > 2^8, so the result is exact whenever no row grew; otherwise the warp
  // redoes half 0 on the exact path below.
  uint32_t pk0[kBN / 4];
  // MUFU turn: slot 0 waits for slot 1's previous exps (the first wait is pre-arrived), slot 1
  // for slot 0's exps of this tile
  if (HPA_SM_SEQ && seq) named_bar_sync((s == 0 ? kSeqBar0 : kSeqBar1) + quarter, 64);
  const bool opt = HPA_OPT_EXP && __all_sync(0xffffffffu, m_run != -CUDART_INF_F);
  bool p0_stored = false;  // P half 0 already in TMEM (not yet published)
  if (opt) {
    exps_half(0, m_run, pk0);
    if (HPA_SPLIT_LD) {  // async store overlapping the second half's load and the max
      tc_st32(tS, pk0);
      p0_stored = true;
    }
  }
  if (HPA_SPLIT_LD) {
    tc_wait_ld();
    if (!all_vis) mask_cols(kLd0, kBN);
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty);  // col[] consumed (masking done)
  }
  if (row == 0) TRACE(31 + s, j);
  // row max as a tree (8 independent partial maxima), not a 64-deep chain
  float pm[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) pm[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
  for (int c = 16; c < kBN; c += 16) {
#pragma unroll
    for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], fmaxf(x[c + k], x[c + k + 8]));
  }
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx *= sl2;
  // lazy rescale: move the running max only when it grows by > 2^8
  const bool grow = mx > m_run + kRescaleThreshold;
  float alpha = 1.f;
  float m_use = m_run;
  if (row == 0) TRACE(33 + s, j);
  if (!opt || __any_sync(0xffffffffu, grow)) {
    if (row == 0) TRACE(37 + s, j);  // exact path taken
    const float m_new = grow ? mx : m_run;
    alpha = grow ? fast_exp2(m_run - m_new) : 1.f;
    m_run = m_new;
    if (j > 0 && __any_sync(0xffffffffu, grow)) {  // O_s is settled: PV_s(j-1) completed before S_s(j)
      float o[32];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        tc_ld32(tO + c * 32, o);
        tc_wait_ld();
#pragma unroll
        for (int y = 0; y < 32; ++y) o[y] *= alpha;
        tc_st32(tO + c * 32, reinterpret_cast<const uint32_t*>(o));
      }
    }
    // a row with nothing visible yet (span-masked leading tiles) keeps p = 0, not NaN
    m_use = m_new == -CUDART_INF_F ? 0.f : m_new;
#pragma unroll
    for (int k = 0; k < 4; ++k) rs4[k] = make_float2(0.f, 0.f);
    exps_half(0, m_use, pk0);
    if (p0_stored) tc_wait_st();  // the optimistic store lands before it is overwritten
    p0_stored = false;
  }
  // P (bf16 pairs) over S: keys [64 half, 64 half + 64) -> columns [128 s + 32 half, +32)
  if (row == 0) TRACE(35 + s, j);
  if (!p0_stored) tc_st32(tS, pk0);
  if (HPA_PV_SPLIT) {
    tc_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&pf[0]);
    if (row == 0) TRACE(11 + 2 * s, j);
    if (lane == 0) TRACE(23 + 4 * s + quarter, j);  // per-warp P half0
  }
  {
    uint32_t pk1[kBN / 4];
    exps_half(1, m_use, pk1);
    // hand the MUFU over (slot 1 skips its last hand-off: slot 0 has no tile left to wait for)
    if (HPA_SM_SEQ && seq && !(s == 1 && seq_last)) named_bar_arrive((s == 0 ? kSeqBar1 : kSeqBar0) + quarter, 64);
    tc_st32(tS + 32, pk1);
    tc_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (!HPA_PV_SPLIT) mbar_arrive(&pf[0]);
      mbar_arrive(&pf[1]);
    }
    if (row == 0) TRACE(12 + 2 * s, j);
    if (lane == 0) TRACE(15 + 4 * s + quarter, j);  // per-warp P completion
  }
  const float2 rsa = fadd2(rs4[0], rs4[1]), rsb = fadd2(rs4[2], rs4[3]);
  l_run = l_run * alpha + ((rsa.x + rsb.x) + (rsa.y + rsb.y));
}

// kCl (HPA_PF1 with G even): the two q-heads of a KV-head pair run as a 2-CTA cluster over
// the same row tile; each CTA issues half of the K/V page boxes and multicasts them to both.
template <int D, bool kCl>
__global__ void __launch_bounds__(kThreads, 1)
prefill_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
               const __grid_constant__ CUtensorMap tm_op, const PrefillArgs a) {
  using L = PSmem<D>;
  constexpr int kHalves = D / 64;
  constexpr uint16_t kPair = 0x3;
  const uint32_t crank = kCl ? cluster_rank() : 0u;
  grid_dependency_wait();  // PDL
  grid_launch_dependents();
#ifdef HPA_TRACE
  if (threadIdx.x == 0) CTA_STAMP(0, gtimer());
#endif
  // unit (b, y, x) and key-range piece: from the work list (plan_prefill) or the grid
  int ux = blockIdx.x, uy = blockIdx.y, piece = 0, part = -1;
  // kCl with HPA_PF1: the PF1 cluster mapping below; kCl without it (HPA_PF_MC2): two listed
  // units of one KV head (consecutive work items) share every K/V box by multicast
  constexpr bool kPf1Cl = kCl && HPA_PF1;
  int b = kPf1Cl ? int(blockIdx.z) / (a.Hq / 2) : int(blockIdx.z);
  const bool listed = !HPA_PF1 && a.work != nullptr;
  // listed: wr = {jb, n_tiles, skip_a, n_skip}, wq = {seq, q_len, q_off, seq_len}, wn = {n_ent}
  // (four independent 16-B loads instead of a chain of dependent metadata loads)
  int4 wr = make_int4(0, 0, 0, 0), wq = make_int4(0, 0, 0, 0), wn = make_int4(0, 0, 0, 0);
  if (listed) {
    const int4 w = a.work[4 * blockIdx.x];
    wr = a.work[4 * blockIdx.x + 1];
    wq = a.work[4 * blockIdx.x + 2];
    wn = a.work[4 * blockIdx.x + 3];
    b = w.x;
    uy = w.y;
    ux = w.z;
    piece = w.w & 15;
    part = ((w.w >> 4) & 15) > 1 ? (w.w >> 8) : -1;
  }
  const int q_len = listed ? wq.y : a.q_len[b];
  // slot -> (q-head, row tile)
  int hq_s[2], mt_s[2];
  if (kPf1Cl) {  // cluster (x = member, y = row tile, z = head pair + Hq/2 * sequence)
    hq_s[0] = hq_s[1] = 2 * (int(blockIdx.z) % (a.Hq / 2)) + int(blockIdx.x);
    mt_s[0] = blockIdx.y;
    mt_s[1] = INT_MAX / kBM;
  } else if (HPA_PF1) {  // one query tile per CTA: (row tile, q-head)
    hq_s[0] = hq_s[1] = blockIdx.y;
    mt_s[0] = blockIdx.x;
    mt_s[1] = INT_MAX / kBM;  // never live
  } else {
    unit_slots(a.G, uy, ux, hq_s, mt_s);
  }
  if (mt_s[0] * kBM >= q_len) return;  // ragged: this sequence has fewer query tiles
  const bool slot1_live = mt_s[1] * kBM < q_len;
  const int h = hq_s[0] / a.G;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + L::oQ;
  uint8_t* sK = sm + L::oK;
  uint8_t* sV = sm + L::oV;
  int32_t* sC = reinterpret_cast<int32_t*>(sm + L::oC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kNK;
  uint64_t* v_full = k_empty + kNK;
  uint64_t* v_empty = v_full + kNV;
  uint64_t* s_full = v_empty + kNV;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 4;
  uint64_t* c_full = o_full + 1;
  uint64_t* c_empty = c_full + kNC;
  uint64_t* o_ready = c_empty + kNC;  // HPA_PF1: one phase per PV(j) completion
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oMisc);
  int32_t* ntiles_slot = reinterpret_cast<int32_t*>(sm + L::oMisc + 4);  // [n_tiles, skip_a, n_skip]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = listed ? wq.x : a.seq_rows[b];
  const int seq_len = listed ? wq.w : a.t.seq_len[seq];
  const int n_ent = listed ? wn.x : a.t.n_entries[seq];
  const int q_off = listed ? wq.z : a.q_off[b];
  const int32_t* bt = a.t.block_table + int64_t(seq) * a.t.max_pages;
  const int32_t* p0 = a.t.pos0 + int64_t(seq) * a.t.max_pages;
  const int32_t* mt_ = a.t.meta + int64_t(seq) * a.t.max_pages;
  const int P = a.P;
  const int lp = a.log2P;
  const int q_base = seq_len - q_len;                         // logical index of query row 0
  const int i_min = q_base + mt_s[0] * kBM;                     // smallest row index in the CTA
  const int last_mt = slot1_live ? mt_s[1] : mt_s[0];
  const int i_max = q_base + min(q_len, (last_mt + 1) * kBM) - 1;
  // GRC mask-out span (NEXT-4a): queries with logical index >= q_from do not see keys in
  // [span_lo, span_hi). The producer tags span columns with kSpanBit in their logical
  // index; a row with i >= q_from compares the tagged index (always > i), other rows
  // compare the index with the tag masked off.
  const int span_from = a.span ? a.span[3 * b + 2] : INT_MAX;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < kNK; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], kCl ? 2 : 1); }
    for (int i = 0; i < kNV; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], kCl ? 2 : 1); }
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 4);  // one arrive per softmax warp
    mbar_init(o_full, 1);
    mbar_init(o_ready, 1);
    for (int i = 0; i < kNC; ++i) { mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], kSoftWarps); }
    fence_barrier_init();
    if (!kPf1Cl) {  // Q tiles in flight while the CTA finishes its setup
      tma_prefetch_desc(&tm_q);
      mbar_arrive_expect_tx(q_full, slot1_live ? 2 * L::kQ : L::kQ);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s == 1 && !slot1_live) break;
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf)
          tma_load_3d(sQ + s * L::kQ + hf * kBM * 128, &tm_q, q_full, hf * 64, hq_s[s], q_off + mt_s[s] * kBM);
      }
    }
    // key slot of a logical index x: the last entry with pos0 <= x, plus the row offset
    auto slot_of = [&](int x) {
      int lo = 0, hi = n_ent - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p0[mid] <= x) lo = mid; else hi = mid - 1;
      }
      return (lo << lp) + (x - p0[lo]);
    };
    if (listed) {  // the host computed the tile range (plan_prefill): no table search here
      ntiles_slot[0] = ntiles_slot[1] = ntiles_slot[2] = 0;
    } else {
    // key tiles needed: up to the tile holding the slot of logical index i_max
    ntiles_slot[0] = slot_of(i_max) / kBN + 1;
    // tiles entirely inside the GRC span are skipped when every query row of the CTA
    // is a span row (their keys are all masked): iteration jj -> tile jj (+ skip)
    int skip_a = 0, skip_b = 0;
    if (a.span && i_min >= span_from && a.span[3 * b + 1] > a.span[3 * b]) {
      skip_a = (slot_of(a.span[3 * b]) + kBN - 1) / kBN;
      skip_b = (slot_of(a.span[3 * b + 1] - 1) + 1) / kBN;
      if (skip_b < skip_a) skip_b = skip_a;
    }
    ntiles_slot[1] = skip_a;
    ntiles_slot[2] = skip_b - skip_a;
    }
  }
  if (warp == kMmaWarp) {  // TMEM: S/P 0 [0,128), S/P 1 [128,256), O0 [256,..), O1 [384,..)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCl) cluster_sync();  // the peer's barriers are initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef HPA_TRACE
  if (threadIdx.x == 0) CTA_STAMP(1, gtimer());
#endif
  // this CTA runs iterations [jb, jb + n_tiles) of its unit; iteration jj loads key tile
  // tile_of(jj) (past the tiles skipped inside the GRC span)
  const int skip_a = listed ? wr.z : ntiles_slot[1], n_skip = listed ? wr.w : ntiles_slot[2];
  const int jb = listed ? wr.x : 0;
  const int n_tiles = listed ? wr.y : ntiles_slot[0] - n_skip;
  auto tile_of = [&](int jj) {
    jj += jb;
    return jj < skip_a ? jj : jj + n_skip;
  };
  if (n_tiles <= 0) {  // an empty split piece (more pieces than key tiles): O = 0, LSE = -inf
    if (warp < 8 && part >= 0) {
      const int s = warp >> 2, row = (warp & 3) * 32 + lane;
      const int pp = (part * a.split_max + piece) * 2 + s;
      float4* orow = reinterpret_cast<float4*>(a.o_part + (int64_t(pp) * kBM + row) * D);
      for (int c = 0; c < D / 4; ++c) orow[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.lse_part[int64_t(pp) * kBM + row] = -CUDART_INF_F;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
    return;
  }

  if (warp >= kSoftWarps) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kOtherRegs));
  if (warp == kProducerWarp) {
    // ================================================================ producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      if (kPf1Cl) {
        tma_prefetch_desc(&tm_q);
        mbar_arrive_expect_tx(q_full, slot1_live ? 2 * L::kQ : L::kQ);
        for (int s = 0; s < (slot1_live ? 2 : 1); ++s) {
          const int q_tok = q_off + mt_s[s] * kBM;
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tma_load_3d(sQ + s * L::kQ + hf * kBM * 128, &tm_q, q_full, hf * 64, hq_s[s], q_tok);
        }
      }
    }
    const int pbox = P < kBN ? P : kBN;
    const int nbox = kBN / pbox;
    constexpr int kOobRow = INT_MAX / 2;  // fully out-of-bounds box -> TMA zero fill
    const int head_row = a.layer * a.NP;
    // The block-table values of tile j+1 are fetched while tile j is processed: their L2
    // latency would otherwise pace this loop (and with it the whole pipeline).
    int nmv[kBN / 32], np0[kBN / 32], nrow = kOobRow;
    auto fetch = [&](int jj, int* mv, int* pv, int& rw) {
      const int tile = tile_of(jj);
      const bool ok = jj < n_tiles;
#pragma unroll
      for (int x = 0; x < kBN / 32; ++x) {
        const int e = (tile * kBN + x * 32 + lane) >> lp;
        mv[x] = ok && e < n_ent ? __ldg(mt_ + e) : 0;
        pv[x] = ok && e < n_ent ? __ldg(p0 + e) : 0;
      }
      rw = kOobRow;
      if (ok && lane < nbox) {
        const int slot = tile * kBN + lane * pbox;
        const int e = slot >> lp;
        if (e < n_ent) rw = ((head_row + __ldg(bt + e)) * a.Hkv + h) * P + (slot & (P - 1));
      }
    };
    fetch(0, nmv, np0, nrow);
    for (int j = 0; j < n_tiles; ++j) {
      const int tile = tile_of(j);
      int cmv[kBN / 32], cp0[kBN / 32];
#pragma unroll
      for (int x = 0; x < kBN / 32; ++x) {
        cmv[x] = nmv[x];
        cp0[x] = np0[x];
      }
      const int row = nrow;
      fetch(j + 1, nmv, np0, nrow);
      // logical index of every key slot (INT_MAX: row >= valid_rows or past the table)
      const int cs = j % kNC;
      if (lane == 0) TRACE(13, j);
      if (j >= kNC) mbar_wait(&c_empty[cs], ((j / kNC) - 1) & 1);
      if (lane == 0) TRACE(14, j);
      int32_t* col = sC + cs * (kBN + 4);
      bool vis = true;
#pragma unroll
      for (int x = 0; x < kBN / 32; ++x) {
        const int c = x * 32 + lane;
        const int slot = tile * kBN + c;
        const int e = slot >> lp, r = slot & (P - 1);
        int v = INT_MAX;
        if (e < n_ent && r < (cmv[x] & kMetaRowsMask)) v = cp0[x] + r;
        if (a.span && v >= a.span[3 * b] && v < a.span[3 * b + 1]) v |= kSpanBit;
        col[c] = v;
        vis &= (v <= i_min);
      }
      vis = __all_sync(0xffffffffu, vis);
      if (lane == 0) col[kBN] = vis ? 1 : 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(&c_full[cs]);
      const int ks = j % kNK;
      if (lane == 0) TRACE(15, j);
      if (j >= kNK) mbar_wait(&k_empty[ks], ((j / kNK) - 1) & 1);
      if (lane == 0) { TRACE(0, j); mbar_arrive_expect_tx(&k_full[ks], L::kKV); }
      __syncwarp();
      if (lane < nbox) {
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf) {
          uint8_t* dst = sK + ks * L::kKV + hf * kBN * 128 + lane * pbox * 128;
          if (!kCl) tma_load_2d(dst, &tm_k, &k_full[ks], hf * 64, row);
          else if (((lane * kHalves + hf) & 1) == int(crank)) tma_load_2d_mc(dst, &tm_k, &k_full[ks], hf * 64, row, kPair);
        }
      }
      __syncwarp();
    }
  } else if (warp == kVProducerWarp) {
    // ================================================================ V producer
    // (decoupled from K so K(j+1) never waits behind V(j)'s ring slot)
    const int pbox = P < kBN ? P : kBN;
    const int nbox = kBN / pbox;
    constexpr int kOobRow = INT_MAX / 2;
    const int head_row = a.layer * a.NP;
    auto vrow = [&](int jj) {  // fetched one tile ahead (see the K producer)
      int rw = kOobRow;
      if (jj < n_tiles && lane < nbox) {
        const int tile = tile_of(jj);
        const int slot = tile * kBN + lane * pbox;
        const int e = slot >> lp;
        if (e < n_ent) rw = ((head_row + __ldg(bt + e)) * a.Hkv + h) * P + (slot & (P - 1));
      }
      return rw;
    };
    int next_row = vrow(0);
    for (int j = 0; j < n_tiles; ++j) {
      const int row = next_row;
      next_row = vrow(j + 1);
      const int vs = j % kNV;
      if (j >= kNV) mbar_wait(&v_empty[vs], ((j / kNV) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&v_full[vs], L::kKV);
      __syncwarp();
      if (lane < nbox) {
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf) {
          uint8_t* dst = sV + vs * L::kKV + hf * kBN * 128 + lane * pbox * 128;
          if (!kCl) tma_load_2d(dst, &tm_v, &v_full[vs], hf * 64, row);
          else if (((lane * kHalves + hf) & 1) == int(crank)) tma_load_2d_mc(dst, &tm_v, &v_full[vs], hf * 64, row, kPair);
        }
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp && HPA_PF1) {
    // ================================================================ MMA issuer (HPA_PF1)
    // One query tile, S double-buffered in TMEM: QK(0), QK(1); then per tile j: PV(j) (two
    // 64-key halves, A = P(j) from buffer j%2) and QK(j+2) into the same buffer (the pipe is
    // in order, so PV(j) has read P(j) before QK(j+2) overwrites it).
    constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
    constexpr uint32_t idO = idesc_bf16(kBM, D, 0, 1);
    const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
    mbar_wait(q_full, 0);
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) tc_commit(bar);
      __syncwarp();
    };
    auto issue_s = [&](int jj) {  // S buffer jj % 2
      mbar_wait(&k_full[jj % kNK], (jj / kNK) & 1);
      if (lane == 0) TRACE(1, jj);
      tc_fence_after();
      const int ks = jj % kNK;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t ad = sdesc(aQ + (k >> 2) * (kBM * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(aK + ks * L::kKV + (k >> 2) * (kBN * 128) + (k & 3) * 32, 16, 1024);
          tc_mma_ss(tmem + (jj & 1) * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[jj & 1]);
        if (kCl) tc_commit_mc(&k_empty[ks], kPair);  // both CTAs' producers may reuse the stage
        else tc_commit(&k_empty[ks]);
      }
      __syncwarp();
    };
    issue_s(0);
    if (n_tiles > 1) issue_s(1);
    for (int j = 0; j < n_tiles; ++j) {
      const int buf = j & 1, vs = j % kNV;
      if (lane == 0) TRACE(5, j);
      mbar_wait(&v_full[vs], (j / kNV) & 1);
      if (lane == 0) TRACE(2, j);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        mbar_wait(&p_full[2 * buf + half], (j >> 1) & 1);
        if (lane == 0) TRACE(3 + half, j);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = half * 4; k < half * 4 + 4; ++k) {
            const uint64_t bd = sdesc(aV + vs * L::kKV + k * 2048, kBN * 128, 1024);
            tc_mma_ts(tmem + 256, tmem + buf * 128 + k * 8, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
      }
      if (kCl) {
        if (elect_one()) tc_commit_mc(&v_empty[vs], kPair);
        __syncwarp();
      } else {
        commit(&v_empty[vs]);
      }
      commit(o_ready);  // PV(j) done -> the softmax of tile j+1 may rescale O
      if (j + 2 < n_tiles) issue_s(j + 2);
    }
    commit(o_full);
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    // All 32 lanes run the loop (warp-uniform waits keep the descriptor math in uniform
    // registers); the elected lane issues every tcgen05.mma and commit (commit tracks the
    // MMAs of the issuing thread, and elect.sync picks the same lowest lane each time).
    {
      constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
      constexpr uint32_t idO = idesc_bf16(kBM, D, 0, 1);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
      const int nslot = slot1_live ? 2 : 1;
      mbar_wait(q_full, 0);
      auto issue_s = [&](int s, int jj) {
        const int ks = jj % kNK;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ad = sdesc(aQ + s * L::kQ + (k >> 2) * (kBM * 128) + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(aK + ks * L::kKV + (k >> 2) * (kBN * 128) + (k & 3) * 32, 16, 1024);
            tc_mma_ss(tmem + s * 128, ad, bd, idS, k > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[s]);
        }
        __syncwarp();
      };
      auto issue_pv_half = [&](int s, int jj, int half) {
        const int vs = jj % kNV;
        if (elect_one()) {
#pragma unroll
          for (int k = half * 4; k < half * 4 + 4; ++k) {
            const uint64_t bd = sdesc(aV + vs * L::kKV + k * 2048, kBN * 128, 1024);
            tc_mma_ts(tmem + 256 + s * 128, tmem + s * 128 + k * 8, bd, idO, (jj > 0 || k > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) tc_commit(bar);
        __syncwarp();
      };
      // a K / V stage is refilled (by multicast into both CTAs) only after both CTAs' MMAs
      // have read it: with kCl the release arrives on both CTAs' barriers (count 2)
      auto release = [&](uint64_t* bar) {
        if (kCl) {
          if (elect_one()) tc_commit_mc(bar, kPair);
          __syncwarp();
        } else {
          commit(bar);
        }
      };
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int s = 0; s < nslot; ++s) issue_s(s, 0);
      release(&k_empty[0]);
      for (int j = 0; j < n_tiles; ++j) {
        const bool more = j + 1 < n_tiles;
        mbar_wait(&v_full[j % kNV], (j / kNV) & 1);
        if (lane == 0) TRACE(2, j);
        bool k_ready = false;
        for (int s = 0; s < nslot; ++s) {
          // PV over keys 0..63 as soon as the first half of P is in TMEM, then 64..127
          mbar_wait(&p_full[2 * s], j & 1);
          if (lane == 0) TRACE(3 + s, j);
          tc_fence_after();
          issue_pv_half(s, j, 0);
          mbar_wait(&p_full[2 * s + 1], j & 1);
          if (lane == 0) TRACE(5 + s, j);
          tc_fence_after();
          issue_pv_half(s, j, 1);
          if (s == nslot - 1) release(&v_empty[j % kNV]);
          if (more) {
            if (!k_ready) {  // K(j+1) is only needed here, not by PV(j)
              mbar_wait(&k_full[(j + 1) % kNK], ((j + 1) / kNK) & 1);
              if (lane == 0) TRACE(1, j);
              tc_fence_after();
              k_ready = true;
            }
            issue_s(s, j + 1);  // overwrites S/P s after PV s has read P (in-order pipe)
          }
        }
        if (more) release(&k_empty[(j + 1) % kNK]);
      }
      commit(o_full);
    }
#if HPA_PF1
  } else if (warp < kSoftWarps) {
    // ================================================================ softmax (HPA_PF1)
    // warp = 4 half + quarter: rows quarter*32 + lane, key columns [64 hc, 64 hc + 64) of the
    // tile's S buffer, P columns [32 hc, +32) of it, O columns [D/2 hc, +D/2).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    constexpr int kCols = kBN / 2, kOCols = D / 2;
    const int hc = (warp >> 2) & 1, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int t = mt_s[0] * kBM + row;
    const int my_i = q_base + t;
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    const uint32_t tO = tmem + lane_base + 256 + hc * kOCols;
    float* xmax = reinterpret_cast<float*>(sm + L::oX);  // [2 buf][2 half][128]
    float* xsum = xmax + 8 * kBM;                        // [2 half][128]
    const float sl2 = a.scale_log2;
    float m_run = -CUDART_INF_F, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int cs = j % kNC, buf = j & 1;
      const uint32_t tS = tmem + lane_base + buf * 128 + hc * kCols;
      const uint32_t tP = tmem + lane_base + buf * 128 + hc * (kCols / 2);
      float x[kCols];
      mbar_wait(&s_full[buf], (j >> 1) & 1);
      if (row == 0) TRACE(7 + hc, j);
      tc_fence_after();
      tc_ld32(tS, x);
      tc_ld32(tS + 32, x + 32);
      mbar_wait(&c_full[cs], (j / kNC) & 1);
      const int32_t* col = sC + cs * (kBN + 4) + hc * kCols;
      const bool all_vis = sC[cs * (kBN + 4) + kBN] != 0;
      tc_wait_ld();
      if (!all_vis) {
        const int cmask = my_i >= span_from ? -1 : ~kSpanBit;
#pragma unroll
        for (int c = 0; c < kCols; c += 4) {
          const int4 ci = *reinterpret_cast<const int4*>(col + c);
          x[c + 0] = (ci.x & cmask) <= my_i ? x[c + 0] : -CUDART_INF_F;
          x[c + 1] = (ci.y & cmask) <= my_i ? x[c + 1] : -CUDART_INF_F;
          x[c + 2] = (ci.z & cmask) <= my_i ? x[c + 2] : -CUDART_INF_F;
          x[c + 3] = (ci.w & cmask) <= my_i ? x[c + 3] : -CUDART_INF_F;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c_empty[cs]);
      float pm[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
      for (int c = 16; c < kCols; c += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], fmaxf(x[c + k], x[c + k + 8]));
      }
      float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      float* xb = xmax + buf * 2 * kBM;
      xb[hc * kBM + row] = mx;
      named_bar_sync(1, 8 * 32);
      mx = fmaxf(mx, xb[(hc ^ 1) * kBM + row]);
      mx *= sl2;
      const bool grow = mx > m_run + kRescaleThreshold;  // lazy rescale (both halves agree)
      const float m_new = grow ? mx : m_run;
      const float alpha = grow ? fast_exp2(m_run - m_new) : 1.f;
      m_run = m_new;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        // S(j) ready only implies PV(j-2) done: wait for PV(j-1) before touching O (phases up
        // to j-2 are complete, so the parity wait for phase j-1 cannot alias)
        mbar_wait(o_ready, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kOCols; c += 16) {
          float o[16];
          tc_ld16(tO + c, o);
          tc_wait_ld();
#pragma unroll
          for (int y = 0; y < 16; ++y) o[y] *= alpha;
          tc_st16(tO + c, reinterpret_cast<const uint32_t*>(o));
        }
      }
      const float m_use = m_new == -CUDART_INF_F ? 0.f : m_new;
      const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m_use, -m_use);
      float2 rs4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[kCols / 2];
#pragma unroll
      for (int c = 0; c < kCols; c += 2) {
        const float2 arg = ffma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
        float2 e;
        e.x = fast_exp2(arg.x);
        e.y = fast_exp2(arg.y);
        rs4[(c >> 1) & 3] = fadd2(rs4[(c >> 1) & 3], e);
        pk[c >> 1] = pack_bf16(e.x, e.y);
      }
      tc_st32(tP, pk);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * buf + hc]);
      if (row == 0) TRACE(11 + hc, j);
      const float2 rsa = fadd2(rs4[0], rs4[1]), rsb = fadd2(rs4[2], rs4[3]);
      l_run = l_run * alpha + ((rsa.x + rsb.x) + (rsa.y + rsb.y));
    }
    // epilogue: l = both halves' sums; this warp's half of O / l -> bf16 -> global
    xsum[hc * kBM + row] = l_run;
    named_bar_sync(1, 8 * 32);
    const float inv = 1.f / (l_run + xsum[(hc ^ 1) * kBM + row]);
    mbar_wait(o_full, 0);
    tc_fence_after();
    __nv_bfloat16* orow =
        static_cast<__nv_bfloat16*>(a.out) + (int64_t(q_off + t) * a.Hq + hq_s[0]) * D + hc * kOCols;
#pragma unroll
    for (int c = 0; c < kOCols; c += 16) {
      float o[16];
      tc_ld16(tO + c, o);
      tc_wait_ld();
      if (t < q_len) {
#pragma unroll
        for (int y = 0; y < 16; y += 8) {
          uint4 v;
          v.x = pack_bf16(o[y + 0] * inv, o[y + 1] * inv);
          v.y = pack_bf16(o[y + 2] * inv, o[y + 3] * inv);
          v.z = pack_bf16(o[y + 4] * inv, o[y + 5] * inv);
          v.w = pack_bf16(o[y + 6] * inv, o[y + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c + y) = v;
        }
      }
    }
  }
#elif HPA_SM16
  } else if (warp < kSoftWarps) {
    // ================================================================ softmax, 16 warps
    // warp = 8 slot + 4 half + quarter: rows quarter*32 + lane of slot `s`, key columns
    // [64 hc, 64 hc + 64) of S, P columns [32 hc, +32) (bf16 pairs), O columns [D/2 hc, +D/2).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    constexpr int kCols = kBN / 2, kOCols = D / 2;
    const int s = warp >> 3, hc = (warp >> 2) & 1, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int t = mt_s[s] * kBM + row;
    const int my_i = q_base + t;
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + s * 128 + hc * kCols;
    const uint32_t tP = tmem + lane_base + s * 128 + hc * (kCols / 2);
    const uint32_t tO = tmem + lane_base + 256 + s * 128 + hc * kOCols;
    float* xmax = reinterpret_cast<float*>(sm + L::oX);             // [2 buf][2 slot][2 half][128]
    float* xsum = xmax + 8 * kBM;                                     // [2 slot][2 half][128]
    const float sl2 = a.scale_log2;
    const bool live = s == 0 || slot1_live;
    float m_run = -CUDART_INF_F, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int cs = j % kNC;
      if (!live) {  // dead slot: still release the mask slot
        mbar_wait(&c_full[cs], (j / kNC) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&c_empty[cs]);
        continue;
      }
      float x[kCols];
      mbar_wait(&s_full[s], j & 1);
      if (row == 0 && hc == 0) TRACE(7 + s, j);
      tc_fence_after();
      tc_ld32(tS, x);
      tc_ld32(tS + 32, x + 32);
      mbar_wait(&c_full[cs], (j / kNC) & 1);
      const int32_t* col = sC + cs * (kBN + 4) + hc * kCols;
      const bool all_vis = sC[cs * (kBN + 4) + kBN] != 0;
      tc_wait_ld();
      if (row == 0 && hc == 0) TRACE(9 + s, j);
      if (!all_vis) {
        const int cmask = my_i >= span_from ? -1 : ~kSpanBit;
#pragma unroll
        for (int c = 0; c < kCols; c += 4) {
          const int4 ci = *reinterpret_cast<const int4*>(col + c);
          x[c + 0] = (ci.x & cmask) <= my_i ? x[c + 0] : -CUDART_INF_F;
          x[c + 1] = (ci.y & cmask) <= my_i ? x[c + 1] : -CUDART_INF_F;
          x[c + 2] = (ci.z & cmask) <= my_i ? x[c + 2] : -CUDART_INF_F;
          x[c + 3] = (ci.w & cmask) <= my_i ? x[c + 3] : -CUDART_INF_F;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c_empty[cs]);
      float pm[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
      for (int c = 16; c < kCols; c += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], fmaxf(x[c + k], x[c + k + 8]));
      }
      float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      // row max over both column halves: exchange with the partner warp (same rows, other half)
      float* xb = xmax + ((j & 1) * 2 + s) * 2 * kBM;
      xb[hc * kBM + row] = mx;
      named_bar_sync(1 + s, 8 * 32);
      mx = fmaxf(mx, xb[(hc ^ 1) * kBM + row]);
      mx *= sl2;
      const bool grow = mx > m_run + kRescaleThreshold;  // lazy rescale (both halves agree)
      const float m_new = grow ? mx : m_run;
      const float alpha = grow ? fast_exp2(m_run - m_new) : 1.f;
      m_run = m_new;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {  // this half of O_s (PV_s(j-1) completed)
#pragma unroll
        for (int c = 0; c < kOCols; c += 16) {
          float o[16];
          tc_ld16(tO + c, o);
          tc_wait_ld();
#pragma unroll
          for (int y = 0; y < 16; ++y) o[y] *= alpha;
          tc_st16(tO + c, reinterpret_cast<const uint32_t*>(o));
        }
      }
      const float m_use = m_new == -CUDART_INF_F ? 0.f : m_new;
      const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m_use, -m_use);
#pragma unroll
      for (int c = 0; c < kCols; c += 2) {  // all ex2 first, in place
        const float2 arg = ffma2(make_float2(x[c], x[c + 1]), sl2x2, negm);
        x[c] = fast_exp2(arg.x);
        x[c + 1] = fast_exp2(arg.y);
      }
      float2 rs4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int ch = 0; ch < kCols / 32; ++ch) {  // sums + bf16 pairs, stored 16 columns at a time
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float2 e = make_float2(x[ch * 32 + 2 * q], x[ch * 32 + 2 * q + 1]);
          rs4[q & 3] = fadd2(rs4[q & 3], e);
          pk[q] = pack_bf16(e.x, e.y);
        }
        tc_st16(tP + ch * 16, pk);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * s + hc]);
      if (row == 0) TRACE(11 + 2 * s + hc, j);
      const float2 rsa = fadd2(rs4[0], rs4[1]), rsb = fadd2(rs4[2], rs4[3]);
      l_run = l_run * alpha + ((rsa.x + rsb.x) + (rsa.y + rsb.y));
    }
    if (live) {
      // epilogue: l = both halves' sums; this warp's half of O / l -> bf16 -> global
      xsum[(s * 2 + hc) * kBM + row] = l_run;
      named_bar_sync(1 + s, 8 * 32);
      const float inv = 1.f / (l_run + xsum[(s * 2 + (hc ^ 1)) * kBM + row]);
      mbar_wait(o_full, 0);
      tc_fence_after();
      __nv_bfloat16* orow =
          static_cast<__nv_bfloat16*>(a.out) + (int64_t(q_off + t) * a.Hq + hq_s[s]) * D + hc * kOCols;
#pragma unroll
      for (int c = 0; c < kOCols; c += 16) {
        float o[16];
        tc_ld16(tO + c, o);
        tc_wait_ld();
        if (t < q_len) {
#pragma unroll
          for (int y = 0; y < 16; y += 8) {
            uint4 v;
            v.x = pack_bf16(o[y + 0] * inv, o[y + 1] * inv);
            v.y = pack_bf16(o[y + 2] * inv, o[y + 3] * inv);
            v.z = pack_bf16(o[y + 4] * inv, o[y + 5] * inv);
            v.w = pack_bf16(o[y + 6] * inv, o[y + 7] * inv);
            *reinterpret_cast<uint4*>(orow + c + y) = v;
          }
        }
      }
    }
  }
#else
  } else if (warp < 8) {
    // ================================================================ softmax (slot = warp / 4)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    const int s = warp >> 2;
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int my_mt = s ? mt_s[1] : mt_s[0], my_hq = s ? hq_s[1] : hq_s[0];  // (no local-memory indexing)
    const int row = quarter * 32 + lane;          // query row within the slot tile == TMEM lane
    const int t = my_mt * kBM + row;
    const int my_i = q_base + t;                  // logical index of this query row
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + s * 128;
    const uint32_t tO = tmem + lane_base + 256 + s * 128;
    const float sl2 = a.scale_log2;
    const bool live = s == 0 || slot1_live;
    float m_run = -CUDART_INF_F, l_run = 0.f;
    const bool seq = HPA_SM_SEQ && slot1_live;  // both slots live: MUFU hand-off
    if (seq && s == 1) named_bar_arrive(kSeqBar0 + quarter, 64);  // slot 0 goes first
    for (int j = 0; j < n_tiles; ++j) {
      const int cs = j % kNC;
      if (!live) {  // dead slot: still release the mask slot
        mbar_wait(&c_full[cs], (j / kNC) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&c_empty[cs]);
        continue;
      }
      mbar_wait(&s_full[s], j & 1);
      if (row == 0) TRACE(7 + s, j);
#ifdef HPA_TRACE
      if (j == 0 && threadIdx.x == 0) CTA_STAMP(2, gtimer());
#endif
      tc_fence_after();
      softmax_tile<D>(a, s, quarter, row, lane, j, tS, tO, sC + cs * (kBN + 4), &c_full[cs], (j / kNC) & 1,
                      &c_empty[cs], &p_full[2 * s], my_i, span_from, sl2, m_run, l_run, seq, j + 1 == n_tiles);
    }
#ifdef HPA_TRACE
    if (threadIdx.x == 0) {
      mbar_wait(o_full, 0);
      CTA_STAMP(3, gtimer());
    }
#endif
    if (live) {
      // Epilogue. O / l is staged in shared memory (the K and V rings are idle once o_full has
      // fired: every MMA has completed) in the 128-B-swizzled box layout and written by TMA
      // stores: bf16 into the output rows, or -- a split piece -- fp32 O / l into the
      // workspace with LSE = m + log2 l (log2 domain; -inf when no key of the piece was
      // visible to the row), merged by prefill_combine_kernel. A ragged last row tile (its
      // box would cover the next sequence's rows) is stored row by row instead.
      mbar_wait(o_full, 0);
      tc_fence_after();
      const bool split = part >= 0;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      if (split || (my_mt + 1) * kBM <= q_len) {
        uint8_t* stage = s == 0 ? sK : sV;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tc_ld32(tO + c * 32, o);
          tc_wait_ld();
          if (split) {  // fp32 box c: columns [32 c, 32 c + 32) = one 128-B row of 8 chunks
            uint8_t* box = stage + c * (kBM * 128);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(box + sw128(row, k)) =
                  make_float4(o[4 * k] * inv, o[4 * k + 1] * inv, o[4 * k + 2] * inv, o[4 * k + 3] * inv);
          } else {  // bf16 box c / 2: columns [64 (c / 2), + 64), chunks 4 (c & 1) .. + 3
            uint8_t* box = stage + (c >> 1) * (kBM * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint4 v;
              v.x = pack_bf16(o[8 * k + 0] * inv, o[8 * k + 1] * inv);
              v.y = pack_bf16(o[8 * k + 2] * inv, o[8 * k + 3] * inv);
              v.z = pack_bf16(o[8 * k + 4] * inv, o[8 * k + 5] * inv);
              v.w = pack_bf16(o[8 * k + 6] * inv, o[8 * k + 7] * inv);
              *reinterpret_cast<uint4*>(box + sw128(row, (c & 1) * 4 + k)) = v;
            }
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1 + s, 128);
        const int pp = (part * a.split_max + piece) * 2 + s;
        if (quarter == 0 && lane == 0) {
          if (split) {
#pragma unroll
            for (int c = 0; c < D / 32; ++c) tma_store_2d(&tm_op, stage + c * (kBM * 128), c * 32, pp * kBM);
          } else {
#pragma unroll
            for (int hf = 0; hf < kHalves; ++hf)
              tma_store_3d(&tm_o, stage + hf * (kBM * 128), hf * 64, my_hq, q_off + my_mt * kBM);
          }
          bulk_commit();
          bulk_wait_read();  // the smem is released at exit
        }
        if (split) a.lse_part[int64_t(pp) * kBM + row] = l_run > 0.f ? m_run + __log2f(l_run) : -CUDART_INF_F;
      } else {
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + (int64_t(q_off + t) * a.Hq + my_hq) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tc_ld32(tO + c * 32, o);
          tc_wait_ld();
          if (t < q_len) {
#pragma unroll
            for (int y = 0; y < 32; y += 8) {
              uint4 v;
              v.x = pack_bf16(o[y + 0] * inv, o[y + 1] * inv);
              v.y = pack_bf16(o[y + 2] * inv, o[y + 3] * inv);
              v.z = pack_bf16(o[y + 4] * inv, o[y + 5] * inv);
              v.w = pack_bf16(o[y + 6] * inv, o[y + 7] * inv);
              *reinterpret_cast<uint4*>(orow + c * 32 + y) = v;
            }
          }
        }
      }
    }
  }
#endif  // HPA_PF1 / HPA_SM16
  tc_fence_before();
  __syncthreads();
#ifdef HPA_TRACE
  if (threadIdx.x == 0) {
    CTA_STAMP(4, gtimer());
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    CTA_STAMP(5, smid);
    CTA_STAMP(6, n_tiles);
    CTA_STAMP(7, 1);
  }
#endif
  if constexpr (kCl) cluster_sync();  // the peer may still multicast into / signal this CTA until here
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent prefill (default configuration): one CTA per SM loops over the work items the host
// assigned to it (PrefillArgs::cta_off, longest-processing-time greedy over estimated tile
// counts). Setup (barrier init, TMEM allocation) happens once; the K/V/mask rings, the
// S/P handshakes and the tile counters run on across items, so the next item's K/V tiles
// stream in while the current item drains, and its Q tiles are loaded (warp 11) as soon as the
// current item's last Q K^T has completed (q_empty; issued by the V producer warp). Per item the
// softmax warps finish with the epilogue (row stores: the shared memory rings stay in use) and
// carry straight on with the next item's first tile. Items never have an empty key range (the host clamps split counts).
struct PItem {
  int b, piece, part, jb, n_tiles, skip_a, n_skip, seq, q_len, q_off, seq_len, n_ent;
  int hq0, hq1, mt0, mt1;
  bool live1;
};
__device__ __forceinline__ PItem load_item(const PrefillArgs& a, int idx) {
  const int4 w = a.work[4 * idx], wr = a.work[4 * idx + 1], wq = a.work[4 * idx + 2], wn = a.work[4 * idx + 3];
  PItem u;
  u.b = w.x;
  u.piece = w.w & 15;
  u.part = ((w.w >> 4) & 15) > 1 ? (w.w >> 8) : -1;
  u.jb = wr.x;
  u.n_tiles = wr.y;
  u.skip_a = wr.z;
  u.n_skip = wr.w;
  u.seq = wq.x;
  u.q_len = wq.y;
  u.q_off = wq.z;
  u.seq_len = wq.w;
  u.n_ent = wn.x;
  int hq[2], mt[2];
  unit_slots(a.G, w.y, w.z, hq, mt);
  u.hq0 = hq[0];
  u.hq1 = hq[1];
  u.mt0 = mt[0];
  u.mt1 = mt[1];
  u.live1 = mt[1] * kBM < u.q_len;
  return u;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
prefill_persistent_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const PrefillArgs a) {
  using L = PSmem<D>;
  constexpr int kHalves = D / 64;
  grid_dependency_wait();  // PDL
  grid_launch_dependents();
  const int beg = a.cta_off[blockIdx.x], end = a.cta_off[blockIdx.x + 1];
  if (beg >= end) return;
#ifdef HPA_TRACE
  if (threadIdx.x == 0) CTA_STAMP(0, gtimer());
#endif

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm + L::oQ;
  uint8_t* sK = sm + L::oK;
  uint8_t* sV = sm + L::oV;
  int32_t* sC = reinterpret_cast<int32_t*>(sm + L::oC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kNK;
  uint64_t* v_full = k_empty + kNK;
  uint64_t* v_empty = v_full + kNV;
  uint64_t* s_full = v_empty + kNV;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 4;
  uint64_t* c_full = o_full + 1;
  uint64_t* c_empty = c_full + kNC;
  uint64_t* q_empty = c_empty + kNC;  // (the o_ready slot of the single-unit kernel)
  uint64_t* o_full1 = q_empty + 1;    // o_full: slot 0's O ready; o_full1: slot 1's (items with slot 1 live)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::oMisc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto issue_q = [&](const PItem& u) {  // one thread
    mbar_arrive_expect_tx(q_full, u.live1 ? 2 * L::kQ : L::kQ);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s == 1 && !u.live1) break;
#pragma unroll
      for (int hf = 0; hf < kHalves; ++hf)
        tma_load_3d(sQ + s * L::kQ + hf * kBM * 128, &tm_q, q_full, hf * 64, s ? u.hq1 : u.hq0,
                    u.q_off + (s ? u.mt1 : u.mt0) * kBM);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < kNK; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < kNV; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 4);  // one arrive per softmax warp
    mbar_init(o_full, 1);
    mbar_init(o_full1, 1);
    for (int i = 0; i < kNC; ++i) { mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], kSoftWarps); }
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    issue_q(load_item(a, beg));  // the first item's Q during setup
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int P = a.P, lp = a.log2P;
#ifdef HPA_TRACE
  if (threadIdx.x == 0) CTA_STAMP(1, gtimer());
#endif

  if (warp >= kSoftWarps) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kOtherRegs));
  if (warp == kProducerWarp) {
    // ================================================================ K producer + mask indices
    if (lane == 0) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
    }
    const int pbox = P < kBN ? P : kBN;
    const int nbox = kBN / pbox;
    constexpr int kOobRow = INT_MAX / 2;
    const int head_row = a.layer * a.NP;
    uint32_t g = 0;  // K tiles issued by this CTA (ring position)
    for (int it = beg; it < end; ++it) {
      const PItem u = load_item(a, it);
      const int32_t* bt = a.t.block_table + int64_t(u.seq) * a.t.max_pages;
      const int32_t* p0 = a.t.pos0 + int64_t(u.seq) * a.t.max_pages;
      const int32_t* mt_ = a.t.meta + int64_t(u.seq) * a.t.max_pages;
      const int h = u.hq0 / a.G;
      const int i_min = u.seq_len - u.q_len + u.mt0 * kBM;
      const int span_lo = a.span ? a.span[3 * u.b] : 0, span_hi = a.span ? a.span[3 * u.b + 1] : 0;
      auto tile_of = [&](int jj) {
        jj += u.jb;
        return jj < u.skip_a ? jj : jj + u.n_skip;
      };
      int nmv[kBN / 32], np0[kBN / 32], nrow = kOobRow;
      auto fetch = [&](int jj, int* mv, int* pv, int& rw) {
        const int tile = tile_of(jj);
        const bool ok = jj < u.n_tiles;
#pragma unroll
        for (int x = 0; x < kBN / 32; ++x) {
          const int e = (tile * kBN + x * 32 + lane) >> lp;
          mv[x] = ok && e < u.n_ent ? __ldg(mt_ + e) : 0;
          pv[x] = ok && e < u.n_ent ? __ldg(p0 + e) : 0;
        }
        rw = kOobRow;
        if (ok && lane < nbox) {
          const int slot = tile * kBN + lane * pbox;
          const int e = slot >> lp;
          if (e < u.n_ent) rw = ((head_row + __ldg(bt + e)) * a.Hkv + h) * P + (slot & (P - 1));
        }
      };
      fetch(0, nmv, np0, nrow);
      for (int j = 0; j < u.n_tiles; ++j, ++g) {
        const int tile = tile_of(j);
        int cmv[kBN / 32], cp0[kBN / 32];
#pragma unroll
        for (int x = 0; x < kBN / 32; ++x) {
          cmv[x] = nmv[x];
          cp0[x] = np0[x];
        }
        const int row = nrow;
        fetch(j + 1, nmv, np0, nrow);
        const int cs = g % kNC;
        if (g >= kNC) mbar_wait(&c_empty[cs], ((g / kNC) - 1) & 1);
        int32_t* col = sC + cs * (kBN + 4);
        bool vis = true;
#pragma unroll
        for (int x = 0; x < kBN / 32; ++x) {
          const int c = x * 32 + lane;
          const int slot = tile * kBN + c;
          const int e = slot >> lp, r = slot & (P - 1);
          int v = INT_MAX;
          if (e < u.n_ent && r < (cmv[x] & kMetaRowsMask)) v = cp0[x] + r;
          if (a.span && v >= span_lo && v < span_hi) v |= kSpanBit;
          col[c] = v;
          vis &= (v <= i_min);
        }
        vis = __all_sync(0xffffffffu, vis);
        if (lane == 0) col[kBN] = vis ? 1 : 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&c_full[cs]);
        const int ks = g % kNK;
        if (g >= kNK) mbar_wait(&k_empty[ks], ((g / kNK) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&k_full[ks], L::kKV);
        __syncwarp();
        if (lane < nbox) {
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tma_load_2d(sK + ks * L::kKV + hf * kBN * 128 + lane * pbox * 128, &tm_k, &k_full[ks], hf * 64, row);
        }
        __syncwarp();
      }
    }
  } else if (warp == kVProducerWarp) {
    // ================================================================ V producer
    const int pbox = P < kBN ? P : kBN;
    const int nbox = kBN / pbox;
    constexpr int kOobRow = INT_MAX / 2;
    const int head_row = a.layer * a.NP;
    uint32_t g = 0;
    for (int it = beg; it < end; ++it) {
      const PItem u = load_item(a, it);
      if (it > beg && lane == 0) {  // this item's Q once every Q K^T of the previous one completed
        mbar_wait(q_empty, (it - beg - 1) & 1);
        issue_q(u);
      }
      const int32_t* bt = a.t.block_table + int64_t(u.seq) * a.t.max_pages;
      const int h = u.hq0 / a.G;
      auto vrow = [&](int jj) {
        int rw = kOobRow;
        if (jj < u.n_tiles && lane < nbox) {
          int tile = jj + u.jb;
          tile = tile < u.skip_a ? tile : tile + u.n_skip;
          const int slot = tile * kBN + lane * pbox;
          const int e = slot >> lp;
          if (e < u.n_ent) rw = ((head_row + __ldg(bt + e)) * a.Hkv + h) * P + (slot & (P - 1));
        }
        return rw;
      };
      int next_row = vrow(0);
      for (int j = 0; j < u.n_tiles; ++j, ++g) {
        const int row = next_row;
        next_row = vrow(j + 1);
        const int vs = g % kNV;
        if (g >= kNV) mbar_wait(&v_empty[vs], ((g / kNV) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&v_full[vs], L::kKV);
        __syncwarp();
        if (lane < nbox) {
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tma_load_2d(sV + vs * L::kKV + hf * kBN * 128 + lane * pbox * 128, &tm_v, &v_full[vs], hf * 64, row);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
    constexpr uint32_t idO = idesc_bf16(kBM, D, 0, 1);
    const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
    auto issue_s = [&](int s, uint32_t gg) {
      const int ks = gg % kNK;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t ad = sdesc(aQ + s * L::kQ + (k >> 2) * (kBM * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(aK + ks * L::kKV + (k >> 2) * (kBN * 128) + (k & 3) * 32, 16, 1024);
          tc_mma_ss(tmem + s * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[s]);
      }
      __syncwarp();
    };
    auto issue_pv_half = [&](int s, uint32_t gg, int half, bool acc0) {
      const int vs = gg % kNV;
      if (elect_one()) {
#pragma unroll
        for (int k = half * 4; k < half * 4 + 4; ++k) {
          const uint64_t bd = sdesc(aV + vs * L::kKV + k * 2048, kBN * 128, 1024);
          tc_mma_ts(tmem + 256 + s * 128, tmem + s * 128 + k * 8, bd, idO, (acc0 || k > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) tc_commit(bar);
      __syncwarp();
    };
    uint32_t g = 0;                // tiles (K and V ring position)
    uint32_t np[2] = {0u, 0u};     // P publications per slot (p_full phase)
    for (int it = beg; it < end; ++it) {
      const PItem u = load_item(a, it);
      const int nslot = u.live1 ? 2 : 1;
      mbar_wait(q_full, (it - beg) & 1);
      mbar_wait(&k_full[g % kNK], (g / kNK) & 1);
      tc_fence_after();
      for (int s = 0; s < nslot; ++s) issue_s(s, g);
      if (u.n_tiles == 1) commit(q_empty);
      commit(&k_empty[g % kNK]);
      for (int j = 0; j < u.n_tiles; ++j, ++g) {
        const bool more = j + 1 < u.n_tiles;
        mbar_wait(&v_full[g % kNV], (g / kNV) & 1);
        bool k_ready = false;
        for (int s = 0; s < nslot; ++s) {
          mbar_wait(&p_full[2 * s], np[s] & 1);
          tc_fence_after();
          issue_pv_half(s, g, 0, j > 0);
          mbar_wait(&p_full[2 * s + 1], np[s] & 1);
          tc_fence_after();
          issue_pv_half(s, g, 1, j > 0);
          ++np[s];
          if (s == nslot - 1) commit(&v_empty[g % kNV]);
          if (more) {
            if (!k_ready) {
              mbar_wait(&k_full[(g + 1) % kNK], ((g + 1) / kNK) & 1);
              tc_fence_after();
              k_ready = true;
            }
            issue_s(s, g + 1);
          }
        }
        if (more) {
          commit(&k_empty[(g + 1) % kNK]);
          if (j + 2 == u.n_tiles) commit(q_empty);  // the item's last Q K^T was just issued
        }
      }
      commit(o_full);
      if (u.live1) commit(o_full1);
    }
  } else if (warp < kSoftWarps) {
    // ================================================================ softmax (slot = warp / 4)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
    const int s = warp >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + s * 128;
    const uint32_t tO = tmem + lane_base + 256 + s * 128;
    const float sl2 = a.scale_log2;
    uint64_t* my_o_full = s ? o_full1 : o_full;
    // tiles seen (mask ring), S tiles of this slot (s_full phase), items with this slot live
    // (o_full phase: a slot waits only for items it takes part in, so it cannot fall two
    // phases behind -- the next such item needs its P)
    uint32_t g = 0, ns = 0, no = 0;
    for (int it = beg; it < end; ++it) {
      const PItem u = load_item(a, it);
      const bool live = s == 0 || u.live1;
      const int mt = s ? u.mt1 : u.mt0;
      const int t = mt * kBM + row;
      const int my_i = u.seq_len - u.q_len + t;
      const int span_from = a.span ? a.span[3 * u.b + 2] : INT_MAX;
      float m_run = -CUDART_INF_F, l_run = 0.f;
      for (int j = 0; j < u.n_tiles; ++j, ++g) {
        const int cs = g % kNC;
        if (!live) {  // dead slot: still release the mask slot
          mbar_wait(&c_full[cs], (g / kNC) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&c_empty[cs]);
          continue;
        }
        mbar_wait(&s_full[s], ns & 1);
#ifdef HPA_TRACE
        if (ns == 0 && threadIdx.x == 0) CTA_STAMP(2, gtimer());
#endif
        ++ns;
        tc_fence_after();
        softmax_tile<D>(a, s, quarter, row, lane, j, tS, tO, sC + cs * (kBN + 4), &c_full[cs], (g / kNC) & 1,
                        &c_empty[cs], &p_full[2 * s], my_i, span_from, sl2, m_run, l_run);
      }
      if (!live) continue;
      mbar_wait(my_o_full, no & 1);
#ifdef HPA_TRACE
      if (threadIdx.x == 0 && it == end - 1) CTA_STAMP(3, gtimer());
#endif
      ++no;
      tc_fence_after();
      // epilogue (row stores: the K/V rings already hold the next item's tiles)
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      if (u.part >= 0) {
        const int pp = (u.part * a.split_max + u.piece) * 2 + s;
        float* orow = a.o_part + (int64_t(pp) * kBM + row) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tc_ld32(tO + c * 32, o);
          tc_wait_ld();
#pragma unroll
          for (int y = 0; y < 32; y += 4)
            *reinterpret_cast<float4*>(orow + c * 32 + y) =
                make_float4(o[y] * inv, o[y + 1] * inv, o[y + 2] * inv, o[y + 3] * inv);
        }
        a.lse_part[int64_t(pp) * kBM + row] = l_run > 0.f ? m_run + __log2f(l_run) : -CUDART_INF_F;
      } else {
        __nv_bfloat16* orow =
            static_cast<__nv_bfloat16*>(a.out) + (int64_t(u.q_off + t) * a.Hq + (s ? u.hq1 : u.hq0)) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tc_ld32(tO + c * 32, o);
          tc_wait_ld();
          if (t < u.q_len) {
#pragma unroll
            for (int y = 0; y < 32; y += 8) {
              uint4 v;
              v.x = pack_bf16(o[y + 0] * inv, o[y + 1] * inv);
              v.y = pack_bf16(o[y + 2] * inv, o[y + 3] * inv);
              v.z = pack_bf16(o[y + 4] * inv, o[y + 5] * inv);
              v.w = pack_bf16(o[y + 6] * inv, o[y + 7] * inv);
              *reinterpret_cast<uint4*>(orow + c * 32 + y) = v;
            }
          }
        }
      }
      tc_fence_before();  // O_s read before the next item's P(0) publication lets PV overwrite it
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef HPA_TRACE
  if (threadIdx.x == 0) {
    CTA_STAMP(4, gtimer());
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    CTA_STAMP(5, smid);
    CTA_STAMP(6, end - beg);
    CTA_STAMP(7, 1);
  }
#endif
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Split-KV merge (the LSE algebra of the decode combine, a5): one warp per (split unit, slot,
// query row); lane l holds the LSE of piece l, every lane accumulates D/32 dims over the pieces.
// out = sum_i 2^(lse_i - M) O_i / sum_i 2^(lse_i - M), bf16, into the caller's output rows.
// kS > 0: compiled for exactly kS pieces (the planner's counts), so every piece's loads are
// issued before the first use; kS = 0: any count <= 15.
template <int D, int kS>
__global__ void __launch_bounds__(128) prefill_combine_kernel(const PrefillArgs a) {
  grid_dependency_wait();
  grid_launch_dependents();
  constexpr int kV = D / 32;
  constexpr int kU = kS > 0 ? kS : 1;  // pieces held in registers at once
  const int lane = threadIdx.x & 31;
  const int64_t rid = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (rid >= int64_t(a.n_parts) * 2 * kBM) return;
  const int part = int(rid / (2 * kBM)), s = int(rid / kBM) & 1, row = int(rid % kBM);
  const int4 u = a.parts[2 * part], uq = a.parts[2 * part + 1];  // {b, y, x, nsplit}, {q_len, q_off}
  int hq_s[2], mt_s[2];
  unit_slots(a.G, u.y, u.z, hq_s, mt_s);
  const int t = mt_s[s] * kBM + row;
  if (t >= uq.x) return;
  const int S = u.w;  // <= kS when kS > 0 (kS = the plan's largest piece count)
  auto pidx = [&](int i) { return (int64_t(part * a.split_max + i) * 2 + s) * kBM + row; };
  auto load = [&](int i, float* v) {
    const float* op = a.o_part + pidx(i) * D + lane * kV;
    if constexpr (kV == 4) {
      const float4 x = *reinterpret_cast<const float4*>(op);
      v[0] = x.x; v[1] = x.y; v[2 % kV] = x.z; v[3 % kV] = x.w;
    } else {
      const float2 x = *reinterpret_cast<const float2*>(op);
      v[0] = x.x; v[1 % kV] = x.y;
    }
  };
  const float l = lane < S ? a.lse_part[pidx(lane)] : -CUDART_INF_F;
  float vals[kU][kV];
  if constexpr (kS > 0) {
#pragma unroll
    for (int i = 0; i < kS; ++i)
      if (i < S) load(i, vals[i]);
  }
  float M = l;
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w = l == -CUDART_INF_F ? 0.f : fast_exp2(l - M);
  float W = w;
#pragma unroll
  for (int o = 16; o; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
  float acc[kV];
#pragma unroll
  for (int v = 0; v < kV; ++v) acc[v] = 0.f;
  if constexpr (kS > 0) {
#pragma unroll
    for (int i = 0; i < kS; ++i) {
      const float wi = __shfl_sync(0xffffffffu, w, i);
      if (i < S) {
#pragma unroll
        for (int v = 0; v < kV; ++v) acc[v] += wi * vals[i][v];
      }
    }
  } else {
    for (int i = 0; i < S; ++i) {
      const float wi = __shfl_sync(0xffffffffu, w, i);
      load(i, vals[0]);
#pragma unroll
      for (int v = 0; v < kV; ++v) acc[v] += wi * vals[0][v];
    }
  }
  const float inv = W > 0.f ? 1.f / W : 0.f;
  __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + (int64_t(uq.y + t) * a.Hq + hq_s[s]) * D + lane * kV;
  if constexpr (kV == 4) {
    uint2 v;
    v.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    v.y = pack_bf16(acc[2 % kV] * inv, acc[3 % kV] * inv);
    *reinterpret_cast<uint2*>(orow) = v;
  } else {
    *reinterpret_cast<uint32_t*>(orow) = pack_bf16(acc[0] * inv, acc[1 % kV] * inv);
  }
}

template <int D>
cudaError_t launch_combine_d(const PrefillArgs& a, cudaStream_t s) {
  const dim3 grid(unsigned((int64_t(a.n_parts) * 2 * kBM + 3) / 4));
  switch (a.split_max) {  // every split unit of a plan has split_max pieces
    case 2: return launch_pdl(prefill_combine_kernel<D, 2>, grid, dim3(128), 0, s, a);
    case 3: return launch_pdl(prefill_combine_kernel<D, 3>, grid, dim3(128), 0, s, a);
    case 4: return launch_pdl(prefill_combine_kernel<D, 4>, grid, dim3(128), 0, s, a);
    case 6: return launch_pdl(prefill_combine_kernel<D, 6>, grid, dim3(128), 0, s, a);
    case 8: return launch_pdl(prefill_combine_kernel<D, 8>, grid, dim3(128), 0, s, a);
    default: return launch_pdl(prefill_combine_kernel<D, 0>, grid, dim3(128), 0, s, a);
  }
}

template <int D>
cudaError_t launch_prefill_d(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                             const CUtensorMap& tm_o, const CUtensorMap& tm_op, const PrefillArgs& a, cudaStream_t s,
                             int* launches) {
  const int mtiles = (a.max_q_len + kBM - 1) / kBM;
  ++*launches;
  if (HPA_PF1 && HPA_PF1_CLUSTER && (a.G & 1) == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2, mtiles, (a.Hq / 2) * a.n_seqs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = PSmem<D>::kBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, prefill_kernel<D, true>, tm_q, tm_k, tm_v, tm_o, tm_op, a);
  }
  if (!HPA_PF1 && a.work) {  // split-KV work list: one CTA per (unit, piece), then the merge
    if (a.n_work == 0) return cudaSuccess;
    cudaError_t e;
    if (a.cta_off) {
      e = launch_pdl(prefill_persistent_kernel<D>, dim3(unsigned(a.n_ctas)), dim3(kThreads), PSmem<D>::kBytes, s,
                     tm_q, tm_k, tm_v, a);
    } else if (HPA_PF_MC2 && a.mc2) {  // consecutive work items pair up as 2-CTA clusters
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(a.n_work));
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = PSmem<D>::kBytes;
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      e = cudaLaunchKernelEx(&cfg, prefill_kernel<D, true>, tm_q, tm_k, tm_v, tm_o, tm_op, a);
    } else {
      e = launch_pdl(prefill_kernel<D, false>, dim3(unsigned(a.n_work)), dim3(kThreads), PSmem<D>::kBytes, s, tm_q,
                     tm_k, tm_v, tm_o, tm_op, a);
    }
    if (e != cudaSuccess || a.n_parts == 0) return e;
    ++*launches;
    return launch_combine_d<D>(a, s);
  }
  dim3 grid;
  if (HPA_PF1) grid = dim3(mtiles, a.Hq, a.n_seqs);
  else if ((a.G & 1) == 0) grid = dim3(mtiles, a.Hkv * (a.G / 2), a.n_seqs);
  else grid = dim3((mtiles + 1) / 2, a.Hq, a.n_seqs);
  return launch_pdl(prefill_kernel<D, false>, grid, dim3(kThreads), PSmem<D>::kBytes, s, tm_q, tm_k, tm_v, tm_o,
                    tm_op, a);
}

}  // namespace

bool prefill_split_supported() { return !HPA_PF1 && !HPA_SM16; }
bool prefill_mc2_supported(int32_t G) { return HPA_PF_MC2 && !HPA_SM16 && G % 4 == 0; }

cudaError_t prefill_init_attributes() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(prefill_kernel<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                PSmem<128>::kBytes)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(prefill_kernel<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                PSmem<64>::kBytes)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(prefill_persistent_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                PSmem<128>::kBytes)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(prefill_persistent_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                PSmem<64>::kBytes)) != cudaSuccess)
    return e;
  if ((HPA_PF1 && HPA_PF1_CLUSTER) || HPA_PF_MC2) {
    if ((e = cudaFuncSetAttribute(prefill_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  PSmem<128>::kBytes)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(prefill_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  PSmem<64>::kBytes)) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

cudaError_t launch_prefill(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                           const CUtensorMap& tm_o, const CUtensorMap& tm_op, const PrefillArgs& a, int32_t D,
                           cudaStream_t s, int* launches) {
  if (a.n_seqs == 0) return cudaSuccess;
  if (D == 128) return launch_prefill_d<128>(tm_q, tm_k, tm_v, tm_o, tm_op, a, s, launches);
  if (D == 64) return launch_prefill_d<64>(tm_q, tm_k, tm_v, tm_o, tm_op, a, s, launches);
  return cudaErrorInvalidValue;
}

}  // namespace hpa
