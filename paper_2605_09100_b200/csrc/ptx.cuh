// ptx.cuh -- thin inline-PTX wrappers for sm_100a (mbarrier, TMA, ldmatrix,
// mma.sync, tcgen05). Only what the HPA kernels use.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>

namespace hpa {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Adds expected transaction bytes to the current phase without arriving.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Arrives `count` times at once (one release standing for several expected arrivals).
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifdef HPA_DEBUG_HANG
// Debug builds: give up after ~2^24 polls and report the stuck barrier (smem offset).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t n = 0; !mbar_try_wait(bar, parity); ++n) {
    if (n == (1u << 24)) {
      printf("HANG block (%d,%d,%d) thread %d bar smem 0x%x parity %u\n", blockIdx.x, blockIdx.y, blockIdx.z,
             threadIdx.x, smem_u32(bar), parity);
      return;
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
#endif

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D tile load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 3-D tile load with an L2 cache-policy hint (e.g. evict-first for streamed KV).
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* m, uint64_t* bar,
                                                 int32_t c0, int32_t c1, int32_t c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
// TMA tile stores shared -> global (bulk-group completion; the smem source may be reused or
// released once bulk_wait_read() returns).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1,
                                             int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- ldmatrix / mma.sync
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulate.
// 8x8 b16 matrix transpose across the warp (fragment layout in, fragment layout out).
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_f16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t f16x2_from_e4m3x2(uint32_t two_codes) {  // low 16 bits: 2 codes
  uint32_t h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(uint16_t(two_codes)));
  return h2;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));  // lo in the low 16 bits
  return r;
}
// bf16x2 -> f16x2 (exact for |x| in the f16 normal range)
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t v) {
  return pack_f16(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}
// bf16x2 -> f16x2 of (x * mul), mul a power of two chosen to keep x * mul in f16's range
__device__ __forceinline__ uint32_t bf16x2_to_f16x2_scaled(uint32_t v, float mul) {
  return pack_f16(__uint_as_float(v << 16) * mul, __uint_as_float(v & 0xffff0000u) * mul);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x = lo (low 16 bits)
  return *reinterpret_cast<uint32_t*>(&v);
}
// 8 codes * scale -> 8 bf16 (fp32 product, bf16 round to nearest even): int4.
__device__ __forceinline__ int4 bf16x8_from_e4m3(uint2 c, float scale) {
  uint32_t in[4] = {c.x & 0xffffu, c.x >> 16, c.y & 0xffffu, c.y >> 16};
  uint32_t out[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(uint16_t(in[i])));
    const float lo = __half2float(__ushort_as_half(uint16_t(h2 & 0xffffu))) * scale;
    const float hi = __half2float(__ushort_as_half(uint16_t(h2 >> 16))) * scale;
    out[i] = pack_bf16(lo, hi);
  }
  return make_int4(int(out[0]), int(out[1]), int(out[2]), int(out[3]));
}

// NEXT-4c fp8 token pool layout: per 16-row group of a (layer, page, head) tile one
// contiguous block [16 x D e4m3 codes | 16 fp32 row scales] (16 D + 64 bytes), so a decode
// chunk is one bulk copy. Pool row prow = ((l * NPt + page) * H_kv + h) * P + r -> block prow/16.
__host__ __device__ __forceinline__ int64_t fp8_block_bytes(int D) { return 16 * int64_t(D) + 64; }
__host__ __device__ __forceinline__ uint8_t* fp8_code_ptr(uint8_t* base, int64_t prow, int D) {
  return base + (prow >> 4) * fp8_block_bytes(D) + (prow & 15) * int64_t(D);
}
// K codes only (HPA_FP8_KSWZ): the 16-byte chunks of a row are XOR-swizzled by the row's
// position in its 16-row block, chunk' = chunk ^ (r & (D/16 - 1)), so that lanes reading the
// same chunk column of 8 different rows hit different banks. Address of K code byte `off`
// (logical column) of pool row prow.
#ifndef HPA_FP8_KSWZ
#define HPA_FP8_KSWZ 1
#endif
__host__ __device__ __forceinline__ int fp8_kswz(int off, int64_t prow, int D) {
  if (!HPA_FP8_KSWZ) return off;
  const int r = int(prow & 15) & (D / 16 - 1);
  return (((off >> 4) ^ r) << 4) | (off & 15);
}
__host__ __device__ __forceinline__ uint8_t* fp8_kcode_ptr(uint8_t* base, int64_t prow, int D, int off) {
  return fp8_code_ptr(base, prow, D) + fp8_kswz(off, prow, D);
}
// V rows (HPA_FP8_VPAIR): the codes of keys 2p and 2p+1 of a 16-row block interleave in
// "pair row" p: dim 16m + 8h + g (g < 8) of row r sits at byte 32m + 4g + 2h + (r & 1), so the
// 4 bytes at 32m + 4g are the (key 2p, key 2p+1) code pairs of dims 16m + g and 16m + g + 8 --
// two f16x2 registers of the V^T MMA operand (rows g and g + 8 of M tile m) from one 32-bit
// load. The pair row's 16-byte chunks are XOR-swizzled by (2p) & 7, which makes those loads
// (lanes (g, t) read pair rows t and t + 4) bank-conflict-free.
#ifndef HPA_FP8_VPAIR
#define HPA_FP8_VPAIR 1
#endif
#if HPA_FP8_F16
#undef HPA_FP8_VPAIR
#define HPA_FP8_VPAIR 0
#endif
__host__ __device__ __forceinline__ int fp8_voff(int r, int d, int D) {  // byte in the block's code area
  if (!HPA_FP8_VPAIR) return r * D + d;
  const int pr = r >> 1, lin = 32 * (d >> 4) + 4 * (d & 7) + 2 * ((d >> 3) & 1) + (r & 1);
  return pr * 2 * D + ((((lin >> 4) ^ ((2 * pr) & 7))) << 4) + (lin & 15);
}
__host__ __device__ __forceinline__ uint8_t* fp8_block_codes(uint8_t* base, int64_t prow, int D) {
  return base + (prow >> 4) * fp8_block_bytes(D);
}
__host__ __device__ __forceinline__ float* fp8_scale_ptr(uint8_t* base, int64_t prow, int D) {
  return reinterpret_cast<float*>(base + (prow >> 4) * fp8_block_bytes(D) + 16 * int64_t(D) + 4 * (prow & 15));
}
// The 8 V codes of block row r, dims d0 .. d0+7 (d0 % 8 == 0), as one uint2 (logical order).
__device__ __forceinline__ uint2 fp8_vcodes8(const uint8_t* blk, int r, int d0, int D) {
  if (!HPA_FP8_VPAIR) return *reinterpret_cast<const uint2*>(blk + r * D + d0);
  // dims d0 + g sit at byte 4 g + b (b = 2 h + (r & 1)) of the 32 bytes of group d0 / 16:
  // byte b of every word of its two chunks
  const int m16 = d0 & ~15, b = 2 * ((d0 >> 3) & 1) + (r & 1);
  const uint4 ca = *reinterpret_cast<const uint4*>(blk + fp8_voff(r & ~1, m16, D));      // dims m16 + 0..3
  const uint4 cb = *reinterpret_cast<const uint4*>(blk + fp8_voff(r & ~1, m16 + 4, D));  // dims m16 + 4..7
  const uint32_t sel = uint32_t(b) | (uint32_t(b + 4) << 4);
  const uint32_t a01 = __byte_perm(ca.x, ca.y, sel), a23 = __byte_perm(ca.z, ca.w, sel);
  const uint32_t b01 = __byte_perm(cb.x, cb.y, sel), b23 = __byte_perm(cb.z, cb.w, sel);
  return make_uint2(__byte_perm(a01, a23, 0x5410), __byte_perm(b01, b23, 0x5410));
}
// Writes 8 V codes (logical order, element i in byte i) of block row r, dims d0 .. d0+7.
__device__ __forceinline__ void fp8_vstore8(uint8_t* blk, int r, int d0, int D, uint2 codes) {
  if (!HPA_FP8_VPAIR) {
    *reinterpret_cast<uint2*>(blk + r * D + d0) = codes;
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    blk[fp8_voff(r, d0 + i, D)] = uint8_t(((i < 4 ? codes.x : codes.y) >> (8 * (i & 3))) & 0xff);
}
// Same packing on the integer ALU pipe (F2FP issues on the XU pipe that MUFU.EX2 also uses):
// round to nearest with ties away from zero (add half an ulp of bf16, keep the upper halves).
// Differs from RNE only on exact ties. For finite non-negative inputs (softmax P).
__device__ __forceinline__ uint32_t pack_bf16_alu(float lo, float hi) {
  return __byte_perm(__float_as_uint(lo) + 0x8000u, __float_as_uint(hi) + 0x8000u, 0x7632);
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Byte offset of (row, 16-byte chunk) inside a tile written by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B: rows are 128 B, chunk index XOR (row % 8).
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels launched with launch_pdl() may start while the previous kernel in the
// stream drains; they must call this before touching global memory it may write.
__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// PDL: let the next kernel in the stream start its prologue now. Safe because every kernel
// this library launches with PDL calls grid_dependency_wait() (full completion + memory
// visibility of the predecessor) before touching memory another kernel uses.
__device__ __forceinline__ void grid_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

// ---------------------------------------------------------------- named barriers
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace hpa
