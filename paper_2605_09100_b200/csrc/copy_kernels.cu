// copy_kernels.cu -- the paper's "store ... into the corresponding blocks" op
// as one sm_100a scatter kernel, plus the logical-KV export
// used by the bit-exact tests.
//
// Roofline: HBM copy. Algorithmic bytes = 2 (K,V) x rows x H_kv x d x 2 B read
// + the same written.
#include "hpa_kernels.h"
#include "ptx.cuh"
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace hpa {

namespace {

// ---- NEXT-4c fp8 token rows (reading A20) --------------------------------------
// 8 e4m3 codes <- 8 fp32 values, round to nearest even, saturating (element i in byte i).
__device__ __forceinline__ uint2 e4m3x8_from_f32(const float* x) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint16_t h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(x[2 * i + 1]), "f"(x[2 * i]));
    w[i] = h;
  }
  return make_uint2(w[0] | (w[1] << 16), w[2] | (w[3] << 16));
}
// Appends record r's rows into the fp8 token pool: one (layer, row, head) unit per group of
// D/8 consecutive lanes (8 elements each); the group reduces the row's amax, then
// s = amax / 448, codes = e4m3(x * (448 / amax)) (s = 1, codes 0 for an all-zero row).
template <int D>
__device__ __forceinline__ void quant_rows(const PoolGeom& g, const ScatterRecord& r, const int32_t* idx) {
  constexpr int kVPR = D / 8;
  const uint32_t units = uint32_t(r.n_rows) * uint32_t(g.Hkv) * uint32_t(g.L);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ustride = gridDim.x * blockDim.x / kVPR;
  const uint32_t c = tid % kVPR;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gmask = ((kVPR == 32 ? 0xffffffffu : ((1u << kVPR) - 1u))) << (lane & ~uint32_t(kVPR - 1));
  const __nv_bfloat16* ksrc = static_cast<const __nv_bfloat16*>(r.k);
  const __nv_bfloat16* vsrc = static_cast<const __nv_bfloat16*>(r.v);
  for (uint32_t unit = tid / kVPR; unit < units; unit += ustride) {
    const uint32_t h = unit % uint32_t(g.Hkv);
    const uint32_t rest = unit / uint32_t(g.Hkv);
    const uint32_t row = rest % uint32_t(r.n_rows);
    const uint32_t l = rest / uint32_t(r.n_rows);
    const int32_t slot = r.page_mode ? (idx[r.idx_off + ((r.row0 + int32_t(row)) >> g.log2P)] << g.log2P) +
                                           ((r.row0 + int32_t(row)) & (g.P - 1))
                                     : idx[r.idx_off + row];
    const int64_t prow = ((int64_t(l) * g.NPt + (slot >> g.log2P)) * g.Hkv + h) * g.P + (slot & (g.P - 1));
    const int64_t src = int64_t(l) * r.stride_l + int64_t(row) * r.stride_r + int64_t(h) * D + c * 8;
    const int4 kraw = __ldg(reinterpret_cast<const int4*>(ksrc + src));
    const int4 vraw = __ldg(reinterpret_cast<const int4*>(vsrc + src));
    float kx[8], vx[8];
    const __nv_bfloat162* kb = reinterpret_cast<const __nv_bfloat162*>(&kraw);
    const __nv_bfloat162* vb = reinterpret_cast<const __nv_bfloat162*>(&vraw);
    float ka = 0.f, va = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 kf = __bfloat1622float2(kb[i]), vf = __bfloat1622float2(vb[i]);
      kx[2 * i] = kf.x; kx[2 * i + 1] = kf.y;
      vx[2 * i] = vf.x; vx[2 * i + 1] = vf.y;
      ka = fmaxf(ka, fmaxf(fabsf(kf.x), fabsf(kf.y)));
      va = fmaxf(va, fmaxf(fabsf(vf.x), fabsf(vf.y)));
    }
#pragma unroll
    for (int o = kVPR / 2; o > 0; o >>= 1) {
      ka = fmaxf(ka, __shfl_xor_sync(gmask, ka, o));
      va = fmaxf(va, __shfl_xor_sync(gmask, va, o));
    }
    const float kinv = ka > 0.f ? __fdiv_rn(448.f, ka) : 1.f, vinv = va > 0.f ? __fdiv_rn(448.f, va) : 1.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      kx[i] = __fmul_rn(kx[i], kinv);
      vx[i] = __fmul_rn(vx[i], vinv);
    }
    *reinterpret_cast<uint2*>(fp8_kcode_ptr(g.k8, prow, D, int(c) * 8)) = e4m3x8_from_f32(kx);
    fp8_vstore8(fp8_block_codes(g.v8, prow, D), int(prow & 15), int(c) * 8, D, e4m3x8_from_f32(vx));
    if (c == 0) {
      *fp8_scale_ptr(g.k8, prow, D) = ka > 0.f ? __fdiv_rn(ka, 448.f) : 1.f;
      *fp8_scale_ptr(g.v8, prow, D) = va > 0.f ? __fdiv_rn(va, 448.f) : 1.f;
    }
  }
}

// Copies record r's rows (all layers, heads, 16-B vectors) into their pool slots,
// grid-stride over this record's CTAs. A unit is one (layer, row, head) = D/8
// 16-byte vectors handled by D/8 consecutive threads (coalesced 256-B rows);
// each thread keeps kU units in flight. 32-bit index math, P a power of two.
template <int D>
__device__ __forceinline__ void copy_rows(const PoolGeom& g, const ScatterRecord& r, const int32_t* idx) {
  constexpr int kVPR = D / 8;
  constexpr int kU = 4;
  const uint32_t units = uint32_t(r.n_rows) * uint32_t(g.Hkv) * uint32_t(g.L);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ustride = gridDim.x * blockDim.x / kVPR;
  const uint32_t c = tid % kVPR;
  const int64_t page_elems = int64_t(g.P) * D;
  const __nv_bfloat16* ksrc = static_cast<const __nv_bfloat16*>(r.k);
  const __nv_bfloat16* vsrc = static_cast<const __nv_bfloat16*>(r.v);
  for (uint32_t u0 = tid / kVPR; u0 < units; u0 += kU * ustride) {
    int4 kv[kU], vv[kU];
    int64_t dst[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t unit = u0 + u * ustride;
      dst[u] = -1;
      if (unit < units) {
        const uint32_t h = unit % uint32_t(g.Hkv);
        const uint32_t rest = unit / uint32_t(g.Hkv);
        const uint32_t row = rest % uint32_t(r.n_rows);
        const uint32_t l = rest / uint32_t(r.n_rows);
        int32_t slot;
        if (r.page_mode) {
          const int32_t gr = r.row0 + int32_t(row);
          slot = (idx[r.idx_off + (gr >> g.log2P)] << g.log2P) + (gr & (g.P - 1));
        } else {
          slot = idx[r.idx_off + row];
        }
        dst[u] = ((int64_t(l) * g.NP + (slot >> g.log2P)) * g.Hkv + h) * page_elems +
                 int64_t(slot & (g.P - 1)) * D + c * 8;
        if (r.src_from_pool && r.src_fp8) {  // move out of the fp8 token pool: dequantize
          const int32_t ss = idx[r.src_off + row];
          const int64_t prow = ((int64_t(l) * g.NPt + (ss >> g.log2P)) * g.Hkv + h) * g.P + (ss & (g.P - 1));
          kv[u] = bf16x8_from_e4m3(*reinterpret_cast<const uint2*>(fp8_kcode_ptr(g.k8, prow, D, int(c) * 8)),
                                   *fp8_scale_ptr(g.k8, prow, D));
          vv[u] = bf16x8_from_e4m3(fp8_vcodes8(fp8_block_codes(g.v8, prow, D), int(prow & 15), int(c) * 8, D),
                                   *fp8_scale_ptr(g.v8, prow, D));
        } else if (r.src_from_pool) {  // in-cache move: source is another pool slot
          const int32_t ss = idx[r.src_off + row];
          const int64_t src = ((int64_t(l) * g.NP + (ss >> g.log2P)) * g.Hkv + h) * page_elems +
                              int64_t(ss & (g.P - 1)) * D + c * 8;
          kv[u] = *reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.k_pool) + src);
          vv[u] = *reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.v_pool) + src);
        } else {
          const int64_t src = int64_t(l) * r.stride_l + int64_t(row) * r.stride_r + int64_t(h) * D + c * 8;
          kv[u] = __ldg(reinterpret_cast<const int4*>(ksrc + src));
          vv[u] = __ldg(reinterpret_cast<const int4*>(vsrc + src));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (dst[u] >= 0) {
        *reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.k_pool) + dst[u]) = kv[u];
        *reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.v_pool) + dst[u]) = vv[u];
      }
    }
  }
}

// Grid: x = CTAs per record (grid-stride), y = record. All CTAs also apply the
// metadata word writes (grid-stride over words) -- the table update rides the
// same launch as the row copy.
template <int D>
__global__ void __launch_bounds__(256) scatter_kernel(PoolGeom g, int32_t* __restrict__ arena,
                                                      const WordWrite* __restrict__ words,
                                                      int32_t n_words,
                                                      const ScatterRecord* __restrict__ recs,
                                                      const int32_t* __restrict__ idx) {
  grid_dependency_wait();
  grid_launch_dependents();
  const int64_t nthreads = int64_t(gridDim.x) * gridDim.y * blockDim.x;
  const int64_t gtid = (int64_t(blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < n_words; i += nthreads) arena[words[i].idx] = words[i].val;
  if (recs == nullptr) return;
  if (recs[blockIdx.y].quant8) quant_rows<D>(g, recs[blockIdx.y], idx);
  else copy_rows<D>(g, recs[blockIdx.y], idx);
}

// Same, with the metadata in the kernel parameters (no H2D copy).
template <int D, int N>
__global__ void __launch_bounds__(256) scatter_inline_kernel(PoolGeom g, int32_t* __restrict__ arena,
                                                             const __grid_constant__ InlineMetaT<N> m) {
  grid_dependency_wait();
  grid_launch_dependents();
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < m.n_words; i += nthreads) arena[m.data[2 * i]] = m.data[2 * i + 1];
  if (!m.has_rec) return;
  if (m.rec.quant8) quant_rows<D>(g, m.rec, m.data + 2 * m.n_words);
  else copy_rows<D>(g, m.rec, m.data + 2 * m.n_words);
}

// NEXT-4c prefill staging: item i = {fp8 token page, bf16 page, valid rows}; CTA (i, h) writes
// rows 0..valid-1 of the (page, head) tile as bf16(fp32(code) * scale) (reading A20) into the
// bf16 page's tile. Page-granular: no per-row index arrays; one 16-B store per thread.
template <int D>
__global__ void __launch_bounds__(256) dequant_pages_kernel(PoolGeom g, const int4* __restrict__ items) {
  grid_dependency_wait();
  grid_launch_dependents();
  constexpr int kVPR = D / 8;
  const int4 it = items[blockIdx.x];
  const int h = blockIdx.y;
  const int64_t row0 = (int64_t(it.x) * g.Hkv + h) * g.P;  // fp8 pool row of the tile's row 0
  const int64_t dst0 = (int64_t(it.y) * g.Hkv + h) * g.P * D;
  for (int v = threadIdx.x; v < it.z * kVPR; v += blockDim.x) {
    const int r = v / kVPR, c = v % kVPR;
    const int64_t prow = row0 + r;
    const uint2 kc = *reinterpret_cast<const uint2*>(fp8_kcode_ptr(g.k8, prow, D, c * 8));
    const uint2 vc = fp8_vcodes8(fp8_block_codes(g.v8, prow, D), int(prow & 15), c * 8, D);
    const float ks = *fp8_scale_ptr(g.k8, prow, D), vs = *fp8_scale_ptr(g.v8, prow, D);
    reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.k_pool) + dst0 + int64_t(r) * D)[c] = bf16x8_from_e4m3(kc, ks);
    reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.v_pool) + dst0 + int64_t(r) * D)[c] = bf16x8_from_e4m3(vc, vs);
  }
}

// NEXT-2 copy-on-write of a token page shared by forked sequences (reading A21): item i =
// {source page, destination page}; CTA (i, l) copies the page's whole layer-l region -- every
// head, all P rows, K and V -- byte for byte: bf16 tiles [H][P][d], or the fp8 pool's 16-row
// blocks [16 x d codes | 16 scales] (the K chunk swizzle and the V pair rows are functions of
// the row index inside its block, so a raw block copy preserves them). Rows past the sharer's
// valid rows are copied too; they stay masked by valid_rows.
__global__ void __launch_bounds__(256) copy_pages_kernel(PoolGeom g, const __grid_constant__ CopyPagesMeta m) {
  grid_dependency_wait();
  grid_launch_dependents();
  const int2 it = m.items[blockIdx.x];
  const int64_t l = blockIdx.y;
  int64_t bytes;
  const int4 *ks, *vs;
  int4 *kd, *vd;
  if (m.fp8) {
    bytes = int64_t(g.Hkv) * g.P / 16 * fp8_block_bytes(g.D);
    const int64_t per_page = bytes;
    ks = reinterpret_cast<const int4*>(g.k8 + (l * g.NPt + it.x) * per_page);
    vs = reinterpret_cast<const int4*>(g.v8 + (l * g.NPt + it.x) * per_page);
    kd = reinterpret_cast<int4*>(g.k8 + (l * g.NPt + it.y) * per_page);
    vd = reinterpret_cast<int4*>(g.v8 + (l * g.NPt + it.y) * per_page);
  } else {
    bytes = int64_t(g.Hkv) * g.P * g.D * 2;
    const int64_t per_page = bytes / 2;  // elements
    ks = reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.k_pool) + (l * g.NP + it.x) * per_page);
    vs = reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.v_pool) + (l * g.NP + it.x) * per_page);
    kd = reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.k_pool) + (l * g.NP + it.y) * per_page);
    vd = reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(g.v_pool) + (l * g.NP + it.y) * per_page);
  }
  for (int64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) {
    kd[i] = ks[i];
    vd[i] = vs[i];
  }
}

// Grid: x = table entry, y = kv head. Copies rows 0..valid-1 of the page tile
// to out[h][pos0 + r][:].
__global__ void __launch_bounds__(128) export_kernel(PoolGeom g, DevTables t, int32_t layer,
                                                     int32_t seq, void* k_out, void* v_out) {
  const int32_t e = blockIdx.x, h = blockIdx.y;
  const int64_t idx = int64_t(seq) * t.max_pages + e;
  const int32_t page = t.block_table[idx];
  const int32_t pos0 = t.pos0[idx];
  const int32_t valid = t.meta[idx] & kMetaRowsMask;
  const int32_t len = t.seq_len[seq];
  const int32_t vec_per_row = g.D / 8;
  if (g.k8 && !(t.meta[idx] & kMetaLatent)) {  // fp8 token page: dequantized to bf16
    const int64_t row0 = ((int64_t(layer) * g.NPt + page) * g.Hkv + h) * g.P;
    const int64_t dst0 = (int64_t(h) * len + pos0) * g.D;
    for (int32_t i = threadIdx.x; i < valid * vec_per_row; i += blockDim.x) {
      const int64_t prow = row0 + i / vec_per_row;
      const int64_t off = int64_t(i % vec_per_row) * 8;
      reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(k_out) + dst0)[i] =
          bf16x8_from_e4m3(*reinterpret_cast<const uint2*>(fp8_kcode_ptr(g.k8, prow, g.D, int(off))),
                           *fp8_scale_ptr(g.k8, prow, g.D));
      reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(v_out) + dst0)[i] =
          bf16x8_from_e4m3(fp8_vcodes8(fp8_block_codes(g.v8, prow, g.D), int(prow & 15), int(off), g.D),
                           *fp8_scale_ptr(g.v8, prow, g.D));
    }
    return;
  }
  const int64_t src0 = ((int64_t(layer) * g.NP + page) * g.Hkv + h) * int64_t(g.P) * g.D;
  const int64_t dst0 = (int64_t(h) * len + pos0) * g.D;
  for (int32_t i = threadIdx.x; i < valid * vec_per_row; i += blockDim.x) {
    const int64_t off = int64_t(i) * 8;
    reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(k_out) + dst0)[i] =
        reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.k_pool) + src0 + off)[0];
    reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(v_out) + dst0)[i] =
        reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(g.v_pool) + src0 + off)[0];
  }
}

}  // namespace

cudaError_t launch_scatter(const PoolGeom& g, int32_t* arena, const WordWrite* words,
                           int32_t n_words, const ScatterRecord* recs, int32_t n_recs,
                           const int32_t* idx, int64_t max_rows_per_rec, cudaStream_t s) {
  if (n_words == 0 && n_recs == 0) return cudaSuccess;
  const int64_t threads = max_rows_per_rec * g.Hkv * g.L * (g.D / 8) / 4;  // 4 units per thread
  int64_t bx = n_recs == 0 ? (n_words + 255) / 256 : (threads + 255) / 256;
  // Enough CTAs to fill 148 SMs several times over; each loops grid-stride.
  const int64_t cap = n_recs > 0 ? (148 * 16 + n_recs - 1) / n_recs : 148 * 4;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  const dim3 grid(unsigned(bx), unsigned(n_recs > 0 ? n_recs : 1));
  const ScatterRecord* r = n_recs > 0 ? recs : static_cast<const ScatterRecord*>(nullptr);
  if (g.D == 128) return launch_pdl(scatter_kernel<128>, grid, dim3(256), 0, s, g, arena, words, n_words, r, idx);
  return launch_pdl(scatter_kernel<64>, grid, dim3(256), 0, s, g, arena, words, n_words, r, idx);
}

template <int N>
cudaError_t launch_scatter_inline_n(const PoolGeom& g, int32_t* arena, const InlineMetaT<N>& m, int64_t max_rows,
                                    cudaStream_t s) {
  int64_t bx = m.has_rec ? (max_rows * g.Hkv * g.L * (g.D / 8) / 4 + 255) / 256 : (m.n_words + 255) / 256;
  if (bx > 148 * 16) bx = 148 * 16;
  if (bx < 1) bx = 1;
  if (g.D == 128) return launch_pdl(scatter_inline_kernel<128, N>, dim3(unsigned(bx)), dim3(256), 0, s, g, arena, m);
  return launch_pdl(scatter_inline_kernel<64, N>, dim3(unsigned(bx)), dim3(256), 0, s, g, arena, m);
}

cudaError_t launch_scatter_inline(const PoolGeom& g, int32_t* arena, const InlineMeta& m, int64_t max_rows,
                                  cudaStream_t s) {
  return launch_scatter_inline_n(g, arena, m, max_rows, s);
}
cudaError_t launch_scatter_inline(const PoolGeom& g, int32_t* arena, const InlineMetaSmall& m, int64_t max_rows,
                                  cudaStream_t s) {
  return launch_scatter_inline_n(g, arena, m, max_rows, s);
}

cudaError_t launch_dequant_pages(const PoolGeom& g, const int4* items, int32_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const dim3 grid(unsigned(n), unsigned(g.Hkv));
  if (g.D == 128) return launch_pdl(dequant_pages_kernel<128>, grid, dim3(256), 0, s, g, items);
  return launch_pdl(dequant_pages_kernel<64>, grid, dim3(256), 0, s, g, items);
}

cudaError_t launch_copy_pages(const PoolGeom& g, const CopyPagesMeta& m, cudaStream_t s) {
  if (m.n == 0) return cudaSuccess;
  return launch_pdl(copy_pages_kernel, dim3(unsigned(m.n), unsigned(g.L)), dim3(256), 0, s, g, m);
}

cudaError_t launch_export(const PoolGeom& g, DevTables t, int32_t layer, int32_t seq,
                          int32_t n_entries_host, void* k_out, void* v_out, cudaStream_t s) {
  if (n_entries_host == 0) return cudaSuccess;
  export_kernel<<<dim3(n_entries_host, g.Hkv), 128, 0, s>>>(g, t, layer, seq, k_out, v_out);
  return cudaGetLastError();
}

}  // namespace hpa
