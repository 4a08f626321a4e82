// copy_kernels.cu -- the paper's "store ... into the corresponding blocks" op
// as one sm_100a scatter kernel, plus the logical-KV export
// used by the bit-exact tests.
//
// Roofline: HBM copy. Algorithmic bytes = 2 (K,V) x rows x H_kv x d x 2 B read
// + the same written.
#include "hpa_kernels.h"
#include "ptx.cuh"
#include <cuda_bf16.h>

namespace hpa {

namespace {

// Copies record r's rows (all layers, heads, 16-B vectors) into their pool slots,
// grid-stride over this record's CTAs.
__device__ __forceinline__ void copy_rows(const PoolGeom& g, const ScatterRecord& r, const int32_t* slots) {
  const int32_t vec_per_row = g.D / 8;  // 16-byte vectors per (row, head)
  const int64_t per_layer = int64_t(r.n_rows) * g.Hkv * vec_per_row;
  const int64_t total = per_layer * g.L;
  const int64_t page_elems = int64_t(g.P) * g.D;
  constexpr int kU = 4;  // vectors in flight per thread
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; base < total; base += stride * kU) {
    int4 kv[kU], vv[kU];
    int64_t dst[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * stride;
      dst[u] = -1;
      if (i < total) {
        const int32_t c = int32_t(i % vec_per_row);
        int64_t rest = i / vec_per_row;
        const int32_t h = int32_t(rest % g.Hkv);
        rest /= g.Hkv;
        const int32_t row = int32_t(rest % r.n_rows);
        const int32_t l = int32_t(rest / r.n_rows);
        const int64_t src = int64_t(l) * r.stride_l + int64_t(row) * r.stride_r + int64_t(h) * g.D + c * 8;
        const int32_t slot = slots[r.slot_off + row];
        const int32_t page = slot / g.P, prow = slot % g.P;
        dst[u] = ((int64_t(l) * g.NP + page) * g.Hkv + h) * page_elems + int64_t(prow) * g.D + c * 8;
        kv[u] = __ldg(reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(r.k) + src));
        vv[u] = __ldg(reinterpret_cast<const int4*>(static_cast<const __nv_bfloat16*>(r.v) + src));
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
__global__ void __launch_bounds__(256) scatter_kernel(PoolGeom g, int32_t* __restrict__ arena,
                                                      const WordWrite* __restrict__ words,
                                                      int32_t n_words,
                                                      const ScatterRecord* __restrict__ recs,
                                                      const int32_t* __restrict__ slots) {
  grid_dependency_wait();
  const int64_t nthreads = int64_t(gridDim.x) * gridDim.y * blockDim.x;
  const int64_t gtid = (int64_t(blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < n_words; i += nthreads) arena[words[i].idx] = words[i].val;
  if (recs == nullptr) return;
  copy_rows(g, recs[blockIdx.y], slots);
}

// Same, with the metadata in the kernel parameters (no H2D copy).
__global__ void __launch_bounds__(256) scatter_inline_kernel(PoolGeom g, int32_t* __restrict__ arena,
                                                             const __grid_constant__ InlineMeta m) {
  grid_dependency_wait();
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < m.n_words; i += nthreads) arena[m.data[2 * i]] = m.data[2 * i + 1];
  if (!m.has_rec) return;
  copy_rows(g, m.rec, m.data + 2 * m.n_words);
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
                           const int32_t* slots, int64_t max_rows_per_rec, cudaStream_t s) {
  if (n_words == 0 && n_recs == 0) return cudaSuccess;
  const int64_t work = max_rows_per_rec * g.Hkv * (g.D / 8) * g.L / 4;  // 4 vectors per thread
  int64_t bx = (work + 255) / 256;
  if (n_recs == 0) bx = (n_words + 255) / 256;
  // Enough CTAs to fill 148 SMs several times over; each loops grid-stride.
  const int64_t cap = n_recs > 0 ? (148 * 16 + n_recs - 1) / n_recs : 148 * 4;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  dim3 grid(unsigned(bx), unsigned(n_recs > 0 ? n_recs : 1));
  return launch_pdl(scatter_kernel, grid, dim3(256), 0, s, g, arena, words, n_words,
                    n_recs > 0 ? recs : static_cast<const ScatterRecord*>(nullptr), slots);
}

cudaError_t launch_scatter_inline(const PoolGeom& g, int32_t* arena, const InlineMeta& m, int64_t max_rows,
                                  cudaStream_t s) {
  int64_t bx = m.has_rec ? (max_rows * g.Hkv * (g.D / 8) * g.L / 4 + 255) / 256 : (m.n_words + 255) / 256;
  if (bx > 148 * 16) bx = 148 * 16;
  if (bx < 1) bx = 1;
  return launch_pdl(scatter_inline_kernel, dim3(unsigned(bx)), dim3(256), 0, s, g, arena, m);
}

cudaError_t launch_export(const PoolGeom& g, DevTables t, int32_t layer, int32_t seq,
                          int32_t n_entries_host, void* k_out, void* v_out, cudaStream_t s) {
  if (n_entries_host == 0) return cudaSuccess;
  export_kernel<<<dim3(n_entries_host, g.Hkv), 128, 0, s>>>(g, t, layer, seq, k_out, v_out);
  return cudaGetLastError();
}

}  // namespace hpa
