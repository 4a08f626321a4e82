// hpa_kernels.h -- internal interface between the host runtime (runtime.cpp)
// and the CUDA kernels. Not part of the public ABI (see include/hpa.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace hpa {

// Device block-table entry meta word: bits 0..15 valid_rows, bit 30 latent.
constexpr int32_t kMetaLatent = 1 << 30;
constexpr int32_t kMetaRowsMask = 0xffff;

// Device metadata arena (one int32 allocation), sliced as:
//   block_table [max_seqs][max_pages]  physical page id per entry
//   pos0        [max_seqs][max_pages]  logical index of the entry's row 0
//   meta        [max_seqs][max_pages]  valid_rows | latent bit
//   seq_len     [max_seqs]
//   n_entries   [max_seqs]
struct DevTables {
  int32_t* block_table;
  int32_t* pos0;
  int32_t* meta;
  int32_t* seq_len;
  int32_t* n_entries;
  int32_t max_pages;
};

// One (index, value) write into the metadata arena.
struct WordWrite {
  int32_t idx;
  int32_t val;
};

// One scatter record: n_rows rows of K and V, copied for every layer into the
// pool slots slots[slot_off .. slot_off + n_rows) (slot = page * P + row).
// Row r's destination: slot mode (append): slot = idx[off + r], slot = page * P + row;
// page mode (latent install): g = row0 + r, slot = idx[off + g / P] * P + g % P.
// Source: the k / v pointers, or (src_from_pool) the pool itself at slot
// idx[src_off + r] (in-cache moves, e.g. hpa_seq_compress).
struct ScatterRecord {
  const void* k;      // bf16, element (l, r, h, x) at k + l*stride_l + r*stride_r + h*d + x
  const void* v;
  int64_t stride_l;   // elements
  int64_t stride_r;   // elements
  int32_t n_rows;
  int32_t idx_off;    // offset into the index array (slots or pages)
  int32_t row0;       // page mode: row offset inside the first page
  int32_t page_mode;
  int32_t src_from_pool;
  int32_t src_off;    // src_from_pool: offset of the source slots in the index array
  int32_t quant8;     // NEXT-4c: destination is the fp8 token pool (rows quantized, reading A20)
  int32_t src_fp8;    // NEXT-4c: source slots are in the fp8 token pool (rows dequantized to bf16)
};

struct PoolGeom {
  void* k_pool;  // bf16 [L][NP][H_kv][P][d]
  void* v_pool;
  int32_t L, NP, Hkv, P, D, log2P;
  // NEXT-4c fp8 token pools (nullptr when the cache stores bf16 token pages), K and V:
  // blocks of [16 x d e4m3 codes | 16 fp32 row scales] (reading A20; fp8_code_ptr / fp8_scale_ptr)
  uint8_t* k8;
  uint8_t* v8;
  int32_t NPt;
};

// Metadata writes + row scatter in one launch (append / install / apply).
cudaError_t launch_scatter(const PoolGeom& g, int32_t* arena, const WordWrite* words,
                           int32_t n_words, const ScatterRecord* recs, int32_t n_recs,
                           const int32_t* idx, int64_t max_rows_per_rec, cudaStream_t s);

// Small metadata shipped as kernel parameters instead of an H2D copy (the
// common decode-step append): table words (2 ints each) then slots (1 int
// each), at most kInlineInts ints, and at most one record.
constexpr int kInlineInts = 1536;
constexpr int kInlineIntsSmall = 224;  // the common case (a decode-step append, a compress) in < 1 KB
template <int N>
struct InlineMetaT {
  int32_t n_words;
  int32_t n_slots;
  int32_t has_rec;
  int32_t pad;
  ScatterRecord rec;
  int32_t data[N];
};
using InlineMeta = InlineMetaT<kInlineInts>;
using InlineMetaSmall = InlineMetaT<kInlineIntsSmall>;  // the launch copies the whole parameter block
cudaError_t launch_scatter_inline(const PoolGeom& g, int32_t* arena, const InlineMetaSmall& m, int64_t max_rows,
                                  cudaStream_t s);
cudaError_t launch_scatter_inline(const PoolGeom& g, int32_t* arena, const InlineMeta& m, int64_t max_rows,
                                  cudaStream_t s);

// NEXT-4c: dequantize whole fp8 token-page tiles into bf16 pages of the main pool;
// items[n] = {fp8 token page, bf16 page, valid rows, 0} (device), g sliced to one layer.
cudaError_t launch_dequant_pages(const PoolGeom& g, const int4* items, int32_t n, cudaStream_t s);

// NEXT-2 copy-on-write: whole-page copies {source page, destination page} in every layer,
// of the bf16 main pools (fp8 = 0) or the fp8 token pools (fp8 = 1). Items travel as kernel
// parameters, kCopyPagesMax per launch.
constexpr int kCopyPagesMax = 128;
struct CopyPagesMeta {
  int32_t n;
  int32_t fp8;
  int2 items[kCopyPagesMax];
};
cudaError_t launch_copy_pages(const PoolGeom& g, const CopyPagesMeta& m, cudaStream_t s);

// Logical K/V export of one (layer, seq): out bf16 [H_kv][len][d].
cudaError_t launch_export(const PoolGeom& g, DevTables t, int32_t layer, int32_t seq,
                          int32_t n_entries_host, void* k_out, void* v_out, cudaStream_t s);

struct DecodeArgs {
  DevTables t;
  const int32_t* seq_rows;  // [n_seqs] device
  const void* q;            // bf16 [n][Hq][d]
  void* out;                // bf16 [n][Hq][d]
  float* o_part;            // fp32 [n][Hq][S][d]   (S > 1)
  float* lse_part;          // fp32 [n][Hq][S]      (log2 domain)
  int32_t* counters;        // [n][Hkv] zero; split-arrival counters for the fused combine
  float* part_o;            // context-parallel partial output (or nullptr): fp32 [n][Hq][d]
  float* part_lse;          //   and log2-sum-exp [n][Hq]
  int32_t n_seqs, Hq, Hkv, G, P, NP, layer, splits;  // splits = S_max (partials stride)
  float scale_log2;         // softmax_scale * log2(e)
  // persistent kernel work list (host-planned, longest unit first):
  // NEXT-4c: token entries read the fp8 pools (16-row blocks of codes + row scales)
  int32_t fp8, NPt;
  const uint8_t* k8;
  const uint8_t* v8;
  const int4* units;        // [n_units] {request b, seq id, h | split << 8 | S_b << 16, r}: entries
                            // [r, n_entries) split S_b ways (r: the request's cascaded shared run)
  const int32_t* nsplit;    // [n] per-request split count S_b (combine); nullptr = uniform `splits`
  int32_t* sched;           // [2] unit ticket / finished-CTA counters, zero between calls
  int32_t n_units;
  long long* trace;         // HPA_TRACE builds only: per-CTA {entry ns, last consumer exit ns, units}
  // cascade decode (NEXT-2): group-piece records [kGroupRec] {e0, e1, n members, -, request
  // index b[kGroupMax], partial slot[kGroupMax]}; a unit {-2 - record, representative seq, h, 0}
  // reads entries [e0, e1) of the representative once for the G query rows of every member.
  // nullptr: no group units in this plan.
  const int32_t* groups;
};
constexpr int kGroupMax = 32;               // members per group record (rows = members x G <= 32)
constexpr int kGroupRec = 4 + 2 * kGroupMax;
// Fused decode-step append (hpa_append_decode): request b of the batch gains one token row,
// written by the decode kernel itself before it reads that row's tile. tail[b] is the
// request's LAST block-table entry after the append, {n_entries, page, meta, pos0}; the new
// row is row (meta & kMetaRowsMask) - 1 of that page. The kernel reads these values instead
// of the device table for that entry (which it writes back for later calls).
struct AppendRows {
  const void* k;        // bf16 [L][n][H_kv][d] (device)
  const void* v;
  void* k_pool;         // the cache's bf16 pools [L][NP][H_kv][P][d]
  void* v_pool;
  int64_t stride_l;     // elements between layers = n * H_kv * d
  int32_t n, L;         // n == n_seqs of the decode call
  const int4* tail;     // [n] (host; travels as kernel parameters)
};
constexpr int kAppendFuseSmall = 64;   // parameter-block variants: 1 KB and 8 KB of tail records
constexpr int kAppendFuseMax = 512;
// Merge of context-parallel partials: out[r][:] = sum_p 2^(lse_p - LSE) o_p / sum_p 2^(lse_p - LSE).
cudaError_t launch_merge(int32_t n_parts, int32_t n_rows, int32_t D, const float* o_parts,
                         const float* lse_parts, void* out, cudaStream_t s);
// tm_k / tm_v: 2-D tensor maps over the pools viewed as [L*NP*H_kv*P][d],
// box {64, 16}, 128-B swizzle.
// ap (or nullptr): the fused append of hpa_append_decode (persistent kernel, ap->n <= kAppendFuseMax).
cudaError_t launch_decode(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const DecodeArgs& a,
                          int32_t D, cudaStream_t s, int* launches, const AppendRows* ap = nullptr);
int decode_ctas_per_sm(int32_t D, int32_t G);
// Persistent decode kernel compiled in (HPA_DECODE_PERSISTENT) and its resident CTA count.
bool decode_persistent();
int decode_slots(int32_t D, int32_t G);
// Per-device one-time setup (dynamic smem opt-in); call with the device current.
cudaError_t decode_init_attributes();
cudaError_t prefill_init_attributes();

struct PrefillArgs {
  DevTables t;
  const int32_t* seq_rows;  // [n] device
  const int32_t* q_len;     // [n] device
  const int32_t* q_off;     // [n] device: first row of sequence i in q / out
  void* out;                // bf16 [sum q][Hq][d]
  int32_t n_seqs, Hq, Hkv, G, P, NP, layer, max_q_len;
  float scale_log2;
  int32_t log2P;
  const int32_t* span;      // [n][3] device (lo, hi, q_from) or nullptr: GRC mask-out span
  long long* trace;         // HPA_TRACE builds only: per-phase clock64 stamps of CTA (0,0,0)
  // Work list (plan_prefill; nullptr: one CTA per (row tile, head pair, sequence) of a grid,
  // each searching the table for its key-tile count). CTA i reads work[4i .. 4i+3] =
  // {seq b, head index y, row-tile index x, piece | nsplit << 4 | part << 8},
  // {first iteration jb, iterations n, skip_a, n_skip} (iteration j loads key tile
  // j < skip_a ? j : j + n_skip), {seq id, q_len, q_off, seq_len}, {n_entries, 0, 0, 0}.
  // nsplit == 1 writes bf16 output directly; nsplit > 1 writes O / l (fp32) and the
  // log2-domain LSE of piece `piece` of split unit `part` to o_part / lse_part, merged by
  // prefill_combine_kernel over parts[2j], parts[2j+1] = {b, y, x, nsplit}, {q_len, q_off, 0, 0}.
  const int4* work;
  int32_t n_work;
  const int4* parts;
  int32_t n_parts, split_max;
  float* o_part;            // [n_parts][split_max][2 slots][128 rows][D]
  float* lse_part;          // [n_parts][split_max][2][128]
  // Persistent launch (nullptr: one CTA per work item): CTA c runs items
  // [cta_off[c], cta_off[c + 1]) of `work`, in order; n_ctas <= #SMs.
  const int32_t* cta_off;
  int32_t n_ctas;
  int32_t mc2;              // HPA_PF_MC2 builds: work items 2k, 2k+1 are a 2-CTA cluster sharing K/V
};
// Split-KV prefill (work lists) is built in the default kernel configuration only.
bool prefill_split_supported();
bool prefill_mc2_supported(int32_t G);
// tm_q / tm_o: 3-D maps over q / out [sum q][Hq][d] with box {64, 1, 128};
// tm_k / tm_v: 2-D maps over the pools with box {64, min(P,128)};
// tm_op: 2-D fp32 map over o_part [rows][d] with box {32, 128} (work lists with splits).
cudaError_t launch_prefill(const CUtensorMap& tm_q, const CUtensorMap& tm_k,
                           const CUtensorMap& tm_v, const CUtensorMap& tm_o, const CUtensorMap& tm_op,
                           const PrefillArgs& a, int32_t D, cudaStream_t s, int* launches);

}  // namespace hpa
