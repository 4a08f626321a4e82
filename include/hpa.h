/*
 * hpa.h -- C ABI of the B200-native hybrid paged attention (HPA) library.
 *
 * What it implements: PAPER.md §3 "Hybrid paged attention for LLM serving"
 * (P:L248-251): vLLM-style paged attention whose blocks hold two kinds of KV
 * cache -- regular (prefix + dynamic) token KV and the compressed KV of the
 * meta latent tokens -- "store[d] ... into the corresponding blocks".
 * HPA computes ordinary causal softmax attention over the *logical* KV
 * sequence (block-table order); paging and the latent/token tag change storage
 * and update cost, not the math.
 *
 * Conventions for every call:
 *   - All calls return hpa_status_t; no C++ exception crosses the ABI.
 *     hpa_last_error() returns a thread-local message for the last failure.
 *   - "device" pointers are CUDA device addresses on the cache's device
 *     (e.g. torch.Tensor.data_ptr()); they must be 16-byte aligned and
 *     contiguous in the documented layout. "host" pointers are CPU memory.
 *   - The caller owns q / k / v / out / payload buffers; the cache owns its K/V
 *     pools, block tables and staging. Device work is enqueued on the caller's
 *     stream (`stream` is a cudaStream_t, NULL = legacy default stream); all
 *     calls on one cache must use the same stream or be ordered by the caller.
 *     Input buffers may be reused once the stream has passed the call.
 *   - Host metadata (allocator, tables) is updated synchronously; the device
 *     copy of the tables is updated stream-ordered before the next kernel.
 *   - One cache = one owner thread; calls on a cache are not
 *     thread-safe. Different caches (e.g. one per GPU) are independent.
 *   - Failure atomicity: a call that returns an error leaves the cache
 *     unchanged (HPA_ERR_OUT_OF_PAGES is the "backpressure" signal of S:L388).
 *   - Calls are not CUDA-graph capturable: each stages its per-call metadata
 *     (table writes, scatter records, work lists) through host memory or
 *     kernel parameters at enqueue time, so a replayed graph would repeat
 *     stale metadata. Kernels use programmatic dependent launch instead.
 *   - bf16 everywhere (KV bytes = 2); fp32 accumulation.
 */
#ifndef HPA_H_
#define HPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpa_cache hpa_cache_t;
typedef void* hpa_stream_t; /* a cudaStream_t */

typedef enum {
  HPA_OK = 0,
  HPA_ERR_INVALID_ARG = 1,   /* bad shape / layer / length / alignment / duplicate seq / q_len > seq_len */
  HPA_ERR_OUT_OF_PAGES = 2,  /* pool exhausted; cache left unchanged (S:L388 backpressure) */
  HPA_ERR_SEQ_CAPACITY = 3,  /* a sequence would exceed max_pages_per_seq */
  HPA_ERR_UNKNOWN_SEQ = 4,
  HPA_ERR_UNKNOWN_SET = 5,
  HPA_ERR_CUDA = 6,          /* message carries the cudaError string */
  HPA_ERR_UNSUPPORTED = 7    /* head_dim not in {64,128}, page_size not in {16,32,64,128,256},
                                G = Hq/H_kv > 16, or device is not sm_100 */
} hpa_status_t;

/* Cache configuration. Invariant: num_q_heads % num_kv_heads == 0. */
typedef struct {
  int32_t num_layers;        /* L: layers held in the pool (one pool for all layers) */
  int32_t num_q_heads;       /* Hq */
  int32_t num_kv_heads;      /* H_kv (8 for Qwen3) */
  int32_t head_dim;          /* d: 64 or 128 */
  int32_t page_size;         /* P rows per page: 16, 32, 64, 128 or 256 (reading A15) */
  int32_t num_pages;         /* NP physical pages, shared by all layers */
  int32_t max_seqs;          /* sequence slots; seq ids are 0..max_seqs-1 */
  int32_t max_pages_per_seq; /* block-table row length */
  int32_t device;            /* CUDA ordinal */
  uint64_t placement_seed;   /* 0: free list in page order; else a seeded shuffle of the
                                free list (physical placement is then a random permutation,
                                SURVEY §8(d) "Physical pages") */
  int32_t token_kv_dtype;    /* SURVEY §8(f) NEXT-4c: 0 = token pages bf16 (default, the paper's
                                storage); 1 = token pages fp8 e4m3 with one fp32 scale
                                per (layer, row, kv-head) for K and for V (reading A20),
                                held in a separate token pool; latent pages stay bf16. With 1,
                                decode reads both kinds; prefill dequantizes the batch's token pages
                                into temporary bf16 pages of the main pool for the call (needs
                                free pages; HPA_ERR_OUT_OF_PAGES otherwise). */
  int32_t num_token_pages;   /* token_kv_dtype = 1: pages of the fp8 token pool (> 0) */
} hpa_config_t;

/* Thread-local message of the last failing call ("" if none). */
const char* hpa_last_error(void);
const char* hpa_status_string(hpa_status_t s);

/* KV size = 2 x L x H_kv x d_h x N x bytes (§3 Eq. "KV size").
 * hpa_kv_bytes(28, 8, 128, 1, 2) == 114688. Pure host arithmetic. */
uint64_t hpa_kv_bytes(int64_t num_layers, int64_t num_kv_heads, int64_t head_dim,
                      int64_t seq_len, int64_t elem_bytes);

/* ---------------------------------------------------------------- lifecycle
 * Allocates K and V pools, each bf16 [L][NP][H_kv][P][d] (zero-filled), plus
 * device block tables (page id, pos0, meta per entry; seq_len; entry count).
 * "pre-allocating KV cache in the device memory and partitioning them into
 * fixed-size non-continuous blocks". */
hpa_status_t hpa_cache_create(const hpa_config_t* cfg, hpa_cache_t** out);
hpa_status_t hpa_cache_destroy(hpa_cache_t* c);

/* Device pool base pointers and the byte size of ONE pool (introspection / tests). */
hpa_status_t hpa_cache_pools(hpa_cache_t* c, void** k_pool, void** v_pool, uint64_t* pool_bytes);

/* Allocator state: free pages, pages referenced by at least one table, live sequences. */
/* NEXT-4c fp8 token pool (token_kv_dtype = 1): device pointers to the K and V token pools
 * and the free token pages. Layout (reading A20): pool row prow = ((layer * num_token_pages +
 * page) * H_kv + h) * P + r; rows are grouped 16 at a time into contiguous blocks of
 * [16 x d e4m3 codes | 16 fp32 scales] (16 d + 64 bytes), block index prow / 16; row r of
 * a block means code * scale. K rows (not V) store their 16-byte code chunks XOR-swizzled:
 * logical chunk c of block row r sits at chunk c ^ (r & (d/16 - 1)) (bank-conflict-free
 * register loads of the K fragments in decode). V rows pair up: the codes of block rows 2p and
 * 2p+1 interleave in "pair row" p (2 d bytes: dim 16 m + 8 h + g, g < 8, of row r at byte
 * 32 m + 4 g + 2 h + (r & 1)), whose 16-byte chunks are XOR-swizzled by (2p) & 7 (one 32-bit
 * load = two V^T operand registers). The cache owns the pools; read-only for callers (tests
 * compare them bit-exactly with the oracle's quantizer). HPA_ERR_INVALID_ARG if the cache
 * stores bf16 token pages. */
hpa_status_t hpa_cache_token_pool(hpa_cache_t* c, void** k8, void** v8, int32_t* free_token_pages);

hpa_status_t hpa_cache_stats(hpa_cache_t* c, int32_t* free_pages, int32_t* used_pages,
                             int32_t* live_seqs);

/* Creates an empty sequence; *seq_id receives the lowest free slot. */
hpa_status_t hpa_seq_create(hpa_cache_t* c, int32_t* seq_id);
/* Drops a sequence and decrements the refcount of each of its pages. */
hpa_status_t hpa_seq_release(hpa_cache_t* c, int32_t seq_id);

/* ---------------------------------------------------------------- append
 * The paper's "store ... into the corresponding blocks" op for regular KV
 * (P:L251). Appends n_new[i] token rows to sequence seq_ids[i] for i < n_seqs.
 * k, v: device bf16 [L][sum(n_new)][H_kv][d], rows of the sequences in call
 * order. Each sequence's trailing TOKEN segment is extended (its last page is
 * filled first); if the sequence ends with a LATENT set (or is empty) a new
 * TOKEN segment starts on a fresh page. Allocation is all-or-nothing across the
 * call. seq_ids must be distinct. One kernel launch (+ one H2D metadata copy). */
hpa_status_t hpa_append_kv(hpa_cache_t* c, int32_t n_seqs, const int32_t* seq_ids /*host*/,
                           const int32_t* n_new /*host*/, const void* k, const void* v,
                           hpa_stream_t stream);

/* ---------------------------------------------------------------- latent sets (a3)
 * Installs or replaces a latent-memory page set: the m_rows-row compressed KV of
 * a document/history ("compressed ... KV cache with O(1) length is used as
 * the updatable memory").
 * kv: device bf16 [L][2][m_rows][H_kv][d] (K then V per layer).
 * set_id == -1: append a new LATENT set at the end of the sequence (new segment
 *   on fresh pages); set ids are a per-sequence counter starting at 0.
 * set_id >= 0: replace that set. Same page count ceil(m/P): the set's pages are
 *   rewritten in place; otherwise its pages are freed/allocated and the
 *   sequence's table is spliced (later entries' pos0 shift). Token pages are
 *   never touched (O(1) update). *set_id_out (may be NULL) receives the id. */
hpa_status_t hpa_latent_set_install(hpa_cache_t* c, int32_t seq_id, int32_t set_id,
                                    int32_t m_rows, const void* kv, hpa_stream_t stream,
                                    int32_t* set_id_out);
/* Batched form: n installs (distinct seq_ids), one kernel launch. kv_ptrs[i] is a
 * device pointer to payload i ([L][2][m_rows[i]][H_kv][d]); set_ids_out may be NULL. */
hpa_status_t hpa_latent_set_install_batch(hpa_cache_t* c, int32_t n, const int32_t* seq_ids,
                                          const int32_t* set_ids, const int32_t* m_rows,
                                          const void* const* kv_ptrs, hpa_stream_t stream,
                                          int32_t* set_ids_out);
/* Shared document memory ("KV cache server for storing
 * and retrieving compressed document memories"): appends to dst_seq a new LATENT
 * set that references the physical pages of src_seq's set src_set_id (page
 * refcounts +1; no copy, O(pages) host work, no kernel). A document retrieved by
 * many requests is stored once. Shared pages are read-only: replacing a shared
 * set in any sequence writes fresh pages for that sequence only (copy-on-write);
 * removing / releasing drops that sequence's references. *set_id_out receives
 * dst's new set id. Errors: HPA_ERR_UNKNOWN_SEQ / _UNKNOWN_SET / _SEQ_CAPACITY. */
hpa_status_t hpa_latent_set_share(hpa_cache_t* c, int32_t dst_seq, int32_t src_seq, int32_t src_set_id,
                                  int32_t* set_id_out);
/* Prefix sharing ("regular KV cache including prefix KV cache
 * for user prompts"; reading A21): creates a new sequence (*dst_seq_out) whose
 * logical rows are the first n_prefix_rows rows of src_seq -- the same segments in order,
 * latent sets with their set ids (dst's set counter continues from src's), the segment
 * holding row n_prefix_rows - 1 cut after it. The new sequence references src's physical
 * pages (refcounts +1; O(pages) host work, no kernel, no copy). Appending to a sequence whose
 * partial last page is shared copies that page first (copy-on-write, one page-copy launch
 * before the append's scatter) unless the appender owns the page's claimed rows; replacing a
 * shared latent set writes fresh pages (as hpa_latent_set_share). Either side can be released
 * first. n_prefix_rows = 0 gives an empty sequence. Errors (cache unchanged): INVALID_ARG
 * (n_prefix_rows outside [0, seq_len], or a cut inside a latent set), UNKNOWN_SEQ,
 * SEQ_CAPACITY (no free sequence slot). */
hpa_status_t hpa_seq_fork(hpa_cache_t* c, int32_t src_seq, int32_t n_prefix_rows, int32_t* dst_seq_out);
/* Memory-server staging ("KV cache server for storing
 * and retrieving compressed document memories"): as hpa_latent_set_install_batch,
 * but payload i is in HOST memory (host_ptrs[i], [L][2][m_rows[i]][H_kv][d] bf16;
 * pinned memory gives asynchronous copies). The library copies the payloads to
 * its device staging buffer on an internal copy stream -- so the transfer overlaps
 * work already queued on `stream` (e.g. the previous step's decode) -- makes
 * `stream` wait for the copies, and installs them with one scatter launch. The
 * host buffers may be reused once `stream` has passed the call. */
hpa_status_t hpa_latent_set_install_host(hpa_cache_t* c, int32_t n, const int32_t* seq_ids,
                                         const int32_t* set_ids, const int32_t* m_rows,
                                         const void* const* host_ptrs, hpa_stream_t stream,
                                         int32_t* set_ids_out);
/* Removes a latent set (frees its pages, splices the table). */
hpa_status_t hpa_latent_set_remove(hpa_cache_t* c, int32_t seq_id, int32_t set_id);

/* In-cache compression: how a latent page set is born.
 * GRC computes a document's compression in the same forward pass that reads it
 * ("three tasks in one forward pass"; the meta latent tokens' KV is the
 * compressed cache): the caller appends the document's token KV, then the
 * m meta latent tokens' KV (as tokens; their queries can be prefetched with
 * hpa_prefill), then calls this. The last m_rows rows of the sequence become a new
 * LATENT set (copied into fresh latent pages, one kernel launch) and the
 * n_doc_rows rows just before them are dropped; their token pages are freed.
 * Both ranges must lie in the sequence's trailing TOKEN segment (else
 * HPA_ERR_INVALID_ARG). Needs ceil(m_rows/P) free pages (else
 * HPA_ERR_OUT_OF_PAGES, cache unchanged). *set_id_out (may be NULL) receives the
 * new set id. Memory for the document goes from O(n_doc) to O(m) rows. */
hpa_status_t hpa_seq_compress(hpa_cache_t* c, int32_t seq_id, int32_t n_doc_rows, int32_t m_rows,
                              hpa_stream_t stream, int32_t* set_id_out);
/* hpa_seq_compress for n distinct sequences at once (one launch for all the moves): request i
 * turns the last m_rows[i] rows of its trailing token segment into a new latent set and drops
 * the n_doc_rows[i] rows before them. All arrays are host arrays of n entries; set_ids_out
 * (may be NULL) receives the new set ids. Checked as a whole before any change: an invalid
 * request, a repeated sequence (HPA_ERR_INVALID_ARG), capacity (HPA_ERR_SEQ_CAPACITY) or
 * sum ceil(m_rows[i]/P) > free pages (HPA_ERR_OUT_OF_PAGES) leave the cache unchanged. */
hpa_status_t hpa_seq_compress_batch(hpa_cache_t* c, int32_t n, const int32_t* seq_ids, const int32_t* n_doc_rows,
                                    const int32_t* m_rows, hpa_stream_t stream, int32_t* set_ids_out);

/* ---------------------------------------------------------------- attention (a4-a6)
 * Decode (a4 + a5): for each listed sequence the query is its LAST logical row
 * (its KV must already be appended; reading A8), so every stored row is visible.
 * q: device bf16 [n_seqs][Hq][d]; out: device bf16 [n_seqs][Hq][d].
 * out[b][hq] = softmax(scale * K_log[h] q^T) V_log[h], h = floor(hq / G).
 * softmax_scale <= 0 selects 1/sqrt(d) (reading A5). Split-KV over pages +
 * LSE combine; the split count depends only on the batch's page counts.
 * Cascade (NEXT-2; "prefix KV cache for user prompts"): requests of the batch whose
 * block tables begin with the same run of pages (a prompt prefix shared by hpa_seq_fork,
 * latent sets shared by hpa_latent_set_share and installed first) read that run once per
 * group of up to 32/G requests -- one work unit holds the G query rows of every member --
 * and each request's own remaining pages as usual; all partials merge in the combine. Same
 * result up to fp32 rounding order; bf16 or fp8 token pages, G <= 8, runs of >= 4 chunks that
 * save >= 1/3 of the batch's reads (hpa_set_decode_cascade switches it off). */
hpa_status_t hpa_decode(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                        const void* q, void* out, float softmax_scale, hpa_stream_t stream);

/* Decode step in one launch (a2 + a4 + a5): the per-token "store ... into the
 * corresponding blocks" of regular KV fused with the decode that follows it.
 * Result and cache state are exactly those of
 *   hpa_append_kv(c, n_seqs, seq_ids, {1, ..., 1}, k, v, stream);
 *   hpa_decode(c, layer, n_seqs, seq_ids, q, out, softmax_scale, stream);
 * k, v: device bf16 [L][n_seqs][H_kv][d] (one new row per sequence, every layer);
 * q, out as hpa_decode. The decode kernel writes each sequence's new row into its pool
 * slot itself (no separate scatter launch) when the cache stores bf16 token pages and
 * n_seqs <= 512; otherwise the call runs the two steps above. Argument errors
 * (INVALID_ARG / OUT_OF_PAGES / SEQ_CAPACITY / UNKNOWN_SEQ) leave the cache unchanged;
 * after HPA_ERR_CUDA the row is allocated but its contents are undefined. */
hpa_status_t hpa_append_decode(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                               const void* k, const void* v, const void* q, void* out,
                               float softmax_scale, hpa_stream_t stream);

/* Context-parallel decode (SURVEY §8(f) NEXT-4b: contexts beyond one GPU's pool,
 * pages sharded by row range across GPUs). As hpa_decode, but over the rows this
 * cache holds for each sequence (a shard of the logical sequence; the query is the
 * LAST row of the full sequence, so every stored row is visible) and the result is
 * a mergeable partial: o_part fp32 [n_seqs][Hq][d] (normalised over the shard) and
 * lse_part fp32 [n_seqs][Hq] = log2 sum_j exp(s_j) over the shard (device). */
hpa_status_t hpa_decode_partial(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                                const void* q, float* o_part, float* lse_part, float softmax_scale,
                                hpa_stream_t stream);
/* Merges n_parts partials (device, laid out [n_parts][n_rows][head_dim] and
 * [n_parts][n_rows], e.g. after an all-gather over NVLink) into bf16
 * out [n_rows][head_dim]: out = sum_p 2^(lse_p - LSE) o_p / sum_p 2^(lse_p - LSE).
 * Stateless; runs on the current CUDA device. n_rows = n_seqs * Hq. */
hpa_status_t hpa_merge_partials(int32_t n_parts, int32_t n_rows, int32_t head_dim, const float* o_parts,
                                const float* lse_parts, void* out, hpa_stream_t stream);

/* Chunked prefill (a6): queries of sequence i are its LAST q_lens[i] logical
 * rows (1 <= q_lens[i] <= seq_len; their KV appended first). Query row t sits at
 * logical index i = seq_len - q_len + t and attends keys j <= i (bottom-right
 * causal; reading A1). q, out: device bf16 [sum(q_lens)][Hq][d] (varlen, in call
 * order). tcgen05/TMEM/TMA kernel. */
hpa_status_t hpa_prefill(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                         const int32_t* q_lens /*host*/, const void* q, void* out,
                         float softmax_scale, hpa_stream_t stream);

/* Chunked prefill with the GRC mask-out span (SURVEY §8(f) NEXT-4a; §2,
 * queries of segment ❸ must not see segment ❶ while the meta latent
 * tokens do). As hpa_prefill, plus span (host int32 [n_seqs][3] = lo, hi, q_from):
 * a query at logical index i >= q_from does not attend keys lo <= j < hi. Requires
 * 0 <= lo <= hi <= q_from (so every query still sees itself). */
hpa_status_t hpa_prefill_span(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                              const int32_t* q_lens /*host*/, const int32_t* span /*host*/,
                              const void* q, void* out, float softmax_scale, hpa_stream_t stream);

/* ---------------------------------------------------------------- introspection / tests
 * Host-side sequence summary. */
hpa_status_t hpa_seq_info(hpa_cache_t* c, int32_t seq_id, int32_t* len, int32_t* n_pages,
                          int32_t* n_latent_rows);
/* Gathers the logical K and V of (layer, seq) into device bf16 [H_kv][len][d]
 * (one kernel; bit-exact copy of the stored rows in block-table order; fp8 token rows are
 * written as bf16(fp32(code) * scale), reading A20). */
hpa_status_t hpa_export_logical_kv(hpa_cache_t* c, int32_t layer, int32_t seq_id, void* k_out,
                                   void* v_out, hpa_stream_t stream);
/* Host copy of a sequence's block table: pages[i], pos0[i] (logical index of the
 * entry's row 0 = sum of earlier valid_rows) and meta[i] (bit 15 = latent page,
 * low 15 bits = valid_rows) for i < *n_out <= cap. */
hpa_status_t hpa_export_table(hpa_cache_t* c, int32_t seq_id, int32_t* pages, int32_t* pos0,
                              uint16_t* meta, int32_t cap, int32_t* n_out);
/* Testing / tuning hook: force the decode split count (0 = planner). */
hpa_status_t hpa_set_decode_splits(hpa_cache_t* c, int32_t splits);
/* Cascade decode of shared leading page runs in hpa_decode / hpa_append_decode /
 * hpa_decode_partial: on = 1 (default: the planner's groups, kept when they save >= 1/3 of
 * the batch's reads), 0 = every request reads its whole table, 2 = every group the planner
 * finds regardless of the saving (testing hook). INVALID_ARG on a NULL cache or on outside
 * [0, 2]. */
hpa_status_t hpa_set_decode_cascade(hpa_cache_t* c, int32_t on);
/* Introspection of the last decode plan (persistent kernel): *n_units work units, of which
 * *n_group_units are cascade group units, *splits_max partial slots per request (1 = no
 * combine). Any output pointer may be NULL. INVALID_ARG on a NULL cache. */
hpa_status_t hpa_decode_plan_info(hpa_cache_t* c, int32_t* n_units, int32_t* n_group_units, int32_t* splits_max);
/* Testing / tuning hook for hpa_prefill / hpa_prefill_span: 0 = planner (stream-K shares, or
 * split-KV for the units of an under-filled last wave; see hpa_set_prefill_ctas), 1 = never
 * split, 2..15 = split every unit's key tiles into that many pieces (merged by LSE), 16 = no
 * host work list (one CTA per unit of a grid; each CTA searches the block table for its
 * key-tile range). INVALID_ARG outside [0, 16]. */
hpa_status_t hpa_set_prefill_splits(hpa_cache_t* c, int32_t splits);
/* Testing / tuning hook: prefill CTAs. -1 = default: batches of >= 4 waves run one CTA per
 * planned item (with G % 4 == 0 as 2-CTA clusters sharing K/V by multicast), smaller ones the
 * persistent kernel on every SM with stream-K shares (whole units round-robin, the last
 * partial wave's key tiles cut into equal-time pieces merged by LSE); -2 = one CTA per item,
 * clusters forced whenever G % 4 == 0; -3 = one CTA per item at every batch size (the
 * last wave's units split into equal pieces); 0 = the persistent kernel, one CTA per SM;
 * n > 0 = persistent with at most n CTAs. With forced splits (hpa_set_prefill_splits 2..15)
 * the persistent kernel takes the equal pieces instead of stream-K shares. INVALID_ARG below -3. */
hpa_status_t hpa_set_prefill_ctas(hpa_cache_t* c, int32_t n);
/* Introspection of the last hpa_prefill / hpa_prefill_span plan: *n_ctas prefill CTAs
 * launched, *n_split_units units split into *splits key ranges each (0 / 1 when none), or
 * *n_ctas = 0 when the grid path ran; *cluster_size = 2 when the items ran as 2-CTA clusters
 * sharing K/V tiles by TMA multicast, else 1. Any output pointer may be NULL. */
hpa_status_t hpa_prefill_plan_info(hpa_cache_t* c, int32_t* n_ctas, int32_t* n_split_units, int32_t* splits,
                                   int32_t* cluster_size);
/* Number of kernels this cache has launched so far (bench "gpu_launches"). */
hpa_status_t hpa_launch_count(hpa_cache_t* c, uint64_t* n);
/* Diagnostics only (scripts/trace_*.py): a device buffer of int64 slots into which kernels
 * built with -DHPA_TRACE write per-CTA / per-phase %globaltimer stamps (layout defined by
 * the trace script that reads it); NULL disables. The default build ignores it. The caller
 * owns the buffer and keeps it alive while traced kernels run. INVALID_ARG on a NULL cache. */
hpa_status_t hpa_debug_trace(hpa_cache_t* c, void* device_buf);

#ifdef __cplusplus
}
#endif
#endif /* HPA_H_ */
