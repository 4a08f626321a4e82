// runtime.cpp -- host runtime of the HPA library and the C ABI (include/hpa.h).
//
// Host side of SURVEY §8(a) a1 (page pool + hybrid block table):
//  * PageAllocator: free-list stack + refcounts over NP physical pages shared by
//    all layers ("pre-allocating KV cache ... fixed-size non-continuous blocks",
//    PAPER.md P:L250). Optional seeded shuffle of the free list so physical
//    placement is a random permutation.
//  * Seq: ordered segment list {TOKEN | LATENT(set_id)}; each segment starts on
//    a fresh page and only its last page may be partial (reading A7).
//    Host mirror of the table row: page id, pos0 (= prefix sum of valid rows,
//    the logical index of the entry's row 0) and meta (valid_rows | latent).
//  * Every mutation is checked first and applied only if it can complete
//    (failure atomicity; HPA_ERR_OUT_OF_PAGES = S:L388 backpressure).
//  * Device table updates are queued as (index, value) word writes and shipped
//    through a pinned staging ring with ONE H2D copy per call; the scatter
//    kernel applies them in the same launch that copies the K/V rows.
#include "../../include/hpa.h"
#include "hpa_kernels.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <deque>
#include <functional>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

using namespace hpa;

namespace {

thread_local std::string g_last_error;

hpa_status_t fail(hpa_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

hpa_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(HPA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define HPA_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda,
// so the library also loads on hosts without a driver).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 map over `rows` x `cols` (row-major), box {64, box_rows}, 128-B swizzle.
bool make_map_2d(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef HPA_DEC_MAP3
#define HPA_DEC_MAP3 1  // decode: one 3-D TMA per 16-row K or V tile (else two 2-D boxes)
#endif
#ifndef HPA_DEC_L2PROMO
#define HPA_DEC_L2PROMO 2  // 0 none, 1 128 B, 2 256 B
#endif

// Decode map over a pool [rows][d]: dims {64, rows, d/64} with the d/64 column halves as the
// outer dim (stride 128 B), box {64, 16, d/64}: one TMA fills the same [half][16][64] smem
// layout the two 2-D boxes did.
bool make_map_dec(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const CUtensorMapL2promotion promo = HPA_DEC_L2PROMO == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : HPA_DEC_L2PROMO == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                              : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (!HPA_DEC_MAP3) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, 16};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, 16, cuuint32_t(cols / 64)};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 map over a [rows][cols] workspace: box {32, 128} (128-B rows), 128-B swizzle.
bool make_map_f32(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// 3-D bf16 map over q [tokens][Hq][d]: box {64, 1, box_tok}, 128-B swizzle.
bool make_map_q(CUtensorMap* m, const void* base, uint64_t tokens, uint64_t heads, uint64_t d,
                uint32_t box_tok) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d, heads, tokens};
  cuuint64_t strides[2] = {d * 2, heads * d * 2};
  cuuint32_t box[3] = {64, 1, box_tok};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ allocator
class PageAllocator {
 public:
  void init(int32_t num_pages, uint64_t seed) {
    refcnt_.assign(num_pages, 0);
    high_.assign(num_pages, 0);
    free_.resize(num_pages);
    for (int32_t i = 0; i < num_pages; ++i) free_[i] = num_pages - 1 - i;  // pop_back -> page 0 first
    if (seed != 0) {
      uint64_t st = seed;
      for (int32_t i = num_pages - 1; i > 0; --i) {
        int32_t j = int32_t(splitmix64(st) % uint64_t(i + 1));
        std::swap(free_[i], free_[j]);
      }
    }
  }
  int32_t num_free() const { return int32_t(free_.size()); }
  int32_t num_pages() const { return int32_t(refcnt_.size()); }
  // caller checked num_free() >= n
  void alloc(int32_t n, std::vector<int32_t>& out) {
    for (int32_t i = 0; i < n; ++i) {
      int32_t p = free_.back();
      free_.pop_back();
      refcnt_[p] = 1;
      high_[p] = 0;
      out.push_back(p);
    }
  }
  void release(int32_t p) {
    if (--refcnt_[p] == 0) free_.push_back(p);
  }
  void retain(int32_t p) { ++refcnt_[p]; }
  int32_t refcount(int32_t p) const { return refcnt_[p]; }
  // Token pages shared by forked sequences (NEXT-2, reading A21): rows claimed so far. A sharer
  // may append in place only when its valid rows equal the watermark (rows beyond it are then
  // nobody's); any other sharer copies the page first.
  int32_t high(int32_t p) const { return high_[p]; }
  void set_high(int32_t p, int32_t rows) { high_[p] = rows; }

 private:
  std::vector<int32_t> free_;
  std::vector<int32_t> refcnt_;
  std::vector<int32_t> high_;
};

struct Segment {
  bool latent;
  int32_t set_id;  // -1 for token segments
  int32_t rows;
  std::vector<int32_t> pages;
};

struct Seq {
  bool live = false;
  int32_t next_set = 0;
  std::vector<Segment> segs;
  // host mirror of the table row (rebuilt from segs)
  std::vector<int32_t> pages, pos0, meta;
  // cascade decode (NEXT-2): ph[k] = hash of entries [0, k] (page, meta), pch[k] = 16-row chunks
  // in entries [0, k]; two sequences share their first k entries iff ph[k - 1] agree
  std::vector<uint64_t> ph;
  std::vector<int32_t> pch;
  int32_t len = 0;
  int32_t chunks = 0;  // number of 16-row decode chunks
};

// Pinned host staging ring mirrored by a device ring of the same size: an
// upload copies [off, off+n) host -> device; the region is reused only after
// the event recorded behind the consuming kernel has completed.
class StagingRing {
 public:
  cudaError_t init(size_t cap) {
    cap_ = cap;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&host_), cap, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    return cudaMalloc(reinterpret_cast<void**>(&dev_), cap);
  }
  void destroy() {
    for (auto& f : inflight_) cudaEventDestroy(f.ev);
    for (auto ev : pool_) cudaEventDestroy(ev);
    inflight_.clear();
    pool_.clear();
    if (host_) cudaFreeHost(host_);
    if (dev_) cudaFree(dev_);
    host_ = dev_ = nullptr;
  }
  size_t cap() const { return cap_; }
  static constexpr size_t kNoRoom = ~size_t(0);
  // Returns the offset of a free region of n bytes, or kNoRoom when n exceeds the capacity
  // (callers go through ring_reserve(), which turns that into HPA_ERR_INVALID_ARG).
  size_t reserve(size_t n) {
    n = (n + 255) & ~size_t(255);
    if (n > cap_) return kNoRoom;
    if (head_ + n > cap_) head_ = 0;
    const size_t lo = head_, hi = head_ + n;
    while (!inflight_.empty() && cudaEventQuery(inflight_.front().ev) == cudaSuccess) pop_front();
    for (auto it = inflight_.begin(); it != inflight_.end();) {
      if (it->lo < hi && lo < it->hi) {
        cudaEventSynchronize(it->ev);
        pool_.push_back(it->ev);
        it = inflight_.erase(it);
      } else {
        ++it;
      }
    }
    head_ = hi;
    return lo;
  }
  char* host(size_t off) { return host_ + off; }
  char* dev(size_t off) { return dev_ + off; }
  cudaError_t upload(size_t off, size_t n, cudaStream_t s) {
    return cudaMemcpyAsync(dev_ + off, host_ + off, n, cudaMemcpyHostToDevice, s);
  }
  // The same copy on a side stream `cs`, with `s` waiting for it: the copy engine can move the
  // metadata while `s` still runs earlier kernels (reserve() already guaranteed that no earlier
  // consumer of this region is still reading it).
  cudaError_t upload_side(size_t off, size_t n, cudaStream_t s, cudaStream_t cs, cudaEvent_t ev) {
    cudaError_t e = cudaMemcpyAsync(dev_ + off, host_ + off, n, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
    return e;
  }
  cudaError_t commit(size_t off, size_t n, cudaStream_t s) {
    cudaEvent_t ev;
    if (!pool_.empty()) {
      ev = pool_.back();
      pool_.pop_back();
    } else {
      cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ev, s);
    inflight_.push_back({off, off + ((n + 255) & ~size_t(255)), ev});
    return e;
  }

 private:
  struct Flight {
    size_t lo, hi;
    cudaEvent_t ev;
  };
  void pop_front() {
    pool_.push_back(inflight_.front().ev);
    inflight_.pop_front();
  }
  char* host_ = nullptr;
  char* dev_ = nullptr;
  size_t cap_ = 0, head_ = 0;
  std::deque<Flight> inflight_;
  std::vector<cudaEvent_t> pool_;
};

// Serialises heterogeneous arrays into one staging upload.
struct Blob {
  std::vector<char> bytes;
  template <class T>
  size_t add(const T* p, size_t n) {
    size_t off = (bytes.size() + 15) & ~size_t(15);
    bytes.resize(off + n * sizeof(T));
    if (n) std::memcpy(bytes.data() + off, p, n * sizeof(T));
    return off;
  }
};

}  // namespace

// Split-KV prefill work list (plan_prefill).
struct PfPlan {
  std::vector<int4> work;   // 4 per CTA (PrefillArgs::work)
  std::vector<int4> parts;  // 2 per split unit: {b, y, x, nsplit}, {q_len, q_off, 0, 0}
  int32_t split_max = 1;
  std::vector<int32_t> cta_off;  // persistent launch: items of CTA c = [cta_off[c], cta_off[c+1])
  bool mc2 = false;              // items 2k, 2k+1 form 2-CTA clusters (HPA_PF_MC2)
};

struct hpa_cache {
  hpa_config_t cfg{};
  PageAllocator alloc;
  std::vector<Seq> seqs;
  int32_t live = 0;
  // device
  void* k_pool = nullptr;
  void* v_pool = nullptr;
  uint64_t pool_bytes = 0;
  // NEXT-4c fp8 token pool (token_kv_dtype = 1): codes + per-row scales, its own allocator
  bool fp8 = false;
  PageAllocator alloc8;
  uint8_t* k8_pool = nullptr;  // 16-row blocks [16 x d codes | 16 fp32 scales] (fp8_code_ptr)
  uint8_t* v8_pool = nullptr;
  // allocator of a segment's pages: token pages live in the fp8 pool when fp8
  PageAllocator& pages_of(bool latent) { return (fp8 && !latent) ? alloc8 : alloc; }
  int32_t* arena = nullptr;
  DevTables dt{};
  CUtensorMap tm_k_dec{}, tm_v_dec{}, tm_k_pre{}, tm_v_pre{};
  CUtensorMap tm_opart{};  // fp32 map over pf_o_part (split-KV prefill workspace)
  StagingRing ring;
  std::vector<WordWrite> pending;  // device table writes not yet shipped
  // decode batch cache
  std::vector<int32_t> batch_host;
  int32_t* batch_dev = nullptr;
  int32_t batch_cap = 0;
  // decode partials
  float* o_part = nullptr;
  float* lse_part = nullptr;
  int32_t* counters = nullptr;  // [max_seqs][H_kv] + 2 (persistent ticket counters), zero between calls
  size_t part_elems = 0;
  // persistent decode work list (rebuilt only when the batch or a split count changes)
  std::vector<int32_t> plan_key;
  int4* units_dev = nullptr;
  int32_t* nsplit_dev = nullptr;
  size_t units_cap = 0, nsplit_cap = 0;
  int32_t plan_units = 0, plan_smax = 1;
  int32_t forced_splits = 0;
  // cascade decode (NEXT-2): group-piece records of the current plan (device), on/off switch
  int32_t cascade = 1;  // hpa_set_decode_cascade: 0 off, 1 planner, 2 every shared run
  int32_t* groups_dev = nullptr;
  size_t groups_cap = 0;
  int32_t plan_group_units = 0;
  bool plan_groups = false;
  // split-KV prefill: forced split count (0 = planner) and the partial workspace
  int32_t pf_forced_splits = 0;
  int32_t pf_ctas = -1;          // prefill CTAs: -1 = one per item (default), 0 = persistent on every SM, n > 0 = at most n
  uint64_t table_version = 0;    // bumped by every block-table rebuild
  std::vector<int32_t> pf_key;   // last prefill plan's inputs (version, forced, batch, q_lens, span)
  PfPlan pf_plan;
  bool pf_listed = false;
  float* pf_o_part = nullptr;
  float* pf_lse_part = nullptr;
  size_t pf_part_rows = 0;
  // host-staged installs (NEXT-3): device payload buffer filled on copy_stream
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t upload_done = nullptr;  // staging-ring metadata copies issued on copy_stream
  cudaEvent_t copy_done = nullptr, payload_free = nullptr;
  char* payload_dev = nullptr;
  size_t payload_cap = 0;
  long long* trace = nullptr;  // prefill phase trace (HPA_TRACE builds; set via hpa_debug_trace)
  int num_sms = 148;
  uint64_t launches = 0;

  int64_t idx(int32_t seq, int32_t e) const { return int64_t(seq) * cfg.max_pages_per_seq + e; }
  int64_t off_pos0() const { return int64_t(cfg.max_seqs) * cfg.max_pages_per_seq; }
  int64_t off_meta() const { return 2 * off_pos0(); }
  int64_t off_len() const { return 3 * off_pos0(); }
  int64_t off_nent() const { return off_len() + cfg.max_seqs; }

  PoolGeom geom() const {
    return PoolGeom{k_pool, v_pool, cfg.num_layers, cfg.num_pages, cfg.num_kv_heads, cfg.page_size,
                    cfg.head_dim, __builtin_ctz(uint32_t(cfg.page_size)), k8_pool, v8_pool,
                    fp8 ? cfg.num_token_pages : 0};
  }

  // Recomputes the host mirror of seq `s` from entry `from_entry` on (entries
  // before it are unchanged by the caller's mutation; only a segment's last page
  // may be partial, so the pages before `from_entry` inside its segment are full)
  // and queues device writes for the fields that changed. O(changed entries).
  void rebuild(int32_t s, int32_t from_entry) {
    ++table_version;
    Seq& q = seqs[s];
    const int32_t P = cfg.page_size;
    const int32_t old_n = int32_t(q.pages.size());
    from_entry = std::max(0, std::min(from_entry, old_n));
    int32_t e = 0;
    size_t gi = 0;
    for (; gi < q.segs.size(); ++gi) {  // segment holding from_entry (O(#segments))
      const int32_t np = int32_t(q.segs[gi].pages.size());
      if (e + np > from_entry) break;
      e += np;
    }
    int32_t pos = from_entry < old_n ? q.pos0[from_entry] : q.len;
    int32_t old_tail_chunks = 0;
    for (int32_t k = from_entry; k < old_n; ++k) old_tail_chunks += ((q.meta[k] & kMetaRowsMask) + 15) / 16;
    std::vector<int32_t> tp, tpos, tmeta;
    int32_t new_tail_chunks = 0;
    int32_t pi = from_entry - e;  // page index inside segment gi
    for (; gi < q.segs.size(); ++gi, pi = 0) {
      const Segment& g = q.segs[gi];
      int32_t left = g.rows - pi * P;
      for (size_t k = size_t(pi); k < g.pages.size(); ++k) {
        const int32_t take = std::min(P, left);
        tp.push_back(g.pages[k]);
        tpos.push_back(pos);
        tmeta.push_back(take | (g.latent ? kMetaLatent : 0));
        new_tail_chunks += (take + 15) / 16;
        pos += take;
        left -= take;
      }
    }
    const int32_t n = from_entry + int32_t(tp.size());
    for (int32_t k = from_entry; k < n; ++k) {  // only the fields that changed
      const int32_t t = k - from_entry;
      const bool fresh = k >= old_n;
      if (fresh || q.pages[k] != tp[t]) pending.push_back({int32_t(idx(s, k)), tp[t]});
      if (fresh || q.pos0[k] != tpos[t]) pending.push_back({int32_t(off_pos0() + idx(s, k)), tpos[t]});
      if (fresh || q.meta[k] != tmeta[t]) pending.push_back({int32_t(off_meta() + idx(s, k)), tmeta[t]});
    }
    if (q.len != pos) pending.push_back({int32_t(off_len() + s), pos});
    if (old_n != n) pending.push_back({int32_t(off_nent() + s), n});
    q.pages.resize(from_entry);
    q.pos0.resize(from_entry);
    q.meta.resize(from_entry);
    q.pages.insert(q.pages.end(), tp.begin(), tp.end());
    q.pos0.insert(q.pos0.end(), tpos.begin(), tpos.end());
    q.meta.insert(q.meta.end(), tmeta.begin(), tmeta.end());
    q.len = pos;
    q.chunks += new_tail_chunks - old_tail_chunks;
    q.ph.resize(size_t(from_entry));
    q.pch.resize(size_t(from_entry));
    for (int32_t k = from_entry; k < n; ++k) {
      uint64_t h = (k ? q.ph[size_t(k - 1)] : 0x9e3779b97f4a7c15ull) ^
                   (uint64_t(uint32_t(q.pages[size_t(k)])) << 20 ^ uint64_t(uint32_t(q.meta[size_t(k)])));
      h ^= h >> 33;  // splitmix64 finalizer
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 33;
      h *= 0xc4ceb9fe1a85ec53ull;
      h ^= h >> 33;
      q.ph.push_back(h);
      q.pch.push_back((k ? q.pch[size_t(k - 1)] : 0) + ((q.meta[size_t(k)] & kMetaRowsMask) + 15) / 16);
    }
  }
};

namespace {

hpa_status_t check_seq(hpa_cache_t* c, int32_t s) {
  if (s < 0 || s >= c->cfg.max_seqs || !c->seqs[s].live)
    return fail(HPA_ERR_UNKNOWN_SEQ, "unknown sequence %d", s);
  return HPA_OK;
}

int32_t seq_entries(const Seq& q) { return int32_t(q.pages.size()); }

// A staging-ring region of n bytes, or INVALID_ARG when one call's upload exceeds the ring.
hpa_status_t ring_reserve(hpa_cache_t* c, size_t n, size_t* off) {
  *off = c->ring.reserve(n);
  if (*off == StagingRing::kNoRoom)
    return fail(HPA_ERR_INVALID_ARG, "staging upload of %zu bytes exceeds the ring capacity %zu", n, c->ring.cap());
  return HPA_OK;
}

// Ships pending word writes (+ optional scatter records/slots) in one upload and
// one scatter launch on `s`.
hpa_status_t ship(hpa_cache_t* c, cudaStream_t s, const std::vector<ScatterRecord>& recs,
                  const std::vector<int32_t>& slots, int64_t max_rows, const PoolGeom* geom = nullptr) {
  const PoolGeom gm = geom ? *geom : c->geom();
  if (c->pending.empty() && recs.empty()) return HPA_OK;
  // The scatter kernel applies words in parallel, so each index may appear at
  // most once: keep the LAST queued write per index (program order).
  if (c->pending.size() > 1) {
    std::stable_sort(c->pending.begin(), c->pending.end(),
                     [](const WordWrite& x, const WordWrite& y) { return x.idx < y.idx; });
    size_t w = 0;
    for (size_t r = 0; r < c->pending.size(); ++r) {
      if (w > 0 && c->pending[w - 1].idx == c->pending[r].idx) c->pending[w - 1] = c->pending[r];
      else c->pending[w++] = c->pending[r];
    }
    c->pending.resize(w);
  }
  const size_t n_ints = 2 * c->pending.size() + slots.size();
  if (recs.size() <= 1 && n_ints <= size_t(kInlineInts)) {
    // metadata as kernel parameters (no H2D copy); the launch copies the whole parameter
    // block, so the common small case uses the small variant
    auto fill_launch = [&](auto& m) -> cudaError_t {
      m.n_words = int32_t(c->pending.size());
      m.n_slots = int32_t(slots.size());
      m.has_rec = recs.empty() ? 0 : 1;
      m.pad = 0;
      if (!recs.empty()) m.rec = recs[0];
      for (size_t i = 0; i < c->pending.size(); ++i) {
        m.data[2 * i] = c->pending[i].idx;
        m.data[2 * i + 1] = c->pending[i].val;
      }
      if (!slots.empty()) std::memcpy(m.data + 2 * c->pending.size(), slots.data(), slots.size() * 4);
      return launch_scatter_inline(gm, c->arena, m, max_rows, s);
    };
    if (n_ints <= size_t(kInlineIntsSmall)) {
      InlineMetaSmall m;
      HPA_CUDA(fill_launch(m));
    } else {
      InlineMeta m;
      HPA_CUDA(fill_launch(m));
    }
    c->launches += 1;
    c->pending.clear();
    return HPA_OK;
  }
  Blob b;
  const size_t o_words = b.add(c->pending.data(), c->pending.size());
  const size_t o_recs = b.add(recs.data(), recs.size());
  const size_t o_slots = b.add(slots.data(), slots.size());
  size_t off;
  if (hpa_status_t st = ring_reserve(c, b.bytes.size(), &off)) return st;
  std::memcpy(c->ring.host(off), b.bytes.data(), b.bytes.size());
  HPA_CUDA(c->ring.upload_side(off, b.bytes.size(), s, c->copy_stream, c->upload_done));
  char* d = c->ring.dev(off);
  HPA_CUDA(launch_scatter(gm, c->arena, reinterpret_cast<const WordWrite*>(d + o_words),
                          int32_t(c->pending.size()), reinterpret_cast<const ScatterRecord*>(d + o_recs),
                          int32_t(recs.size()), reinterpret_cast<const int32_t*>(d + o_slots), max_rows, s));
  c->launches += 1;
  HPA_CUDA(c->ring.commit(off, b.bytes.size(), s));
  c->pending.clear();
  return HPA_OK;
}

// Device copy of the batch's seq rows (re-uploaded only when the list changes).
hpa_status_t upload_batch(hpa_cache_t* c, int32_t n, const int32_t* seq_ids, cudaStream_t s) {
  if (int32_t(c->batch_host.size()) == n && std::equal(seq_ids, seq_ids + n, c->batch_host.begin()))
    return HPA_OK;
  if (n > c->batch_cap) {
    if (c->batch_dev) cudaFree(c->batch_dev);
    c->batch_cap = std::max(n, 1024);
    HPA_CUDA(cudaMalloc(&c->batch_dev, size_t(c->batch_cap) * 4));
  }
  size_t off;
  if (hpa_status_t st = ring_reserve(c, size_t(n) * 4, &off)) return st;
  std::memcpy(c->ring.host(off), seq_ids, size_t(n) * 4);
  HPA_CUDA(cudaMemcpyAsync(c->batch_dev, c->ring.host(off), size_t(n) * 4, cudaMemcpyHostToDevice, s));
  HPA_CUDA(c->ring.commit(off, size_t(n) * 4, s));
  c->batch_host.assign(seq_ids, seq_ids + n);
  return HPA_OK;
}

// Split planner: splits depend only on the batch's table sizes (never on
// physical placement). Minimises the wave-quantised time of equal-length
// units plus a small per-split cost.
int32_t plan_splits(hpa_cache_t* c, int32_t n, int32_t max_entries, int32_t max_chunks) {
  if (c->forced_splits > 0) return std::max(1, std::min(c->forced_splits, std::max(1, max_entries)));
  const int64_t units = int64_t(n) * c->cfg.num_kv_heads;
  const int64_t slots = int64_t(c->num_sms) * decode_ctas_per_sm(c->cfg.head_dim, 1);
  int32_t best = 1;
  double best_cost = 1e30;
  const int32_t smax = std::max(1, std::min<int32_t>(64, std::max(1, max_entries)));
  for (int32_t S = 1; S <= smax; ++S) {
    if (max_chunks / S < 8 && S > 1) break;  // keep >= 8 chunks (128 rows) per split
    const int64_t ctas = units * S;
    const double waves = std::ceil(double(ctas) / double(slots));
    const double cost = waves * (double(max_chunks) / S + 6.0) + (S > 1 ? 2.0 : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = S;
    }
  }
  return best;
}

// Persistent decode: per-request split counts S_b so that every (request, kv-head, split)
// work unit covers about the same number of 16-row chunks (ragged batches stay balanced),
// chosen by a makespan estimate over the resident CTA slots:
//   cost = total / slots + max_unit / 2 + combine,   total = H_kv * sum_b (chunks_b + c0 * S_b).
// The units go to the kernel longest first (it fetches them dynamically), so the tail is
// about half a unit.  Returns S_max and fills splits[] (one per request).
int32_t plan_splits_core(const hpa_cache_t* c, int32_t n, std::vector<int32_t> ch, std::vector<int32_t> ne,
                         int32_t slots, std::vector<int32_t>& splits) {
  splits.assign(n, 1);
  int32_t cmax = 0;
  for (int32_t i = 0; i < n; ++i) {
    ch[i] = std::max(1, ch[i]);
    ne[i] = std::max(1, ne[i]);
    cmax = std::max(cmax, ch[i]);
  }
  if (c->forced_splits > 0) {
    int32_t smax = 1;
    for (int32_t i = 0; i < n; ++i) {
      splits[i] = std::min(std::min(c->forced_splits, 64), ne[i]);
      smax = std::max(smax, splits[i]);
    }
    return smax;
  }
  // per-unit cost in chunks (Q load, end-of-unit consumer barrier and merge, partial write) and
  // the combine's fixed cost; HPA_PLAN_C0 / HPA_PLAN_COMBINE override them (tuning knobs, read
  // once). c0 measured at configs[1] (profiles/r2_decode_plan_c0.log): bf16 0.5 (3.0 gave the
  // fused step at most 1 % on one box, none in the bench, and cost 7 % at P = 64); an fp8 chunk
  // costs ~0.6 of a bf16 one, so the per-unit time is several chunks there: 5.0 (S = 4 instead
  // of 10 at configs[1]: 170 -> 152.6 us).
  static const double c0_env = std::getenv("HPA_PLAN_C0") ? std::atof(std::getenv("HPA_PLAN_C0")) : -1.0;
  // round 2, with the 10-stage ring: bf16 P = 16 runs the configs[1] step 1.3 % and the ragged
  // batch 1 % faster at 3.0 (S = 5) than at 0.5 (S = 10), while P = 64 runs 3.5 % slower there
  // (profiles/r2_decode_plan_c0_ring10.log): 3.0 for pages of <= 32 rows, 0.5 above
  const double c0 = c0_env >= 0.0 ? c0_env : (c->fp8 ? 5.0 : (c->cfg.page_size <= 32 ? 3.0 : 0.5));
  static const double k_comb = std::getenv("HPA_PLAN_COMBINE") ? std::atof(std::getenv("HPA_PLAN_COMBINE")) : 4.0;
  const double hkv = c->cfg.num_kv_heads;
  const double part_chunks = double(c->cfg.num_q_heads) * (c->cfg.head_dim + 1) * 8 / 8192.0;
  double best_cost = 1e300;
  int32_t best_E = cmax;
  int32_t prevE = -1;
  for (int32_t sref = 1; sref <= 64; ++sref) {
    const int32_t E = (cmax + sref - 1) / sref;        // chunk budget per unit
    if (E == prevE) continue;
    if (sref > 1 && E < 4) break;
    prevE = E;
    double total = 0, maxu = 0;
    int32_t smax = 1;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t sb = std::min(std::min(64, ne[i]), std::max(1, (ch[i] + E - 1) / E));
      total += ch[i] + c0 * sb;
      maxu = std::max(maxu, double(ch[i]) / sb);
      smax = std::max(smax, sb);
    }
    total *= hkv;
    double cost = total / slots + 0.5 * (maxu + c0);
    if (smax > 1) cost += k_comb + n * smax * part_chunks / slots;  // combine launch + partial traffic
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best_E = E;
    }
  }
  int32_t smax = 1;
  for (int32_t i = 0; i < n; ++i) {
    splits[i] = std::min(std::min(64, ne[i]), std::max(1, (ch[i] + best_E - 1) / best_E));
    smax = std::max(smax, splits[i]);
  }
  return smax;
}

int32_t plan_request_splits(const hpa_cache_t* c, int32_t n, const int32_t* seq_ids, int32_t slots,
                            std::vector<int32_t>& splits) {
  std::vector<int32_t> ch(n), ne(n);
  for (int32_t i = 0; i < n; ++i) {
    ch[i] = c->seqs[seq_ids[i]].chunks;
    ne[i] = seq_entries(c->seqs[seq_ids[i]]);
  }
  return plan_splits_core(c, n, std::move(ch), std::move(ne), slots, splits);
}

// ---- cascade decode (NEXT-2: "prefix KV cache for user prompts"; shared latent sets)
// Requests of one batch whose block tables start with the same entries (a forked prompt
// prefix, shared latent sets installed first) read that run once per group of up to 32 / G
// members: one group unit per (group, KV head, piece) holds the G query rows of every member
// and writes each member a partial (O, LSE) of the run; the member's own entries [r, n) are
// split as usual and the combine merges all partials (same LSE algebra as the split-KV a5).
struct CGroup {
  int32_t r = 0;    // shared run: entries [0, r)
  int32_t rch = 0;  // its 16-row chunks
  std::vector<int32_t> mem;  // batch indices; mem[0] is the representative
  int32_t pieces = 1;
};

// longest common prefix (in entries) of two sequences' tables, from the prefix hashes
int32_t lcp_entries(const Seq& a, const Seq& b) {
  int32_t lo = 0, hi = int32_t(std::min(a.ph.size(), b.ph.size()));
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) / 2;
    if (a.ph[size_t(mid - 1)] == b.ph[size_t(mid - 1)]) lo = mid;
    else hi = mid - 1;
  }
  while (lo > 0 && (a.pages[size_t(lo - 1)] != b.pages[size_t(lo - 1)] || a.meta[size_t(lo - 1)] != b.meta[size_t(lo - 1)]))
    --lo;  // (a 64-bit hash collision: never seen, kept exact anyway)
  return lo;
}

constexpr int32_t kCascadeMinChunks = 4;  // shorter shared runs are decoded per request

std::vector<CGroup> find_cascade_groups(const hpa_cache_t* c, int32_t n, const int32_t* seq_ids) {
  std::vector<CGroup> out;
  const int32_t G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  if (!c->cascade || G > 8 || !decode_persistent()) return out;
  std::vector<std::pair<int32_t, int32_t>> fp;  // (first page, batch index)
  fp.reserve(size_t(n));
  for (int32_t i = 0; i < n; ++i) {
    const Seq& q = c->seqs[seq_ids[i]];
    if (!q.pages.empty()) fp.emplace_back(q.pages[0], i);
  }
  std::sort(fp.begin(), fp.end());
  const int32_t cap = std::min(kGroupMax, 32 / G);  // members per group unit (32 query rows)
  for (size_t a = 0; a < fp.size();) {
    size_t b = a;
    while (b < fp.size() && fp[b].first == fp[a].first) ++b;
    if (b - a >= 2) {
      // Members ordered so that those sharing long prefixes are adjacent: by their common
      // prefix with the bucket's longest table (desc), then by the entry where they leave it
      // (in a fork tree: the fork point, then the branch). Any order is correct -- members j..k
      // share min(adjacent LCPs) entries -- this one makes the shared runs long.
      std::vector<int32_t> mem;
      for (size_t k = a; k < b; ++k) mem.push_back(fp[k].second);
      auto lcp_of = [&](int32_t x, int32_t y) { return lcp_entries(c->seqs[seq_ids[x]], c->seqs[seq_ids[y]]); };
      int32_t ref = mem[0];
      for (int32_t x : mem)
        if (c->seqs[seq_ids[x]].pages.size() > c->seqs[seq_ids[ref]].pages.size()) ref = x;
      struct Key {
        int32_t lcp, page, meta, idx;
      };
      std::vector<Key> keys;
      keys.reserve(mem.size());
      for (int32_t x : mem) {
        const Seq& X = c->seqs[seq_ids[x]];
        const int32_t l = x == ref ? int32_t(X.pages.size()) : lcp_of(ref, x);
        const bool more = l < int32_t(X.pages.size());
        keys.push_back({l, more ? X.pages[size_t(l)] : -1, more ? X.meta[size_t(l)] : -1, x});
      }
      std::sort(keys.begin(), keys.end(), [](const Key& x, const Key& y) {
        if (x.lcp != y.lcp) return x.lcp > y.lcp;
        if (x.page != y.page) return x.page < y.page;
        if (x.meta != y.meta) return x.meta < y.meta;
        return x.idx < y.idx;
      });
      for (size_t k = 0; k < keys.size(); ++k) mem[k] = keys[k].idx;
      const size_t m = mem.size();
      std::vector<int32_t> adj(m - 1);
      for (size_t k = 0; k + 1 < m; ++k) adj[k] = lcp_of(mem[k], mem[k + 1]);
      // chunks in the first r entries of member k (which has at least r entries)
      auto chunks_of = [&](int32_t r, size_t k) { return r > 0 ? c->seqs[seq_ids[mem[k]]].pch[size_t(r - 1)] : 0; };
      // the threshold t (entries) that saves the most chunk reads: runs of adjacent LCP >= t,
      // each cut into groups of <= cap members sharing the run's minimum LCP
      auto plan_t = [&](int32_t t, std::vector<CGroup>* outg) {
        int64_t saved = 0;
        size_t j = 0;
        while (j + 1 < m) {
          if (adj[j] < t) {
            ++j;
            continue;
          }
          size_t k = j;
          while (k + 1 < m && adj[k] >= t) ++k;  // members j..k share >= t entries
          for (size_t g0 = j; g0 <= k; g0 += size_t(cap)) {
            const size_t g1 = std::min(k, g0 + size_t(cap) - 1);
            if (g1 == g0) break;  // a lone member reads its run itself
            int32_t r = adj[g0];
            for (size_t q = g0; q < g1; ++q) r = std::min(r, adj[q]);
            const int32_t rch = chunks_of(r, g0);
            if (rch < kCascadeMinChunks) continue;
            saved += int64_t(g1 - g0) * rch;
            if (outg) {
              CGroup g;
              g.r = r;
              g.rch = rch;
              g.mem.assign(mem.begin() + int64_t(g0), mem.begin() + int64_t(g1) + 1);
              std::sort(g.mem.begin(), g.mem.end());
              outg->push_back(std::move(g));
            }
          }
          j = k + 1;
        }
        return saved;
      };
      int64_t best = 0;
      int32_t best_t = -1;
      std::vector<int32_t> ts;
      for (size_t k = 0; k + 1 < m; ++k)
        if (adj[k] > 0 && chunks_of(adj[k], k) >= kCascadeMinChunks) ts.push_back(adj[k]);
      std::sort(ts.begin(), ts.end());
      ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
      if (ts.size() > 16) {  // at most 16 candidate thresholds (each costs a pass over the bucket)
        std::vector<int32_t> sub;
        for (size_t k = 0; k < 16; ++k) sub.push_back(ts[k * (ts.size() - 1) / 15]);
        sub.erase(std::unique(sub.begin(), sub.end()), sub.end());
        ts.swap(sub);
      }
      for (int32_t t : ts) {
        const int64_t sv = plan_t(t, nullptr);
        if (sv > best) {
          best = sv;
          best_t = t;
        }
      }
      if (best_t > 0) plan_t(best_t, &out);
    }
    a = b;
  }
  // worth it only when the reads saved are a real share of the batch's: a group chunk costs
  // ~1.75 normal chunks of CTA time (every consumer works through it), and short shared runs
  // are L2-resident for the plain path anyway (8 latent sets shared by 64 requests, 17 % of
  // the reads: 7 % slower with cascade; a 2K prompt + 4K own, 29 %: 3 % slower; a 1K prompt +
  // 1K own, 44 %: 1.12x faster; profiles/r2_cascade_cases.log)
  int64_t saved = 0, total = 0;
  for (const CGroup& g : out) saved += int64_t(g.mem.size() - 1) * g.rch;
  for (int32_t i = 0; i < n; ++i) total += c->seqs[seq_ids[i]].chunks;
  static const double min_saved = std::getenv("HPA_CASC_MIN_SAVED") ? std::atof(std::getenv("HPA_CASC_MIN_SAVED")) : 1.0 / 3;
  static const bool trace = std::getenv("HPA_CASC_TRACE") != nullptr;
  if (trace && !out.empty())
    std::fprintf(stderr, "cascade: %zu groups, saved %lld of %lld chunk reads (min %.3f)\n", out.size(),
                 (long long)saved, (long long)total, min_saved);
  if (c->cascade < 2 && double(saved) < min_saved * double(total)) out.clear();
  return out;
}

// Split-KV prefill plan. The prefill kernel owns all 512 TMEM columns, so one CTA runs per SM
// and U units (two 128-row query tiles sharing K/V) take ceil(U / W) waves of about equal
// length: B = 1 of configs[2] is 256 units on 148 SMs, 1.73 waves of work in 2 waves. The
// plan keeps the L2-friendly dispatch order and splits the units dispatched last -- those of
// the under-filled last wave, optionally one more wave's worth -- into s key ranges whose
// pieces fill the SMs; each split unit's pieces are merged by LSE (prefill_combine_kernel).
// Chosen by a greedy list-scheduling simulation of the hardware's in-order CTA dispatch, in
// key tiles: unit = tiles(i_max) + o, piece = tiles / s + o', merge = c_m + partial bytes /
// bandwidth (o, o' measured per CTA).

// Greedy in-order dispatch onto W SMs (min-heap of the times the SMs become free): `items`
// are appended to the state `heap` (W entries); returns the makespan of the state.
double list_schedule(std::vector<double>& heap, const double* items, size_t n) {
  auto gt = std::greater<double>();
  for (size_t k = 0; k < n; ++k) {
    std::pop_heap(heap.begin(), heap.end(), gt);
    heap.back() += items[k];
    std::push_heap(heap.begin(), heap.end(), gt);
  }
  return *std::max_element(heap.begin(), heap.end());
}

// Stream-K tail for the persistent prefill kernel (the default for batches under 4 waves:
// configs[2] B = 1, 256 units on 148 SMs, 1202 vs 1174 TFLOP/s for the list-scheduled split
// tail of one CTA per item; profiles/r2_prefill_streamk_ab.log). The first floor(nU / W) * W units (in
// dispatch order) go round-robin to the W CTAs, whole -- as the hardware would dispatch them,
// so the CTAs running at one time work on neighbouring units and share K/V tiles in L2. The
// remaining nU mod W units are cut, in order, into W consecutive shares that fill every CTA
// to the same estimated end time (tiles + per-item cost; water-filling over the CTAs' loads
// after the whole units), so all CTAs finish together; a unit straddling share boundaries
// becomes pieces merged by LSE (at most 15; none shorter than kMin tiles).
// unit(k) -> (b, y, x, n, skip_a, n_skip).
template <class UnitFn>
bool plan_prefill_streamk(const hpa_cache_t* c, const int32_t* seq_ids, const int32_t* q_lens, const int32_t* q_off,
                          int64_t nU, int32_t W, double o_item, double o_piece, UnitFn unit, PfPlan& plan) {
  const int64_t R = nU % W, whole = nU - R;
  std::vector<double> load(size_t(W), 0.0);
  for (int64_t k = 0; k < whole; ++k) load[size_t(k % W)] += std::get<3>(unit(k)) + o_item;
  int64_t Tt = 0;  // tail tiles
  for (int64_t k = whole; k < nU; ++k) Tt += std::get<3>(unit(k));
  const double per = o_piece * (1.0 + double(R) / W);  // piece cost per CTA (~1 + R/W pieces each)
  // end time E: sum_c max(0, E - load_c - per) = Tt (bisection)
  double lo = *std::min_element(load.begin(), load.end()),
         hi = *std::max_element(load.begin(), load.end()) + double(Tt) + per;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    double f = 0;
    for (double l : load) f += std::max(0.0, mid - l - per);
    (f < double(Tt) ? lo : hi) = mid;
  }
  const double E = hi;
  // a tail unit longer than 15 shares would need more pieces than the item format holds: the
  // caller falls back to the list-scheduled plan (equal pieces of the last wave's units)
  {
    const double share = double(Tt) / W;
    for (int64_t k = whole; k < nU; ++k)
      if (double(std::get<3>(unit(k))) > 14.0 * std::max(1.0, share)) return false;
  }
  // shortest piece: 12 tiles, or the tail's per-CTA share when that is smaller (small batches)
  const int32_t kMin = int32_t(std::max<int64_t>(4, std::min<int64_t>(12, Tt / W)));
  struct Item { int32_t cta; int4 w0, w1, wq, wn; };
  std::vector<Item> items;
  plan.work.clear();
  plan.parts.clear();
  plan.mc2 = false;
  plan.split_max = 1;
  auto wq_of = [&](int32_t b) { return make_int4(seq_ids[b], q_lens[b], q_off[b], c->seqs[seq_ids[b]].len); };
  auto wn_of = [&](int32_t b) { return make_int4(int32_t(c->seqs[seq_ids[b]].pages.size()), 0, 0, 0); };
  for (int64_t k = 0; k < whole; ++k) {
    const auto [b, y, x, n, skip_a, n_skip] = unit(k);
    items.push_back({int32_t(k % W), make_int4(b, y, x, 1 << 4), make_int4(0, n, skip_a, n_skip), wq_of(b), wn_of(b)});
  }
  // CTA c takes tail tiles [bnd[c], bnd[c+1]) of the concatenated tail units: its room up to
  // E minus about one piece's cost, scaled so the shares cover the tail exactly
  std::vector<int64_t> bnd(size_t(W) + 1, 0);
  {
    std::vector<double> room(static_cast<size_t>(W));
    double sum = 0;
    for (int32_t i = 0; i < W; ++i) sum += room[size_t(i)] = std::max(0.0, E - load[size_t(i)] - per);
    double acc = 0;
    for (int32_t i = 0; i < W; ++i) {
      acc += room[size_t(i)];
      bnd[size_t(i) + 1] = sum > 0 ? int64_t(std::llround(acc / sum * double(Tt))) : Tt;
    }
    bnd[size_t(W)] = Tt;
  }
  int64_t g = 0;
  std::vector<int4> pcs;  // {cta, first tile, tiles, -}
  for (int64_t k = whole; k < nU; ++k) {
    const auto [b, y, x, n, skip_a, n_skip] = unit(k);
    const int64_t u0 = g, u1 = g + n;
    g = u1;
    pcs.clear();
    int32_t ci = int32_t(std::upper_bound(bnd.begin(), bnd.end(), u0) - bnd.begin()) - 1;
    for (; ci < W && bnd[size_t(ci)] < u1; ++ci) {
      const int64_t lo = std::max(u0, bnd[size_t(ci)]), hi = std::min(u1, bnd[size_t(ci) + 1]);
      if (hi > lo) pcs.push_back(make_int4(ci, int32_t(lo - u0), int32_t(hi - lo), 0));
    }
    if (pcs.empty())  // a unit without key tiles (not produced by the planner today) still writes its rows
      pcs.push_back(make_int4(std::min(std::max(ci, 0), W - 1), 0, n, 0));
    // slivers shorter than kMin join their neighbour (at most 15 pieces)
    for (size_t i = 0; pcs.size() > 1 && i < pcs.size();) {
      if (pcs[i].z < kMin || pcs.size() > 15) {
        if (i > 0) {
          pcs[i - 1].z += pcs[i].z;
        } else {
          pcs[1].y = pcs[0].y;
          pcs[1].z += pcs[0].z;
        }
        pcs.erase(pcs.begin() + std::ptrdiff_t(i));
      } else {
        ++i;
      }
    }
    const int32_t ns = int32_t(pcs.size());
    const int32_t part = int32_t(plan.parts.size() / 2);
    if (ns > 1) {
      plan.parts.push_back(make_int4(b, y, x, ns));
      plan.parts.push_back(make_int4(q_lens[b], q_off[b], 0, 0));
      plan.split_max = std::max(plan.split_max, ns);
    }
    for (int32_t p = 0; p < ns; ++p)
      items.push_back({pcs[size_t(p)].x, make_int4(b, y, x, ns > 1 ? (p | (ns << 4) | (part << 8)) : (1 << 4)),
                       make_int4(pcs[size_t(p)].y, pcs[size_t(p)].z, skip_a, n_skip), wq_of(b), wn_of(b)});
  }
  // each CTA's list: its whole units in dispatch order, then its tail pieces
  std::stable_sort(items.begin(), items.end(), [](const Item& u, const Item& v) { return u.cta < v.cta; });
  std::vector<int32_t> count(size_t(W), 0);
  for (const Item& it : items) {
    ++count[size_t(it.cta)];
    plan.work.insert(plan.work.end(), {it.w0, it.w1, it.wq, it.wn});
  }
  int32_t n_ctas = W;
  while (n_ctas > 1 && count[size_t(n_ctas) - 1] == 0) --n_ctas;
  plan.cta_off.assign(size_t(n_ctas) + 1, 0);
  for (int32_t i = 0; i < n_ctas; ++i) plan.cta_off[size_t(i) + 1] = plan.cta_off[size_t(i)] + count[size_t(i)];
  return true;
}

// Key-tile iterations of every unit, computed here from the host mirror of the table exactly
// as the kernel would (so the kernel needs no table search before its pipeline starts):
// n = slot(i_max) / 128 + 1 tiles, minus the tiles wholly inside the GRC span when every
// query row of the unit is a span row. Returns false when the legacy grid (no work list) is
// used (HPA_PF1 / HPA_SM16 builds, or hpa_set_prefill_splits(c, 16)).
bool plan_prefill(const hpa_cache_t* c, int32_t n_seqs, const int32_t* seq_ids, const int32_t* q_lens,
                  const int32_t* q_off, const int32_t* span, PfPlan& plan) {
  const int32_t forced = c->pf_forced_splits;
  if (forced == 16 || !prefill_split_supported()) return false;
  // persistent launch (one CTA per SM looping over its items): selected with
  // hpa_set_prefill_ctas(c, n >= 0) (a positive value caps the CTA count), and by default for
  // batches of fewer than 4 waves (stream-K shares, below); larger batches run one CTA per item
  // (2-3 % faster there, with 2-CTA clusters)
  const int32_t max_ctas = c->pf_ctas > 0 ? std::min(c->pf_ctas, c->num_sms) : c->num_sms;
  // per-item fixed cost in key tiles: a launched CTA (setup, pipeline fill, epilogue, CTA
  // switch; scripts/trace_prefill_ctas.py) vs a persistent item (Q reload bubble and the
  // epilogue, partly overlapped by the other slot's work)
  static const double o_item_p = std::getenv("HPA_PF_OVH_P") ? std::atof(std::getenv("HPA_PF_OVH_P")) : 1.5;
  static const double o_piece_p = o_item_p + 1.5;
  const int32_t Hq = c->cfg.num_q_heads, Hkv = c->cfg.num_kv_heads, G = Hq / Hkv;
  const int32_t lp = __builtin_ctz(uint32_t(c->cfg.page_size));
  const int32_t Y = (G & 1) == 0 ? Hkv * (G / 2) : Hq;
  struct U { int32_t b, x, n, skip_a, n_skip; };
  std::vector<U> rows;  // one per (sequence, row-tile index); the Y head units share it
  for (int32_t i = 0; i < n_seqs; ++i) {
    const Seq& q = c->seqs[seq_ids[i]];
    const int32_t ql = q_lens[i], mt = (ql + 127) / 128, X = (G & 1) == 0 ? mt : (mt + 1) / 2;
    const int32_t ne = int32_t(q.pages.size());
    auto slot_of = [&](int32_t x) {
      const int32_t e = std::max<int32_t>(
          0, int32_t(std::upper_bound(q.pos0.begin(), q.pos0.begin() + ne, x) - q.pos0.begin()) - 1);
      return (int64_t(e) << lp) + (x - q.pos0[size_t(e)]);
    };
    const int32_t q_base = q.len - ql;
    for (int32_t x = 0; x < X; ++x) {
      const int32_t first_mt = (G & 1) == 0 ? x : 2 * x;
      const int32_t last_mt = (G & 1) == 0 ? x : std::min(2 * x + 1, mt - 1);
      const int32_t i_min = q_base + first_mt * 128;
      const int32_t i_max = q_base + std::min(ql, (last_mt + 1) * 128) - 1;
      const int32_t total = int32_t(slot_of(i_max) / 128 + 1);
      int32_t skip_a = 0, skip_b = 0;
      if (span && i_min >= span[3 * i + 2] && span[3 * i + 1] > span[3 * i]) {
        skip_a = int32_t((slot_of(span[3 * i]) + 127) / 128);
        skip_b = int32_t((slot_of(span[3 * i + 1] - 1) + 1) / 128);
        if (skip_b < skip_a) skip_b = skip_a;
      }
      rows.push_back({i, x, total - (skip_b - skip_a), skip_a, skip_b - skip_a});
    }
  }
  // Dispatch order (the hardware starts CTAs in order): sequence, then head index y, then row
  // tile x fastest -- the CTAs running at the same time then share K/V tiles in L2 (all row
  // tiles of one KV head read the same keys). Ordering units by length instead scattered a
  // wave over every (sequence, KV head) and re-read K/V from HBM (-4 % at configs[2] B = 4).
  const int64_t nU = int64_t(rows.size()) * Y;
  const bool persistent = c->pf_ctas >= 0 || (c->pf_ctas == -1 && forced == 0 && nU < int64_t(4) * c->num_sms);
  const int32_t W = persistent ? max_ctas : c->num_sms;
  // The two head-pair units of a KV head as a 2-CTA cluster (consecutive work items, identical
  // key ranges) sharing every K/V box by TMA multicast: +1.3 % at configs[2] B=4, but pairing
  // constrains the split plan (-1.2 % at B=1), so only for batches of >= 4 waves (or forced by
  // the testing hook hpa_set_prefill_ctas(c, -2)).
  const bool mc2 = !persistent && prefill_mc2_supported(G) && (c->pf_ctas == -2 || nU >= int64_t(4) * W);
  std::vector<std::pair<int32_t, int32_t>> order;  // (row index, y)
  order.reserve(size_t(nU));
  for (size_t r0 = 0; r0 < rows.size();) {
    size_t r1 = r0;
    while (r1 < rows.size() && rows[r1].b == rows[r0].b) ++r1;
    if (mc2) {  // y = h * G/2 + pair, pair fastest: cluster partners adjacent
      const int32_t np = G / 2;
      for (int32_t h = 0; h < Hkv; ++h)
        for (size_t r = r0; r < r1; ++r)
          for (int32_t pr = 0; pr < np; ++pr) order.push_back({int32_t(r), h * np + pr});
    } else {
      for (int32_t y = 0; y < Y; ++y)
        for (size_t r = r0; r < r1; ++r) order.push_back({int32_t(r), y});
    }
    r0 = r1;
  }
  auto unit = [&](int64_t k) -> const U& { return rows[size_t(order[size_t(k)].first)]; };
  if (persistent && forced == 0 &&
      plan_prefill_streamk(c, seq_ids, q_lens, q_off, nU, W, o_item_p, o_piece_p,
                                [&](int64_t k) { return std::make_tuple(unit(k).b, order[size_t(k)].second, unit(k).x,
                                                                        unit(k).n, unit(k).skip_a, unit(k).n_skip); },
                                plan))
    return true;  // else (a unit would need more than 15 pieces) the list-scheduled plan below
  int64_t best_tail = 0;
  int32_t best_s = 1;
  if (forced > 1) {
    best_tail = nU;
    best_s = forced;
  } else if (forced == 0 && nU < int64_t(16) * W) {  // beyond 16 waves the tail loss is < 1/16
    // measured per-CTA fixed cost (scripts/trace_prefill_ctas.py: setup, pipeline fill, epilogue,
    // CTA switch) ~6.6 us = 3.3 key tiles; a split piece's fp32 epilogue adds ~1.4 us
    static const double o_launch = std::getenv("HPA_PF_OVH") ? std::atof(std::getenv("HPA_PF_OVH")) : 3.3;
    const double o = persistent ? o_item_p : o_launch;
    const double o_piece = persistent ? o_piece_p : o_launch + 0.7;
    static const double c_m = std::getenv("HPA_PF_MERGE") ? std::atof(std::getenv("HPA_PF_MERGE")) : 2.0;
    const double tile_us = 1.95 * c->cfg.head_dim / 128.0;
    const double part_tiles = 2.0 * 128 * c->cfg.head_dim * 4 / 5e6 / tile_us;  // one piece's partial read
    std::vector<double> items(static_cast<size_t>(nU)), base(static_cast<size_t>(W), 0.0), heap, pieces;
    for (int64_t k = 0; k < nU; ++k) items[size_t(k)] = unit(k).n + o;
    heap = base;
    const double t0 = list_schedule(heap, items.data(), items.size());
    double best = t0;
    const int64_t R = mc2 ? ((nU % W) + 1) / 2 * 2 : nU % W;  // whole clusters
    for (int64_t tail : {R, R + W}) {
      if (tail <= 0 || tail > nU) continue;
      std::vector<double> head = base;  // the unsplit units
      list_schedule(head, items.data(), size_t(nU - tail));
      for (int32_t s : {2, 3, 4, 6, 8}) {
        pieces.clear();
        for (int64_t k = nU - tail; k < nU; ++k)
          for (int32_t p = 0; p < s; ++p) pieces.push_back(double(unit(k).n) / s + o_piece);
        heap = head;
        const double t = list_schedule(heap, pieces.data(), pieces.size()) + c_m + double(tail) * s * part_tiles / W;
        if (t < best && t < 0.98 * t0) {
          best = t;
          best_tail = tail;
          best_s = s;
        }
      }
    }
  }
  plan.work.clear();
  plan.parts.clear();
  plan.split_max = best_s;
  plan.work.reserve(size_t(4 * (nU + best_tail * (best_s - 1))));
  for (int64_t k = 0; k < nU; ++k) {
    const U& u = unit(k);
    const int32_t y = order[size_t(k)].second;
    const Seq& q = c->seqs[seq_ids[u.b]];
    const int4 wq = make_int4(seq_ids[u.b], q_lens[u.b], q_off[u.b], q.len);
    const int4 wn = make_int4(int32_t(q.pages.size()), 0, 0, 0);
    if (k < nU - best_tail) {
      plan.work.push_back(make_int4(u.b, y, u.x, 0 | (1 << 4)));
      plan.work.push_back(make_int4(0, u.n, u.skip_a, u.n_skip));
      plan.work.push_back(wq);
      plan.work.push_back(wn);
      continue;
    }
    // persistent items never have an empty key range: a unit gets at most n pieces
    const int32_t ns = persistent ? std::max(1, std::min(best_s, u.n)) : best_s;
    if (ns == 1) {
      plan.work.push_back(make_int4(u.b, y, u.x, 0 | (1 << 4)));
      plan.work.push_back(make_int4(0, u.n, u.skip_a, u.n_skip));
      plan.work.push_back(wq);
      plan.work.push_back(wn);
      continue;
    }
    if (mc2) {  // units k, k + 1 are cluster partners: emit their pieces interleaved
      const int32_t y2 = order[size_t(k + 1)].second;
      const int32_t part = int32_t(plan.parts.size() / 2);
      plan.parts.push_back(make_int4(u.b, y, u.x, ns));
      plan.parts.push_back(make_int4(q_lens[u.b], q_off[u.b], 0, 0));
      plan.parts.push_back(make_int4(u.b, y2, u.x, ns));
      plan.parts.push_back(make_int4(q_lens[u.b], q_off[u.b], 0, 0));
      for (int32_t p = 0; p < ns; ++p) {
        const int32_t jb = int32_t(int64_t(u.n) * p / ns), je = int32_t(int64_t(u.n) * (p + 1) / ns);
        for (int32_t m = 0; m < 2; ++m) {
          plan.work.push_back(make_int4(u.b, m ? y2 : y, u.x, p | (ns << 4) | ((part + m) << 8)));
          plan.work.push_back(make_int4(jb, je - jb, u.skip_a, u.n_skip));
          plan.work.push_back(wq);
          plan.work.push_back(wn);
        }
      }
      ++k;
      continue;
    }
    const int32_t part = int32_t(plan.parts.size() / 2);
    plan.parts.push_back(make_int4(u.b, y, u.x, ns));
    plan.parts.push_back(make_int4(q_lens[u.b], q_off[u.b], 0, 0));
    for (int32_t p = 0; p < ns; ++p) {
      const int32_t jb = int32_t(int64_t(u.n) * p / ns), je = int32_t(int64_t(u.n) * (p + 1) / ns);
      plan.work.push_back(make_int4(u.b, y, u.x, p | (ns << 4) | (part << 8)));
      plan.work.push_back(make_int4(jb, je - jb, u.skip_a, u.n_skip));
      plan.work.push_back(wq);
      plan.work.push_back(wn);
    }
  }
  plan.mc2 = mc2;
  plan.cta_off.clear();
  if (persistent) {
    // Items go, in dispatch order, to the CTA that is free first (estimated key tiles + the
    // per-item cost), as the hardware would dispatch them; each CTA's list keeps that order.
    const size_t n_items = plan.work.size() / 4;
    const int32_t n_ctas = int32_t(std::min<size_t>(size_t(max_ctas), n_items));
    std::vector<std::pair<double, int32_t>> heap;
    for (int32_t i = 0; i < n_ctas; ++i) heap.push_back({0.0, i});
    std::vector<int32_t> owner(n_items);
    std::vector<int32_t> count(size_t(n_ctas), 0);
    auto gt = std::greater<std::pair<double, int32_t>>();
    std::make_heap(heap.begin(), heap.end(), gt);
    for (size_t k = 0; k < n_items; ++k) {
      std::pop_heap(heap.begin(), heap.end(), gt);
      const bool piece = ((plan.work[4 * k].w >> 4) & 15) > 1;
      heap.back().first += plan.work[4 * k + 1].y + (piece ? o_piece_p : o_item_p);
      owner[k] = heap.back().second;
      ++count[size_t(owner[k])];
      std::push_heap(heap.begin(), heap.end(), gt);
    }
    plan.cta_off.assign(size_t(n_ctas) + 1, 0);
    for (int32_t i = 0; i < n_ctas; ++i) plan.cta_off[size_t(i) + 1] = plan.cta_off[size_t(i)] + count[size_t(i)];
    std::vector<int4> sorted(plan.work.size());
    std::vector<int32_t> fill(plan.cta_off.begin(), plan.cta_off.end() - 1);
    for (size_t k = 0; k < n_items; ++k) {
      const int32_t dst = fill[size_t(owner[k])]++;
      for (int f = 0; f < 4; ++f) sorted[4 * size_t(dst) + f] = plan.work[4 * k + f];
    }
    plan.work.swap(sorted);
  }
  return true;
}

// Pages needed to append n rows to seq q.
int32_t pages_for_append(const hpa_cache_t* c, const Seq& q, int32_t n) {
  if (n <= 0) return 0;
  const int32_t P = c->cfg.page_size;
  if (!q.segs.empty() && !q.segs.back().latent) {
    const Segment& g = q.segs.back();
    const int32_t room = int32_t(g.pages.size()) * P - g.rows;
    return n <= room ? 0 : (n - room + P - 1) / P;
  }
  return (n + P - 1) / P;
}

// Whether appending n rows to q must first copy its trailing token segment's last page: the
// page is partial, shared (refcount > 1), and some sharer has claimed rows beyond q's valid rows
// (watermark != valid; `claimed` holds watermarks raised earlier in the same call, and this
// call's claim is recorded in it when q appends in place). NEXT-2, reading A21.
bool append_needs_copy(const hpa_cache_t* c, const Seq& q, int32_t n,
                       std::vector<std::pair<int32_t, int32_t>>& claimed) {
  if (n <= 0 || q.segs.empty() || q.segs.back().latent) return false;
  const int32_t P = c->cfg.page_size;
  const Segment& g = q.segs.back();
  const int32_t vl = g.rows % P;
  if (vl == 0) return false;  // the last page is full: the rows go to fresh pages
  const PageAllocator& tok = const_cast<hpa_cache_t*>(c)->pages_of(false);
  const int32_t pl = g.pages.back();
  int32_t high = tok.high(pl);
  for (const auto& cl : claimed)
    if (cl.first == pl) high = cl.second;
  if (tok.refcount(pl) > 1 && high != vl) return true;
  claimed.emplace_back(pl, std::min(P, vl + n));
  return false;
}

bool valid_dims(const hpa_config_t* g) {
  auto p2 = [](int x) { return x == 16 || x == 32 || x == 64 || x == 128 || x == 256; };
  return (g->head_dim == 64 || g->head_dim == 128) && p2(g->page_size);
}

}  // namespace

// ========================================================================= C ABI
extern "C" {

const char* hpa_last_error(void) { return g_last_error.c_str(); }

const char* hpa_status_string(hpa_status_t s) {
  switch (s) {
    case HPA_OK: return "HPA_OK";
    case HPA_ERR_INVALID_ARG: return "HPA_ERR_INVALID_ARG";
    case HPA_ERR_OUT_OF_PAGES: return "HPA_ERR_OUT_OF_PAGES";
    case HPA_ERR_SEQ_CAPACITY: return "HPA_ERR_SEQ_CAPACITY";
    case HPA_ERR_UNKNOWN_SEQ: return "HPA_ERR_UNKNOWN_SEQ";
    case HPA_ERR_UNKNOWN_SET: return "HPA_ERR_UNKNOWN_SET";
    case HPA_ERR_CUDA: return "HPA_ERR_CUDA";
    case HPA_ERR_UNSUPPORTED: return "HPA_ERR_UNSUPPORTED";
  }
  return "HPA_ERR_?";
}

uint64_t hpa_kv_bytes(int64_t num_layers, int64_t num_kv_heads, int64_t head_dim, int64_t seq_len,
                      int64_t elem_bytes) {
  return 2ull * uint64_t(num_layers) * uint64_t(num_kv_heads) * uint64_t(head_dim) * uint64_t(seq_len) *
         uint64_t(elem_bytes);
}

hpa_status_t hpa_cache_create(const hpa_config_t* cfg, hpa_cache_t** out) {
  if (!cfg || !out) return fail(HPA_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  const hpa_config_t& g = *cfg;
  if (g.num_layers <= 0 || g.num_q_heads <= 0 || g.num_kv_heads <= 0 || g.num_pages <= 0 ||
      g.max_seqs <= 0 || g.max_pages_per_seq <= 0)
    return fail(HPA_ERR_INVALID_ARG, "all config counts must be positive");
  if (g.num_q_heads % g.num_kv_heads != 0)
    return fail(HPA_ERR_INVALID_ARG, "num_q_heads %% num_kv_heads != 0 (S:L25)");
  if (!valid_dims(cfg))
    return fail(HPA_ERR_UNSUPPORTED, "head_dim must be 64/128 and page_size 16..256 (power of 2)");
  if (g.num_q_heads / g.num_kv_heads > 16) return fail(HPA_ERR_UNSUPPORTED, "GQA group > 16");
  const int64_t rows = int64_t(g.num_layers) * g.num_pages * g.num_kv_heads * g.page_size;
  if (rows >= (int64_t(1) << 31)) return fail(HPA_ERR_UNSUPPORTED, "pool too large for 32-bit TMA row index");
  if (g.token_kv_dtype != 0 && g.token_kv_dtype != 1)
    return fail(HPA_ERR_INVALID_ARG, "token_kv_dtype must be 0 (bf16) or 1 (fp8 e4m3)");
  const int64_t rows8 = g.token_kv_dtype == 1 ? int64_t(g.num_layers) * g.num_token_pages * g.num_kv_heads * g.page_size : 0;
  if (g.token_kv_dtype == 1 && g.num_token_pages <= 0)
    return fail(HPA_ERR_INVALID_ARG, "token_kv_dtype = 1 needs num_token_pages > 0");
  if (rows8 >= (int64_t(1) << 31)) return fail(HPA_ERR_UNSUPPORTED, "token pool too large for 32-bit TMA row index");
  if (int64_t(g.max_seqs) * g.max_pages_per_seq * 3 + 2 * g.max_seqs >= (int64_t(1) << 31))
    return fail(HPA_ERR_UNSUPPORTED, "table too large");
  if (int64_t(g.max_pages_per_seq) * g.page_size >= (int64_t(1) << 30))
    return fail(HPA_ERR_UNSUPPORTED, "sequences must stay below 2^30 rows");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || g.device < 0 || g.device >= ndev)
    return fail(HPA_ERR_INVALID_ARG, "CUDA device %d not available", g.device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, g.device) != cudaSuccess)
    return fail(HPA_ERR_CUDA, "cudaGetDeviceProperties failed");
  if (prop.major != 10 || prop.minor != 0)
    return fail(HPA_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a", g.device,
                prop.major, prop.minor);
  DeviceGuard dg(g.device);
  std::unique_ptr<hpa_cache> c(new hpa_cache());
  c->cfg = g;
  c->num_sms = prop.multiProcessorCount;
  c->alloc.init(g.num_pages, g.placement_seed);
  c->fp8 = g.token_kv_dtype == 1;
  if (c->fp8) c->alloc8.init(g.num_token_pages, g.placement_seed ? g.placement_seed ^ 0x5bd1e995ull : 0);
  c->seqs.resize(g.max_seqs);
  c->pool_bytes = uint64_t(rows) * g.head_dim * 2;
  auto cleanup = [&]() {
    if (c->k_pool) cudaFree(c->k_pool);
    if (c->v_pool) cudaFree(c->v_pool);
    if (c->k8_pool) cudaFree(c->k8_pool);
    if (c->v8_pool) cudaFree(c->v8_pool);
    if (c->arena) cudaFree(c->arena);
    if (c->counters) cudaFree(c->counters);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->upload_done) cudaEventDestroy(c->upload_done);
    if (c->copy_done) cudaEventDestroy(c->copy_done);
    if (c->payload_free) cudaEventDestroy(c->payload_free);
    c->copy_stream = nullptr;
    c->upload_done = c->copy_done = c->payload_free = nullptr;
    c->ring.destroy();
  };
  cudaError_t e;
  if ((e = cudaMalloc(&c->k_pool, c->pool_bytes)) != cudaSuccess ||
      (e = cudaMalloc(&c->v_pool, c->pool_bytes)) != cudaSuccess ||
      (e = cudaMemset(c->k_pool, 0, c->pool_bytes)) != cudaSuccess ||
      (e = cudaMemset(c->v_pool, 0, c->pool_bytes)) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "pool allocation");
  }
  if (c->fp8) {
    const size_t b8 = size_t(rows8) * (g.head_dim + 4);  // codes + one fp32 scale per row
    if ((e = cudaMalloc(&c->k8_pool, b8)) != cudaSuccess || (e = cudaMalloc(&c->v8_pool, b8)) != cudaSuccess ||
        (e = cudaMemset(c->k8_pool, 0, b8)) != cudaSuccess || (e = cudaMemset(c->v8_pool, 0, b8)) != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "fp8 token pool allocation");
    }
  }
  const int64_t arena_words = c->off_nent() + g.max_seqs;
  if ((e = cudaMalloc(&c->arena, size_t(arena_words) * 4)) != cudaSuccess ||
      (e = cudaMemset(c->arena, 0, size_t(arena_words) * 4)) != cudaSuccess ||
      (e = c->ring.init(size_t(64) << 20)) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "table allocation");
  }
  // [max_seqs][H_kv] fused-combine counters, then the persistent decode's 2 ticket counters
  const size_t n_counters = size_t(g.max_seqs) * g.num_kv_heads + 2;
  if ((e = cudaMalloc(&c->counters, n_counters * 4)) != cudaSuccess ||
      (e = cudaMemset(c->counters, 0, n_counters * 4)) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "counter allocation");
  }
  c->dt = DevTables{c->arena, c->arena + c->off_pos0(), c->arena + c->off_meta(), c->arena + c->off_len(),
                    c->arena + c->off_nent(), g.max_pages_per_seq};
  if (!make_map_dec(&c->tm_k_dec, c->k_pool, uint64_t(rows), uint64_t(g.head_dim)) ||
      !make_map_dec(&c->tm_v_dec, c->v_pool, uint64_t(rows), uint64_t(g.head_dim)) ||
      !make_map_2d(&c->tm_k_pre, c->k_pool, uint64_t(rows), uint64_t(g.head_dim), uint32_t(std::min(g.page_size, 128))) ||
      !make_map_2d(&c->tm_v_pre, c->v_pool, uint64_t(rows), uint64_t(g.head_dim), uint32_t(std::min(g.page_size, 128)))) {
    cleanup();
    return fail(HPA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the KV pools");
  }
  if ((e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->upload_done, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->payload_free, cudaEventDisableTiming)) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "copy stream setup");
  }
  if ((e = decode_init_attributes()) != cudaSuccess || (e = prefill_init_attributes()) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "kernel attribute setup");
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cache init");
  }
  *out = c.release();
  return HPA_OK;
}

hpa_status_t hpa_cache_destroy(hpa_cache_t* c) {
  if (!c) return HPA_OK;
  DeviceGuard dg(c->cfg.device);
  cudaDeviceSynchronize();
  cudaFree(c->k_pool);
  cudaFree(c->v_pool);
  if (c->k8_pool) cudaFree(c->k8_pool);
  if (c->v8_pool) cudaFree(c->v8_pool);
  cudaFree(c->arena);
  if (c->batch_dev) cudaFree(c->batch_dev);
  if (c->o_part) cudaFree(c->o_part);
  if (c->lse_part) cudaFree(c->lse_part);
  if (c->pf_o_part) cudaFree(c->pf_o_part);
  if (c->pf_lse_part) cudaFree(c->pf_lse_part);
  if (c->counters) cudaFree(c->counters);
  if (c->units_dev) cudaFree(c->units_dev);
  if (c->nsplit_dev) cudaFree(c->nsplit_dev);
  if (c->groups_dev) cudaFree(c->groups_dev);
  if (c->payload_dev) cudaFree(c->payload_dev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->upload_done) cudaEventDestroy(c->upload_done);
  if (c->copy_done) cudaEventDestroy(c->copy_done);
  if (c->payload_free) cudaEventDestroy(c->payload_free);
  c->ring.destroy();
  delete c;
  return HPA_OK;
}

hpa_status_t hpa_cache_pools(hpa_cache_t* c, void** k_pool, void** v_pool, uint64_t* pool_bytes) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (k_pool) *k_pool = c->k_pool;
  if (v_pool) *v_pool = c->v_pool;
  if (pool_bytes) *pool_bytes = c->pool_bytes;
  return HPA_OK;
}

hpa_status_t hpa_cache_token_pool(hpa_cache_t* c, void** k8, void** v8, int32_t* free_token_pages) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (!c->fp8) return fail(HPA_ERR_INVALID_ARG, "this cache stores bf16 token pages (token_kv_dtype = 0)");
  if (k8) *k8 = c->k8_pool;
  if (v8) *v8 = c->v8_pool;
  if (free_token_pages) *free_token_pages = c->alloc8.num_free();
  return HPA_OK;
}

hpa_status_t hpa_cache_stats(hpa_cache_t* c, int32_t* free_pages, int32_t* used_pages, int32_t* live_seqs) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  int32_t used = 0;
  for (int32_t p = 0; p < c->alloc.num_pages(); ++p) used += c->alloc.refcount(p) > 0;
  if (free_pages) *free_pages = c->alloc.num_free();
  if (used_pages) *used_pages = used;
  if (live_seqs) *live_seqs = c->live;
  return HPA_OK;
}

hpa_status_t hpa_seq_create(hpa_cache_t* c, int32_t* seq_id) {
  if (!c || !seq_id) return fail(HPA_ERR_INVALID_ARG, "null argument");
  for (int32_t s = 0; s < c->cfg.max_seqs; ++s) {
    if (!c->seqs[s].live) {
      c->seqs[s] = Seq();
      c->seqs[s].live = true;
      c->pending.push_back({int32_t(c->off_len() + s), 0});
      c->pending.push_back({int32_t(c->off_nent() + s), 0});
      ++c->live;
      *seq_id = s;
      return HPA_OK;
    }
  }
  return fail(HPA_ERR_SEQ_CAPACITY, "all %d sequence slots are in use", c->cfg.max_seqs);
}

hpa_status_t hpa_seq_release(hpa_cache_t* c, int32_t seq_id) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (hpa_status_t st = check_seq(c, seq_id)) return st;
  Seq& q = c->seqs[seq_id];
  for (const Segment& g : q.segs)
    for (int32_t p : g.pages) c->pages_of(g.latent).release(p);
  q = Seq();
  c->pending.push_back({int32_t(c->off_len() + seq_id), 0});
  c->pending.push_back({int32_t(c->off_nent() + seq_id), 0});
  --c->live;
  return HPA_OK;
}

namespace {
// hpa_append_kv in two halves. append_check validates the call without mutating anything and
// returns the number of rows; append_apply then allocates, updates the host tables (their
// device words go to c->pending) and enqueues any copy-on-write page copies on `s`, filling
// `slots` with each new row's pool slot.
hpa_status_t append_check(hpa_cache_t* c, int32_t n_seqs, const int32_t* seq_ids, const int32_t* n_new,
                          const void* k, const void* v, int64_t* rows_out) {
  *rows_out = 0;
  if (!seq_ids || !n_new) return fail(HPA_ERR_INVALID_ARG, "null seq_ids / n_new");
  int64_t total_rows = 0;
  int32_t need = 0;
  std::vector<char> seen(c->cfg.max_seqs, 0);
  for (int32_t i = 0; i < n_seqs; ++i) {
    if (hpa_status_t st = check_seq(c, seq_ids[i])) return st;
    if (seen[seq_ids[i]]) return fail(HPA_ERR_INVALID_ARG, "sequence %d listed twice", seq_ids[i]);
    seen[seq_ids[i]] = 1;
    if (n_new[i] < 0) return fail(HPA_ERR_INVALID_ARG, "n_new[%d] < 0", i);
    const Seq& q = c->seqs[seq_ids[i]];
    const int32_t np = pages_for_append(c, q, n_new[i]);
    if (seq_entries(q) + np > c->cfg.max_pages_per_seq)
      return fail(HPA_ERR_SEQ_CAPACITY, "sequence %d would exceed %d pages", seq_ids[i], c->cfg.max_pages_per_seq);
    need += np;
    total_rows += n_new[i];
  }
  if (total_rows == 0) return HPA_OK;
  if (!k || !v) return fail(HPA_ERR_INVALID_ARG, "null k / v");
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return fail(HPA_ERR_INVALID_ARG, "k / v must be 16-byte aligned");
  PageAllocator& tok = c->pages_of(false);
  // copy-on-write of shared partial last pages (forked prefixes, reading A21), decided in call
  // order with the watermarks this call claims: one more page per copied sequence
  {
    std::vector<std::pair<int32_t, int32_t>> claimed;  // (page, watermark) claimed by this call
    for (int32_t i = 0; i < n_seqs; ++i) need += append_needs_copy(c, c->seqs[seq_ids[i]], n_new[i], claimed);
  }
  if (need > tok.num_free())
    return fail(HPA_ERR_OUT_OF_PAGES, "append needs %d pages, %d free", need, tok.num_free());
  *rows_out = total_rows;
  return HPA_OK;
}

hpa_status_t append_apply(hpa_cache_t* c, int32_t n_seqs, const int32_t* seq_ids, const int32_t* n_new,
                          int64_t total_rows, cudaStream_t s, std::vector<int32_t>& slots) {
  PageAllocator& tok = c->pages_of(false);
  const int32_t P = c->cfg.page_size;
  slots.reserve(size_t(total_rows));
  CopyPagesMeta cow{};
  cow.fp8 = c->fp8 ? 1 : 0;
  for (int32_t i = 0; i < n_seqs; ++i) {
    Seq& q = c->seqs[seq_ids[i]];
    int32_t n = n_new[i];
    if (n == 0) continue;
    const int32_t first_entry = std::max(0, seq_entries(q) - 1);
    std::vector<std::pair<int32_t, int32_t>> none;
    if (append_needs_copy(c, q, n, none)) {  // watermarks of earlier sequences are already applied
      Segment& g = q.segs.back();
      std::vector<int32_t> fresh;
      tok.alloc(1, fresh);
      const int32_t old = g.pages.back();
      if (cow.n == kCopyPagesMax) {
        HPA_CUDA(launch_copy_pages(c->geom(), cow, s));
        c->launches += 1;
        cow.n = 0;
      }
      cow.items[cow.n++] = make_int2(old, fresh[0]);
      tok.release(old);
      g.pages.back() = fresh[0];
    }
    if (q.segs.empty() || q.segs.back().latent) q.segs.push_back(Segment{false, -1, 0, {}});
    Segment& g = q.segs.back();
    const int32_t np = pages_for_append(c, q, n);
    tok.alloc(np, g.pages);
    for (int32_t r = 0; r < n; ++r) {
      const int32_t row = g.rows + r;
      slots.push_back(g.pages[row / P] * P + row % P);
    }
    for (int32_t pg = g.rows / P; pg < int32_t(g.pages.size()); ++pg)  // watermarks of the written pages
      tok.set_high(g.pages[pg], std::min(P, g.rows + n - pg * P));
    g.rows += n;
    c->rebuild(seq_ids[i], first_entry);
  }
  if (cow.n) {  // stream order: the copies land before the scatter writes the new rows
    HPA_CUDA(launch_copy_pages(c->geom(), cow, s));
    c->launches += 1;
  }
  return HPA_OK;
}
}  // namespace

hpa_status_t hpa_append_kv(hpa_cache_t* c, int32_t n_seqs, const int32_t* seq_ids, const int32_t* n_new,
                           const void* k, const void* v, hpa_stream_t stream) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n_seqs < 0) return fail(HPA_ERR_INVALID_ARG, "n_seqs < 0");
  if (n_seqs == 0) return HPA_OK;
  int64_t total_rows = 0;
  if (hpa_status_t st = append_check(c, n_seqs, seq_ids, n_new, k, v, &total_rows)) return st;
  if (total_rows == 0) return HPA_OK;
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int32_t> slots;
  if (hpa_status_t st = append_apply(c, n_seqs, seq_ids, n_new, total_rows, s, slots)) return st;
  const int64_t Hd = int64_t(c->cfg.num_kv_heads) * c->cfg.head_dim;
  std::vector<ScatterRecord> recs{
      ScatterRecord{k, v, total_rows * Hd, Hd, int32_t(total_rows), 0, 0, 0, 0, 0, c->fp8 ? 1 : 0, 0}};
  return ship(c, s, recs, slots, total_rows);
}

hpa_status_t hpa_seq_fork(hpa_cache_t* c, int32_t src_seq, int32_t n_prefix_rows, int32_t* dst_seq_out) {
  if (!c || !dst_seq_out) return fail(HPA_ERR_INVALID_ARG, "null argument");
  if (hpa_status_t st = check_seq(c, src_seq)) return st;
  const Seq& src = c->seqs[src_seq];
  if (n_prefix_rows < 0 || n_prefix_rows > src.len)
    return fail(HPA_ERR_INVALID_ARG, "n_prefix_rows %d outside [0, %d]", n_prefix_rows, src.len);
  const int32_t P = c->cfg.page_size;
  std::vector<Segment> segs;
  int32_t left = n_prefix_rows;
  for (const Segment& g : src.segs) {
    if (left == 0) break;
    if (g.rows > left && g.latent)
      return fail(HPA_ERR_INVALID_ARG, "fork cut at row %d falls inside latent set %d", n_prefix_rows, g.set_id);
    const int32_t take = std::min(g.rows, left);
    segs.push_back(Segment{g.latent, g.set_id, take,
                           std::vector<int32_t>(g.pages.begin(), g.pages.begin() + (take + P - 1) / P)});
    left -= take;
  }
  int32_t d = -1;
  for (int32_t s = 0; s < c->cfg.max_seqs && d < 0; ++s)
    if (!c->seqs[s].live) d = s;
  if (d < 0) return fail(HPA_ERR_SEQ_CAPACITY, "all %d sequence slots are in use", c->cfg.max_seqs);
  for (const Segment& g : segs)
    for (int32_t p : g.pages) c->pages_of(g.latent).retain(p);
  Seq& q = c->seqs[d];
  q = Seq();
  q.live = true;
  q.next_set = c->seqs[src_seq].next_set;
  q.segs = std::move(segs);
  c->pending.push_back({int32_t(c->off_len() + d), 0});
  c->pending.push_back({int32_t(c->off_nent() + d), 0});
  c->rebuild(d, 0);
  ++c->live;
  *dst_seq_out = d;
  return HPA_OK;
}

namespace {

struct InstallPlan {
  int32_t seq, set_id, m;
  const void* kv;
  bool is_new;
  int32_t seg_index;  // existing segment (replace)
  int32_t new_pages;  // pages to allocate
  int32_t old_pages;
};

hpa_status_t plan_install(hpa_cache_t* c, int32_t seq, int32_t set_id, int32_t m, const void* kv,
                          InstallPlan* p) {
  if (hpa_status_t st = check_seq(c, seq)) return st;
  if (m <= 0) return fail(HPA_ERR_INVALID_ARG, "m_rows must be positive");
  if (!kv || (reinterpret_cast<uintptr_t>(kv) & 15)) return fail(HPA_ERR_INVALID_ARG, "kv must be a 16-byte aligned device pointer");
  const Seq& q = c->seqs[seq];
  const int32_t P = c->cfg.page_size;
  const int32_t np = (m + P - 1) / P;
  *p = InstallPlan{seq, set_id, m, kv, set_id < 0, -1, np, 0};
  if (set_id >= 0) {
    for (int32_t i = 0; i < int32_t(q.segs.size()); ++i)
      if (q.segs[i].latent && q.segs[i].set_id == set_id) p->seg_index = i;
    if (p->seg_index < 0) return fail(HPA_ERR_UNKNOWN_SET, "sequence %d has no latent set %d", seq, set_id);
    const Segment& g = q.segs[p->seg_index];
    p->old_pages = int32_t(g.pages.size());
    bool shared = false;
    for (int32_t pg : g.pages) shared |= c->alloc.refcount(pg) > 1;
    if (p->old_pages == np && !shared) p->new_pages = 0;  // rewrite in place (never into shared pages)
  }
  const int32_t delta = p->new_pages - (p->new_pages ? p->old_pages : 0);
  if (seq_entries(q) + delta > c->cfg.max_pages_per_seq)
    return fail(HPA_ERR_SEQ_CAPACITY, "sequence %d would exceed %d pages", seq, c->cfg.max_pages_per_seq);
  return HPA_OK;
}

// Applies a checked plan; appends the set's slots; returns the set id.
int32_t apply_install(hpa_cache_t* c, const InstallPlan& p, std::vector<int32_t>& slots) {
  Seq& q = c->seqs[p.seq];
  const int32_t P = c->cfg.page_size;
  int32_t seg_i, first_entry = 0;
  if (p.is_new) {
    first_entry = seq_entries(q);
    q.segs.push_back(Segment{true, q.next_set++, 0, {}});
    seg_i = int32_t(q.segs.size()) - 1;
    c->alloc.alloc(p.new_pages, q.segs[seg_i].pages);
  } else {
    seg_i = p.seg_index;
    for (int32_t i = 0; i < seg_i; ++i) first_entry += int32_t(q.segs[i].pages.size());
    Segment& g = q.segs[seg_i];
    if (p.new_pages > 0) {  // different page count: free + allocate + splice
      for (int32_t pg : g.pages) c->alloc.release(pg);
      g.pages.clear();
      c->alloc.alloc(p.new_pages, g.pages);
    }
  }
  Segment& g = q.segs[seg_i];
  const bool same_rows = !p.is_new && g.rows == p.m;
  g.rows = p.m;
  slots.insert(slots.end(), g.pages.begin(), g.pages.end());  // page mode: one index per page
  (void)P;
  if (!same_rows) c->rebuild(p.seq, first_entry);  // same rows in the same pages: table unchanged
  return g.set_id;
}

}  // namespace

hpa_status_t hpa_latent_set_install_batch(hpa_cache_t* c, int32_t n, const int32_t* seq_ids,
                                          const int32_t* set_ids, const int32_t* m_rows,
                                          const void* const* kv_ptrs, hpa_stream_t stream,
                                          int32_t* set_ids_out) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n < 0) return fail(HPA_ERR_INVALID_ARG, "n < 0");
  if (n == 0) return HPA_OK;
  if (!seq_ids || !set_ids || !m_rows || !kv_ptrs) return fail(HPA_ERR_INVALID_ARG, "null argument");
  std::vector<InstallPlan> plans(n);
  std::vector<char> seen(c->cfg.max_seqs, 0);
  int32_t need = 0, freed = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (hpa_status_t st = plan_install(c, seq_ids[i], set_ids[i], m_rows[i], kv_ptrs[i], &plans[i])) return st;
    if (seen[seq_ids[i]]) return fail(HPA_ERR_INVALID_ARG, "sequence %d listed twice", seq_ids[i]);
    seen[seq_ids[i]] = 1;
    need += plans[i].new_pages;
    if (plans[i].new_pages && !plans[i].is_new) {  // only sole references return pages to the pool
      for (int32_t pg : c->seqs[seq_ids[i]].segs[plans[i].seg_index].pages) freed += c->alloc.refcount(pg) == 1;
    }
  }
  // replaced sets free their pages before allocating (all-or-nothing budget)
  if (need > c->alloc.num_free() + freed)
    return fail(HPA_ERR_OUT_OF_PAGES, "install needs %d pages, %d free", need, c->alloc.num_free() + freed);
  DeviceGuard dg(c->cfg.device);
  // release replaced pages first so their pages are reusable within this call
  std::vector<int32_t> slots;
  std::vector<ScatterRecord> recs;
  const int64_t Hd = int64_t(c->cfg.num_kv_heads) * c->cfg.head_dim;
  int64_t max_rows = 0;
  for (int32_t i = 0; i < n; ++i) {
    const InstallPlan& p = plans[i];
    if (p.new_pages && !p.is_new) {
      Segment& g = c->seqs[p.seq].segs[p.seg_index];
      for (int32_t pg : g.pages) c->alloc.release(pg);
      g.pages.clear();
    }
  }
  for (int32_t i = 0; i < n; ++i) {
    InstallPlan p = plans[i];
    const int32_t slot_off = int32_t(slots.size());
    if (p.new_pages && !p.is_new) {
      // pages already released above: allocate + splice
      Seq& q = c->seqs[p.seq];
      int32_t first_entry = 0;
      for (int32_t s = 0; s < p.seg_index; ++s) first_entry += int32_t(q.segs[s].pages.size());
      Segment& g = q.segs[p.seg_index];
      c->alloc.alloc(p.new_pages, g.pages);
      g.rows = p.m;
      slots.insert(slots.end(), g.pages.begin(), g.pages.end());  // page mode
      c->rebuild(p.seq, first_entry);
      if (set_ids_out) set_ids_out[i] = g.set_id;
    } else {
      const int32_t id = apply_install(c, p, slots);
      if (set_ids_out) set_ids_out[i] = id;
    }
    const char* kv = static_cast<const char*>(p.kv);
    recs.push_back(ScatterRecord{kv, kv + size_t(p.m) * Hd * 2, 2 * int64_t(p.m) * Hd, Hd, p.m, slot_off, 0, 1, 0, 0});
    max_rows = std::max<int64_t>(max_rows, p.m);
  }
  return ship(c, static_cast<cudaStream_t>(stream), recs, slots, max_rows);
}

hpa_status_t hpa_latent_set_install_host(hpa_cache_t* c, int32_t n, const int32_t* seq_ids,
                                         const int32_t* set_ids, const int32_t* m_rows,
                                         const void* const* host_ptrs, hpa_stream_t stream,
                                         int32_t* set_ids_out) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n < 0) return fail(HPA_ERR_INVALID_ARG, "n < 0");
  if (n == 0) return HPA_OK;
  if (!seq_ids || !set_ids || !m_rows || !host_ptrs) return fail(HPA_ERR_INVALID_ARG, "null argument");
  const size_t row_bytes = size_t(c->cfg.num_kv_heads) * c->cfg.head_dim * 2;
  std::vector<size_t> off(n);
  size_t total = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (m_rows[i] <= 0 || !host_ptrs[i]) return fail(HPA_ERR_INVALID_ARG, "bad payload %d", i);
    off[i] = total;
    total += (size_t(c->cfg.num_layers) * 2 * m_rows[i] * row_bytes + 255) & ~size_t(255);
  }
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (total > c->payload_cap) {  // grow (rare): wait for the previous user of the buffer
    HPA_CUDA(cudaStreamSynchronize(c->copy_stream));
    HPA_CUDA(cudaEventSynchronize(c->payload_free));
    if (c->payload_dev) cudaFree(c->payload_dev);
    c->payload_dev = nullptr;
    HPA_CUDA(cudaMalloc(&c->payload_dev, total));
    c->payload_cap = total;
  }
  // copies wait (on the GPU) until the previous host install's scatter has read the buffer
  HPA_CUDA(cudaStreamWaitEvent(c->copy_stream, c->payload_free, 0));
  // payloads that lie back to back in host memory (and so in the device buffer) go as one copy:
  // one DMA per request cost ~1 us each at 256 requests
  std::vector<const void*> dev_ptrs(n);
  for (int32_t i = 0; i < n;) {
    size_t bytes = size_t(c->cfg.num_layers) * 2 * m_rows[i] * row_bytes;
    int32_t j = i + 1;
    for (; j < n; ++j) {
      const size_t bj = size_t(c->cfg.num_layers) * 2 * m_rows[j] * row_bytes;
      if (off[j] != off[i] + bytes || static_cast<const char*>(host_ptrs[j]) != static_cast<const char*>(host_ptrs[i]) + bytes)
        break;
      bytes += bj;
    }
    HPA_CUDA(cudaMemcpyAsync(c->payload_dev + off[i], host_ptrs[i], bytes, cudaMemcpyHostToDevice, c->copy_stream));
    for (int32_t k = i; k < j; ++k) dev_ptrs[k] = c->payload_dev + off[k];
    i = j;
  }
  HPA_CUDA(cudaEventRecord(c->copy_done, c->copy_stream));
  HPA_CUDA(cudaStreamWaitEvent(s, c->copy_done, 0));
  hpa_status_t st = hpa_latent_set_install_batch(c, n, seq_ids, set_ids, m_rows, dev_ptrs.data(), stream,
                                                 set_ids_out);
  HPA_CUDA(cudaEventRecord(c->payload_free, s));
  return st;
}

hpa_status_t hpa_latent_set_install(hpa_cache_t* c, int32_t seq_id, int32_t set_id, int32_t m_rows,
                                    const void* kv, hpa_stream_t stream, int32_t* set_id_out) {
  int32_t out = -1;
  hpa_status_t st = hpa_latent_set_install_batch(c, 1, &seq_id, &set_id, &m_rows, &kv, stream, &out);
  if (st == HPA_OK && set_id_out) *set_id_out = out;
  return st;
}

hpa_status_t hpa_latent_set_share(hpa_cache_t* c, int32_t dst_seq, int32_t src_seq, int32_t src_set_id,
                                  int32_t* set_id_out) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (hpa_status_t st = check_seq(c, dst_seq)) return st;
  if (hpa_status_t st = check_seq(c, src_seq)) return st;
  const Segment* src = nullptr;
  for (const Segment& g : c->seqs[src_seq].segs)
    if (g.latent && g.set_id == src_set_id) src = &g;
  if (!src) return fail(HPA_ERR_UNKNOWN_SET, "sequence %d has no latent set %d", src_seq, src_set_id);
  Seq& d = c->seqs[dst_seq];
  if (seq_entries(d) + int32_t(src->pages.size()) > c->cfg.max_pages_per_seq)
    return fail(HPA_ERR_SEQ_CAPACITY, "sequence %d would exceed %d pages", dst_seq, c->cfg.max_pages_per_seq);
  Segment g{true, d.next_set++, src->rows, src->pages};  // copy first: src may live in d.segs
  for (int32_t pg : g.pages) c->alloc.retain(pg);
  const int32_t first_entry = seq_entries(d);
  d.segs.push_back(std::move(g));
  c->rebuild(dst_seq, first_entry);
  if (set_id_out) *set_id_out = d.segs.back().set_id;
  return HPA_OK;
}

hpa_status_t hpa_latent_set_remove(hpa_cache_t* c, int32_t seq_id, int32_t set_id) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (hpa_status_t st = check_seq(c, seq_id)) return st;
  Seq& q = c->seqs[seq_id];
  int32_t first_entry = 0;
  for (int32_t i = 0; i < int32_t(q.segs.size()); ++i) {
    if (q.segs[i].latent && q.segs[i].set_id == set_id) {
      for (int32_t pg : q.segs[i].pages) c->alloc.release(pg);
      q.segs.erase(q.segs.begin() + i);
      c->rebuild(seq_id, first_entry);
      return HPA_OK;
    }
    first_entry += int32_t(q.segs[i].pages.size());
  }
  return fail(HPA_ERR_UNKNOWN_SET, "sequence %d has no latent set %d", seq_id, set_id);
}

hpa_status_t hpa_seq_compress(hpa_cache_t* c, int32_t seq_id, int32_t n_doc_rows, int32_t m_rows,
                              hpa_stream_t stream, int32_t* set_id_out) {
  return hpa_seq_compress_batch(c, 1, &seq_id, &n_doc_rows, &m_rows, stream, set_id_out);
}

hpa_status_t hpa_seq_compress_batch(hpa_cache_t* c, int32_t n, const int32_t* seq_ids, const int32_t* n_doc_rows,
                                    const int32_t* m_rows, hpa_stream_t stream, int32_t* set_ids_out) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n < 0) return fail(HPA_ERR_INVALID_ARG, "n < 0");
  if (n == 0) return HPA_OK;
  if (!seq_ids || !n_doc_rows || !m_rows) return fail(HPA_ERR_INVALID_ARG, "null argument");
  const int32_t P = c->cfg.page_size;
  // every check before any change (the cache is unchanged on error)
  int32_t need = 0;
  std::vector<int32_t> sorted(seq_ids, seq_ids + n);
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
    return fail(HPA_ERR_INVALID_ARG, "a sequence appears twice in the batch");
  for (int32_t i = 0; i < n; ++i) {
    if (hpa_status_t st = check_seq(c, seq_ids[i])) return st;
    const Seq& q = c->seqs[seq_ids[i]];
    if (n_doc_rows[i] < 0 || m_rows[i] <= 0) return fail(HPA_ERR_INVALID_ARG, "need n_doc_rows >= 0 and m_rows > 0");
    if (q.segs.empty() || q.segs.back().latent || q.segs.back().rows < n_doc_rows[i] + m_rows[i])
      return fail(HPA_ERR_INVALID_ARG, "document + latent rows must lie in the trailing token segment");
    const Segment& T = q.segs.back();
    const int32_t np = (m_rows[i] + P - 1) / P;
    const int32_t keep = T.rows - n_doc_rows[i] - m_rows[i];
    const int32_t n_before = seq_entries(q) - int32_t(T.pages.size());
    if (n_before + (keep + P - 1) / P + np > c->cfg.max_pages_per_seq)
      return fail(HPA_ERR_SEQ_CAPACITY, "sequence %d would exceed %d pages", seq_ids[i], c->cfg.max_pages_per_seq);
    need += np;
  }
  // Pages: a request's trailing token pages past its kept rows hold either only document rows
  // (freed before the destinations are allocated, so the batch can reuse them) or some of the
  // m source rows (freed after the move is queued: no destination may overlap a source).
  auto is_src_page = [&](int32_t i, int32_t k) {  // page k of request i's trailing segment
    const Segment& T = c->seqs[seq_ids[i]].segs.back();
    const int32_t lo = T.rows - m_rows[i];  // first source row
    return (k + 1) * P > lo;                // page k covers rows [kP, kP + P)
  };
  int32_t reusable = 0;  // document-only pages that return to the latent pages' pool
  if (!c->fp8) {
    for (int32_t i = 0; i < n; ++i) {
      const Segment& T = c->seqs[seq_ids[i]].segs.back();
      const int32_t keep_pages = (T.rows - n_doc_rows[i] - m_rows[i] + P - 1) / P;
      for (int32_t k = keep_pages; k < int32_t(T.pages.size()); ++k)
        if (!is_src_page(i, k) && c->alloc.refcount(T.pages[size_t(k)]) == 1) ++reusable;
    }
  }
  if (need > c->alloc.num_free() + reusable)
    return fail(HPA_ERR_OUT_OF_PAGES, "compress needs %d pages, %d free", need, c->alloc.num_free() + reusable);
  DeviceGuard dg(c->cfg.device);
  for (int32_t i = 0; i < n; ++i) {  // document-only pages first
    Segment& T = c->seqs[seq_ids[i]].segs.back();
    const int32_t keep_pages = (T.rows - n_doc_rows[i] - m_rows[i] + P - 1) / P;
    for (int32_t k = keep_pages; k < int32_t(T.pages.size()); ++k)
      if (!is_src_page(i, k)) c->pages_of(false).release(T.pages[size_t(k)]);
  }
  // destination pages of every request, then one page-mode move record per request, all in
  // one launch; the source pages are released once the records are built
  std::vector<Segment> lat(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    Seq& q = c->seqs[seq_ids[i]];
    lat[size_t(i)] = Segment{true, q.next_set++, m_rows[i], {}};
    c->alloc.alloc((m_rows[i] + P - 1) / P, lat[size_t(i)].pages);
  }
  std::vector<int32_t> idx;
  std::vector<ScatterRecord> recs;
  std::vector<int32_t> src_pages;
  for (int32_t i = 0; i < n; ++i) {
    Seq& q = c->seqs[seq_ids[i]];
    Segment& T = q.segs.back();
    const int32_t keep = T.rows - n_doc_rows[i] - m_rows[i];
    const int32_t keep_pages = (keep + P - 1) / P;
    const int32_t n_before = seq_entries(q) - int32_t(T.pages.size());
    const int32_t dst_off = int32_t(idx.size());
    idx.insert(idx.end(), lat[size_t(i)].pages.begin(), lat[size_t(i)].pages.end());  // page-mode destination
    const int32_t src_off = int32_t(idx.size());
    for (int32_t r = 0; r < m_rows[i]; ++r) {
      const int32_t row = keep + n_doc_rows[i] + r;
      idx.push_back(T.pages[row / P] * P + row % P);
    }
    recs.push_back(ScatterRecord{nullptr, nullptr, 0, 0, m_rows[i], dst_off, 0, 1, 1, src_off, 0, c->fp8 ? 1 : 0});
    for (int32_t k = keep_pages; k < int32_t(T.pages.size()); ++k)
      if (is_src_page(i, k)) src_pages.push_back(T.pages[size_t(k)]);
    T.pages.resize(size_t(keep_pages));
    T.rows = keep;
    if (keep % P && c->pages_of(false).refcount(T.pages.back()) == 1)  // sole owner: rows past keep are free again
      c->pages_of(false).set_high(T.pages.back(), keep % P);
    if (keep == 0) q.segs.pop_back();
    q.segs.push_back(std::move(lat[size_t(i)]));
    c->rebuild(seq_ids[i], n_before + std::max(0, keep_pages - 1));
    if (set_ids_out) set_ids_out[i] = q.segs.back().set_id;
  }
  for (int32_t pg : src_pages) c->pages_of(false).release(pg);
  int64_t rows = 0;  // the scatter grid is sized by the largest record
  for (int32_t i = 0; i < n; ++i) rows = std::max<int64_t>(rows, m_rows[i]);
  return ship(c, static_cast<cudaStream_t>(stream), recs, idx, rows);
}

namespace {
hpa_status_t decode_impl(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids, const void* q,
                         void* out, float* part_o, float* part_lse, float softmax_scale, hpa_stream_t stream,
                         const AppendRows* ap = nullptr);
}

hpa_status_t hpa_decode(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids, const void* q,
                        void* out, float softmax_scale, hpa_stream_t stream) {
  if (!out) return fail(HPA_ERR_INVALID_ARG, "null out");
  return decode_impl(c, layer, n_seqs, seq_ids, q, out, nullptr, nullptr, softmax_scale, stream);
}

#ifdef HPA_HOST_PROF  // diagnostics build: per-phase host time of hpa_append_decode, printed at exit
namespace {
struct HostProf {
  double t[16] = {0};
  long n = 0;
  ~HostProf() {
    if (n)
      std::fprintf(stderr,
                   "host prof (%ld calls, us): check %.2f ship %.2f apply %.2f tail %.2f decode %.2f "
                   "[decode: checks+ship+batch %.2f groups %.2f splits %.2f upload %.2f launch %.2f]\n",
                   n, t[0] / n, t[1] / n, t[2] / n, t[3] / n, t[4] / n, t[8] / n, t[9] / n, t[10] / n, t[11] / n,
                   t[12] / n);
  }
} g_hprof;
inline double hp_now() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace
#define HP_MARK(i) do { const double _t = hp_now(); g_hprof.t[i] += _t - hp_last; hp_last = _t; } while (0)
#else
#define HP_MARK(i) do {} while (0)
#endif

hpa_status_t hpa_append_decode(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                               const void* k, const void* v, const void* q, void* out, float softmax_scale,
                               hpa_stream_t stream) {
#ifdef HPA_HOST_PROF
  double hp_last = hp_now();
  ++g_hprof.n;
#endif
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n_seqs < 0) return fail(HPA_ERR_INVALID_ARG, "n_seqs < 0");
  if (n_seqs == 0) return HPA_OK;
  // everything decode_impl would reject is checked before the append mutates the cache
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(HPA_ERR_INVALID_ARG, "layer %d out of range", layer);
  if (n_seqs > c->cfg.max_seqs) return fail(HPA_ERR_INVALID_ARG, "n_seqs > max_seqs");
  if (!seq_ids || !q || !out) return fail(HPA_ERR_INVALID_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(HPA_ERR_INVALID_ARG, "q / out must be 16-byte aligned");
  if (c->fp8 && !decode_persistent())
    return fail(HPA_ERR_UNSUPPORTED, "fp8 token pages need the persistent decode kernel");
  if (decode_persistent() && c->cfg.num_kv_heads > 255)
    return fail(HPA_ERR_UNSUPPORTED, "persistent decode supports H_kv <= 255");
  const std::vector<int32_t> ones(size_t(n_seqs), 1);
  int64_t rows = 0;
  if (hpa_status_t st = append_check(c, n_seqs, seq_ids, ones.data(), k, v, &rows)) return st;
  HP_MARK(0);
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // fp8 token pages quantize on append (copy_kernels.cu); larger batches exceed the kernel's
  // parameter block: both take the two-launch path
  static const bool no_fuse = std::getenv("HPA_NO_FUSE") != nullptr;  // A/B knob: the two-launch step
  const bool fuse = !c->fp8 && decode_persistent() && n_seqs <= kAppendFuseMax && !no_fuse;
  if (fuse) {
    if (hpa_status_t st = ship(c, s, {}, {}, 0)) return st;  // earlier calls' table words first
  }
  HP_MARK(1);
  std::vector<int32_t> slots;
  if (hpa_status_t st = append_apply(c, n_seqs, seq_ids, ones.data(), rows, s, slots)) return st;
  HP_MARK(2);
  if (!fuse) {
    const int64_t Hd = int64_t(c->cfg.num_kv_heads) * c->cfg.head_dim;
    std::vector<ScatterRecord> recs{
        ScatterRecord{k, v, rows * Hd, Hd, int32_t(rows), 0, 0, 0, 0, 0, c->fp8 ? 1 : 0, 0}};
    if (hpa_status_t st = ship(c, s, recs, slots, rows)) return st;
    return decode_impl(c, layer, n_seqs, seq_ids, q, out, nullptr, nullptr, softmax_scale, stream);
  }
  // The append changed only each sequence's last entry, its length and its entry count
  // (rebuild from the old last entry); the kernel takes those from the tail records and
  // writes them back, so the queued words are dropped -- unless something else is queued.
  std::vector<int4> tail(static_cast<size_t>(n_seqs));
  std::vector<int32_t> own;
  own.reserve(size_t(n_seqs) * 5);
  for (int32_t i = 0; i < n_seqs; ++i) {
    const int32_t sid = seq_ids[i];
    const Seq& sq = c->seqs[sid];
    const int32_t e = seq_entries(sq) - 1;
    tail[i] = make_int4(e + 1, sq.pages[e], sq.meta[e], sq.pos0[e]);
    own.insert(own.end(), {int32_t(c->idx(sid, e)), int32_t(c->off_pos0() + c->idx(sid, e)),
                           int32_t(c->off_meta() + c->idx(sid, e)), int32_t(c->off_len() + sid),
                           int32_t(c->off_nent() + sid)});
  }
  std::sort(own.begin(), own.end());
  bool only_own = true;
  for (const WordWrite& w : c->pending) only_own = only_own && std::binary_search(own.begin(), own.end(), w.idx);
  if (only_own) c->pending.clear();  // else decode_impl ships them (the same values) first
  const PoolGeom g = c->geom();
  const AppendRows ap{k, v, g.k_pool, g.v_pool, rows * c->cfg.num_kv_heads * c->cfg.head_dim, n_seqs,
                      c->cfg.num_layers, tail.data()};
  HP_MARK(3);
  const hpa_status_t st = decode_impl(c, layer, n_seqs, seq_ids, q, out, nullptr, nullptr, softmax_scale, stream, &ap);
  HP_MARK(4);
  return st;
}

hpa_status_t hpa_decode_partial(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                                const void* q, float* o_part, float* lse_part, float softmax_scale,
                                hpa_stream_t stream) {
  if (!o_part || !lse_part || (reinterpret_cast<uintptr_t>(o_part) & 15))
    return fail(HPA_ERR_INVALID_ARG, "o_part / lse_part must be device pointers (o_part 16-byte aligned)");
  return decode_impl(c, layer, n_seqs, seq_ids, q, nullptr, o_part, lse_part, softmax_scale, stream);
}

hpa_status_t hpa_merge_partials(int32_t n_parts, int32_t n_rows, int32_t head_dim, const float* o_parts,
                                const float* lse_parts, void* out, hpa_stream_t stream) {
  if (n_parts <= 0 || n_rows < 0 || !o_parts || !lse_parts || !out)
    return fail(HPA_ERR_INVALID_ARG, "bad merge arguments");
  if (head_dim != 64 && head_dim != 128) return fail(HPA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  cudaError_t e = launch_merge(n_parts, n_rows, head_dim, o_parts, lse_parts, out,
                               static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "merge launch");
  return HPA_OK;
}

namespace {
// Work list of a batch with cascade groups: own units {b, seq, h | split << 8 | S_b << 16, r_b}
// over entries [r_b, n_b) and group units {-2 - record, representative, h, 0}, longest first;
// a member's partial slots are its S_b own splits, then its group's pieces. Uploaded only when
// the plan changes (key: batch, splits, runs, groups).
hpa_status_t plan_cascade(hpa_cache_t* c, int32_t n, const int32_t* seq_ids, std::vector<CGroup>& groups,
                          cudaStream_t s, int32_t* S_out) {
  const int32_t D = c->cfg.head_dim, Hq = c->cfg.num_q_heads, Hkv = c->cfg.num_kv_heads;
  const int32_t slots = decode_slots(D, Hq / Hkv);
  std::vector<int32_t> r(size_t(n), 0), gof(size_t(n), -1);
  std::vector<int32_t> ch(r.size()), ne(r.size());
  for (size_t g = 0; g < groups.size(); ++g)
    for (int32_t i : groups[g].mem) {
      r[size_t(i)] = groups[g].r;
      gof[size_t(i)] = int32_t(g);
    }
  for (int32_t i = 0; i < n; ++i) {
    const Seq& q = c->seqs[seq_ids[i]];
    ne[size_t(i)] = seq_entries(q) - r[size_t(i)];
    ch[size_t(i)] = q.chunks - (r[size_t(i)] ? q.pch[size_t(r[size_t(i)] - 1)] : 0);
  }
  std::vector<int32_t> sp;
  plan_splits_core(c, n, ch, ne, slots, sp);
  int32_t E = kCascadeMinChunks;  // chunk budget of an own unit
  for (int32_t i = 0; i < n; ++i) {
    if (ne[size_t(i)] <= 0) sp[size_t(i)] = 0;  // nothing of its own: the group covers it
    else E = std::max(E, (std::max(1, ch[size_t(i)]) + sp[size_t(i)] - 1) / sp[size_t(i)]);
  }
  // a group piece reads its chunks once but every consumer of the CTA works through all of
  // them (for its own query columns): ~1.75 chunk times per chunk (configs[1]-shaped forks,
  // scripts/time_cascade.py). Pieces: no group unit longer than the per-slot share of the
  // batch's work, and about one group unit per CTA slot (profiles/r2_cascade_pieces.log:
  // fewer, longer pieces leave the group units on the critical path; more add partials)
  double work = 0;
  for (int32_t i = 0; i < n; ++i) work += double(std::max(0, ch[size_t(i)])) * Hkv;
  static const double kappa = std::getenv("HPA_CASC_KAPPA") ? std::atof(std::getenv("HPA_CASC_KAPPA")) : 1.75;
  for (const CGroup& g : groups) work += kappa * g.rch * Hkv;
  // The group units run first (longest first) and all have about one length, so their count
  // is kept just under a whole number k of CTA waves (320 units on 296 slots ran 1.3x slower
  // than 256): the smallest k whose pieces are no longer than the per-slot share of the work.
  const double share = std::max(double(E), work / slots);
  const int32_t gh = std::max<int32_t>(1, int32_t(groups.size()) * Hkv);
  int32_t rmax = 0;
  for (const CGroup& g : groups) rmax = std::max(rmax, g.rch);
  int32_t pk = 64;
  for (int32_t k = 1; k <= 64; ++k) {
    const int32_t p = std::max(1, k * slots / gh);
    if (kappa * rmax / p <= share || p >= 64) {
      pk = std::min(64, p);
      break;
    }
  }
  for (CGroup& g : groups) g.pieces = std::max(1, std::min({pk, g.r, std::max(1, g.rch / 4)}));
  if (const char* fp = std::getenv("HPA_CASC_PIECES"))  // tuning knob: forced pieces per group
    for (CGroup& g : groups) g.pieces = std::max(1, std::min(g.r, std::atoi(fp)));
  std::vector<int32_t> nsplit(r.size());
  int32_t S = 2;  // every request goes through the combine
  for (int32_t i = 0; i < n; ++i) {
    nsplit[size_t(i)] = sp[size_t(i)] + (gof[size_t(i)] >= 0 ? groups[size_t(gof[size_t(i)])].pieces : 0);
    S = std::max(S, nsplit[size_t(i)]);
  }
  if (S > 255) return fail(HPA_ERR_UNSUPPORTED, "cascade plan needs %d partial slots (max 255)", S);
  std::vector<int32_t> key{-7, S};
  key.insert(key.end(), seq_ids, seq_ids + n);
  key.insert(key.end(), sp.begin(), sp.end());
  key.insert(key.end(), r.begin(), r.end());
  for (const CGroup& g : groups) {
    key.push_back(g.pieces);
    key.push_back(int32_t(g.mem.size()));
    key.insert(key.end(), g.mem.begin(), g.mem.end());
  }
  *S_out = S;
  if (key == c->plan_key) return HPA_OK;
  std::vector<int32_t> rec;
  std::vector<std::pair<double, int4>> list;
  for (const CGroup& g : groups) {
    const Seq& rep = c->seqs[seq_ids[g.mem[0]]];
    for (int32_t pc = 0; pc < g.pieces; ++pc) {
      const int32_t ri = int32_t(rec.size()) / kGroupRec;
      const int32_t e0 = int32_t(int64_t(pc) * g.r / g.pieces), e1 = int32_t(int64_t(pc + 1) * g.r / g.pieces);
      rec.resize(rec.size() + kGroupRec, 0);
      int32_t* w = rec.data() + size_t(ri) * kGroupRec;
      w[0] = e0;
      w[1] = e1;
      w[2] = int32_t(g.mem.size());
      for (size_t m = 0; m < g.mem.size(); ++m) {
        w[4 + m] = g.mem[m];
        w[4 + kGroupMax + m] = sp[size_t(g.mem[m])] + pc;
      }
      const double cost = kappa * (rep.pch[size_t(e1 - 1)] - (e0 ? rep.pch[size_t(e0 - 1)] : 0));
      for (int32_t h = 0; h < Hkv; ++h) list.emplace_back(-cost, int4{-2 - ri, seq_ids[g.mem[0]], h, 0});
    }
  }
  for (int32_t i = 0; i < n; ++i) {
    if (sp[size_t(i)] == 0) continue;
    const double cost = double(std::max(1, ch[size_t(i)])) / sp[size_t(i)];
    for (int32_t h = 0; h < Hkv; ++h)
      for (int32_t k = 0; k < sp[size_t(i)]; ++k)
        list.emplace_back(-cost, int4{i, seq_ids[i], h | (k << 8) | (sp[size_t(i)] << 16), r[size_t(i)]});
  }
  std::stable_sort(list.begin(), list.end(), [](const std::pair<double, int4>& x, const std::pair<double, int4>& y) {
    return x.first < y.first;
  });
  const size_t U = list.size();
  if (U > (size_t(1) << 30)) return fail(HPA_ERR_INVALID_ARG, "too many decode work units");
  if (U > c->units_cap) {
    if (c->units_dev) cudaFree(c->units_dev);
    c->units_dev = nullptr;
    c->units_cap = std::max<size_t>(U, 4096);
    HPA_CUDA(cudaMalloc(&c->units_dev, c->units_cap * sizeof(int4)));
  }
  if (size_t(n) > c->nsplit_cap) {
    if (c->nsplit_dev) cudaFree(c->nsplit_dev);
    c->nsplit_dev = nullptr;
    c->nsplit_cap = std::max<size_t>(size_t(n), 1024);
    HPA_CUDA(cudaMalloc(&c->nsplit_dev, c->nsplit_cap * 4));
  }
  if (rec.size() > c->groups_cap) {
    if (c->groups_dev) cudaFree(c->groups_dev);
    c->groups_dev = nullptr;
    c->groups_cap = std::max<size_t>(rec.size(), 64 * kGroupRec);
    HPA_CUDA(cudaMalloc(&c->groups_dev, c->groups_cap * 4));
  }
  const size_t ub = U * sizeof(int4), nb = size_t(n) * 4, gb = rec.size() * 4;
  size_t off;
  if (hpa_status_t st = ring_reserve(c, ub + nb + gb, &off)) return st;
  int4* hu = reinterpret_cast<int4*>(c->ring.host(off));
  for (size_t k = 0; k < U; ++k) hu[k] = list[k].second;
  std::memcpy(c->ring.host(off) + ub, nsplit.data(), nb);
  std::memcpy(c->ring.host(off) + ub + nb, rec.data(), gb);
  HPA_CUDA(cudaMemcpyAsync(c->units_dev, c->ring.host(off), ub, cudaMemcpyHostToDevice, s));
  HPA_CUDA(cudaMemcpyAsync(c->nsplit_dev, c->ring.host(off) + ub, nb, cudaMemcpyHostToDevice, s));
  HPA_CUDA(cudaMemcpyAsync(c->groups_dev, c->ring.host(off) + ub + nb, gb, cudaMemcpyHostToDevice, s));
  HPA_CUDA(c->ring.commit(off, ub + nb + gb, s));
  c->plan_key.swap(key);
  c->plan_units = int32_t(U);
  c->plan_smax = S;
  c->plan_groups = true;
  c->plan_group_units = int32_t(rec.size() / kGroupRec) * Hkv;
  return HPA_OK;
}

hpa_status_t decode_impl(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids, const void* q,
                         void* out, float* part_o, float* part_lse, float softmax_scale, hpa_stream_t stream,
                         const AppendRows* ap) {
#ifdef HPA_HOST_PROF
  double hp_last = hp_now();
#endif
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(HPA_ERR_INVALID_ARG, "layer %d out of range", layer);
  if (n_seqs < 0) return fail(HPA_ERR_INVALID_ARG, "n_seqs < 0");
  if (n_seqs == 0) return HPA_OK;
  if (n_seqs > c->cfg.max_seqs) return fail(HPA_ERR_INVALID_ARG, "n_seqs > max_seqs");
  if (!seq_ids || !q) return fail(HPA_ERR_INVALID_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(HPA_ERR_INVALID_ARG, "q / out must be 16-byte aligned");
  int32_t max_entries = 0, max_chunks = 0;
  for (int32_t i = 0; i < n_seqs; ++i) {
    if (hpa_status_t st = check_seq(c, seq_ids[i])) return st;
    const Seq& s = c->seqs[seq_ids[i]];
    if (s.len == 0) return fail(HPA_ERR_INVALID_ARG, "sequence %d is empty (reading A11)", seq_ids[i]);
    max_entries = std::max(max_entries, seq_entries(s));
    max_chunks = std::max(max_chunks, s.chunks);
  }
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (hpa_status_t st = ship(c, s, {}, {}, 0)) return st;
  if (hpa_status_t st = upload_batch(c, n_seqs, seq_ids, s)) return st;
  HP_MARK(8);
  const int32_t D = c->cfg.head_dim, Hq = c->cfg.num_q_heads, Hkv = c->cfg.num_kv_heads;
  int32_t S = 1;
  if (decode_persistent()) {
    if (Hkv > 255) return fail(HPA_ERR_UNSUPPORTED, "persistent decode supports H_kv <= 255");
    std::vector<CGroup> groups;
    groups = find_cascade_groups(c, n_seqs, seq_ids);
    HP_MARK(9);
    std::vector<int32_t> sp;
    std::vector<int32_t> key;
    if (!groups.empty()) {
      if (hpa_status_t st = plan_cascade(c, n_seqs, seq_ids, groups, s, &S)) return st;
    } else {
      S = plan_request_splits(c, n_seqs, seq_ids, decode_slots(D, Hq / Hkv), sp);
      key.assign(seq_ids, seq_ids + n_seqs);
      key.insert(key.end(), sp.begin(), sp.end());
    }
    HP_MARK(10);
    if (groups.empty() && key != c->plan_key) {
      // unit list, longest unit first (the kernel fetches units dynamically in this order)
      std::vector<std::pair<double, int32_t>> order;  // (-size, request)
      int64_t U = 0;
      for (int32_t i = 0; i < n_seqs; ++i) {
        order.emplace_back(-double(std::max(1, c->seqs[seq_ids[i]].chunks)) / sp[i], i);
        U += int64_t(sp[i]) * Hkv;
      }
      std::stable_sort(order.begin(), order.end(),
                       [](const std::pair<double, int32_t>& x, const std::pair<double, int32_t>& y) {
                         return x.first < y.first;
                       });
      if (U > (int64_t(1) << 30)) return fail(HPA_ERR_INVALID_ARG, "too many decode work units");
      if (size_t(U) > c->units_cap) {
        if (c->units_dev) cudaFree(c->units_dev);
        c->units_dev = nullptr;
        c->units_cap = std::max<size_t>(size_t(U), 4096);
        HPA_CUDA(cudaMalloc(&c->units_dev, c->units_cap * sizeof(int4)));
      }
      if (size_t(n_seqs) > c->nsplit_cap) {
        if (c->nsplit_dev) cudaFree(c->nsplit_dev);
        c->nsplit_dev = nullptr;
        c->nsplit_cap = std::max<size_t>(size_t(n_seqs), 1024);
        HPA_CUDA(cudaMalloc(&c->nsplit_dev, c->nsplit_cap * 4));
      }
      const size_t ub = size_t(U) * sizeof(int4), nb = size_t(n_seqs) * 4;
      size_t off;
      if (hpa_status_t st = ring_reserve(c, ub + nb, &off)) return st;
      int4* hu = reinterpret_cast<int4*>(c->ring.host(off));
      size_t k = 0;
      for (const auto& o : order) {
        const int32_t i = o.second;
        // splits of one (request, head) adjacent: concurrently running units read unrelated
        // pages (heads of one page adjacent measured 7 % slower: HBM channel locality)
        for (int32_t h = 0; h < Hkv; ++h)
          for (int32_t sp_i = 0; sp_i < sp[i]; ++sp_i) hu[k++] = int4{i, seq_ids[i], h | (sp_i << 8) | (sp[i] << 16), 0};
      }
      std::memcpy(c->ring.host(off) + ub, sp.data(), nb);
      HPA_CUDA(cudaMemcpyAsync(c->units_dev, c->ring.host(off), ub, cudaMemcpyHostToDevice, s));
      HPA_CUDA(cudaMemcpyAsync(c->nsplit_dev, c->ring.host(off) + ub, nb, cudaMemcpyHostToDevice, s));
      HPA_CUDA(c->ring.commit(off, ub + nb, s));
      c->plan_key.swap(key);
      c->plan_units = int32_t(U);
      c->plan_smax = S;
      c->plan_groups = false;
      c->plan_group_units = 0;
    }
    HP_MARK(11);
  } else {
    S = plan_splits(c, n_seqs, max_entries, max_chunks);
  }
  if (S > 1 || part_o) {
    const size_t need = size_t(n_seqs) * Hq * S;
    if (need > c->part_elems) {
      if (c->o_part) cudaFree(c->o_part);
      if (c->lse_part) cudaFree(c->lse_part);
      c->o_part = nullptr;
      c->lse_part = nullptr;
      HPA_CUDA(cudaMalloc(&c->o_part, need * D * 4));
      HPA_CUDA(cudaMalloc(&c->lse_part, need * 4));
      c->part_elems = need;
    }
  }
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(float(D));
  DecodeArgs a{c->dt, c->batch_dev, q, out, c->o_part, c->lse_part, c->counters, part_o, part_lse, n_seqs, Hq,
               c->cfg.num_kv_heads,
               Hq / c->cfg.num_kv_heads, c->cfg.page_size, c->cfg.num_pages, layer, S,
               scale * 1.4426950408889634f, c->fp8 ? 1 : 0, c->fp8 ? c->cfg.num_token_pages : 0,
               c->k8_pool, c->v8_pool, c->units_dev, c->nsplit_dev,
               c->counters + size_t(c->cfg.max_seqs) * Hkv, c->plan_units, c->trace,
               decode_persistent() && c->plan_groups ? c->groups_dev : nullptr};
  static const bool force_cs = std::getenv("HPA_FORCE_CS") != nullptr;  // A/B knob: the cascade kernel variant
  if (force_cs && !a.groups && !c->fp8 && decode_persistent() && !ap) a.groups = reinterpret_cast<const int32_t*>(c->units_dev);
  if (c->fp8 && !decode_persistent())
    return fail(HPA_ERR_UNSUPPORTED, "fp8 token pages need the persistent decode kernel");
  int launched = 0;
  cudaError_t e = launch_decode(c->tm_k_dec, c->tm_v_dec, a, D, s, &launched, ap);
  HP_MARK(12);
  c->launches += launched;
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  return HPA_OK;
}
}  // namespace

namespace {
hpa_status_t prefill_impl(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                          const int32_t* q_lens, const int32_t* span, const void* q, void* out,
                          float softmax_scale, hpa_stream_t stream);
}

hpa_status_t hpa_prefill(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                         const int32_t* q_lens, const void* q, void* out, float softmax_scale,
                         hpa_stream_t stream) {
  return prefill_impl(c, layer, n_seqs, seq_ids, q_lens, nullptr, q, out, softmax_scale, stream);
}

hpa_status_t hpa_prefill_span(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                              const int32_t* q_lens, const int32_t* span, const void* q, void* out,
                              float softmax_scale, hpa_stream_t stream) {
  if (!span) return fail(HPA_ERR_INVALID_ARG, "null span");
  return prefill_impl(c, layer, n_seqs, seq_ids, q_lens, span, q, out, softmax_scale, stream);
}

namespace {
hpa_status_t prefill_impl(hpa_cache_t* c, int32_t layer, int32_t n_seqs, const int32_t* seq_ids,
                          const int32_t* q_lens, const int32_t* span, const void* q, void* out,
                          float softmax_scale, hpa_stream_t stream) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(HPA_ERR_INVALID_ARG, "layer %d out of range", layer);
  if (n_seqs < 0) return fail(HPA_ERR_INVALID_ARG, "n_seqs < 0");
  if (n_seqs == 0) return HPA_OK;
  if (!seq_ids || !q_lens || !q || !out) return fail(HPA_ERR_INVALID_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(HPA_ERR_INVALID_ARG, "q / out must be 16-byte aligned");
  std::vector<int32_t> meta(size_t(span ? 6 : 3) * n_seqs);  // rows | q_len | q_off [| span lo,hi,from]
  int64_t total_q = 0;
  int32_t max_q = 0;
  for (int32_t i = 0; i < n_seqs; ++i) {
    if (hpa_status_t st = check_seq(c, seq_ids[i])) return st;
    const Seq& s = c->seqs[seq_ids[i]];
    if (q_lens[i] < 1 || q_lens[i] > s.len)
      return fail(HPA_ERR_INVALID_ARG, "q_lens[%d]=%d must be in [1, seq_len=%d]", i, q_lens[i], s.len);
    meta[i] = seq_ids[i];
    meta[n_seqs + i] = q_lens[i];
    meta[2 * n_seqs + i] = int32_t(total_q);
    if (span) {
      const int32_t lo = span[3 * i], hi = span[3 * i + 1], from = span[3 * i + 2];
      if (lo < 0 || hi < lo || from < hi)
        return fail(HPA_ERR_INVALID_ARG, "span %d must satisfy 0 <= lo <= hi <= q_from", i);
      meta[3 * n_seqs + 3 * i] = lo;
      meta[3 * n_seqs + 3 * i + 1] = hi;
      meta[3 * n_seqs + 3 * i + 2] = from;
    }
    total_q += q_lens[i];
    max_q = std::max(max_q, q_lens[i]);
  }
  if (total_q >= (int64_t(1) << 31)) return fail(HPA_ERR_INVALID_ARG, "too many query rows");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (hpa_status_t st = ship(c, s, {}, {}, 0)) return st;
  // NEXT-4c: the tcgen05 prefill reads bf16 tiles, so a cache with fp8 token pages first
  // dequantizes this layer's token pages of the batch into temporary bf16 pages of the main
  // pool (the pool-to-pool scatter, rows bf16(fp32(code) * scale) as in reading A20) and
  // points the device table entries at them; after the launch the entries are restored and
  // the pages returned (stream order: the host mirror never changes). Same-stream semantics.
  std::vector<int32_t> tmp_pages;
  std::vector<WordWrite> restore;
  // Failure atomicity (include/hpa.h): once table entries may point at temporary pages, every
  // exit -- an error return included -- queues the restoring writes, ships them and returns
  // the temporaries to the allocator. The success path does the same at the end and disarms.
  struct TmpRedirect {
    hpa_cache_t* c;
    cudaStream_t s;
    std::vector<int32_t>& pages;
    std::vector<WordWrite>& restore;
    bool armed = false;
    hpa_status_t undo() {
      armed = false;
      c->pending.insert(c->pending.end(), restore.begin(), restore.end());
      const hpa_status_t st = ship(c, s, {}, {}, 0);
      for (int32_t p : pages) c->alloc.release(p);
      pages.clear();
      return st;
    }
    ~TmpRedirect() {
      if (armed) undo();
    }
  } redirect{c, s, tmp_pages, restore};
  if (c->fp8) {
    const int32_t P = c->cfg.page_size;
    std::vector<char> seen(c->cfg.max_seqs, 0);
    int32_t need = 0;
    for (int32_t i = 0; i < n_seqs; ++i) {
      if (seen[seq_ids[i]]) continue;
      seen[seq_ids[i]] = 1;
      for (const Segment& g : c->seqs[seq_ids[i]].segs)
        if (!g.latent) need += int32_t(g.pages.size());
    }
    if (need > c->alloc.num_free())
      return fail(HPA_ERR_OUT_OF_PAGES, "prefill over fp8 token pages needs %d temporary pages, %d free", need,
                  c->alloc.num_free());
    if (need > 0) {
      c->alloc.alloc(need, tmp_pages);
      redirect.armed = true;
      std::vector<int4> items;  // {fp8 token page, temporary bf16 page, valid rows, 0}
      int32_t k = 0;
      std::fill(seen.begin(), seen.end(), 0);
      for (int32_t i = 0; i < n_seqs; ++i) {
        const int32_t sq = seq_ids[i];
        if (seen[sq]) continue;
        seen[sq] = 1;
        const Seq& q = c->seqs[sq];
        for (size_t e = 0; e < q.pages.size(); ++e) {
          if (q.meta[e] & kMetaLatent) continue;
          const int32_t t = tmp_pages[size_t(k++)], valid = q.meta[e] & kMetaRowsMask;
          items.push_back(make_int4(q.pages[e], t, valid, 0));
          c->pending.push_back({int32_t(c->idx(sq, int32_t(e))), t});
          restore.push_back({int32_t(c->idx(sq, int32_t(e))), q.pages[e]});
        }
      }
      // table entries -> temporary pages (one scatter launch), then the page-granular
      // dequantization of this layer's tiles
      if (hpa_status_t st = ship(c, s, {}, {}, 0)) return st;
      PoolGeom gl = c->geom();  // this layer only
      const int64_t bf_off = int64_t(layer) * c->cfg.num_pages * c->cfg.num_kv_heads * P * c->cfg.head_dim;
      const int64_t f8_rows = int64_t(layer) * c->cfg.num_token_pages * c->cfg.num_kv_heads * P;
      gl.k_pool = static_cast<__nv_bfloat16_raw*>(c->k_pool) + bf_off;
      gl.v_pool = static_cast<__nv_bfloat16_raw*>(c->v_pool) + bf_off;
      gl.k8 = c->k8_pool + f8_rows * (c->cfg.head_dim + 4);  // whole 16-row blocks per layer
      gl.v8 = c->v8_pool + f8_rows * (c->cfg.head_dim + 4);
      gl.L = 1;
      const size_t ib = items.size() * sizeof(int4);
      size_t ioff;
      if (hpa_status_t st = ring_reserve(c, ib, &ioff)) return st;
      std::memcpy(c->ring.host(ioff), items.data(), ib);
      HPA_CUDA(c->ring.upload_side(ioff, ib, s, c->copy_stream, c->upload_done));
      int launched = 1;
      cudaError_t ed = launch_dequant_pages(gl, reinterpret_cast<const int4*>(c->ring.dev(ioff)),
                                            int32_t(items.size()), s);
      c->launches += launched;
      if (ed != cudaSuccess) return cuda_fail(ed, "dequant launch");
      HPA_CUDA(c->ring.commit(ioff, ib, s));
    }
  }
  const int32_t D = c->cfg.head_dim, Hq = c->cfg.num_q_heads;
  // work list (plan_prefill) + per-sequence metadata in one staged upload
  // the plan depends only on the tables, the batch and the split setting: reuse it when those
  // are unchanged since the last call (repeated chunks over a fixed batch skip the simulation)
  std::vector<int32_t> key{int32_t(c->table_version), int32_t(c->table_version >> 32), c->pf_forced_splits,
                           c->pf_ctas, n_seqs, span ? 1 : 0};
  key.insert(key.end(), seq_ids, seq_ids + n_seqs);
  key.insert(key.end(), q_lens, q_lens + n_seqs);
  if (span) key.insert(key.end(), span, span + 3 * size_t(n_seqs));
  if (key != c->pf_key) {
    c->pf_listed = plan_prefill(c, n_seqs, seq_ids, q_lens, meta.data() + 2 * n_seqs, span, c->pf_plan);
    c->pf_key.swap(key);
  }
  const PfPlan& plan = c->pf_plan;
  const bool listed = c->pf_listed;
  const size_t wbytes = listed ? (plan.work.size() + plan.parts.size()) * sizeof(int4) : 0;
  const size_t cbytes = listed ? plan.cta_off.size() * 4 : 0;
  const size_t bytes = wbytes + cbytes + meta.size() * 4;
  size_t off;
  if (hpa_status_t st = ring_reserve(c, bytes, &off)) return st;
  if (listed) {
    std::memcpy(c->ring.host(off), plan.work.data(), plan.work.size() * sizeof(int4));
    std::memcpy(c->ring.host(off) + plan.work.size() * sizeof(int4), plan.parts.data(),
                plan.parts.size() * sizeof(int4));
    if (cbytes) std::memcpy(c->ring.host(off) + wbytes, plan.cta_off.data(), cbytes);
  }
  std::memcpy(c->ring.host(off) + wbytes + cbytes, meta.data(), meta.size() * 4);
  HPA_CUDA(c->ring.upload_side(off, bytes, s, c->copy_stream, c->upload_done));
  const int32_t* dmeta = reinterpret_cast<const int32_t*>(c->ring.dev(off) + wbytes + cbytes);
  CUtensorMap tm_q, tm_o;
  if (!make_map_q(&tm_q, q, uint64_t(total_q), uint64_t(Hq), uint64_t(D), 128) ||
      !make_map_q(&tm_o, out, uint64_t(total_q), uint64_t(Hq), uint64_t(D), 128))
    return fail(HPA_ERR_CUDA, "cuTensorMapEncodeTiled failed for q / out");
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(float(D));
  PrefillArgs a{c->dt, dmeta, dmeta + n_seqs, dmeta + 2 * n_seqs, out, n_seqs, Hq, c->cfg.num_kv_heads,
                Hq / c->cfg.num_kv_heads, c->cfg.page_size, c->cfg.num_pages, layer, max_q,
                scale * 1.4426950408889634f, __builtin_ctz(uint32_t(c->cfg.page_size)),
                span ? dmeta + 3 * n_seqs : nullptr, c->trace, nullptr, 0, nullptr, 0, 1, nullptr, nullptr, nullptr, 0, 0};
  if (listed) {
    const size_t rows = plan.parts.size() / 2 * size_t(plan.split_max) * 2 * 128;
    if (rows > c->pf_part_rows) {  // split workspace (grown on demand) and its fp32 TMA map
      if (c->pf_o_part) cudaFree(c->pf_o_part);
      if (c->pf_lse_part) cudaFree(c->pf_lse_part);
      c->pf_o_part = nullptr;
      c->pf_lse_part = nullptr;
      c->pf_part_rows = 0;
      HPA_CUDA(cudaMalloc(&c->pf_o_part, rows * D * 4));
      HPA_CUDA(cudaMalloc(&c->pf_lse_part, rows * 4));
      if (!make_map_f32(&c->tm_opart, c->pf_o_part, rows, uint64_t(D)))
        return fail(HPA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the prefill workspace");
      c->pf_part_rows = rows;
    }
    const int4* dwork = reinterpret_cast<const int4*>(c->ring.dev(off));
    a.work = dwork;
    a.n_work = int32_t(plan.work.size() / 4);
    a.parts = dwork + plan.work.size();
    a.n_parts = int32_t(plan.parts.size() / 2);
    a.split_max = plan.split_max;
    a.o_part = c->pf_o_part;
    a.lse_part = c->pf_lse_part;
    a.mc2 = plan.mc2 ? 1 : 0;
    if (cbytes) {
      a.cta_off = reinterpret_cast<const int32_t*>(c->ring.dev(off) + wbytes);
      a.n_ctas = int32_t(plan.cta_off.size()) - 1;
    }
  }
  int launched = 0;
  cudaError_t e = launch_prefill(tm_q, c->tm_k_pre, c->tm_v_pre, tm_o, c->tm_opart, a, D, s, &launched);
  c->launches += launched;
  if (e != cudaSuccess) return cuda_fail(e, "prefill launch");
  HPA_CUDA(c->ring.commit(off, bytes, s));
  if (redirect.armed) return redirect.undo();  // NEXT-4c: entries back to the fp8 pages, temporaries freed
  return HPA_OK;
}
}  // namespace

hpa_status_t hpa_seq_info(hpa_cache_t* c, int32_t seq_id, int32_t* len, int32_t* n_pages, int32_t* n_latent_rows) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (hpa_status_t st = check_seq(c, seq_id)) return st;
  const Seq& q = c->seqs[seq_id];
  int32_t lat = 0;
  for (const Segment& g : q.segs) lat += g.latent ? g.rows : 0;
  if (len) *len = q.len;
  if (n_pages) *n_pages = seq_entries(q);
  if (n_latent_rows) *n_latent_rows = lat;
  return HPA_OK;
}

hpa_status_t hpa_export_logical_kv(hpa_cache_t* c, int32_t layer, int32_t seq_id, void* k_out, void* v_out,
                                   hpa_stream_t stream) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(HPA_ERR_INVALID_ARG, "layer %d out of range", layer);
  if (hpa_status_t st = check_seq(c, seq_id)) return st;
  if (!k_out || !v_out || ((reinterpret_cast<uintptr_t>(k_out) | reinterpret_cast<uintptr_t>(v_out)) & 15))
    return fail(HPA_ERR_INVALID_ARG, "k_out / v_out must be 16-byte aligned device pointers");
  DeviceGuard dg(c->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (hpa_status_t st = ship(c, s, {}, {}, 0)) return st;
  HPA_CUDA(launch_export(c->geom(), c->dt, layer, seq_id, seq_entries(c->seqs[seq_id]), k_out, v_out, s));
  c->launches += seq_entries(c->seqs[seq_id]) > 0;
  return HPA_OK;
}

hpa_status_t hpa_export_table(hpa_cache_t* c, int32_t seq_id, int32_t* pages, int32_t* pos0, uint16_t* meta,
                              int32_t cap, int32_t* n_out) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (hpa_status_t st = check_seq(c, seq_id)) return st;
  const Seq& q = c->seqs[seq_id];
  const int32_t n = seq_entries(q);
  if (n_out) *n_out = n;
  if (cap < n) return fail(HPA_ERR_INVALID_ARG, "cap %d < %d entries", cap, n);
  for (int32_t e = 0; e < n; ++e) {
    if (pages) pages[e] = q.pages[e];
    if (pos0) pos0[e] = q.pos0[e];
    if (meta)
      meta[e] = uint16_t((q.meta[e] & kMetaRowsMask) | ((q.meta[e] & kMetaLatent) ? 0x8000 : 0));
  }
  return HPA_OK;
}

hpa_status_t hpa_prefill_plan_info(hpa_cache_t* c, int32_t* n_ctas, int32_t* n_split_units, int32_t* splits,
                                   int32_t* cluster_size) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  const bool l = c->pf_listed;
  if (n_ctas)
    *n_ctas = !l ? 0
              : c->pf_plan.cta_off.empty() ? int32_t(c->pf_plan.work.size() / 4)
                                           : int32_t(c->pf_plan.cta_off.size()) - 1;
  if (n_split_units) *n_split_units = l ? int32_t(c->pf_plan.parts.size() / 2) : 0;
  if (splits) *splits = l ? c->pf_plan.split_max : 1;
  if (cluster_size) *cluster_size = l && c->pf_plan.mc2 ? 2 : 1;
  return HPA_OK;
}

hpa_status_t hpa_set_prefill_ctas(hpa_cache_t* c, int32_t n) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n < -3) return fail(HPA_ERR_INVALID_ARG, "prefill ctas %d < -3", n);
  c->pf_ctas = n;
  return HPA_OK;
}

hpa_status_t hpa_set_prefill_splits(hpa_cache_t* c, int32_t splits) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (splits < 0 || splits > 16) return fail(HPA_ERR_INVALID_ARG, "prefill splits %d outside [0, 16]", splits);
  c->pf_forced_splits = splits;
  return HPA_OK;
}

hpa_status_t hpa_set_decode_splits(hpa_cache_t* c, int32_t splits) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (splits < 0) return fail(HPA_ERR_INVALID_ARG, "splits < 0");
  c->forced_splits = splits;
  return HPA_OK;
}

hpa_status_t hpa_set_decode_cascade(hpa_cache_t* c, int32_t on) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (on < 0 || on > 2) return fail(HPA_ERR_INVALID_ARG, "cascade mode %d outside [0, 2]", on);
  c->cascade = on;
  return HPA_OK;
}

hpa_status_t hpa_decode_plan_info(hpa_cache_t* c, int32_t* n_units, int32_t* n_group_units, int32_t* splits_max) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  if (n_units) *n_units = c->plan_units;
  if (n_group_units) *n_group_units = c->plan_groups ? c->plan_group_units : 0;
  if (splits_max) *splits_max = c->plan_smax;
  return HPA_OK;
}

// Diagnostics (include/hpa.h): device buffer for the HPA_TRACE phase stamps.
hpa_status_t hpa_debug_trace(hpa_cache_t* c, void* device_buf) {
  if (!c) return fail(HPA_ERR_INVALID_ARG, "null cache");
  c->trace = static_cast<long long*>(device_buf);
  return HPA_OK;
}

hpa_status_t hpa_launch_count(hpa_cache_t* c, uint64_t* n) {
  if (!c || !n) return fail(HPA_ERR_INVALID_ARG, "null argument");
  *n = c->launches;
  return HPA_OK;
}

}  // extern "C"
