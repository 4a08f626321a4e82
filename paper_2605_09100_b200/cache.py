"""`Cache`: Python handle over one hpa_cache_t (one GPU). Marshalling only."""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from ._lib import LIB, HPAConfig, c_i32, c_vp, check


def _i32(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs, dtype=np.int32).reshape(-1))


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # the handle without a Stream object


def _stream(device: int, stream) -> c_vp:
    if stream is None:
        if _raw_stream is not None:
            return c_vp(_raw_stream(device))
        stream = torch.cuda.current_stream(device)
    return c_vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class _CAI:
    """Zero-copy __cuda_array_interface__ view of cache-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str = "<i2"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def merge_partials(o_parts: torch.Tensor, lse_parts: torch.Tensor, stream=None) -> torch.Tensor:
    """hpa_merge_partials: o_parts fp32 [P][n][Hq][d], lse_parts fp32 [P][n][Hq] (CUDA) ->
    bf16 [n][Hq][d]."""
    if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32 or o_parts.device.type != "cuda":
        raise ValueError("partials must be fp32 CUDA tensors")
    o_parts = o_parts.contiguous()
    lse_parts = lse_parts.contiguous()
    n_parts, d = o_parts.shape[0], o_parts.shape[-1]
    rows = lse_parts[0].numel()
    out = torch.empty(o_parts.shape[1:], dtype=torch.bfloat16, device=o_parts.device)
    check(LIB.hpa_merge_partials(n_parts, rows, d, c_vp(o_parts.data_ptr()), c_vp(lse_parts.data_ptr()),
                                 c_vp(out.data_ptr()), _stream(o_parts.device.index, stream)))
    return out


class Cache:
    """Hybrid paged KV cache on one B200 (include/hpa.h, hpa_cache_create).

    Pools: K and V, each bf16 [L][num_pages][H_kv][P][d]; block tables on the
    device; allocator + segment lists on the host.
    """

    def __init__(self, num_layers: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
                 page_size: int, num_pages: int, max_seqs: int, max_pages_per_seq: int,
                 device: int = 0, placement_seed: int = 0, token_kv_dtype: str = "bf16",
                 num_token_pages: int = 0):
        """token_kv_dtype "fp8" (NEXT-4c): token pages are e4m3 + per-row scales in a separate
        pool of num_token_pages pages; latent pages stay bf16 (reading A20)."""
        if token_kv_dtype not in ("bf16", "fp8"):
            raise ValueError("token_kv_dtype must be 'bf16' or 'fp8'")
        self.token_fp8 = token_kv_dtype == "fp8"
        self.num_token_pages = num_token_pages
        self.cfg = HPAConfig(num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages,
                             max_seqs, max_pages_per_seq, device, placement_seed,
                             1 if self.token_fp8 else 0, num_token_pages)
        self.device = device
        self.L, self.Hq, self.Hkv, self.d, self.P = (num_layers, num_q_heads, num_kv_heads,
                                                      head_dim, page_size)
        self.num_pages = num_pages
        h = c_vp()
        check(LIB.hpa_cache_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self._h = h

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            check(LIB.hpa_cache_destroy(self._h))
            self._h = c_vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def seq_create(self) -> int:
        s = c_i32()
        check(LIB.hpa_seq_create(self._h, ctypes.byref(s)))
        return s.value

    def seq_release(self, seq: int) -> None:
        check(LIB.hpa_seq_release(self._h, seq))

    def stats(self) -> Tuple[int, int, int]:
        f, u, l = c_i32(), c_i32(), c_i32()
        check(LIB.hpa_cache_stats(self._h, ctypes.byref(f), ctypes.byref(u), ctypes.byref(l)))
        return f.value, u.value, l.value

    # ------------------------------------------------------------------ checks
    def _dev_tensor(self, t: torch.Tensor, name: str, shape=None) -> int:
        # fast path (one expression, the per-call cost of the decode step's four tensors)
        if (type(t) is torch.Tensor and t.is_cuda and t.dtype is torch.bfloat16 and t.get_device() == self.device
                and t.is_contiguous() and (shape is None or t.shape == shape)):
            return t.data_ptr()
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.device.index != self.device:
            raise ValueError(f"{name} must be a CUDA tensor on cuda:{self.device}")
        if t.dtype != torch.bfloat16:
            raise ValueError(f"{name} must be bf16")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        return t.data_ptr()

    # ------------------------------------------------------------------ a2: append
    def append_kv(self, seq_ids: Sequence[int], n_new: Sequence[int], k: torch.Tensor,
                  v: torch.Tensor, stream=None) -> None:
        """k, v: bf16 [L][sum(n_new)][H_kv][d] on the cache's device (hpa_append_kv)."""
        ids, ns = _i32(seq_ids), _i32(n_new)
        if ids.size != ns.size:
            raise ValueError("seq_ids and n_new differ in length")
        shape = (self.L, int(ns.sum()), self.Hkv, self.d)
        kp = self._dev_tensor(k, "k", shape)
        vp = self._dev_tensor(v, "v", shape)
        check(LIB.hpa_append_kv(self._h, ids.size, _p32(ids), _p32(ns), c_vp(kp), c_vp(vp),
                                _stream(self.device, stream)))

    # ------------------------------------------------------------------ a3: latent sets
    def latent_install(self, seq: int, set_id: int, kv: torch.Tensor, stream=None) -> int:
        """kv: bf16 [L][2][m][H_kv][d]; set_id = -1 appends a new set. Returns the set id."""
        m = kv.shape[2]
        p = self._dev_tensor(kv, "kv", (self.L, 2, m, self.Hkv, self.d))
        out = c_i32()
        check(LIB.hpa_latent_set_install(self._h, seq, set_id, m, c_vp(p),
                                         _stream(self.device, stream), ctypes.byref(out)))
        return out.value

    def latent_install_batch(self, seq_ids: Sequence[int], set_ids: Sequence[int],
                             kvs: Sequence[torch.Tensor], stream=None) -> List[int]:
        """One launch for many installs; kvs[i] bf16 [L][2][m_i][H_kv][d]."""
        ids, sids = _i32(seq_ids), _i32(set_ids)
        ms = _i32([kv.shape[2] for kv in kvs])
        ptrs = (c_vp * len(kvs))(*[self._dev_tensor(kv, "kv", (self.L, 2, kv.shape[2], self.Hkv, self.d))
                                   for kv in kvs])
        out = np.zeros(len(kvs), dtype=np.int32)
        check(LIB.hpa_latent_set_install_batch(self._h, ids.size, _p32(ids), _p32(sids), _p32(ms), ptrs,
                                               _stream(self.device, stream), _p32(out)))
        return out.tolist()

    def latent_install_packed(self, seq_ids, set_ids, kv: torch.Tensor, stream=None) -> np.ndarray:
        """Batched install from one packed payload kv bf16 [n][L][2][m][H_kv][d] (payload i
        installs into seq_ids[i]); one launch, pointer arithmetic done vectorised."""
        ids, sids = _i32(seq_ids), _i32(set_ids)
        n = ids.size
        if kv.dim() != 6 or kv.shape[0] != n:
            raise ValueError("kv must be [n][L][2][m][H_kv][d]")
        m = kv.shape[3]
        self._dev_tensor(kv, "kv", (n, self.L, 2, m, self.Hkv, self.d))
        ptrs = (kv.data_ptr() + np.arange(n, dtype=np.uint64) * np.uint64(kv[0].numel() * 2)).astype(np.uint64)
        ms = np.full(n, m, dtype=np.int32)
        out = np.zeros(n, dtype=np.int32)
        check(LIB.hpa_latent_set_install_batch(self._h, n, _p32(ids), _p32(sids), _p32(ms),
                                               ptrs.ctypes.data_as(ctypes.POINTER(c_vp)),
                                               _stream(self.device, stream), _p32(out)))
        return out

    def compress(self, seq: int, n_doc_rows: int, m_rows: int, stream=None) -> int:
        """In-cache compression (hpa_seq_compress): the last m_rows rows become a LATENT set,
        the n_doc_rows rows before them are dropped. Returns the new set id."""
        out = c_i32()
        check(LIB.hpa_seq_compress(self._h, seq, n_doc_rows, m_rows, _stream(self.device, stream),
                                   ctypes.byref(out)))
        return out.value

    def compress_batch(self, seq_ids, n_doc_rows, m_rows, stream=None) -> np.ndarray:
        """hpa_seq_compress_batch: in-cache compression of several requests, one launch."""
        ids, nd, ms = _i32(seq_ids), _i32(n_doc_rows), _i32(m_rows)
        if not (ids.size == nd.size == ms.size):
            raise ValueError("seq_ids, n_doc_rows and m_rows differ in length")
        out = np.zeros(ids.size, dtype=np.int32)
        check(LIB.hpa_seq_compress_batch(self._h, ids.size, _p32(ids), _p32(nd), _p32(ms),
                                         _stream(self.device, stream), _p32(out)))
        return out

    def latent_install_host(self, seq_ids, set_ids, kv: torch.Tensor, stream=None) -> np.ndarray:
        """hpa_latent_set_install_host: kv is a (preferably pinned) CPU tensor
        [n][L][2][m][H_kv][d] bf16; copied on the cache's copy stream, then installed."""
        ids, sids = _i32(seq_ids), _i32(set_ids)
        n = ids.size
        if kv.device.type != "cpu" or kv.dtype != torch.bfloat16 or not kv.is_contiguous():
            raise ValueError("kv must be a contiguous bf16 CPU tensor")
        if kv.dim() != 6 or kv.shape[0] != n or tuple(kv.shape[1:3]) != (self.L, 2) \
                or tuple(kv.shape[4:]) != (self.Hkv, self.d):
            raise ValueError("kv must be [n][L][2][m][H_kv][d]")
        m = kv.shape[3]
        ptrs = (kv.data_ptr() + np.arange(n, dtype=np.uint64) * np.uint64(kv[0].numel() * 2)).astype(np.uint64)
        ms = np.full(n, m, dtype=np.int32)
        out = np.zeros(n, dtype=np.int32)
        check(LIB.hpa_latent_set_install_host(self._h, n, _p32(ids), _p32(sids), _p32(ms),
                                              ptrs.ctypes.data_as(ctypes.POINTER(c_vp)),
                                              _stream(self.device, stream), _p32(out)))
        return out

    def seq_fork(self, src_seq: int, n_prefix_rows: int) -> int:
        """hpa_seq_fork: a new sequence sharing the first n_prefix_rows rows of src_seq
        (prefix pages referenced, copy-on-write on append). Returns the new sequence id."""
        out = c_i32()
        check(LIB.hpa_seq_fork(self._h, src_seq, n_prefix_rows, ctypes.byref(out)))
        return out.value

    def latent_share(self, dst_seq: int, src_seq: int, src_set_id: int) -> int:
        """hpa_latent_set_share: dst gets a new LATENT set referencing src's pages."""
        out = c_i32()
        check(LIB.hpa_latent_set_share(self._h, dst_seq, src_seq, src_set_id, ctypes.byref(out)))
        return out.value

    def latent_remove(self, seq: int, set_id: int) -> None:
        check(LIB.hpa_latent_set_remove(self._h, seq, set_id))

    # ------------------------------------------------------------------ a4-a6: attention
    def decode(self, layer: int, seq_ids: Sequence[int], q: torch.Tensor,
               out: Optional[torch.Tensor] = None, scale: float = 0.0, stream=None) -> torch.Tensor:
        """q: bf16 [n][Hq][d] -> out bf16 [n][Hq][d] (hpa_decode)."""
        ids = seq_ids if isinstance(seq_ids, np.ndarray) and seq_ids.dtype == np.int32 else _i32(seq_ids)
        shape = (ids.size, self.Hq, self.d)
        qp = self._dev_tensor(q, "q", shape)
        if out is None:
            out = torch.empty(shape, dtype=torch.bfloat16, device=q.device)
        op = self._dev_tensor(out, "out", shape)
        check(LIB.hpa_decode(self._h, layer, ids.size, _p32(ids), c_vp(qp), c_vp(op), float(scale),
                             _stream(self.device, stream)))
        return out

    def append_decode(self, layer: int, seq_ids: Sequence[int], k: torch.Tensor, v: torch.Tensor,
                      q: torch.Tensor, out: Optional[torch.Tensor] = None, scale: float = 0.0,
                      stream=None) -> torch.Tensor:
        """One decode step (hpa_append_decode): append one row per sequence (k, v bf16
        [L][n][H_kv][d]) and decode q bf16 [n][Hq][d] -> out, in one kernel launch."""
        ids = seq_ids if isinstance(seq_ids, np.ndarray) and seq_ids.dtype == np.int32 else _i32(seq_ids)
        n = ids.size
        kp = self._dev_tensor(k, "k", (self.L, n, self.Hkv, self.d))
        vp = self._dev_tensor(v, "v", (self.L, n, self.Hkv, self.d))
        shape = (n, self.Hq, self.d)
        qp = self._dev_tensor(q, "q", shape)
        if out is None:
            out = torch.empty(shape, dtype=torch.bfloat16, device=q.device)
        op = self._dev_tensor(out, "out", shape)
        check(LIB.hpa_append_decode(self._h, layer, n, _p32(ids), c_vp(kp), c_vp(vp), c_vp(qp), c_vp(op),
                                    float(scale), _stream(self.device, stream)))
        return out

    def decode_partial(self, layer: int, seq_ids: Sequence[int], q: torch.Tensor, scale: float = 0.0,
                       stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
        """hpa_decode_partial: (o fp32 [n][Hq][d], lse2 fp32 [n][Hq]) over this cache's shard."""
        ids = _i32(seq_ids)
        qp = self._dev_tensor(q, "q", (ids.size, self.Hq, self.d))
        o = torch.empty((ids.size, self.Hq, self.d), dtype=torch.float32, device=q.device)
        lse = torch.empty((ids.size, self.Hq), dtype=torch.float32, device=q.device)
        check(LIB.hpa_decode_partial(self._h, layer, ids.size, _p32(ids), c_vp(qp), c_vp(o.data_ptr()),
                                     c_vp(lse.data_ptr()), float(scale), _stream(self.device, stream)))
        return o, lse

    def prefill(self, layer: int, seq_ids: Sequence[int], q_lens: Sequence[int], q: torch.Tensor,
                out: Optional[torch.Tensor] = None, scale: float = 0.0, stream=None) -> torch.Tensor:
        """q: bf16 [sum(q_lens)][Hq][d] -> out (hpa_prefill); bottom-right causal."""
        ids, ql = _i32(seq_ids), _i32(q_lens)
        shape = (int(ql.sum()), self.Hq, self.d)
        qp = self._dev_tensor(q, "q", shape)
        if out is None:
            out = torch.empty(shape, dtype=torch.bfloat16, device=q.device)
        op = self._dev_tensor(out, "out", shape)
        check(LIB.hpa_prefill(self._h, layer, ids.size, _p32(ids), _p32(ql), c_vp(qp), c_vp(op),
                              float(scale), _stream(self.device, stream)))
        return out

    def prefill_span(self, layer: int, seq_ids: Sequence[int], q_lens: Sequence[int], spans,
                     q: torch.Tensor, out: Optional[torch.Tensor] = None, scale: float = 0.0,
                     stream=None) -> torch.Tensor:
        """hpa_prefill_span: spans[i] = (lo, hi, q_from) -- GRC mask-out span per sequence."""
        ids, ql = _i32(seq_ids), _i32(q_lens)
        sp = _i32(spans)
        if sp.size != 3 * ids.size:
            raise ValueError("spans must be [n][3]")
        shape = (int(ql.sum()), self.Hq, self.d)
        qp = self._dev_tensor(q, "q", shape)
        if out is None:
            out = torch.empty(shape, dtype=torch.bfloat16, device=q.device)
        op = self._dev_tensor(out, "out", shape)
        check(LIB.hpa_prefill_span(self._h, layer, ids.size, _p32(ids), _p32(ql), _p32(sp), c_vp(qp),
                                   c_vp(op), float(scale), _stream(self.device, stream)))
        return out

    # ------------------------------------------------------------------ introspection
    def seq_info(self, seq: int) -> Tuple[int, int, int]:
        a, b, c = c_i32(), c_i32(), c_i32()
        check(LIB.hpa_seq_info(self._h, seq, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def export_logical_kv(self, layer: int, seq: int, stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
        n, _, _ = self.seq_info(seq)
        k = torch.empty((self.Hkv, n, self.d), dtype=torch.bfloat16, device=f"cuda:{self.device}")
        v = torch.empty_like(k)
        if n:
            check(LIB.hpa_export_logical_kv(self._h, layer, seq, c_vp(k.data_ptr()), c_vp(v.data_ptr()),
                                            _stream(self.device, stream)))
        return k, v

    def export_table(self, seq: int):
        _, n, _ = self.seq_info(seq)
        pages = np.zeros(n, np.int32)
        pos0 = np.zeros(n, np.int32)
        meta = np.zeros(n, np.uint16)
        cnt = c_i32()
        check(LIB.hpa_export_table(self._h, seq, _p32(pages), _p32(pos0),
                                   meta.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), n,
                                   ctypes.byref(cnt)))
        return pages, pos0, meta

    def pools(self) -> Tuple[torch.Tensor, torch.Tensor]:
        """Zero-copy views of the K and V pools, bf16 [L][NP][H_kv][P][d]."""
        kp, vp, nb = c_vp(), c_vp(), ctypes.c_uint64()
        check(LIB.hpa_cache_pools(self._h, ctypes.byref(kp), ctypes.byref(vp), ctypes.byref(nb)))
        shape = (self.L, self.num_pages, self.Hkv, self.P, self.d)
        dev = torch.device(f"cuda:{self.device}")
        k = torch.as_tensor(_CAI(kp.value, shape), device=dev).view(torch.bfloat16)
        v = torch.as_tensor(_CAI(vp.value, shape), device=dev).view(torch.bfloat16)
        return k, v

    def token_pool(self):
        """NEXT-4c fp8 token pool views (include/hpa.h hpa_cache_token_pool): (k codes, v codes)
        uint8 [L][NPt][H_kv][P][d], (k scales, v scales) fp32 [L][NPt][H_kv][P], free token pages.
        The scales are strided views of the 16-row [codes | scales] blocks; K and V codes are
        copies in logical order (the pool stores K chunk-swizzled and V as swizzled key pairs)."""
        k8, v8, free = c_vp(), c_vp(), c_i32()
        check(LIB.hpa_cache_token_pool(self._h, ctypes.byref(k8), ctypes.byref(v8), ctypes.byref(free)))
        dev = torch.device(f"cuda:{self.device}")
        nblk = self.L * self.num_token_pages * self.Hkv * self.P // 16
        blk = 16 * self.d + 64
        views = []
        nch = self.d // 16
        # K rows store their 16-byte chunks XOR-swizzled by the row's index in its 16-row block
        # (include/hpa.h): physical chunk of logical chunk c in row r is c ^ (r & (d/16 - 1))
        r = torch.arange(16, device=dev)[:, None]
        swz = torch.arange(nch, device=dev)[None, :] ^ (r & (nch - 1))
        for ptr, is_k in ((k8.value, True), (v8.value, False)):
            raw = torch.as_tensor(_CAI(ptr, (nblk, blk), "|u1"), device=dev)
            codes = raw[:, :16 * self.d]
            if is_k:  # a logical-order copy
                codes = codes.reshape(nblk, 16, nch, 16)[:, r, swz, :]
            else:
                # V: pair row p holds keys 2p, 2p + 1: dim 16 m + 8 h + g of row r at byte
                # 32 m + 4 g + 2 h + (r & 1), in 2 d/16 chunks of 16 bytes, chunk c at c ^ ((2 p) & 7)
                pr = torch.arange(8, device=dev)[:, None]
                vsw = torch.arange(2 * nch, device=dev)[None, :] ^ ((2 * pr) & 7)
                lin = codes.reshape(nblk, 8, 2 * nch, 16)[:, pr, vsw, :].reshape(nblk, 8, nch, 8, 2, 2)
                # (block, p, m, g, h, parity) -> (block, p, parity, m, h, g)
                codes = lin.permute(0, 1, 5, 2, 4, 3).reshape(nblk, 16, self.d)
            codes = codes.reshape(self.L, self.num_token_pages, self.Hkv, self.P, self.d)
            scales = raw[:, 16 * self.d:].contiguous().view(torch.float32).reshape(
                self.L, self.num_token_pages, self.Hkv, self.P)
            views.append((codes, scales))
        return views[0][0], views[1][0], views[0][1], views[1][1], free.value

    def set_decode_splits(self, splits: int) -> None:
        check(LIB.hpa_set_decode_splits(self._h, splits))

    def set_decode_cascade(self, on) -> None:
        """Cascade decode of shared leading page runs: True / 1 = planner (default), False / 0 =
        off, 2 = every group the planner finds, whatever it saves (testing hook)."""
        check(LIB.hpa_set_decode_cascade(self._h, int(on)))

    def decode_plan_info(self) -> dict:
        """The last decode's plan: work units, cascade group units, partial slots per request."""
        u, g, s = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(LIB.hpa_decode_plan_info(self._h, ctypes.byref(u), ctypes.byref(g), ctypes.byref(s)))
        return {"units": u.value, "group_units": g.value, "splits": s.value}

    def set_prefill_splits(self, splits: int) -> None:
        """0 = planner, 1 = never split, 2..15 = every unit split into that many key ranges,
        16 = the grid kernel without a host work list."""
        check(LIB.hpa_set_prefill_splits(self._h, splits))

    def set_prefill_ctas(self, n: int) -> None:
        """-1 = default (one CTA per item from 4 waves up, else the persistent kernel with stream-K
        shares), -2 = one CTA per item as forced 2-CTA clusters (G % 4 == 0), -3 = one CTA per
        item at every size, 0 = persistent prefill on every SM, n > 0 = at most n CTAs."""
        check(LIB.hpa_set_prefill_ctas(self._h, n))

    def prefill_plan_info(self) -> dict:
        """The last prefill's plan: CTAs launched, units split, key ranges per split unit."""
        n, u, s, cl = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(LIB.hpa_prefill_plan_info(self._h, ctypes.byref(n), ctypes.byref(u), ctypes.byref(s),
                                        ctypes.byref(cl)))
        return {"ctas": n.value, "split_units": u.value, "splits": s.value, "cluster": cl.value}

    def launch_count(self) -> int:
        n = ctypes.c_uint64()
        check(LIB.hpa_launch_count(self._h, ctypes.byref(n)))
        return n.value
