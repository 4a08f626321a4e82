"""Plain, slow, obviously-correct fp64 oracle for hybrid paged attention.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Citations: `P:Lnnn` is a
line of the paper text, `S:Lnnn` a line of SPEC.md, `§8(c) Ax` a
reading listed in SURVEY.md §8(c) and DESIGN.md "Readings of the paper".
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Tuple

import numpy as np

META_LATENT_BIT = 1 << 15  # export-table encoding: bit 15 = latent page, low bits = valid rows


def kv_cache_bytes(num_layers: int, num_kv_heads: int, head_dim: int, seq_len: int,
                   elem_bytes: int) -> int:
    """KV size = 2 x L x H_kv x d_h x N x bytes.

    PAPER.md P:L232-235 (§3 "KV cache cost", Eq. KV size); the factor 2 is K and V.
    """
    return 2 * num_layers * num_kv_heads * head_dim * seq_len * elem_bytes


# --------------------------------------------------------------------------- fp8 token pages
# SURVEY §8(f) NEXT-4c ("fp8 token pages with bf16 latent pages"); the paper fixes no fp8
# scheme (it stores bf16), so the scheme is DESIGN.md reading A20:
#   per (layer, token row, kv-head) and per tensor (K, V): amax = max_d |x|,
#   s = fp32(amax / 448) (1 if amax = 0), code = e4m3 RNE-satfinite of fp32(x * fp32(448 / amax));
#   the stored row means code * s. Latent pages stay bf16.
E4M3_MAX = 448.0


def e4m3_values() -> np.ndarray:
    """Value of every e4m3 ("e4m3fn": 1-4-3, bias 7, no inf, S.1111.111 = NaN) code, by the
    format's definition; index = code byte."""
    out = np.zeros(256)
    for c in range(256):
        sign = -1.0 if c & 0x80 else 1.0
        e, m = (c >> 3) & 0xF, c & 0x7
        if e == 0xF and m == 0x7:
            out[c] = np.nan
        elif e == 0:
            out[c] = sign * (m / 8.0) * 2.0 ** -6
        else:
            out[c] = sign * (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return out


def e4m3_encode(y: np.ndarray) -> np.ndarray:
    """float32 -> e4m3 code bytes, round to nearest even, saturating to +-448 (the
    library cast; pinned against a brute-force nearest-value search in the tests)."""
    import torch
    t = torch.from_numpy(np.clip(np.asarray(y, dtype=np.float32), -E4M3_MAX, E4M3_MAX))
    return t.to(torch.float8_e4m3fn).view(torch.uint8).numpy()


def quantize_rows_e4m3(x: np.ndarray):
    """x: [..., d] holding bf16 values. Returns (codes uint8 [..., d], scales float32 [...])
    following reading A20 in fp32, the precision the kernel uses."""
    x32 = np.asarray(x, dtype=np.float32)
    amax = np.max(np.abs(x32), axis=-1)
    pos = amax > 0
    safe = np.where(pos, amax, np.float32(1.0)).astype(np.float32)
    scale = np.where(pos, safe / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    inv = np.where(pos, np.float32(E4M3_MAX) / safe, np.float32(1.0)).astype(np.float32)
    y = (x32 * inv[..., None]).astype(np.float32)
    return e4m3_encode(y), scale


def dequantize_rows_e4m3(codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """code value * scale, exact in fp64 (4-bit x 24-bit significands)."""
    return e4m3_values()[codes] * np.asarray(scales, dtype=np.float64)[..., None]


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16, round to nearest even (torch's cast), returned as fp64 values."""
    import torch
    t = torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.to(torch.float64).numpy()


class _Segment:
    """One segment of a sequence: a run of TOKEN rows or one LATENT set.

    P:L251: "two types of KV cache": regular (prefix + dynamic) KV and the
    compressed KV of meta latent tokens, both stored in blocks.
    K, V: fp64 arrays [L][n][H_kv][d] holding the exact bf16 values.
    """

    def __init__(self, kind: str, set_id: int, k: np.ndarray, v: np.ndarray, q8=None):
        self.kind = kind
        self.set_id = set_id
        self.k = k
        self.v = v
        # fp8 token rows (A20): (k codes, k scales, v codes, v scales), [L][n][H_kv][d] / [L][n][H_kv]
        self.q8 = q8

    @property
    def rows(self) -> int:
        return self.k.shape[1]


class OracleCache:
    """Independent model of the hybrid paged cache at the level of logical rows.

    It never looks at pages; it only records, per sequence, the ordered list of
    segments that the op log produces. Rules:
      * append extends the trailing TOKEN segment, or opens a new one after a
        LATENT set (§8(b) "Append");
      * install with set_id = -1 appends a new LATENT set at the end; set ids are
        a per-sequence counter starting at 0 (reading "set ids");
      * install with an existing set_id replaces that set's rows in place in the
        logical order ("updatable memory", §8(c) A13);
      * remove drops the set; release drops the sequence.
    """

    def __init__(self, num_layers: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
                 page_size: int, token_fp8: bool = False):
        if num_q_heads % num_kv_heads != 0:
            raise ValueError("num_q_heads must be a multiple of num_kv_heads (S:L25)")
        self.L = num_layers
        self.Hq = num_q_heads
        self.Hkv = num_kv_heads
        self.d = head_dim
        self.P = page_size
        self.seqs: Dict[int, List[_Segment]] = {}
        self.next_set: Dict[int, int] = {}
        self.token_fp8 = token_fp8  # NEXT-4c: token rows stored as e4m3 + per-row scales (A20)

    # -- op log ---------------------------------------------------------------
    def create_seq(self, seq_id: int) -> None:
        self.seqs[seq_id] = []
        self.next_set[seq_id] = 0

    def release(self, seq_id: int) -> None:
        del self.seqs[seq_id]
        del self.next_set[seq_id]

    def append(self, seq_id: int, k: np.ndarray, v: np.ndarray) -> None:
        """k, v: [L][n][H_kv][d] (values of the bf16 inputs). With token_fp8 the rows are
        quantized (A20) and the segment holds their dequantized values."""
        k = np.asarray(k, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        q8 = None
        if self.token_fp8:
            kc, ks = quantize_rows_e4m3(k)
            vc, vs = quantize_rows_e4m3(v)
            q8 = (kc, ks, vc, vs)
            k = dequantize_rows_e4m3(kc, ks)
            v = dequantize_rows_e4m3(vc, vs)
        segs = self.seqs[seq_id]
        if segs and segs[-1].kind == "token":
            last = segs[-1]
            last.k = np.concatenate([last.k, k], axis=1)
            last.v = np.concatenate([last.v, v], axis=1)
            if q8 is not None:
                last.q8 = tuple(np.concatenate([a, b], axis=1) for a, b in zip(last.q8, q8))
        else:
            segs.append(_Segment("token", -1, k.copy(), v.copy(), q8))

    def install(self, seq_id: int, set_id: int, kv: np.ndarray) -> int:
        """kv: [L][2][m][H_kv][d] (SPEC CompressedMemory payload)."""
        kv = np.asarray(kv, dtype=np.float64)
        k = kv[:, 0].copy()
        v = kv[:, 1].copy()
        segs = self.seqs[seq_id]
        if set_id < 0:
            set_id = self.next_set[seq_id]
            self.next_set[seq_id] += 1
            segs.append(_Segment("latent", set_id, k, v))
            return set_id
        for s in segs:
            if s.kind == "latent" and s.set_id == set_id:
                s.k, s.v = k, v
                return set_id
        raise KeyError(f"unknown latent set {set_id}")

    def compress(self, seq_id: int, n_doc_rows: int, m_rows: int) -> int:
        """In-cache compression (P:L251 / P:L973: the meta latent
        tokens' KV, computed in the same forward pass as the document, becomes the
        document's compressed memory). Both ranges lie at the end of the trailing
        TOKEN segment: [.., doc (n_doc_rows), latents (m_rows)] ->
        [.., LATENT set (the same m rows)]. Returns the new set id."""
        segs = self.seqs[seq_id]
        if not segs or segs[-1].kind != "token" or segs[-1].rows < n_doc_rows + m_rows or m_rows <= 0:
            raise ValueError("compress needs doc + latent rows at the end of a token segment")
        last = segs[-1]
        keep = last.rows - n_doc_rows - m_rows
        lat_k = last.k[:, keep + n_doc_rows:].copy()
        lat_v = last.v[:, keep + n_doc_rows:].copy()
        if self.token_fp8:  # latent pages are bf16: the moved rows become bf16(fp32(code) * scale)
            kc, ks, vc, vs = (a[:, keep + n_doc_rows:] for a in last.q8)
            lat_k = bf16_round(e4m3_values()[kc].astype(np.float32) * ks[..., None])
            lat_v = bf16_round(e4m3_values()[vc].astype(np.float32) * vs[..., None])
        if keep > 0:
            last.k = last.k[:, :keep].copy()
            last.v = last.v[:, :keep].copy()
            if last.q8 is not None:
                last.q8 = tuple(a[:, :keep].copy() for a in last.q8)
        else:
            segs.pop()
        set_id = self.next_set[seq_id]
        self.next_set[seq_id] += 1
        segs.append(_Segment("latent", set_id, lat_k, lat_v))
        return set_id

    def share(self, dst_seq: int, src_seq: int, src_set_id: int) -> int:
        """Shared document memory ("KV cache server for storing
        and retrieving compressed document memories"): dst_seq gets a new LATENT set whose
        rows are those of src_seq's set src_set_id (the logical model copies the values;
        physical sharing is the cache's business). Returns dst's new set id."""
        for sg in self.seqs[src_seq]:
            if sg.kind == "latent" and sg.set_id == src_set_id:
                set_id = self.next_set[dst_seq]
                self.next_set[dst_seq] += 1
                self.seqs[dst_seq].append(_Segment("latent", set_id, sg.k.copy(), sg.v.copy()))
                return set_id
        raise KeyError(f"unknown latent set {src_set_id}")

    def fork(self, src_seq: int, n_prefix_rows: int, dst_seq: int) -> None:
        """Prefix sharing ("regular KV cache including prefix KV
        cache for user prompts"; reading A21): a new sequence dst_seq whose logical
        content is the first n_prefix_rows rows of src_seq -- the same segments in the same
        order (latent sets keep their set ids; dst's set counter continues from src's), the
        segment holding row n_prefix_rows - 1 cut after it. A cut inside a latent set is
        invalid (a latent set is one compressed memory). The model copies values; physical
        sharing is the cache's business."""
        if dst_seq in self.seqs:
            raise KeyError(f"sequence {dst_seq} exists")
        if not 0 <= n_prefix_rows <= self.seq_len(src_seq):
            raise ValueError("n_prefix_rows outside [0, seq_len]")
        segs, left = [], n_prefix_rows
        for sg in self.seqs[src_seq]:
            if left == 0:
                break
            if sg.rows <= left:
                take = sg.rows
            elif sg.kind == "latent":
                raise ValueError("fork cut inside a latent set")
            else:
                take = left
            q8 = None if sg.q8 is None else tuple(a[:, :take].copy() for a in sg.q8)
            segs.append(_Segment(sg.kind, sg.set_id, sg.k[:, :take].copy(), sg.v[:, :take].copy(), q8))
            left -= take
        self.seqs[dst_seq] = segs
        self.next_set[dst_seq] = self.next_set[src_seq]

    def remove(self, seq_id: int, set_id: int) -> None:
        segs = self.seqs[seq_id]
        for i, s in enumerate(segs):
            if s.kind == "latent" and s.set_id == set_id:
                del segs[i]
                return
        raise KeyError(f"unknown latent set {set_id}")

    # -- views ----------------------------------------------------------------
    def seq_len(self, seq_id: int) -> int:
        return sum(s.rows for s in self.seqs[seq_id])

    def latent_rows(self, seq_id: int) -> int:
        return sum(s.rows for s in self.seqs[seq_id] if s.kind == "latent")

    def logical_kv(self, seq_id: int, layer: int, fp8_staged: bool = False) -> Tuple[np.ndarray, np.ndarray]:
        """Gather route 1: concatenate segments in order -> K, V [H_kv][Lb][d].

        fp8_staged (fp8 token pages only): the rows chunked prefill attends over. Reading A20:
        prefill reads token pages through bf16 staging pages holding bf16(fp32(code) * scale),
        the same conversion as compress; decode reads code * scale directly (the default)."""
        segs = self.seqs[seq_id]
        if not segs:
            z = np.zeros((self.Hkv, 0, self.d))
            return z, z.copy()

        def rows(s, which):
            if fp8_staged and s.q8 is not None:
                codes, scales = (s.q8[0], s.q8[1]) if which == 0 else (s.q8[2], s.q8[3])
                return bf16_round(e4m3_values()[codes[layer]].astype(np.float32) * scales[layer][..., None])
            return (s.k if which == 0 else s.v)[layer]
        k = np.concatenate([rows(s, 0) for s in segs], axis=0)  # [Lb][H_kv][d]
        v = np.concatenate([rows(s, 1) for s in segs], axis=0)
        return k.transpose(1, 0, 2).copy(), v.transpose(1, 0, 2).copy()

    def token_codes(self, seq_id: int, layer: int):
        """fp8 mode: per TOKEN segment in order, (k codes, k scales, v codes, v scales) of
        one layer, [n][H_kv][d] / [n][H_kv] -- for bit-exact checks of the token pools."""
        return [tuple(a[layer] for a in sg.q8) for sg in self.seqs[seq_id] if sg.kind == "token"]

    def expected_table(self, seq_id: int) -> List[Tuple[str, int, int]]:
        """Expected block-table entries (kind, valid_rows, pos0) for this sequence."""
        return expected_table([(s.kind, s.rows) for s in self.seqs[seq_id]], self.P)


def expected_table(segments: List[Tuple[str, int]], page_size: int) -> List[Tuple[str, int, int]]:
    """Block-table entries implied by an ordered segment list.

    SURVEY §8(a) a1 / DESIGN.md reading A7: every segment starts on a fresh page,
    only the last page of a segment may be partial, and pos0 of an entry (the
    logical index of its row 0) is the sum of valid_rows over earlier entries.
    """
    out = []
    pos = 0
    for kind, rows in segments:
        left = rows
        while left > 0:
            take = min(page_size, left)
            out.append((kind, take, pos))
            pos += take
            left -= take
    return out


def gather_physical(k_pool: np.ndarray, v_pool: np.ndarray, pages: List[int],
                    meta: List[int], layer: int) -> Tuple[np.ndarray, np.ndarray]:
    """Gather route 2: walk the block table in order and
    take rows 0..valid_rows-1 of pool[layer][page][h] for each entry.

    k_pool, v_pool: [L][NP][H_kv][P][d] (the device pool layout).
    meta: export-table encoding (bit 15 latent, low 15 bits valid_rows).
    Returns K, V [H_kv][Lb][d].
    """
    ks, vs = [], []
    for page, m in zip(pages, meta):
        valid = m & (META_LATENT_BIT - 1)
        ks.append(k_pool[layer, page, :, :valid, :])
        vs.append(v_pool[layer, page, :, :valid, :])
    if not ks:
        h, d = k_pool.shape[2], k_pool.shape[4]
        z = np.zeros((h, 0, d))
        return z, z.copy()
    return np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)


def attend(q: np.ndarray, k_log: np.ndarray, v_log: np.ndarray, scale: float) -> np.ndarray:
    """fp64 softmax attention of the last Tq logical rows.

    q: [Tq][Hq][d]; k_log, v_log: [H_kv][Lb][d]; returns o [Tq][Hq][d].
    Query row t sits at logical index i = Lb - Tq + t and sees keys j <= i
    (reading A1: mask by logical index in block-table order, bottom-right).
    q-head hq reads kv-head floor(hq / G), G = Hq / H_kv (reading A6).
      s_j = scale * sum_d q[t,hq,d] K[h,j,d];  p_j = exp(s_j - max_j s_j);
      o   = sum_j p_j V[h,j] / sum_j p_j.
    Decode is Tq = 1; chunked prefill is Tq = C.
    """
    q = np.asarray(q, dtype=np.float64)
    k_log = np.asarray(k_log, dtype=np.float64)
    v_log = np.asarray(v_log, dtype=np.float64)
    tq, hq_n, d = q.shape
    hkv, lb, _ = k_log.shape
    if tq > lb or lb == 0:
        raise ValueError("need 1 <= Tq <= Lb (reading A11)")
    group = hq_n // hkv
    out = np.zeros((tq, hq_n, d), dtype=np.float64)
    for hq in range(hq_n):
        h = hq // group
        for t in range(tq):
            i = lb - tq + t
            keys = k_log[h, : i + 1]          # [i+1][d]
            vals = v_log[h, : i + 1]
            s = scale * (keys @ q[t, hq])      # K q^T orientation
            p = np.exp(s - s.max())
            out[t, hq] = (p @ vals) / p.sum()
    return out


def attend_span(q: np.ndarray, k_log: np.ndarray, v_log: np.ndarray, scale: float,
                span_lo: int, span_hi: int, q_from: int) -> np.ndarray:
    """attend() with the GRC mask-out span (SURVEY §8(f) NEXT-4a; §2, P:L177-183:
    "we mask out the k vectors in the first segment when computing attention scores from
    the segment ❸ so that q vectors in segment ❸ only attend to the k vectors of meta
    latent tokens ... while q vectors of meta latent tokens can attend to the k vectors
    in segment ❶"). A query at logical index i >= q_from does not see keys j with
    span_lo <= j < span_hi; other queries follow the plain causal rule (reading A1)."""
    q = np.asarray(q, dtype=np.float64)
    k_log = np.asarray(k_log, dtype=np.float64)
    v_log = np.asarray(v_log, dtype=np.float64)
    tq, hq_n, d = q.shape
    hkv, lb, _ = k_log.shape
    group = hq_n // hkv
    out = np.zeros((tq, hq_n, d), dtype=np.float64)
    for hq in range(hq_n):
        h = hq // group
        for t in range(tq):
            i = lb - tq + t
            keys = [j for j in range(i + 1) if not (i >= q_from and span_lo <= j < span_hi)]
            s = scale * (k_log[h, keys] @ q[t, hq])
            p = np.exp(s - s.max())
            out[t, hq] = (p @ v_log[h, keys]) / p.sum()
    return out


def partial_attend(q: np.ndarray, k_part: np.ndarray, v_part: np.ndarray, scale: float):
    """Context-parallel decode, one shard (SURVEY §8(f) NEXT-4b): attention of one query
    row per head over a shard of the logical keys (all visible: the query is the
    sequence's last row). Returns (o [Hq][d] normalised over the shard,
    lse2 [Hq] = log2 sum_j exp(s_j))."""
    q = np.asarray(q, dtype=np.float64)
    hq_n, d = q.shape
    hkv = k_part.shape[0]
    group = hq_n // hkv
    o = np.zeros((hq_n, d))
    lse2 = np.zeros(hq_n)
    for hq in range(hq_n):
        s = scale * (k_part[hq // group] @ q[hq])
        mx = s.max()
        p = np.exp(s - mx)
        o[hq] = (p @ v_part[hq // group]) / p.sum()
        lse2[hq] = (mx + math.log(p.sum())) / math.log(2.0)
    return o, lse2


def merge_partials(o_parts: np.ndarray, lse2_parts: np.ndarray) -> np.ndarray:
    """o = sum_r 2^(lse_r - LSE) o_r / sum_r 2^(lse_r - LSE): exact recombination of
    shard softmaxes (the same identity as the split combine, a5)."""
    m = lse2_parts.max(axis=0)
    w = np.exp2(lse2_parts - m)                       # [R][Hq]
    return (w[..., None] * o_parts).sum(axis=0) / w.sum(axis=0)[..., None]


def decode_reference(cache: OracleCache, seq_id: int, layer: int, q: np.ndarray,
                     scale: float) -> np.ndarray:
    """Decode: the query is the last logical row (reading A8). q: [Hq][d]."""
    k, v = cache.logical_kv(seq_id, layer)
    return attend(np.asarray(q)[None], k, v, scale)[0]


def prefill_reference(cache: OracleCache, seq_id: int, layer: int, q: np.ndarray,
                      scale: float) -> np.ndarray:
    """Chunked prefill: queries are the last Tq logical rows. q: [Tq][Hq][d]."""
    k, v = cache.logical_kv(seq_id, layer)
    return attend(q, k, v, scale)


def default_scale(head_dim: int) -> float:
    """Reading A5: softmax scale 1/sqrt(d) when the caller passes none."""
    return 1.0 / math.sqrt(head_dim)
