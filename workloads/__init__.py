"""Seeded synthetic workload generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no attention, no paging, no
masking). It only describes the BASELINE.json configurations as op scripts and
draws the seeded bf16 inputs (q, token K/V, latent K/V payloads) that both the
oracle (`oracle/`) and the CUDA path (`paper_2605_09100_b200`) consume.

Input recipe (SURVEY.md §8(d) "Configs as concrete
synthetic inputs"):
  * q, k, v ~ N(0, 1), rounded to bf16 (RNE, torch's conversion).
  * latent payloads come from a separate stream (seed + 1).
  * scale = 1/sqrt(d) (SURVEY §8(c) reading A5).
  * shapes are Qwen3-8B-like GQA: Hq = 32, H_kv = 8, d = 128 (BASELINE.json
    configs[1..4]); the tiny config is 2 q-heads / 1 kv-head, d = 64.
  * a latent set holds m = 128 rows.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

import torch

DATA_SEED = 1234
PLACEMENT_SEED = 99
LATENT_ROWS = 128  # m = N_r, PAPER.md P:L238 (§3 "KV cache cost")


@dataclass
class Shape:
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.head_dim)


# One sequence's build script: list of ("latent", m) / ("tokens", n) segments in
# order, followed by the number of query rows (1 for decode, C for prefill).
@dataclass
class SeqScript:
    segments: List[Tuple[str, int]]
    q_len: int = 1

    @property
    def total_rows(self) -> int:
        return sum(n for _, n in self.segments)


@dataclass
class Workload:
    name: str
    shape: Shape
    seqs: List[SeqScript]
    mode: str  # "decode" | "prefill"
    extra: dict = field(default_factory=dict)


def tiny_decode(variant: str = "a") -> Workload:
    """BASELINE.json configs[0]: 1 sequence, 2 q-heads/1 kv-head, d=64, page 16,
    1 latent page + 3 token pages. Variant b: partial latent page (m=8);
    variant c: prefill of the last 16 rows."""
    shape = Shape(num_layers=1, num_q_heads=2, num_kv_heads=1, head_dim=64, page_size=16)
    m = 8 if variant == "b" else 16
    q_len = 16 if variant == "c" else 1
    seq = SeqScript([("latent", m), ("tokens", 48)], q_len=q_len)
    return Workload(f"tiny_{variant}", shape, [seq], "prefill" if variant == "c" else "decode")


def qwen3_8b_shape(page_size: int = 16, num_layers: int = 1) -> Shape:
    return Shape(num_layers=num_layers, num_q_heads=32, num_kv_heads=8, head_dim=128,
                 page_size=page_size)


def rag_decode(batch: int = 64, docs: int = 8, reasoning: int = 4096, page_size: int = 16,
               ragged: bool = False, seed: int = DATA_SEED) -> Workload:
    """BASELINE.json configs[1]: B=64 decode, 8 retrieved docs compressed to
    m=128-row latent sets + 4K reasoning-token rows (current token included)."""
    g = torch.Generator().manual_seed(seed + 7)
    seqs = []
    for _ in range(batch):
        n_tok = reasoning
        if ragged:
            n_tok = int(torch.randint(1024, 8193, (1,), generator=g).item())
        seqs.append(SeqScript([("latent", LATENT_ROWS)] * docs + [("tokens", n_tok)], 1))
    return Workload(f"rag_decode_b{batch}", qwen3_8b_shape(page_size), seqs, "decode")


def rag_prefill(batch: int = 1, docs: int = 8, cached: int = 16384, chunk: int = 2048,
                page_size: int = 16) -> Workload:
    """BASELINE.json configs[2]: chunked prefill, C=2048 over 8 latent sets
    (1024 rows) + 16384 cached token rows; the chunk's rows are appended and
    are the queries (bottom-right causal)."""
    seqs = [SeqScript([("latent", LATENT_ROWS)] * docs + [("tokens", cached + chunk)], chunk)
            for _ in range(batch)]
    return Workload(f"rag_prefill_b{batch}", qwen3_8b_shape(page_size), seqs, "prefill")


def lmag_decode(batch: int = 256, docs: int = 8, reasoning: int = 4096,
                page_size: int = 16) -> Workload:
    """BASELINE.json configs[3]: batch-256 decode with per-request latent-memory
    replacement between steps (set `step mod docs` replaced each step)."""
    w = rag_decode(batch, docs, reasoning, page_size)
    w.name = f"lmag_b{batch}"
    w.extra["replace_sets"] = docs
    return w


def sweep_decode(batch: int, context: int, latent_ratio: float, page_size: int = 16) -> Workload:
    """BASELINE.json configs[4] (per-rank shard of the 8-GPU sweep). Latent rows =
    floor(r*ctx/128)*128 as whole sets placed first."""
    n_sets = int(latent_ratio * context) // LATENT_ROWS
    tok = context - n_sets * LATENT_ROWS
    seqs = [SeqScript([("latent", LATENT_ROWS)] * n_sets + [("tokens", tok)], 1)
            for _ in range(batch)]
    return Workload(f"sweep_b{batch}_ctx{context}_r{latent_ratio}", qwen3_8b_shape(page_size),
                    seqs, "decode")


class Draw:
    """Seeded bf16 draws. Token KV / q from `seed`, latent payloads from `seed+1`
    (separate streams). `device` may be "cpu" or "cuda"; the same seed on a
    different device gives different values, so parity tests copy the drawn
    inputs (never the kernel outputs) to the host for the oracle."""

    def __init__(self, seed: int = DATA_SEED, device: str = "cpu"):
        self.device = device
        self.g_tok = torch.Generator(device=device).manual_seed(seed)
        self.g_lat = torch.Generator(device=device).manual_seed(seed + 1)
        self.g_q = torch.Generator(device=device).manual_seed(seed + 2)

    def _randn(self, shape, g, scale=1.0):
        x = torch.randn(*shape, generator=g, device=self.device, dtype=torch.float32)
        if scale != 1.0:
            x = x * scale
        return x.to(torch.bfloat16)

    def tokens(self, shape: Shape, n: int, v_scale: float = 1.0):
        """Token K, V, each bf16 [L][n][H_kv][d] (the hpa_append_kv layout)."""
        s = (shape.num_layers, n, shape.num_kv_heads, shape.head_dim)
        return self._randn(s, self.g_tok), self._randn(s, self.g_tok, v_scale)

    def latent(self, shape: Shape, m: int, v_scale: float = 1.0):
        """Latent payload bf16 [L][2][m][H_kv][d] (SPEC payload layout)."""
        s = (shape.num_layers, m, shape.num_kv_heads, shape.head_dim)
        k = self._randn(s, self.g_lat)
        v = self._randn(s, self.g_lat, v_scale)
        return torch.stack([k, v], dim=1).contiguous()

    def queries(self, shape: Shape, n: int):
        """q bf16 [n][Hq][d]."""
        return self._randn((n, shape.num_q_heads, shape.head_dim), self.g_q)
