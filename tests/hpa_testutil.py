"""Shared helpers for the GPU parity tests: drive the CUDA cache and the oracle
cache with the same op log on the same seeded inputs (workloads.Draw, CPU)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import OracleCache
from workloads import Draw, Shape

# BASELINE.json north_star tolerance: max abs <= 1e-2, relative L2 <= 5e-3
MAX_ABS = 1e-2
REL_L2 = 5e-3


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def check_close(got: torch.Tensor, ref: np.ndarray, what: str = ""):
    g = f64(got)
    err = np.abs(g - ref)
    max_abs = float(err.max()) if err.size else 0.0
    rel = float(np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30))
    assert np.all(np.isfinite(g)), f"{what}: non-finite output"
    assert max_abs <= MAX_ABS and rel <= REL_L2, f"{what}: max_abs={max_abs:.3e} rel_l2={rel:.3e}"
    return max_abs, rel


class Pair:
    """A CUDA `Cache` and an `OracleCache` fed the same ops."""

    def __init__(self, shape: Shape, num_pages: int, max_seqs: int, max_pages_per_seq: int,
                 placement_seed: int = 99, seed: int = 1234, v_scale: float = 1.0,
                 token_fp8: bool = False, num_token_pages: int = 0):
        from paper_2605_09100_b200 import Cache
        self.shape = shape
        self.cache = Cache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                           shape.page_size, num_pages, max_seqs, max_pages_per_seq, 0, placement_seed,
                           "fp8" if token_fp8 else "bf16", num_token_pages)
        self.orc = OracleCache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads,
                               shape.head_dim, shape.page_size, token_fp8=token_fp8)
        self.draw = Draw(seed)
        self.v_scale = v_scale

    def new_seq(self) -> int:
        s = self.cache.seq_create()
        self.orc.create_seq(s)
        return s

    def latent(self, s: int, m: int, set_id: int = -1) -> int:
        kv = self.draw.latent(self.shape, m, self.v_scale)
        got = self.cache.latent_install(s, set_id, kv.cuda())
        exp = self.orc.install(s, set_id, f64(kv))
        assert got == exp
        return got

    def tokens(self, seqs, ns):
        k, v = self.draw.tokens(self.shape, int(sum(ns)), self.v_scale)
        self.cache.append_kv(seqs, ns, k.cuda(), v.cuda())
        off = 0
        for s, n in zip(seqs, ns):
            self.orc.append(s, f64(k[:, off:off + n]), f64(v[:, off:off + n]))
            off += n

    def build(self, script) -> int:
        s = self.new_seq()
        for kind, n in script:
            if kind == "latent":
                self.latent(s, n)
            else:
                self.tokens([s], [n])
        return s

    def queries(self, n: int) -> torch.Tensor:
        return self.draw.queries(self.shape, n)
