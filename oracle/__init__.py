"""CPU oracle for hybrid paged attention (HPA) -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product path (`paper_2605_09100_b200`) never imports it and has no CPU
fallback; the two share no code (only the input generators in `workloads/`).

What it computes (§3 "Hybrid paged attention for LLM serving",
P:L248-251): HPA is ordinary causal softmax attention over the
*logical* KV sequence of a request; paging and the latent/token tagging change
storage and update cost, not the math ("retain the benefits of paged blocks",
P:L251). So the oracle is the plain definition:

  1. an independent segment-list cache model driven by the same op log as the
     GPU (append / latent install / replace / remove / release);
  2. gather route 1 (model) and route 2 (from a physical pool dump + table);
  3. fp64 softmax attention with the logical-index causal rule (reading A1)
     and GQA head mapping hq -> floor(hq / G) (reading A6).

Pins (tests/test_oracle_*.py, `-m "not gpu"`): pure-Python brute force on tiny
inputs, torch fp64 SDPA with an explicit bottom-right mask, closed forms,
paged == contiguous under random physical permutations, uncompressed
replacement == plain causal attention, chunk == sequential decodes, and the
paper's KV-bytes numbers. Parity of the *values* a trained GRC
model would write into latent pages is unpinned (no weights; synthetic data).
"""
from .hpa_oracle import (  # noqa: F401
    OracleCache,
    attend,
    attend_span,
    merge_partials,
    partial_attend,
    gather_physical,
    kv_cache_bytes,
    expected_table,
    META_LATENT_BIT,
    E4M3_MAX,
    e4m3_values,
    e4m3_encode,
    quantize_rows_e4m3,
    dequantize_rows_e4m3,
    bf16_round,
)
