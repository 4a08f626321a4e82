"""Short all-API random fuzz against the oracle (tests/hpa_fuzz_all.py): create / release, bulk
append, the fused step, latent install / replace / remove / share, fork, compress and
compress-batch, host-staged install; bit-exact views and decode (cascade on and off),
decode_partial, prefill, prefill_span and fused-step parity every 25 ops, at the north_star
tolerance. scripts/fuzz_all.py runs the long version (profiles/r2_fuzz_all.log)."""
import pytest

from tests.hpa_fuzz_all import run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,fp8", [(1, False), (3, False), (6, False), (1, True), (5, True)])
def test_fuzz_all_api(seed, fp8):
    _, st = run(seed, 250, fp8, 25, strict=True)
    assert st["checks"] >= 8, st
