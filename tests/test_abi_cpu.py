"""CPU-only checks of the C-ABI boundary: the library builds/loads without a GPU,
exports every symbol include/hpa.h declares, the binding declares each one,
and the pure host arithmetic matches the paper (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hpa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2605_09100_b200 import _lib
    names = header_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(_lib.lib_path())
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.SIGNATURES) == names  # binding mirrors the header one to one


def test_kv_bytes_through_the_abi():
    """hpa_kv_bytes (host arithmetic) vs the numbers printed in the paper."""
    from paper_2605_09100_b200 import kv_bytes
    assert kv_bytes(28, 8, 128, 1, 2) == 114688
    assert kv_bytes(28, 8, 128, 1024, 2) == 112 * 2 ** 20
    assert kv_bytes(28, 8, 128, 128, 2) == 14 * 2 ** 20


def test_status_strings_and_no_silent_cpu_path():
    """Without a usable sm_100 GPU, cache creation must fail loudly (no fallback)."""
    import torch
    from paper_2605_09100_b200 import Cache, HPAError
    from paper_2605_09100_b200._lib import LIB
    assert LIB.hpa_status_string(2) == b"HPA_ERR_OUT_OF_PAGES"
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by -m gpu tests")
    with pytest.raises(HPAError):
        Cache(1, 2, 1, 64, 16, 8, 1, 8)


def test_sass_contains_blackwell_instructions():
    """The built library holds tcgen05 MMA (UTCHMMA), TMEM ld/st and TMA loads."""
    import shutil
    import subprocess
    from paper_2605_09100_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", _lib.lib_path()], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "UTMALDG", "HMMA.16816.F32.BF16"):
        assert mnemonic in sass, mnemonic
