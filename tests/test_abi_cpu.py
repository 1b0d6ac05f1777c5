"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU, exports every entry point include/swb200.h declares, the ctypes
signatures cover all of them, and argument validation maps onto the
reference's exception types (errors.py) without touching a device."""

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "swb200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(swb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert len(names) >= 25
    for must in ("swb_gemm_bf16", "swb_gemv_bf16", "swb_attn_prefill", "swb_attn_decode",
                 "swb_kv_push_layer", "swb_block_alloc", "swb_kv_pool_ipc_open"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2311_18677_b200 import _abi
    lib = C.CDLL(_abi.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(_abi.SIGNATURES), \
        set(_declared()) ^ set(_abi.SIGNATURES)
    assert _abi.lib.swb_abi_version() == 1


def test_validation_errors_map_to_reference_types():
    from paper_2311_18677_b200 import _abi
    from paper_2311_18677_b200.errors import ValidationError
    # bad shapes are rejected on the host before any launch
    with pytest.raises(ValidationError):
        _abi.call("swb_gemm_bf16", 16, 16, 16, None, 0, 256, 64, 0, 0)
    with pytest.raises(ValidationError):
        _abi.call("swb_gemm_bf16", 16, 16, 16, None, 128, 256, 60, 0, 0)   # K % 8
    with pytest.raises(ValidationError):
        _abi.call("swb_gemv_bf16", 16, 16, 16, None, 33, 256, 64, 0, 0)    # M > 32
    with pytest.raises(ValidationError):
        _abi.call("swb_attn_decode", 16, 8, 16, 16, 16, 4, 16, None, None, 1e4, None, 1, 8, 8,
                  64, 16, 1.0, 64, 64, 16, 16, 0)                           # dh != 128
    with pytest.raises(ValidationError):
        _abi.call("swb_gemm_bf16_bias", 16, 16, 16, None, 16, 128, 256, 64, 3, 0)  # bias+SwiGLU
    with pytest.raises(ValidationError):
        _abi.call("swb_layernorm", 16, None, 16, 16, 16, 4, 30, 1e-5, 0, 0)       # d % 4
    with pytest.raises(ValidationError):
        _abi.call("swb_kv_pool_create", 0, 10, 1, 16, 128, 1, 1, C.byref(C.c_void_p()))
    assert "K=60" in _abi.last_error() or "positive" in _abi.last_error()


def test_sass_contains_tcgen05_and_tma():
    """The shipped library is sm_100a code: tcgen05 MMA / TMEM loads / TMA."""
    import shutil
    import subprocess
    from paper_2311_18677_b200 import _abi
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "sm_100a" in subprocess.run([tool, "-lelf", _abi.LIB_PATH], capture_output=True,
                                       text=True).stdout
