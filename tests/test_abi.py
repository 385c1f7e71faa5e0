"""The C-ABI library builds, loads without a GPU and exports every symbol in include/vx_api.h."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "vx_api.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char\*|void)\s+(vx_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("vx_gemm", "vx_attention", "vx_layernorm", "vx_patchify", "vx_special_tokens", "vx_last_error"):
        assert s in syms


def test_library_exports_all_declared_symbols():
    from paper_2509_25191_b200 import build, ops
    build.build()
    lib = ops.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(ops.EXPORTED_SYMBOLS) == set(declared_symbols())
    assert b"sm_100a" in lib.vx_version()


def test_argument_errors_are_reported_without_gpu():
    """Shape validation happens before any CUDA call and surfaces through vx_last_error."""
    from paper_2509_25191_b200 import ops
    lib = ops.load_library()
    ep = ops.Epilogue()
    rc = lib.vx_gemm(0, ctypes.c_void_p(16), 64, ctypes.c_void_p(16), 64, 128, 128, 100, ctypes.byref(ep), None)
    assert rc == -1
    assert b"multiple of 64" in lib.vx_last_error()
    rc = lib.vx_attention(None, None, None, None, 64, None, 64, 1, 1, 1, 1, 1, 1, None)
    assert rc == -1 and b"null" in lib.vx_last_error()
    rc = lib.vx_layernorm(ctypes.c_void_p(16), 0, 1000, ctypes.c_void_p(16), 1, 1000, None, None, 4, 1000, 1e-5, None)
    assert rc == -1


def test_sass_contains_tcgen05_and_tma():
    """Blackwell-native evidence: UTC*MMA (tcgen05.mma), LDTM (tcgen05.ld), UTMALDG (TMA) in the .so."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump") and not Path("/usr/local/cuda/bin/cuobjdump").exists():
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", str(ROOT / "paper_2509_25191_b200" / "libvx.so")],
                          capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass
    assert "LDTM" in sass
    assert "UTMALDG" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_launch_counter_ignores_rejected_calls():
    """vx_launch_count (bench.py's gpu_launches) counts kernels, not calls: a call rejected by
    argument validation launches nothing."""
    from paper_2509_25191_b200 import ops
    lib = ops.load_library()
    before = ops.kernel_launches()
    rc = lib.vx_layernorm(None, 0, 0, None, 0, 0, None, None, 0, 0, 1e-5, None)
    assert rc != 0
    assert ops.kernel_launches() == before == lib.vx_launch_count()
