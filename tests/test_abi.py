"""The C-ABI shared library loads on a CPU-only box and exports every symbol
include/ckks_b200.h declares (no compute calls)."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "ckks_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ckks_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_loads_and_exports_header_symbols():
    from paper_2512_18345_b200 import _lib

    _lib.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 19
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert sorted(_lib.SYMBOLS) == names
    lib.ckks_abi_version.restype = ctypes.c_int
    assert lib.ckks_abi_version() == _lib.ABI_VERSION


def test_ctx_create_without_gpu_reports_error_not_fallback():
    import torch

    from paper_2512_18345_b200 import _lib

    if torch.cuda.is_available():
        return
    lib = _lib.load()
    h = ctypes.c_void_p()
    status = lib.ckks_ctx_create(0, ctypes.byref(h))
    assert status == 2 and not h.value
    assert b"no CPU fallback" in lib.ckks_last_error()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2512_18345_b200"
    for path in pkg.rglob("*.py"):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path
