"""The C ABI library loads and exports every symbol its headers declare (CPU only)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared(header):
    text = Path(header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ptb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paratime_b200 as B

    lib = B.lib()  # raises when the library was not built: no fallback
    names = declared(ROOT / "include" / "paratime_b200.h")
    assert len(names) > 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_reports_version_and_errors_without_gpu():
    import paratime_b200 as B

    lib = B.lib()
    assert b"sm_100a" in lib.ptb_version()
    h = ctypes.c_void_p()
    # no device in this container (or a bad ordinal): a clean error, not a crash
    st = lib.ptb_context_create(ctypes.c_int(10_000), ctypes.byref(h))
    assert st != 0
    assert lib.ptb_last_error()


def test_oracle_ref_library_exports():
    from oracle import refbind

    if not refbind.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    lib = refbind.lib()
    for n in ["ref_propagate", "ref_parareal_run", "ref_update_svd", "ref_build_setup", "ref_interpolate"]:
        assert hasattr(lib, n)
