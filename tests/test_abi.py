"""The C-ABI boundary: the product library loads without a GPU and exports
every function include/*.h declares; the oracle libraries are present; the
product path refuses to run without its native library (no CPU fallback)."""
import ctypes
import pathlib
import re
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        syms |= set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text))
    return syms


def test_header_declares_the_abi():
    syms = declared_symbols()
    for name in ("hs_query", "hs_ctx_create", "hs_stream_create", "hs_event_record", "hs_stream_wait", "hs_launch",
                 "hs_memcpy_h2d", "hs_memcpy_peer", "hs_capture_begin", "hs_graph_launch", "hs_engine_run"):
        assert name in syms


def test_library_exports_every_declared_symbol(native):
    lib = ctypes.CDLL(str(ROOT / "paper_2009_07482_b200" / "libhetsim.so"))
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2009_07482_b200" / "libhetsim.so")],
                        capture_output=True, text=True).stdout
    assert "hs_launch" in nm


def test_python_binding_covers_the_abi(native):
    from paper_2009_07482_b200 import _native
    assert set(_native.EXPORTED_SYMBOLS) == declared_symbols()


def test_version_and_errors_without_gpu(native):
    assert native.hs_version().decode().startswith("hetsim-b200")
    from paper_2009_07482_b200._native import HetsimError, query
    with pytest.raises(HetsimError) as e:
        query({"op": "parse", "spec": "{", "params": {}})
    assert e.value.errc == "MalformedSpec" and e.value.exit_code == 2


def test_launch_rejects_null_arguments(native):
    assert native.hs_launch(None, 0, None, 0, 1) != 0
    assert b"InvalidParam" in native.hs_last_error()


def test_oracle_libraries_present():
    assert (ROOT / "oracle" / "liboracle.so").exists()


def test_no_fallback_without_native_library(tmp_path):
    code = ("import os,sys; os.environ['HETSIM_LIB']='/nonexistent/libhetsim.so'; sys.path.insert(0, %r)\n"
            "from paper_2009_07482_b200 import _native\n"
            "try:\n    _native.lib()\nexcept _native.NativeLibraryMissing:\n    print('refused')\n") % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert "refused" in out.stdout
