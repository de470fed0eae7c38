"""CPU-side checks of the C ABI: the in-tree library loads and exports every entry
point declared in include/zeco_gla.h (no compute calls: there is no GPU here)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "zeco_gla.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zgla_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for required in ("zgla_zeco_fwd_local", "zgla_zeco_fwd_output", "zgla_zeco_bwd_local", "zgla_zeco_bwd_output",
                     "zgla_allscan_local", "zgla_allscan_run", "zgla_local_state_scan", "zgla_backward"):
        assert required in syms


def test_library_exports_every_declared_symbol():
    from paper_2507_01004_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run make)")
    lib = _native.load()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers the header too
    assert set(header_symbols()) <= set(_native.EXPORTED)


def test_version_and_error_string_without_gpu():
    from paper_2507_01004_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run make)")
    lib = _native.load()
    assert b"sm_100a" in lib.zgla_version()
    assert isinstance(lib.zgla_last_error(), bytes)


def test_status_codes_map_to_reference_exceptions():
    from paper_2507_01004_b200 import _native, errors

    for code, exc in ((-1, errors.DimsError), (-2, errors.DomainError), (-3, errors.LayoutError),
                      (-4, errors.ConfigError), (-5, errors.StateError), (-6, errors.DeadlockError)):
        if not os.path.exists(_native.LIB_PATH):
            pytest.skip("library not built")
        with pytest.raises(exc):
            _native.check(code, "probe")


def test_invalid_shapes_rejected_before_any_launch():
    """Argument validation happens on the host side of the C ABI (no device needed)."""
    import ctypes

    from paper_2507_01004_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load()
    bad = _native.Shape(heads=2, key_dim=4, value_dim=4, chunk_len=3, seq_len=8, dtype=_native.ZGLA_F64)
    assert lib.zgla_workspace_bytes(ctypes.byref(bad)) == -1           # chunk does not divide L
    assert lib.zgla_zeco_workspace_bytes(ctypes.byref(bad), 148) == -1
    ok = _native.Shape(heads=16, key_dim=128, value_dim=128, chunk_len=64, seq_len=16384, dtype=_native.ZGLA_BF16)
    assert lib.zgla_zeco_workspace_bytes(ctypes.byref(ok), 148) > 0
    assert lib.zgla_allscan_local(2, 1, 4, 4, _native.ZGLA_F32, 3, 0, None, None, None, None, None) == -4


def test_plain_c_client_compiles_and_links(tmp_path):
    """The header is plain C99 and the library links into a C program (no torch / C++ in the ABI)."""
    import os
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "client.c"
    src.write_text(
        '#include "zeco_gla.h"\n#include <stdio.h>\n'
        "int main(void) {\n"
        "  zgla_shape s = {16, 128, 128, 64, 16384, ZGLA_BF16};\n"
        "  zgla_tensor t = {0, 0, 0};\n  (void)t;\n"
        "  long long ws = zgla_zeco_workspace_bytes(&s, 148);\n"
        '  printf("%s %lld\\n", zgla_version(), ws);\n'
        "  return ws > 0 ? 0 : 1;\n}\n")
    lib = os.path.join(root, "paper_2507_01004_b200")
    exe = tmp_path / "client"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"), str(src),
                    "-L", lib, "-lzeco_gla", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert out.startswith("zeco-gla-b200")


def test_integration_ctypes_stub_matches_header():
    """The ctypes binding shown in INTEGRATION.md declares the same arity as include/zeco_gla.h."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    header = open(os.path.join(root, "include", "zeco_gla.h")).read()
    doc = open(os.path.join(root, "INTEGRATION.md")).read()
    stub = re.findall(r'"(zgla_\w+)":\s*\[ctypes\.POINTER\(_Shape\), ctypes\.c_int\](?:\s*\+\s*\[_V\]\s*\*\s*(\d+))?', doc)
    assert len(stub) >= 5
    for name, n in stub:
        m = re.search(r"\b" + name + r"\s*\(([^;]*?)\)\s*;", header, re.S)
        assert m, name
        assert len(m.group(1).split(",")) == 2 + int(n or 0), name
