"""C ABI: libpmg.so loads and exports every symbol include/pmg.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pmg.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    names = declared()
    for must in ("pmg_level_create", "pmg_apply", "pmg_residual", "pmg_half_sweep",
                 "pmg_restrict", "pmg_prolong", "pmg_halo_self", "pmg_dot",
                 "pmg_residual_restrict", "pmg_cg_update"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1307_2036_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpmg.so not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(declared()) <= set(_lib.SIGNATURES)


def test_version_and_error_string_without_gpu():
    from paper_1307_2036_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpmg.so not built")
    lib = _lib.load()
    assert lib.pmg_version() >= 1
    assert lib.pmg_partials_size() > 0
    # a value error path that never touches the device
    rc = lib.pmg_level_create(None, None)
    assert rc == _lib.PMG_ERR_VALUE
    assert b"null" in lib.pmg_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "pmg_level_create")


def test_sm100a_cubin():
    """The library carries sm_100a machine code (cuobjdump --list-elf)."""
    import shutil
    import subprocess
    from paper_1307_2036_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH) or shutil.which("cuobjdump") is None:
        pytest.skip("no library or cuobjdump")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_tracing_switch_without_gpu():
    """The tracing mode is host state: set, read back, refused out of range,
    and a null driver handle reports -1 cycle times."""
    import paper_1307_2036_b200 as pmg
    from paper_1307_2036_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpmg.so not built")
    lib = _lib.load()
    assert not pmg.tracing_enabled()
    with pmg.tracing():
        assert pmg.tracing_enabled() and lib.pmg_get_tracing() == 1
    assert not pmg.tracing_enabled()
    assert lib.pmg_set_tracing(2) == _lib.PMG_ERR_VALUE
    assert lib.pmg_hier_cycle_times(None, None, 0) == -1
    assert lib.pmg_phier_cycle_times(None, None, 0) == -1
