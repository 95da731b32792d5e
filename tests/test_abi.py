"""C-ABI library: loads on CPU and exports every symbol include/nysb200.h declares."""
import os
import re

from paper_2510_04094_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "nysb200.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|size_t|unsigned long long|const char\*)\s+(nys_[a-z0-9_]+)\(", txt, re.M)))


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    assert lib.nys_abi_version() == 1
    for name in _header_symbols():
        assert hasattr(lib, name), name
    assert set(_header_symbols()) == set(_lib.exported_symbols())


def test_status_strings():
    lib = _lib.load()
    assert lib.nys_status_string(0) == b"ok"
    assert b"workspace" in lib.nys_status_string(3)


def test_workspace_queries_are_host_only():
    lib = _lib.load()
    assert lib.nys_batch_gram_workspace_bytes(4095, 64, 2, 4096) > 0
    assert lib.nys_fused_gram_workspace_bytes(9999, 50, 50, 2) > 0
    assert lib.nys_kkt_workspace_bytes(64, 2, 4096) == 0          # fits shared memory
    assert lib.nys_kkt_workspace_bytes(256, 2, 1) > 0             # config 4: L2 workspace
