"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every entry point include/mlck_b200.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlck_b200.h")
LIB = os.path.join(ROOT, "paper_2412_15411_b200", "_build", "libmlck_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mlck_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared()
    for must in ("mlck_snapshot_record", "mlck_fnv1a64", "mlck_parse_record", "mlck_check_coverage",
                 "mlck_sparse_to_dense_convert", "mlck_optimizer_step_adam", "mlck_log_put", "mlck_gc_logs",
                 "mlck_state_serialize", "mlck_dense_checkpoint"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libmlck_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_last_error_is_callable_without_gpu():
    if not os.path.exists(LIB):
        pytest.skip("libmlck_b200.so not built")
    lib = ctypes.CDLL(LIB)
    lib.mlck_last_error.restype = ctypes.c_char_p
    assert lib.mlck_last_error() == b""
