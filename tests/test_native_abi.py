"""The C-ABI library: it loads, exports every symbol include/kmerscan_b200.h
declares, reports CUDA absence as an error (no crash, no CPU fallback), and the
product package never touches the oracle.  No GPU needed."""

import ctypes
import re
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1509_01506_b200 import _native

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "kmerscan_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^KS_API\s+[\w\s\*]+?\b(ks_\w+)\(", text, flags=re.M)))


def test_header_declares_api():
    syms = header_symbols()
    assert "ks_count" in syms and "ks_locate" in syms and "ks_dfa_upload" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_native.EXPORTED)


def test_version_and_errors_without_device():
    lib = _native.library()
    assert b"sm_100a" in lib.ks_version()
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.ks_open(0, ctypes.byref(h))
    assert rc != 0
    assert lib.ks_last_error()


def test_product_fails_loudly_without_library():
    code = ("import paper_1509_01506_b200 as ks\n"
            "try:\n"
            "    ks.run(ks.build_dfa(ks.expand_to_literals(ks.parse_expressions('acg'))), "
            "ks.sequence_from_text('acgt'))\n"
            "except RuntimeError as e:\n"
            "    print('RAISED', e)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         env={"KMERSCAN_B200_LIB": "/nonexistent/libkmerscan_b200.so", "PATH": "/usr/bin"})
    assert "RAISED" in out.stdout, out.stderr
    assert "native library not found" in out.stdout


def test_product_never_imports_oracle():
    for path in (REPO / "paper_1509_01506_b200").rglob("*.py"):
        text = path.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), path
