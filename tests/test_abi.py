"""The C-ABI library loads, exports every symbol include/ldpc.h declares, and
validates codes on the host (no GPU needed for these checks)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import ldpcgen as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import paper_cs_0609090_b200 as P
    if not os.path.exists(P.LIB_PATH):
        subprocess.check_call(["make", "-C", ROOT, "paper_cs_0609090_b200/libldpc.so"])
    return P


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "ldpc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ldpc_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported(L):
    syms = _header_symbols()
    assert len(syms) >= 12
    assert sorted(L.EXPORTS) == syms
    lib = L.lib()
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_library_has_sm100a_code(L):
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(L):
    assert L.ldpc_status_string(0) == "LDPC_OK"
    assert L.ldpc_status_string(3) == "LDPC_ERR_UNSUPPORTED"
    assert L.ldpc_version() >= 100


def _create(L, code):
    d, keep = L.make_desc(code)
    h = ctypes.c_void_p()
    st = L.lib().ldpc_code_create(ctypes.byref(d), 0, ctypes.byref(h))
    return st, L.ldpc_last_error_detail()


class _C:
    def __init__(self, N, M, rp, ci, **kw):
        self.n_vars, self.n_checks = N, M
        self.row_ptr, self.col_idx = np.array(rp, np.int32), np.array(ci, np.int32)
        self.qc_z = kw.get("qc_z", 0)
        self.qc_rows, self.qc_cols, self.qc_shift = kw.get("qc_rows", 0), kw.get("qc_cols", 0), kw.get("qc_shift")


@pytest.mark.parametrize("code,msg", [
    (_C(3, 2, [0, 2, 4], [0, 0, 1, 2]), "duplicate column"),
    (_C(3, 2, [0, 2, 4], [1, 0, 1, 2]), "not strictly increasing"),
    (_C(3, 2, [0, 1, 3], [0, 1, 2]), "degree 1 < 2"),
    (_C(4, 2, [0, 2, 4], [0, 1, 1, 2]), "column 3 has degree 0"),
    (_C(3, 2, [0, 2, 4], [0, 1, 1, 7]), "out of range"),
    (_C(3, 2, [1, 2, 4], [0, 1, 1, 2]), "row_ptr[0]"),
])
def test_invalid_codes_rejected_on_host(L, code, msg):
    st, detail = _create(L, code)
    assert st == L.LDPC_ERR_INVALID_CODE
    assert msg in detail


def test_qc_mismatch_rejected(L):
    c = g.qc(2, 4, 5, np.array([1, 2, 1, 2], np.int32), seed=1)
    bad = _C(c.n_vars, c.n_checks, c.row_ptr, c.col_idx, qc_z=5, qc_rows=2, qc_cols=4,
             qc_shift=np.where(c.qc_shift >= 0, (c.qc_shift + 1) % 5, -1).astype(np.int16))
    st, detail = _create(L, bad)
    assert st == L.LDPC_ERR_INVALID_CODE and "QC" in detail


def test_valid_code_without_gpu_reports_cuda(L):
    """On a host without a GPU a valid code passes validation and fails at the device step."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    st, detail = _create(L, g.regular(48, 3, 6, seed=1))
    assert st == L.LDPC_ERR_CUDA


def test_product_path_does_not_import_oracle():
    """The product package never imports the oracle (or any CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_cs_0609090_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src and "engine.inc" not in src, f
