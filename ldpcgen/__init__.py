"""Seeded synthetic inputs (parity-check matrices and channel LLRs).

This module holds NONE of the decoding method's arithmetic.  It is the only code
shared by the CPU oracle side (``oracle/``, tests) and the CUDA side
(``paper_cs_0609090_b200``, bench): it builds the codes of BASELINE.json's five
configs and the AWGN channel LLRs they are decoded from.

Channel model: BPSK over AWGN, all-zero codeword, y = 1 + sigma*g,
Z0 = 2y/sigma^2 (§2); quantisation is round-half-even of
Z0*2^f then a symmetric clamp +-Q.
The paper's workloads (China-DTMB QC codes, DVB-S2 codes, MacKay codes --
PAPER.md:72-75, §1) are not available; the synthetic codes below have their
shapes.
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libldpcgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile libldpcgen.so in-tree with gcc (plain C, pthreads, libm)."""
    src = os.path.join(_HERE, "ldpcgen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _LIB_PATH, src, "-lm", "-lpthread"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.lg_regular.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, i32p, i32p]
        L.lg_regular.restype = ctypes.c_int
        L.lg_qc_base.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, ctypes.c_uint64,
                                 ctypes.POINTER(ctypes.c_int16)]
        L.lg_qc_base.restype = ctypes.c_int
        L.lg_qc_expand.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int16), i32p, i32p]
        L.lg_qc_expand.restype = ctypes.c_int
        L.lg_dvbs2like.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_uint64, i32p, i32p]
        L.lg_dvbs2like.restype = ctypes.c_int
        L.lg_llr.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        L.lg_llr.restype = ctypes.c_int
        L.lg_gauss_pair.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.lg_splitmix64.argtypes = [ctypes.c_uint64]
        L.lg_splitmix64.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


@dataclass
class Code:
    """H as CSR over check rows (0-based, columns strictly increasing per row),
    plus the optional quasi-cyclic description (base shift table, -1 = empty)."""
    n_vars: int
    n_checks: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    qc_z: int = 0
    qc_rows: int = 0
    qc_cols: int = 0
    qc_shift: Optional[np.ndarray] = None
    name: str = ""

    @property
    def n_edges(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def K(self) -> int:
        """Information bits per frame for the design rate R = 1 - M/N."""
        return self.n_vars - self.n_checks

    @property
    def rate(self) -> float:
        return 1.0 - self.n_checks / self.n_vars

    def row_degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def col_degrees(self) -> np.ndarray:
        return np.bincount(self.col_idx, minlength=self.n_vars)

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.array([self.n_vars, self.n_checks], np.int64).tobytes())
        h.update(self.row_ptr.astype(np.int32).tobytes())
        h.update(self.col_idx.astype(np.int32).tobytes())
        return h.hexdigest()

    def dense(self) -> np.ndarray:
        H = np.zeros((self.n_checks, self.n_vars), np.uint8)
        for m in range(self.n_checks):
            H[m, self.col_idx[self.row_ptr[m]:self.row_ptr[m + 1]]] = 1
        return H


def from_dense(H: np.ndarray, name: str = "") -> Code:
    H = np.asarray(H, dtype=np.uint8)
    M, N = H.shape
    rp = [0]
    ci = []
    for m in range(M):
        cols = np.nonzero(H[m])[0]
        ci.extend(int(c) for c in cols)
        rp.append(len(ci))
    return Code(N, M, np.array(rp, np.int32), np.array(ci, np.int32), name=name)


def regular(N: int, dv: int, dc: int, seed: int, remove_4cycles: bool = True) -> Code:
    M = N * dv // dc
    rp = np.zeros(M + 1, np.int32)
    ci = np.zeros(N * dv, np.int32)
    rc = lib().lg_regular(N, dv, dc, seed, int(remove_4cycles), _p(rp, ctypes.c_int32), _p(ci, ctypes.c_int32))
    if rc < 0:
        raise RuntimeError(f"regular code construction failed (N={N}, dv={dv}, dc={dc})")
    return Code(N, M, rp, ci, name=f"reg({dv},{dc}) N={N} seed={seed}")


def qc(mb: int, nb: int, Z: int, col_w, seed: int) -> Code:
    col_w = np.ascontiguousarray(col_w, np.int32)
    sh = np.zeros(mb * nb, np.int16)
    if lib().lg_qc_base(mb, nb, Z, _p(col_w, ctypes.c_int32), seed, _p(sh, ctypes.c_int16)) != 0:
        raise RuntimeError("QC base construction failed")
    return qc_from_shifts(mb, nb, Z, sh.reshape(mb, nb), name=f"QC {mb}x{nb} Z={Z} seed={seed}")


def qc_from_shifts(mb: int, nb: int, Z: int, shifts: np.ndarray, name: str = "") -> Code:
    sh = np.ascontiguousarray(shifts, np.int16).reshape(-1)
    E = int((sh >= 0).sum()) * Z
    rp = np.zeros(mb * Z + 1, np.int32)
    ci = np.zeros(E, np.int32)
    lib().lg_qc_expand(mb, nb, Z, _p(sh, ctypes.c_int16), _p(rp, ctypes.c_int32), _p(ci, ctypes.c_int32))
    return Code(nb * Z, mb * Z, rp, ci, qc_z=Z, qc_rows=mb, qc_cols=nb, qc_shift=sh.reshape(mb, nb).copy(),
                name=name)


def dvbs2like(N: int, M: int, n_hi: int, w_hi: int, w_lo: int, seed: int) -> Code:
    K = N - M
    Ei = n_hi * w_hi + (K - n_hi) * w_lo
    E = Ei + 2 * M - 1
    rp = np.zeros(M + 1, np.int32)
    ci = np.zeros(E, np.int32)
    if lib().lg_dvbs2like(N, M, n_hi, w_hi, w_lo, seed, _p(rp, ctypes.c_int32), _p(ci, ctypes.c_int32)) != 0:
        raise RuntimeError("DVB-S2-like construction failed")
    return Code(N, M, rp, ci, name=f"DVB-S2-like N={N} M={M} seed={seed}")


def ebn0_to_sigma2(ebn0_db: float, rate: float) -> float:
    """sigma^2 = 1 / (2 R 10^(EbN0/10)) for unit-energy BPSK."""
    return 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))


LLR_F64, LLR_F32, LLR_I16, LLR_I8 = 0, 1, 2, 3


def llr(noise_seed: int, f0: int, nf: int, N: int, sigma2: float, kind: int,
        frac_bits: int = 0, clamp: int = 0, out: Optional[np.ndarray] = None, nthreads: int = 0) -> np.ndarray:
    """Channel LLRs for global frames [f0, f0+nf) as a [nf][N] array."""
    dt = {LLR_F64: np.float64, LLR_F32: np.float32, LLR_I16: np.int16, LLR_I8: np.int8}[kind]
    if out is None:
        out = np.empty((nf, N), dt)
    assert out.dtype == dt and out.flags["C_CONTIGUOUS"] and out.size == nf * N
    if nthreads <= 0:
        nthreads = max(1, min(64, os.cpu_count() or 1))
    lib().lg_llr(noise_seed, f0, nf, N, float(sigma2), kind, frac_bits, clamp,
                 out.ctypes.data_as(ctypes.c_void_p), nthreads)
    return out


def gauss_pair(noise_seed: int, f: int, i: int):
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().lg_gauss_pair(noise_seed, f, i, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


# ----------------------------------------------------------------- configs
@dataclass
class Config:
    """One of BASELINE.json's five configs with SURVEY.md §8(c)/(d) decisions applied."""
    idx: int
    code_kind: str
    code_seed: int
    noise_seed: int
    ebn0_db: float
    llr_kind: int
    frac_bits: int
    clamp: int
    variant: str          # "offset" | "normalized"
    offset_raw: int
    alpha: float
    max_iter: int
    early_stop: int
    msg_format: str       # "compact" | "1bit"
    frames: int           # per GPU
    parity_frames: int    # frames the oracle decodes for parity
    extra: dict = field(default_factory=dict)

    def code(self) -> Code:
        return make_code(self.code_kind, self.code_seed)

    def sigma2(self, code: Code) -> float:
        return ebn0_to_sigma2(self.ebn0_db, code.rate)

    def llrs(self, code: Code, f0: int, nf: int, out=None) -> np.ndarray:
        return llr(self.noise_seed, f0, nf, code.n_vars, self.sigma2(code), self.llr_kind,
                   self.frac_bits, self.clamp, out=out)


_CODE_CACHE: dict = {}


def make_code(kind: str, seed: int) -> Code:
    key = (kind, seed)
    if key in _CODE_CACHE:
        return _CODE_CACHE[key]
    if kind == "reg36_1008":
        c = regular(1008, 3, 6, seed, remove_4cycles=True)
    elif kind == "qc_dtmb":
        # D18: 35 base columns of weight 3, 24 of weight 4, chosen by a seeded shuffle
        rng = np.random.default_rng(seed)
        w = np.array([3] * 35 + [4] * 24, np.int32)
        rng.shuffle(w)
        c = qc(35, 59, 127, w, seed)
    elif kind == "dvbs2_64800":
        c = dvbs2like(64800, 32400, 12960, 8, 3, seed)
    else:
        raise KeyError(kind)
    c.name = kind
    _CODE_CACHE[key] = c
    return c


CONFIGS = {
    1: Config(1, "reg36_1008", 1001, 2001, 2.5, LLR_I16, 3, 511, "offset", 1, 1.0, 20, 0, "compact", 1024, 1024),
    2: Config(2, "qc_dtmb", 1002, 2002, 1.5, LLR_I16, 3, 511, "offset", 1, 1.0, 15, 1, "compact", 8192, 1024),
    3: Config(3, "qc_dtmb", 1002, 2003, 2.0, LLR_I8, 2, 127, "offset", 1, 1.0, 30, 0, "1bit", 65536, 2048),
    4: Config(4, "dvbs2_64800", 1004, 2004, 1.0, LLR_I16, 3, 511, "offset", 1, 1.0, 50, 0, "compact", 512, 64),
    5: Config(5, "dvbs2_64800", 1004, 2005, 1.0, LLR_F32, 0, 0, "normalized", 0, 0.75, 50, 0, "compact", 8192, 64),
}
