"""CPU ORACLE for the single-scan min-sum LDPC decoder -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_cs_0609090_b200``) never imports it, and the two share no code: the
oracle is plain C (``oracle.c`` + ``engine.inc``) written from PAPER.md, compiled
with gcc, loaded here with ctypes.  Its inputs come from ``ldpcgen`` (seeded
input generation only) or from the tests.

Engines (PAPER.md section / lines):
  TWOSCAN_NAIVE  §3 Eq.(1)/(2), O(dc^2) check rule -- the plain definition
  TWOSCAN        §3 with the two-minima check rule
  SINGLESCAN     §4 single-scan, per-edge L storage
  COMPACT        §5 memory-efficient single-scan -- the GPU's parity target
  LAYERED_FULL   Eq.(3) with ONE in-place posterior array, rows in ascending m (layered /
                 Gauss-Seidel reading D25); per-edge L, Eq.(1) literally
  LAYERED        the same schedule over the §5 compact state -- the GPU layered target
Numeric modes: "int" (int32 raw LSBs; offset beta + clamp Q), "f64", "f32" (one rounding per
operation, reading D11; posterior sums exact and rounded once, reading D28).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

TWOSCAN_NAIVE, TWOSCAN, SINGLESCAN, COMPACT, LAYERED_FULL, LAYERED = 0, 1, 2, 3, 4, 5
ENGINES = {"twoscan_naive": TWOSCAN_NAIVE, "twoscan": TWOSCAN, "singlescan": SINGLESCAN, "compact": COMPACT,
           "layered_full": LAYERED_FULL, "layered": LAYERED}


class Params(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("early_stop", ctypes.c_int32),
                ("beta_i", ctypes.c_int32), ("clamp_i", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("beta_f", ctypes.c_double),
                ("beta_i_sched", ctypes.c_void_p), ("alpha_sched", ctypes.c_void_p),
                ("beta_f_sched", ctypes.c_void_p)]


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "engine.inc")]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(s) for s in srcs):
        # -ffp-contract=off: no FMA contraction (reading D11); -O2 only, never tuned.
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _LIB, srcs[0], "-lm", "-lpthread"])
    return _LIB


_TYPES = {"int": (np.int32, "i32"), "f64": (np.float64, "f64"), "f32": (np.float32, "f32")}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = ctypes.CDLL(_LIB)
        vp = ctypes.c_void_p
        for mode, (_, suf) in _TYPES.items():
            f = getattr(L, f"orc_decode_{suf}")
            f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.POINTER(Params), ctypes.c_int64,
                          vp, vp, vp, vp, vp, vp, vp, ctypes.c_int]
            f.restype = ctypes.c_int
            g = getattr(L, f"orc_check_naive_{suf}")
            g.argtypes = [ctypes.c_int, vp, ctypes.POINTER(Params), vp]
            h = getattr(L, f"orc_check_compact_{suf}")
            h.argtypes = [ctypes.c_int, vp, ctypes.POINTER(Params), vp, vp, vp, vp, vp]
        L.orc_hardware_threads.restype = ctypes.c_int
        L.orc_f32_exact_sum.argtypes = [ctypes.c_int, vp]
        L.orc_f32_exact_sum.restype = ctypes.c_float
        _lib = L
    return _lib


def hardware_threads() -> int:
    return lib().orc_hardware_threads()


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def make_params(max_iter: int = 1, early_stop: int = 0, beta: float = 0, clamp: int = 0,
                alpha: float = 1.0) -> Params:
    """Integer modes use beta (LSBs), clamp and alpha (normalized: floor(alpha |L|),
    reading D27); float modes use alpha and beta."""
    return Params(int(max_iter), int(early_stop), int(beta), int(clamp), float(alpha), float(beta), None, None, None)


def check_naive(q, mode="int", beta=0, clamp=0, alpha=1.0) -> np.ndarray:
    """Eq.(1) on one check row, literally, plus the variant."""
    dt, suf = _TYPES[mode]
    q = np.ascontiguousarray(q, dt)
    out = np.empty_like(q)
    p = make_params(beta=beta, clamp=clamp, alpha=alpha)
    getattr(lib(), f"orc_check_naive_{suf}")(len(q), _ptr(q), ctypes.byref(p), _ptr(out))
    return out


def check_compact(q, mode="int", beta=0, clamp=0, alpha=1.0):
    """§5 compact form of one check row: (messages, A, B, idx, signs)."""
    dt, suf = _TYPES[mode]
    q = np.ascontiguousarray(q, dt)
    out = np.empty_like(q)
    A = np.zeros(1, dt)
    B = np.zeros(1, dt)
    idx = np.zeros(1, np.int32)
    s = np.zeros(len(q), np.int8)
    p = make_params(beta=beta, clamp=clamp, alpha=alpha)
    getattr(lib(), f"orc_check_compact_{suf}")(len(q), _ptr(q), ctypes.byref(p), _ptr(out), _ptr(A), _ptr(B),
                                               _ptr(idx), _ptr(s))
    return out, A[0], B[0], int(idx[0]), s


@dataclass
class Result:
    post: np.ndarray       # [F][N] posteriors Z^(k)_n at exit
    bits: np.ndarray       # [F][N] uint8 hard decisions
    ok: np.ndarray         # [F] uint8, 1 iff H x̂ = 0 at exit
    iters: np.ndarray      # [F] int32 iterations used
    trace_post: Optional[np.ndarray] = None   # [F][K][N]
    trace_msg: Optional[np.ndarray] = None    # [F][K][E]
    threads: int = 1


def decode(code, z0: np.ndarray, engine="compact", mode="int", max_iter=10, early_stop=0,
           beta=0, clamp=0, alpha=1.0, trace=False, nthreads: int = 1, beta_sched=None, alpha_sched=None) -> Result:
    """Decode frames z0 ([F][N]) of ``code`` (any object with n_vars, n_checks,
    row_ptr, col_idx) with one of the oracle engines.  beta_sched / alpha_sched: optional
    per-iteration offsets / normalization factors (max_iter entries)."""
    dt, suf = _TYPES[mode]
    eng = ENGINES[engine] if isinstance(engine, str) else int(engine)
    z0 = np.ascontiguousarray(np.atleast_2d(z0), dt)
    F, N = z0.shape
    assert N == code.n_vars
    E = int(code.row_ptr[-1])
    rp = np.ascontiguousarray(code.row_ptr, np.int32)
    ci = np.ascontiguousarray(code.col_idx, np.int32)
    post = np.empty((F, N), dt)
    bits = np.empty((F, N), np.uint8)
    ok = np.empty(F, np.uint8)
    iters = np.empty(F, np.int32)
    tp = tm = None
    if trace:
        sentinel = np.iinfo(np.int32).min if mode == "int" else np.nan
        tp = np.full((F, max_iter, N), sentinel, dt)
        tm = np.full((F, max_iter, E), sentinel, dt)
    p = make_params(max_iter, early_stop, beta, clamp, alpha)
    keep = []
    if beta_sched is not None:
        bs = np.ascontiguousarray(beta_sched, np.int32 if mode == "int" else np.float64)
        assert bs.size >= max_iter
        keep.append(bs)
        if mode == "int":
            p.beta_i_sched = bs.ctypes.data
        else:
            p.beta_f_sched = bs.ctypes.data
    if alpha_sched is not None:
        a_s = np.ascontiguousarray(alpha_sched, np.float64)
        assert a_s.size >= max_iter
        keep.append(a_s)
        p.alpha_sched = a_s.ctypes.data
    nt = getattr(lib(), f"orc_decode_{suf}")(eng, N, code.n_checks, _ptr(rp), _ptr(ci), ctypes.byref(p), F,
                                             _ptr(z0), _ptr(post), _ptr(bits), _ptr(ok), _ptr(iters),
                                             _ptr(tp), _ptr(tm), int(nthreads))
    if nt < 0:
        raise ValueError("invalid code")
    return Result(post, bits, ok, iters, tp, tm, nt)


def f32_exact_sum(x) -> np.float32:
    """The fp32 posterior-sum rule of reading D28 on one list of terms: each term saturated
    to [-2^20, 2^20] and placed on the 2^-34 grid, summed exactly, rounded once to fp32."""
    x = np.ascontiguousarray(x, np.float32)
    return np.float32(lib().orc_f32_exact_sum(len(x), _ptr(x)))


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """[F][N] uint8 -> [F][ceil(N/32)] uint32, bit n%32 of word n/32 (LSB first),
    the hard-bit layout of the C-ABI (include/ldpc.h)."""
    F, N = bits.shape
    W = (N + 31) // 32
    padded = np.zeros((F, W * 32), np.uint64)
    padded[:, :N] = bits
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return (padded.reshape(F, W, 32) * weights).sum(axis=2).astype(np.uint32)
