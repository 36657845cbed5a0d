"""B200-native single-scan min-sum LDPC decoder -- Python binding of libldpc.so.

Thin ctypes marshalling over the C ABI declared in ``include/ldpc.h`` (same names).
Every step of the decode runs in the library's CUDA kernels for sm_100a; PyTorch is
used only for device memory, streams and (in bench.py) process groups.  There is no
CPU fallback: if ``libldpc.so`` is missing or cannot be loaded this module raises.

Paper: X. Huang, "Single-Scan Min-Sum Algorithms for Fast Decoding of LDPC Codes"
(ITW 2006) -- §4 single-scan, §5 compact state.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
# LDPC_LIBRARY selects another build of the same library (tests: the bounds-checked build,
# `make checked`); default: the in-tree libldpc.so
LIB_PATH = os.environ.get("LDPC_LIBRARY") or os.path.join(_HERE, "libldpc.so")

LDPC_OK, LDPC_ERR_INVALID_ARG, LDPC_ERR_INVALID_CODE, LDPC_ERR_UNSUPPORTED, LDPC_ERR_CUDA, LDPC_ERR_NO_MEMORY = range(6)
LDPC_LLR_I16, LDPC_LLR_I8, LDPC_LLR_F32 = 0, 1, 2
LDPC_MINSUM_OFFSET, LDPC_MINSUM_NORMALIZED = 0, 1
LDPC_MSG_COMPACT, LDPC_MSG_1BIT, LDPC_MSG_FULL = 0, 1, 2
LDPC_SCHED_SINGLESCAN, LDPC_SCHED_TWOSCAN, LDPC_SCHED_LAYERED = 0, 1, 2
LDPC_PATH_AUTO, LDPC_PATH_STREAM, LDPC_PATH_RESIDENT_BATCHED = 0, 1, 2

# every symbol include/ldpc.h declares
EXPORTS = [
    "ldpc_code_create", "ldpc_code_destroy", "ldpc_code_query", "ldpc_decode_workspace_size",
    "ldpc_decode_batch", "ldpc_decode_batch_messages", "ldpc_decode_host_workspace_size", "ldpc_decode_batch_host",
    "ldpc_count_errors",
    "ldpc_last_launch_count", "ldpc_status_string", "ldpc_last_error_detail", "ldpc_version",
]


class ldpc_code_desc(ctypes.Structure):
    _fields_ = [("n_vars", ctypes.c_int32), ("n_checks", ctypes.c_int32),
                ("row_ptr", ctypes.POINTER(ctypes.c_int32)), ("col_idx", ctypes.POINTER(ctypes.c_int32)),
                ("qc_z", ctypes.c_int32), ("qc_rows", ctypes.c_int32), ("qc_cols", ctypes.c_int32),
                ("qc_shift", ctypes.POINTER(ctypes.c_int16))]


class ldpc_tuning(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("resident_waves", ctypes.c_int32),
                ("stream_chunk_tiles", ctypes.c_int32), ("stream_register_kernels", ctypes.c_int32),
                ("host_chunks", ctypes.c_int32), ("host_streams", ctypes.c_int32),
                ("resident_threads", ctypes.c_int32),
                ("resident_fixed_bases", ctypes.c_int32)]


class ldpc_decode_params(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("early_stop", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("offset_raw", ctypes.c_int32), ("offset_f", ctypes.c_float), ("alpha", ctypes.c_float),
                ("clamp_raw", ctypes.c_int32), ("llr_type", ctypes.c_int32), ("msg_format", ctypes.c_int32),
                ("schedule", ctypes.c_int32),
                ("offset_per_iter", ctypes.POINTER(ctypes.c_int32)),
                ("offset_f_per_iter", ctypes.POINTER(ctypes.c_float)),
                ("alpha_per_iter", ctypes.POINTER(ctypes.c_float)),
                ("tuning", ctypes.POINTER(ldpc_tuning))]


class LdpcError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {_STATUS_NAMES.get(status, status)}: {detail}")
        self.status = status


_STATUS_NAMES = {0: "LDPC_OK", 1: "LDPC_ERR_INVALID_ARG", 2: "LDPC_ERR_INVALID_CODE", 3: "LDPC_ERR_UNSUPPORTED",
                 4: "LDPC_ERR_CUDA", 5: "LDPC_ERR_NO_MEMORY"}
_lib = None


def lib():
    """Load libldpc.so (built in-tree by `make` / __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.ldpc_code_create.argtypes = [ctypes.POINTER(ldpc_code_desc), ctypes.c_int, ctypes.POINTER(vp)]
        L.ldpc_code_destroy.argtypes = [vp]
        L.ldpc_code_destroy.restype = None
        L.ldpc_code_query.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i64),
                                      ctypes.POINTER(i32), ctypes.POINTER(i32)]
        PP = ctypes.POINTER(ldpc_decode_params)
        L.ldpc_decode_workspace_size.argtypes = [vp, i64, PP, ctypes.POINTER(sz)]
        L.ldpc_decode_host_workspace_size.argtypes = [vp, i64, PP, ctypes.POINTER(sz)]
        L.ldpc_decode_batch.argtypes = [vp, PP, i64, vp, vp, vp, vp, vp, vp, sz, vp]
        L.ldpc_decode_batch_messages.argtypes = [vp, PP, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.ldpc_decode_batch_host.argtypes = [vp, PP, i64, vp, vp, vp, vp, vp, vp, sz, vp]
        L.ldpc_count_errors.argtypes = [vp, i64, vp, vp, vp, vp, vp]
        for f in ("ldpc_code_create", "ldpc_code_query", "ldpc_decode_workspace_size", "ldpc_decode_host_workspace_size",
                  "ldpc_decode_batch", "ldpc_decode_batch_messages", "ldpc_decode_batch_host", "ldpc_count_errors"):
            getattr(L, f).restype = ctypes.c_int
        L.ldpc_status_string.argtypes = [ctypes.c_int]
        L.ldpc_status_string.restype = ctypes.c_char_p
        L.ldpc_last_error_detail.restype = ctypes.c_char_p
        L.ldpc_version.restype = i32
        L.ldpc_last_launch_count.restype = i32
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != LDPC_OK:
        raise LdpcError(status, where, lib().ldpc_last_error_detail().decode())


def ldpc_status_string(status: int) -> str:
    return lib().ldpc_status_string(status).decode()


def ldpc_last_error_detail() -> str:
    return lib().ldpc_last_error_detail().decode()


def ldpc_version() -> int:
    return lib().ldpc_version()


def ldpc_last_launch_count() -> int:
    return lib().ldpc_last_launch_count()


def _np_ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def make_desc(code):
    """ldpc_code_desc from any object with n_vars, n_checks, row_ptr, col_idx (numpy) and
    optional qc_z / qc_rows / qc_cols / qc_shift.  Returns (desc, keepalive)."""
    import numpy as np
    rp = np.ascontiguousarray(code.row_ptr, np.int32)
    ci = np.ascontiguousarray(code.col_idx, np.int32)
    keep = [rp, ci]
    d = ldpc_code_desc(int(code.n_vars), int(code.n_checks), _np_ptr(rp, ctypes.c_int32), _np_ptr(ci, ctypes.c_int32),
                       0, 0, 0, None)
    if getattr(code, "qc_z", 0):
        sh = np.ascontiguousarray(code.qc_shift, np.int16).reshape(-1)
        keep.append(sh)
        d.qc_z, d.qc_rows, d.qc_cols = int(code.qc_z), int(code.qc_rows), int(code.qc_cols)
        d.qc_shift = _np_ptr(sh, ctypes.c_int16)
    return d, keep


def ldpc_code_create(code, cuda_device: int = 0) -> int:
    """Returns the opaque handle (int).  Raises LdpcError on failure."""
    d, keep = make_desc(code)
    h = ctypes.c_void_p()
    _check(lib().ldpc_code_create(ctypes.byref(d), int(cuda_device), ctypes.byref(h)), "ldpc_code_create")
    return h.value


def ldpc_code_destroy(handle: int) -> None:
    lib().ldpc_code_destroy(ctypes.c_void_p(handle))


def ldpc_code_query(handle: int):
    N, M, dc, dv = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    E = ctypes.c_int64()
    _check(lib().ldpc_code_query(ctypes.c_void_p(handle), ctypes.byref(N), ctypes.byref(M), ctypes.byref(E),
                                 ctypes.byref(dc), ctypes.byref(dv)), "ldpc_code_query")
    return N.value, M.value, E.value, dc.value, dv.value


def make_params(max_iter=10, early_stop=0, variant=LDPC_MINSUM_OFFSET, offset_raw=0, offset_f=0.0, alpha=1.0,
                clamp_raw=0, llr_type=LDPC_LLR_I16, msg_format=LDPC_MSG_COMPACT,
                schedule=None, offset_per_iter=None, offset_f_per_iter=None,
                alpha_per_iter=None, tuning=None) -> ldpc_decode_params:
    """ldpc_decode_params; the optional per-iteration arrays (max_iter entries) and the
    optional plan overrides (``tuning``: an ldpc_tuning or a dict of its fields) are kept
    alive on the returned object."""
    import numpy as np
    sched = LDPC_SCHED_SINGLESCAN if schedule is None else int(schedule)
    p = ldpc_decode_params(int(max_iter), int(early_stop), int(variant), int(offset_raw), float(offset_f),
                           float(alpha), int(clamp_raw), int(llr_type), int(msg_format), sched)
    p._keep = []
    for name, arr, dt, ct in (("offset_per_iter", offset_per_iter, np.int32, ctypes.c_int32),
                              ("offset_f_per_iter", offset_f_per_iter, np.float32, ctypes.c_float),
                              ("alpha_per_iter", alpha_per_iter, np.float32, ctypes.c_float)):
        if arr is not None:
            a = np.ascontiguousarray(arr, dt)
            if a.size < max_iter:
                raise ValueError(f"{name} needs max_iter = {max_iter} entries")
            p._keep.append(a)
            setattr(p, name, a.ctypes.data_as(ctypes.POINTER(ct)))
    if tuning is not None:
        set_tuning(p, tuning)
    return p


def set_tuning(params: ldpc_decode_params, tuning) -> ldpc_decode_params:
    """Attach plan overrides (include/ldpc.h ldpc_tuning) to params: an ldpc_tuning, a dict of
    its fields, or None to clear."""
    if tuning is None:
        params.tuning = None
        return params
    t = tuning if isinstance(tuning, ldpc_tuning) else ldpc_tuning(**tuning)
    params._tuning = t
    params.tuning = ctypes.pointer(t)
    return params


def ldpc_decode_workspace_size(handle: int, n_frames: int, params: ldpc_decode_params) -> int:
    b = ctypes.c_size_t()
    _check(lib().ldpc_decode_workspace_size(ctypes.c_void_p(handle), int(n_frames), ctypes.byref(params),
                                            ctypes.byref(b)), "ldpc_decode_workspace_size")
    return b.value


def ldpc_decode_host_workspace_size(handle: int, n_frames: int, params: ldpc_decode_params) -> int:
    b = ctypes.c_size_t()
    _check(lib().ldpc_decode_host_workspace_size(ctypes.c_void_p(handle), int(n_frames), ctypes.byref(params),
                                                 ctypes.byref(b)), "ldpc_decode_host_workspace_size")
    return b.value


def ldpc_decode_batch(handle: int, params: ldpc_decode_params, n_frames: int, llr: int, hard_bits: int,
                      posteriors: int, syndrome_ok: int, iterations_used: int, workspace: int, workspace_bytes: int,
                      stream: int) -> None:
    """All pointer arguments are raw device addresses (ints, 0 = NULL); stream is a cudaStream_t."""
    _check(lib().ldpc_decode_batch(ctypes.c_void_p(handle), ctypes.byref(params), int(n_frames), llr or None,
                                   hard_bits or None, posteriors or None, syndrome_ok or None,
                                   iterations_used or None, workspace or None, int(workspace_bytes), stream or None),
           "ldpc_decode_batch")


def ldpc_decode_batch_messages(handle: int, params: ldpc_decode_params, n_frames: int, llr: int, hard_bits: int,
                               posteriors: int, syndrome_ok: int, iterations_used: int, messages: int, workspace: int,
                               workspace_bytes: int, stream: int) -> None:
    """ldpc_decode_batch plus the exit check messages [n_frames][E] (device address)."""
    _check(lib().ldpc_decode_batch_messages(ctypes.c_void_p(handle), ctypes.byref(params), int(n_frames), llr or None,
                                            hard_bits or None, posteriors or None, syndrome_ok or None,
                                            iterations_used or None, messages or None, workspace or None,
                                            int(workspace_bytes), stream or None), "ldpc_decode_batch_messages")


def ldpc_decode_batch_host(handle: int, params: ldpc_decode_params, n_frames: int, llr_host: int,
                           hard_bits_host: int, posteriors_host: int, syndrome_ok_host: int,
                           iterations_used_host: int, workspace: int, workspace_bytes: int, stream: int) -> None:
    """Host-buffer variant: the copies are enqueued on `stream` with the decode."""
    _check(lib().ldpc_decode_batch_host(ctypes.c_void_p(handle), ctypes.byref(params), int(n_frames),
                                        llr_host or None, hard_bits_host or None, posteriors_host or None,
                                        syndrome_ok_host or None, iterations_used_host or None, workspace or None,
                                        int(workspace_bytes), stream or None), "ldpc_decode_batch_host")


def ldpc_count_errors(handle: int, n_frames: int, hard_bits: int, syndrome_ok: int, iterations_used: int,
                      counters: int, stream: int) -> None:
    _check(lib().ldpc_count_errors(ctypes.c_void_p(handle), int(n_frames), hard_bits or None, syndrome_ok or None,
                                   iterations_used or None, counters or None, stream or None), "ldpc_count_errors")


# ------------------------------------------------------------------ convenience
LLR_TYPES = {"i16": LDPC_LLR_I16, "i8": LDPC_LLR_I8, "f32": LDPC_LLR_F32}


@dataclass
class DecodeOutputs:
    hard_bits: "object"      # torch.uint32-as-int32 [F][ceil(N/32)]
    syndrome_ok: "object"    # torch.uint8 [F]
    iterations: "object"     # torch.int32 [F]
    posteriors: Optional["object"] = None


class Decoder:
    """Owns one ldpc_code and a workspace; decodes torch tensors on the current stream."""

    def __init__(self, code, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        self.handle = ldpc_code_create(code, device)
        self.N, self.M, self.E, self.max_dc, self.max_dv = ldpc_code_query(self.handle)
        self.wpf = (self.N + 31) // 32
        self._ws = None
        self._ws_host = None

    def close(self):
        if self.handle:
            ldpc_code_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace(self, n_frames: int, params: ldpc_decode_params, host: bool = False):
        torch = self.torch
        nbytes = (ldpc_decode_host_workspace_size if host else ldpc_decode_workspace_size)(self.handle, n_frames,
                                                                                             params)
        attr = "_ws_host" if host else "_ws"
        ws = getattr(self, attr)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            setattr(self, attr, ws)
        return ws, nbytes

    def alloc_outputs(self, n_frames: int, llr_type: int, posteriors: bool = True) -> DecodeOutputs:
        torch = self.torch
        dev = f"cuda:{self.device}"
        hb = torch.empty((n_frames, self.wpf), dtype=torch.int32, device=dev)
        ok = torch.empty(n_frames, dtype=torch.uint8, device=dev)
        it = torch.empty(n_frames, dtype=torch.int32, device=dev)
        post = None
        if posteriors:
            post = torch.empty((n_frames, self.N), dtype=torch.float32 if llr_type == LDPC_LLR_F32 else torch.int16,
                               device=dev)
        return DecodeOutputs(hb, ok, it, post)

    def decode(self, llr, params: ldpc_decode_params, out: Optional[DecodeOutputs] = None,
               posteriors: bool = True) -> DecodeOutputs:
        """llr: CUDA tensor [F][N] (int16 / int8 / float32 matching params.llr_type)."""
        torch = self.torch
        assert llr.is_cuda and llr.is_contiguous() and llr.shape[1] == self.N
        F = llr.shape[0]
        if out is None:
            out = self.alloc_outputs(F, params.llr_type, posteriors)
        ws, nbytes = self.workspace(F, params)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ldpc_decode_batch(self.handle, params, F, llr.data_ptr(), out.hard_bits.data_ptr(),
                          out.posteriors.data_ptr() if out.posteriors is not None else 0,
                          out.syndrome_ok.data_ptr(), out.iterations.data_ptr(), ws.data_ptr(), nbytes, stream)
        return out

    def decode_messages(self, llr, params: ldpc_decode_params, out: Optional[DecodeOutputs] = None):
        """decode() plus the exit check messages: returns (outputs, messages [F][E] int16 / float32)."""
        torch = self.torch
        assert llr.is_cuda and llr.is_contiguous() and llr.shape[1] == self.N
        F = llr.shape[0]
        if out is None:
            out = self.alloc_outputs(F, params.llr_type, True)
        msg = torch.empty((F, self.E), dtype=torch.float32 if params.llr_type == LDPC_LLR_F32 else torch.int16,
                          device=f"cuda:{self.device}")
        ws, nbytes = self.workspace(F, params)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ldpc_decode_batch_messages(self.handle, params, F, llr.data_ptr(), out.hard_bits.data_ptr(),
                                   out.posteriors.data_ptr() if out.posteriors is not None else 0,
                                   out.syndrome_ok.data_ptr(), out.iterations.data_ptr(), msg.data_ptr(),
                                   ws.data_ptr(), nbytes, stream)
        return out, msg

    def decode_host(self, llr_host, params: ldpc_decode_params, hb_host, ok_host, it_host=None, post_host=None):
        """Host (pinned) tensors in/out; copies + decode enqueued on the current stream."""
        torch = self.torch
        F = llr_host.shape[0]
        ws, nbytes = self.workspace(F, params, host=True)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ldpc_decode_batch_host(self.handle, params, F, llr_host.data_ptr(), hb_host.data_ptr(),
                               post_host.data_ptr() if post_host is not None else 0, ok_host.data_ptr(),
                               it_host.data_ptr() if it_host is not None else 0, ws.data_ptr(), nbytes, stream)

    def count_errors(self, out: DecodeOutputs, counters=None):
        torch = self.torch
        if counters is None:
            counters = torch.zeros(5, dtype=torch.int64, device=f"cuda:{self.device}")
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ldpc_count_errors(self.handle, out.syndrome_ok.numel(), out.hard_bits.data_ptr(), out.syndrome_ok.data_ptr(),
                          out.iterations.data_ptr(), counters.data_ptr(), stream)
        return counters


def params_for_config(cfg, schedule=LDPC_SCHED_SINGLESCAN, msg_format=None) -> ldpc_decode_params:
    """Decode parameters of one of ldpcgen.CONFIGS (BASELINE.json configs).
    schedule=LDPC_SCHED_TWOSCAN gives the paper's two-scan baseline on the same workload
    (full per-edge messages, so the message format is COMPACT)."""
    import ldpcgen
    llr_type = {ldpcgen.LLR_I16: LDPC_LLR_I16, ldpcgen.LLR_I8: LDPC_LLR_I8, ldpcgen.LLR_F32: LDPC_LLR_F32}[cfg.llr_kind]
    if cfg.variant == "normalized":
        return make_params(cfg.max_iter, cfg.early_stop, LDPC_MINSUM_NORMALIZED, 0, 0.0, cfg.alpha, 0, llr_type,
                           LDPC_MSG_COMPACT if msg_format is None else int(msg_format), schedule)
    fmt = LDPC_MSG_1BIT if cfg.msg_format == "1bit" and schedule == LDPC_SCHED_SINGLESCAN else LDPC_MSG_COMPACT
    if msg_format is not None:
        fmt = int(msg_format)
    return make_params(cfg.max_iter, cfg.early_stop, LDPC_MINSUM_OFFSET, cfg.offset_raw, 0.0, 1.0, cfg.clamp,
                       llr_type, fmt, schedule)
