"""Parity-check matrix I/O and the paper's storage arithmetic.

Host-side helpers around the C ABI; nothing here decodes.

* ``read_alist`` / ``write_alist``: MacKay's "alist" text format, the format of the
  regular codes "from Dr. MacKay's website" the paper decodes, so a
  user who has a real matrix can load it.  None ships with this repository.
* ``ParityCheck``: a minimal H in CSR form with the attributes ``Decoder`` /
  ``make_desc`` take (n_vars, n_checks, row_ptr, col_idx, optional QC description).
* ``storage_report``: the paper's memory claims as arithmetic on a given code --
  single-scan stores Z_n (N items) instead of Z_mn (N * d_v items), needs
  only the check->variable addressing, half of two-scan's, and the compact
  form keeps per check two magnitudes, a position and one sign bit per edge instead of
  a fixed-point value per edge.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class ParityCheck:
    n_vars: int
    n_checks: int
    row_ptr: np.ndarray              # int32 [M+1]
    col_idx: np.ndarray              # int32 [E], strictly increasing per row
    name: str = ""
    qc_z: int = 0
    qc_rows: int = 0
    qc_cols: int = 0
    qc_shift: Optional[np.ndarray] = field(default=None, repr=False)

    @property
    def n_edges(self) -> int:
        return int(self.row_ptr[-1])

    def row_degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def col_degrees(self) -> np.ndarray:
        return np.bincount(self.col_idx, minlength=self.n_vars)

    @staticmethod
    def from_rows(n_vars: int, rows, name: str = "") -> "ParityCheck":
        rows = [sorted(int(c) for c in r) for r in rows]
        rp = np.zeros(len(rows) + 1, np.int32)
        rp[1:] = np.cumsum([len(r) for r in rows])
        ci = np.array([c for r in rows for c in r], np.int32)
        return ParityCheck(int(n_vars), len(rows), rp, ci, name)


def read_alist(path: str, name: Optional[str] = None) -> ParityCheck:
    """Parse an alist file: "N M", "max col weight, max row weight", N column weights,
    M row weights, then N lines of 1-based row indices (0-padded) and M lines of 1-based
    column indices (0-padded).  The row lists define H; the column lists must agree
    (ValueError otherwise)."""
    with open(path) as f:
        tok = [int(t) for t in f.read().split()]
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(tok):
            raise ValueError(f"{path}: truncated alist")
        out = tok[pos:pos + n]
        pos += n
        return out

    N, M = take(2)
    mcw, mrw = take(2)
    cw = take(N)
    rw = take(M)
    if max(cw, default=0) > mcw or max(rw, default=0) > mrw:
        raise ValueError(f"{path}: weights exceed the stated maxima")
    cols_of = []
    for n in range(N):
        lst = take(mcw)
        ent = [x for x in lst if x != 0]
        if len(ent) != cw[n]:
            raise ValueError(f"{path}: column {n} lists {len(ent)} rows, weight says {cw[n]}")
        cols_of.append(ent)
    rows = []
    for m in range(M):
        lst = take(mrw)
        ent = [x for x in lst if x != 0]
        if len(ent) != rw[m]:
            raise ValueError(f"{path}: row {m} lists {len(ent)} columns, weight says {rw[m]}")
        if any(c < 1 or c > N for c in ent):
            raise ValueError(f"{path}: row {m} has a column index out of 1..{N}")
        rows.append([c - 1 for c in ent])
    # the two descriptions of H must match
    from_cols = [[] for _ in range(M)]
    for n, lst in enumerate(cols_of):
        for r in lst:
            if r < 1 or r > M:
                raise ValueError(f"{path}: column {n} has a row index out of 1..{M}")
            from_cols[r - 1].append(n)
    for m in range(M):
        if sorted(from_cols[m]) != sorted(rows[m]):
            raise ValueError(f"{path}: row {m} disagrees with the column lists")
    return ParityCheck.from_rows(N, rows, name or path)


def write_alist(path: str, code) -> None:
    """Write any object with n_vars, n_checks, row_ptr, col_idx in alist form."""
    N, M = int(code.n_vars), int(code.n_checks)
    rp = np.asarray(code.row_ptr)
    ci = np.asarray(code.col_idx)
    rows = [ci[rp[m]:rp[m + 1]].tolist() for m in range(M)]
    cols = [[] for _ in range(N)]
    for m, r in enumerate(rows):
        for n in r:
            cols[n].append(m)
    mcw = max(len(c) for c in cols)
    mrw = max(len(r) for r in rows)
    lines = [f"{N} {M}", f"{mcw} {mrw}", " ".join(str(len(c)) for c in cols), " ".join(str(len(r)) for r in rows)]
    for c in cols:
        lines.append(" ".join(str(x + 1) for x in c) + "".join(" 0" for _ in range(mcw - len(c))))
    for r in rows:
        lines.append(" ".join(str(x + 1) for x in r) + "".join(" 0" for _ in range(mrw - len(r))))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def storage_report(code, value_bits: int = 8, index_bits: int = 32) -> dict:
    """Items and bits each algorithm keeps per frame (the paper's memory comparison).

    value_bits: width b of a stored message / posterior (the paper's b = 6~8).
    index_bits: width of one addressing entry.
    """
    N, M = int(code.n_vars), int(code.n_checks)
    E = int(np.asarray(code.row_ptr)[-1])
    dv_avg = E / N
    dc_max = int(np.max(np.diff(np.asarray(code.row_ptr))))
    pos_bits = max(1, math.ceil(math.log2(dc_max)))
    b = value_bits
    return {
        "N": N, "M": M, "E": E, "avg_dv": dv_avg,
        # variable-side storage: Z_mn (N * d_v items) vs Z_n (N items)
        "twoscan_Zmn_items": E, "singlescan_Zn_items": N, "Z_item_ratio": E / N,
        # addressing: both directions vs check->variable only, P:217-224 ("by half")
        "twoscan_addressing_entries": 2 * E, "singlescan_addressing_entries": E,
        "addressing_bits": {"twoscan": 2 * E * index_bits, "singlescan": E * index_bits},
        # check messages: a b-bit value per edge vs (A, B, position, 1 sign bit / edge)
        "message_bits": {"per_edge_fixed_point": E * b,
                         "compact": M * (2 * b + pos_bits) + E},
        "message_bit_ratio": (E * b) / (M * (2 * b + pos_bits) + E),
        # everything persistent per frame (posteriors/extrinsics + messages + channel), in bits
        "persistent_bits": {"twoscan": E * b + E * b + N * b,          # L_mn, Z_mn, Z0_n
                            "singlescan_full_L": E * b + N * b + N * b,  # L_mn, Z_n, Z0_n
                            "singlescan_compact": M * (2 * b + pos_bits) + E + N * b + N * b},
    }
