"""alist I/O and the storage arithmetic; host-only."""
import os

import numpy as np
import pytest

import ldpcgen as g
from paper_cs_0609090_b200.codeio import ParityCheck, read_alist, storage_report, write_alist


def test_alist_hand_written(tmp_path):
    """A hand-written alist of H = [[1,1,0,1],[0,1,1,1]] (1-based, zero-padded)."""
    p = tmp_path / "toy.alist"
    p.write_text("4 2\n2 3\n1 2 1 2\n3 3\n1 0\n1 2\n2 0\n1 2\n1 2 4\n2 3 4\n")
    c = read_alist(str(p))
    assert (c.n_vars, c.n_checks, c.n_edges) == (4, 2, 6)
    assert c.row_ptr.tolist() == [0, 3, 6] and c.col_idx.tolist() == [0, 1, 3, 1, 2, 3]


@pytest.mark.parametrize("code", [g.CONFIGS[1].code(), g.CONFIGS[2].code(), g.dvbs2like(600, 300, 120, 8, 3, seed=6)],
                         ids=lambda c: c.name)
def test_alist_roundtrip(code, tmp_path):
    p = str(tmp_path / "c.alist")
    write_alist(p, code)
    c = read_alist(p)
    assert c.n_vars == code.n_vars and c.n_checks == code.n_checks
    assert np.array_equal(c.row_ptr, code.row_ptr) and np.array_equal(c.col_idx, code.col_idx)


def test_alist_rejects_inconsistent(tmp_path):
    p = tmp_path / "bad.alist"
    p.write_text("3 2\n2 2\n1 2 1\n2 2\n1 0\n1 2\n2 0\n1 2\n1 3\n")   # row 2 lists col 3, col lists say col 2
    with pytest.raises(ValueError):
        read_alist(str(p))


def test_storage_report_matches_the_papers_counts():
    """N vs N*d_v items; addressing halves; compact messages."""
    code = g.CONFIGS[1].code()                   # (3,6)-regular N=1008
    r = storage_report(code, value_bits=8)
    assert r["twoscan_Zmn_items"] == 3 * 1008 and r["singlescan_Zn_items"] == 1008
    assert r["Z_item_ratio"] == pytest.approx(3.0)
    assert r["twoscan_addressing_entries"] == 2 * r["singlescan_addressing_entries"]
    # compact: per check 2 b-bit magnitudes + a 3-bit position (dc = 6) + 6 sign bits
    assert r["message_bits"]["compact"] == 504 * (16 + 3) + 3024
    assert r["message_bits"]["per_edge_fixed_point"] == 3024 * 8


def test_parity_check_from_rows_decoder_interface():
    c = ParityCheck.from_rows(5, [[0, 3, 1], [4, 2]])
    assert c.row_ptr.tolist() == [0, 3, 5] and c.col_idx.tolist() == [0, 1, 3, 2, 4]
    assert c.col_degrees().tolist() == [1, 1, 1, 1, 1]
