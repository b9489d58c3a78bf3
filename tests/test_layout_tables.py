"""Host side of the table-driven entry layout (scba.EntryLayout table mode,
negf_pack_lg_table / negf_unpack_table): the per-entry (block, kind, offset)
tables must address exactly the pattern's (row, col) in the target blocking --
the r_cut subset of the band and the coarser W grid
bs_w = k bs (scba.py:893-937, _scatter_groups(pat_g, bs_w)). No GPU needed
(tables are built on the CPU device)."""

import numpy as np
import pytest

from paper_2508_19138_b200.results import EntryPattern
from paper_2508_19138_b200.scba import EntryLayout


@pytest.mark.parametrize("n_b,bs,cutoff,k", [(6, 4, None, 2), (6, 4, 5, 1), (6, 4, 0, 1), (8, 3, 7, 4),
                                             (4, 5, 3, 2), (5, 4, None, 5)])
def test_tables_address_the_pattern(n_b, bs, cutoff, k):
    lay = EntryLayout(n_b, bs, "cpu", cutoff=cutoff, target_bs=k * bs)
    assert lay.table
    pat = EntryPattern(n_b, bs, 3, True, cutoff)
    assert lay.n_entries == pat.n_entries
    code, q = lay.code.numpy(), lay.q.numpy()
    bt = k * bs
    bi, kind = code >> 1, code & 1
    r, c = np.divmod(q, bt)
    rows, cols = bi * bt + r, (bi + kind) * bt + c
    assert np.array_equal(rows, pat.rows) and np.array_equal(cols, pat.cols)
    assert np.all((kind == 0) | (kind == 1)) and np.all(bi + kind < n_b * bs // bt)
    # the diagonal entries of every G block survive any cutoff (the residual traces)
    dr = lay.diag_rows.numpy()
    assert dr.shape == (n_b, bs)
    assert np.array_equal(pat.rows[dr.reshape(-1)], np.arange(n_b * bs))
    assert np.array_equal(pat.cols[dr.reshape(-1)], np.arange(n_b * bs))
    assert int(lay.diag.sum()) == n_b * bs


def test_cutoff_keeps_the_band_inside_the_radius():
    pat = EntryPattern(5, 6, 3, True, 4)
    assert np.all(np.abs(pat.rows - pat.cols) <= 4) and np.all(pat.rows <= pat.cols)
    full = EntryPattern(5, 6)
    keep = np.abs(full.rows - full.cols) <= 4
    assert np.array_equal(pat.rows, full.rows[keep]) and pat.n_entries == int(keep.sum())


def test_invalid_target_blocking():
    with pytest.raises(ValueError):
        EntryLayout(6, 4, "cpu", target_bs=6)
