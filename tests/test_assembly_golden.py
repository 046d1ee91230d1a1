"""The repo's vectorised input producer against the reference's assembly.

Blocks must have identical sparsity patterns and values within 1e-13
relative (the reference's per-cell BLAS dot products and numpy's einsum
round differently in the last bit); restriction-set generation is integer
work and must match exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import g_blocks, g_sets, golden, same_csr
from paper_2009_13916_b200 import configs


@pytest.mark.parametrize("fname,idx,n", [("config1_n6", 1, 6), ("config2_n8", 2, 8),
                                         ("config3_n5", 3, 5)])
def test_assembly_matches_reference(fname, idx, n):
    d = golden(fname)
    mine = configs.make(idx, n=n).system
    for name, R in zip(("A_ff", "A_fc", "A_cf", "A_cc"), g_blocks(d)):
        M = getattr(mine, name)
        assert same_csr(M, R), name
        scale = np.abs(R.data).max()
        assert np.abs(M.data - R.data).max() <= 1e-13 * scale, name
    assert np.array_equal(mine.free_faces, d["free_faces"])
    assert np.array_equal(mine.face_index, d["face_index"])
    rhs = mine.rhs()
    assert np.abs(rhs - d["rhs"]).max() <= 1e-13 * max(np.abs(d["rhs"]).max(), 1.0)


def test_base_sets_equal_acf_pattern():
    d = golden("config1_n6")
    ref = g_sets(d, "base_Q")
    A_cf = g_blocks(d)[2]
    for m, s in enumerate(ref):
        assert np.array_equal(s, A_cf.indices[A_cf.indptr[m]:A_cf.indptr[m + 1]])
