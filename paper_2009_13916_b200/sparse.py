"""Host-side helpers of ``hexflow.sparse`` the drop-in keeps (hx/sparse.py).

``canonical`` is the CSR normal form every block and artefact of the path is
compared in (hx/sparse.py:28-34); ``mm_write`` / ``mm_read`` are the Matrix
Market exchange format for blocks, vectors and parity artefacts
(hx/sparse.py:302-317).  File I/O is host work by nature; nothing here is on
the device path.
"""

from __future__ import annotations

import numpy as np
import scipy.io
import scipy.sparse as sp


def canonical(A) -> sp.csr_matrix:
    """CSR copy with sorted column indices, duplicates summed and explicit
    zeros removed (hx/sparse.py:28-34)."""
    M = sp.csr_matrix(A, copy=True)
    M.sum_duplicates()
    M.eliminate_zeros()
    M.sort_indices()
    return M


def mm_write(A, path, symmetric: bool = False) -> None:
    """Write a matrix or vector in Matrix Market format, 17 significant digits
    (hx/sparse.py:302-309); 1-D arrays are written as n x 1 columns."""
    if isinstance(A, np.ndarray):
        scipy.io.mmwrite(path, A.reshape(-1, 1) if A.ndim == 1 else A, precision=17)
        return
    scipy.io.mmwrite(path, A, precision=17, symmetry="symmetric" if symmetric else "general")


def mm_read(path) -> sp.csr_matrix:
    """Read a Matrix Market file as canonical CSR; vectors come back n x 1
    (hx/sparse.py:312-317)."""
    M = scipy.io.mmread(path)
    if isinstance(M, np.ndarray):
        return canonical(sp.csr_matrix(M))
    return canonical(M)
