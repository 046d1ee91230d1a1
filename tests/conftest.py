"""Shared fixtures: golden-file loaders and GPU gating."""

from __future__ import annotations

import pathlib
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libedfa.so")
    config.addinivalue_line("markers", "slow: larger-than-unit parity case")


def golden(name: str) -> dict:
    return dict(np.load(GOLDEN / f"{name}.npz"))


def g_csr(d, name):
    return sp.csr_matrix((d[name + "_val"], d[name + "_idx"].astype(np.int32),
                          d[name + "_ptr"].astype(np.int32)),
                         shape=tuple(int(v) for v in d[name + "_shape"]))


def g_sets(d, name):
    p, i = d[name + "_ptr"], d[name + "_idx"]
    return [i[p[k]:p[k + 1]] for k in range(len(p) - 1)]


def g_blocks(d):
    return tuple(g_csr(d, n) for n in ("A_ff", "A_fc", "A_cf", "A_cc"))


class GoldenSystem:
    """Minimal BlockSystem look-alike built from a golden file."""

    def __init__(self, d):
        self.A_ff, self.A_fc, self.A_cf, self.A_cc = g_blocks(d)
        self._rhs = d["rhs"]
        self.free_faces = d["free_faces"]
        self.face_index = d["face_index"]

    @property
    def n_free_faces(self):
        return self.A_ff.shape[0]

    @property
    def n_cells(self):
        return self.A_cc.shape[0]

    @property
    def n_unknowns(self):
        return self.n_free_faces + self.n_cells

    def rhs(self):
        return self._rhs

    def full_matrix(self):
        return sp.bmat([[self.A_ff, self.A_fc], [self.A_cf, self.A_cc]], format="csr")


def same_csr(A, B):
    A, B = A.tocsr(), B.tocsr()
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr)
            and np.array_equal(A.indices, B.indices))


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:   # pragma: no cover
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda:0")
