"""Sampled parity fixture of BASELINE config 5 (256^3) from the pinned oracle.

    python tests/golden/make_oracle_c5.py

A full 256^3 CPU run takes hours, so config 5 is gated on
samples, as §8(d) prescribes:

* stage-1 rows of 10,240 seeded random cells: the oracle computes them on
  z-slabs of the same generator (configs.slab_case: 9 cell layers around the
  sampled layer, so the sampled rows -- pattern reach 2 -- see exactly the
  full system's A_ff / A_cf / A_fc rows) and stores the sets and G~/F~ rows;
* ILU(0) on a sub-block of S~: the oracle's S~ restricted to a 64 x 64 patch
  of one cell layer (its H~ rows from the slab's stage 1), with the oracle's
  ILU(0) factors of that block -- the GPU factorisation fed the same block
  must reproduce them bit for bit.
"""

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import edfa_oracle as O                     # noqa: E402
from paper_2009_13916_b200 import configs                # noqa: E402

N = 256
LAYERS = (7, 96, 181, 252)        # sampled cell layers (one next to the top boundary)
PER_LAYER = 2560


def main():
    rng = np.random.default_rng(2009)
    nxy = N * N
    out = {"rows": [], "set_ptr": [0], "set_idx": [], "G_ptr": [0], "G_idx": [], "G_val": [],
           "F_ptr": [0], "F_idx": [], "F_val": []}
    for L in LAYERS:
        s0, s1 = max(0, L - 4), min(N, L + 5)
        sub = configs.slab_case(5, N, s0, s1).system
        cells = np.sort(rng.choice(nxy, size=PER_LAYER, replace=False)) + (L - s0) * nxy
        sets = O.static_sets(sub.grid, sub.face_index, "A")
        # stage-1 rows of the sampled cells only (the oracle's per-row kernel)
        keep = set(cells.tolist())
        o1 = O.build_stage1(sub.A_ff, sub.A_fc, sub.A_cf,
                            sets=[sets[m] if m in keep else np.empty(0, np.int64) for m in range(sub.n_cells)],
                            no_fill=True, n_workers=8)
        G, FT = o1.G.tocsr(), o1.F.T.tocsr()
        # global numbering: cells shift by s0 layers; faces are stored as global
        # face ids (hx/grid.py:97-107), the test maps the GPU's free indices to them
        from paper_2009_13916_b200.parallel import _sub_face_keys
        gkey, _ = _sub_face_keys(N, N, N, s0, s1 - s0)
        fk = gkey[sub.free_faces]                                     # sub free face -> global face id
        for m in cells:
            q = np.asarray(o1.sets[m], dtype=np.int64)
            out["rows"].append(m + s0 * nxy)
            out["set_idx"].append(fk[q])
            out["set_ptr"].append(out["set_ptr"][-1] + q.size)
            for M, nm in ((G, "G"), (FT, "F")):
                lo, hi = M.indptr[m], M.indptr[m + 1]
                out[nm + "_idx"].append(fk[M.indices[lo:hi]])
                out[nm + "_val"].append(M.data[lo:hi])
                out[nm + "_ptr"].append(out[nm + "_ptr"][-1] + hi - lo)
        print("layer", L, "done", flush=True)
    # ILU(0) of a 64 x 64 patch of S~ in layer 96 (H~ rows need the whole slab's stage 1)
    L = 96
    s0, s1 = L - 4, L + 5
    sub = configs.slab_case(5, N, s0, s1).system
    o1 = O.build_stage1(sub.A_ff, sub.A_fc, sub.A_cf, sets=O.static_sets(sub.grid, sub.face_index, "A"),
                        no_fill=True, n_workers=8)
    patch = ((L - s0) * nxy + np.arange(64)[:, None] * N + np.arange(64)[None, :]).ravel()
    S = O.canonical(O.canonical(sub.A_cc - o1.H).tocsr()[patch][:, patch])
    fac = O.ilu(S, 0.0, no_fill=True)
    Lf, Uf = fac.L.tocsr(), fac.U.tocsr()
    np.savez_compressed(
        HERE / "oracle_c5_sample.npz",
        rows=np.array(out["rows"], np.int64), set_ptr=np.array(out["set_ptr"]), set_idx=np.concatenate(out["set_idx"]),
        G_ptr=np.array(out["G_ptr"]), G_idx=np.concatenate(out["G_idx"]), G_val=np.concatenate(out["G_val"]),
        F_ptr=np.array(out["F_ptr"]), F_idx=np.concatenate(out["F_idx"]), F_val=np.concatenate(out["F_val"]),
        S_ptr=S.indptr, S_idx=S.indices, S_val=S.data, S_n=S.shape[0],
        L_ptr=Lf.indptr, L_idx=Lf.indices, L_val=Lf.data, U_ptr=Uf.indptr, U_idx=Uf.indices, U_val=Uf.data)
    print("rows", len(out["rows"]), "S patch", S.shape, S.nnz)


if __name__ == "__main__":
    main()
