"""Z-slab partition, halo exchange and the distributed GMRES driver on CPU.

The partition/halo bookkeeping and ``parallel.slab_gmres`` are product code;
here every slab's arithmetic is done by ``tests/slab_cpu.CpuSlab`` (oracle /
scipy) so the multi-rank path runs with the gloo backend, world_size 2, on
CPU.  The reference for the partitioned solve is the oracle's EDFA with
slab-block-diagonal inner factors (``block_jacobi_reference``).
"""

from __future__ import annotations

import os
import pathlib
import socket
import sys

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import edfa_oracle as O
from paper_2009_13916_b200 import configs, parallel
from paper_2009_13916_b200.precond import DynamicConfig
from slab_cpu import CpuSlab, block_jacobi_reference, ext_stage1

ROOT = pathlib.Path(__file__).resolve().parents[1]


def small_system(n=6, which=2):
    return (configs.config2(n=n) if which == 2 else configs.config1(n=n)).system


def global_sets(system, proto):
    if proto == "base":
        return O.base_sets(system.A_cf)
    return O.static_sets(system.grid, system.face_index, proto)


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_partition_covers_and_halo_consistent(parts):
    s = small_system(6)
    lays = parallel.build_layouts(s, parts, halo=3)
    faces = np.concatenate([l.own_faces for l in lays])
    cells = np.concatenate([l.own_cells for l in lays])
    assert np.array_equal(np.sort(faces), np.arange(s.n_free_faces))
    assert np.array_equal(np.sort(cells), np.arange(s.n_cells))
    for l in lays:
        for q, (a, b) in l.recv_faces.items():
            assert q != l.rank
            assert lays[q].send_faces[l.rank].size == b - a
            assert np.array_equal(lays[q].own_faces[lays[q].send_faces[l.rank]], l.halo_faces[a:b])
        for q, (a, b) in l.recv_cells.items():
            assert np.array_equal(lays[q].own_cells[lays[q].send_cells[l.rank]], l.halo_cells[a:b])
        if parts > 1:
            # z-slabs: only the slabs directly above / below are neighbours
            assert set(l.recv_faces) | set(l.recv_cells) <= {l.rank - 1, l.rank + 1}


@pytest.mark.parametrize("parts", [2, 3])
def test_local_blocks_reproduce_global_spmv(parts):
    s = small_system(6)
    lays = parallel.build_layouts(s, parts, halo=3)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(s.n_unknowns)
    y = s.full_matrix() @ x
    nf = s.n_free_faces
    for l in lays:
        xe = np.concatenate([x[l.own_faces], x[nf + l.own_cells], x[l.halo_faces], x[nf + l.halo_cells]])
        yl = l.blocks["A_loc"] @ xe
        # same entries, columns reordered (halo last): equal up to summation order
        ref = np.concatenate([y[l.own_faces], y[nf + l.own_cells]])
        assert np.abs(yl - ref).max() <= 1e-13 * np.abs(y).max()
        # the apply's off-diagonal blocks
        tf = np.concatenate([x[l.own_faces], x[l.halo_faces]])
        assert np.allclose(l.blocks["A_cf_loc"] @ tf, (s.A_cf @ x[:nf])[l.own_cells], rtol=0, atol=1e-12)
        yc = np.concatenate([x[nf + l.own_cells], x[nf + l.halo_cells]])
        assert np.allclose(l.blocks["A_fc_loc"] @ yc, (s.A_fc @ x[nf:])[l.own_faces], rtol=0, atol=1e-12)


@pytest.mark.parametrize("kind,proto,dyn", [("base", "base", None), ("static", "A", None),
                                            ("static", "B", None), ("static", "E", None),
                                            ("dynamic", None, (1, 4, None))])
def test_extended_stage1_rows_are_exact(kind, proto, dyn):
    """Own rows of G~/F~ and H~[own, own] from the extended subsystem equal
    the global stage 1 (so slab setup needs no communication after the
    one-time halo copy)."""
    s = small_system(8)
    halo = parallel.halo_layers(kind, proto or "A", DynamicConfig(1, 4) if dyn else None)
    lays = parallel.build_layouts(s, 3, halo=halo)
    sets = None if dyn else global_sets(s, proto)
    if dyn:
        g = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, dynamic=dyn, no_fill=True)
    else:
        g = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, sets=sets, no_fill=True)
    for l in lays:
        e = ext_stage1(l, sets, dyn)
        own = l.blocks["own_cells_in_ext"]
        Ge = e.G.tocsr()[own]
        Gg = g.G.tocsr()[l.own_cells]
        Ge_glob = sp.csr_matrix((Ge.data, l.ext_faces[Ge.indices], Ge.indptr), shape=Gg.shape)
        assert (abs(Ge_glob - Gg)).max() <= 1e-14 * abs(Gg).max()
        He = e.H.tocsr()[own][:, own]
        Hg = g.H.tocsr()[l.own_cells][:, l.own_cells]
        assert (abs(He - Hg)).max() <= 1e-13 * abs(Hg).max()
        Fe = e.F.tocsc()[:, own]
        Fg = g.F.tocsc()[:, l.own_cells]
        Fe_glob = sp.csc_matrix((Fe.data, l.ext_faces[Fe.indices], Fe.indptr), shape=Fg.shape)
        assert (abs(Fe_glob - Fg)).max() <= 1e-14 * abs(Fg).max()


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_slab_gmres_single_process_matches_block_jacobi_oracle(parts):
    s = small_system(6)
    lays = parallel.build_layouts(s, parts, halo=parallel.halo_layers("static", "A"))
    sets = global_sets(s, "A")
    slabs = [CpuSlab(l, sets) for l in lays]
    op = parallel.SlabOperator(slabs, parallel.LocalComm(parts))
    xs, rep = parallel.slab_gmres(op, [p.rhs for p in slabs], tol=1e-8, restart=50)
    x = parallel.scatter_solution(lays, xs, s.n_free_faces, s.n_cells)
    x_ref, rep_ref, _ = block_jacobi_reference(s, lays, sets)
    assert rep.converged and rep_ref.converged
    assert abs(rep.n_it - rep_ref.n_it) <= 2
    assert rep.final_relres <= 1e-8
    true = np.linalg.norm(s.rhs() - s.full_matrix() @ x) / np.linalg.norm(s.rhs())
    assert true <= 1e-8
    assert np.linalg.norm(x - x_ref) <= 1e-7 * np.linalg.norm(x_ref)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _gloo_worker(rank, world, port, parts, out_dir):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT / "tests"))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        s = small_system(6)
        mine = [q for q in range(parts) if q % world == rank]
        lays = parallel.build_layouts(s, parts, halo=parallel.halo_layers("static", "A"), ranks=mine)
        sets = global_sets(s, "A")
        slabs = [CpuSlab(lays[q], sets) for q in mine]
        comm = parallel.TorchComm([q % world for q in range(parts)])
        op = parallel.SlabOperator(slabs, comm)
        xs, rep = parallel.slab_gmres(op, [p.rhs for p in slabs], tol=1e-8, restart=50)
        for q, x in zip(mine, xs):
            np.save(os.path.join(out_dir, f"x{q}.npy"), x.numpy())
        np.save(os.path.join(out_dir, f"rep{rank}.npy"), np.array([rep.n_it, rep.converged, rep.final_relres]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("parts", [2, 4])
def test_slab_gmres_gloo_world2(tmp_path, parts):
    """Two processes over gloo (the NCCL path's host logic on CPU)."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_gloo_worker, args=(2, port, parts, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    s = small_system(6)
    lays = parallel.build_layouts(s, parts, halo=parallel.halo_layers("static", "A"))
    xs = [np.load(tmp_path / f"x{q}.npy") for q in range(parts)]
    x = parallel.scatter_solution(lays, xs, s.n_free_faces, s.n_cells)
    reps = [np.load(tmp_path / f"rep{r}.npy") for r in range(2)]
    assert reps[0][0] == reps[1][0] and reps[0][1] == 1
    x_ref, rep_ref, _ = block_jacobi_reference(s, lays, global_sets(s, "A"))
    assert abs(int(reps[0][0]) - rep_ref.n_it) <= 2
    assert np.linalg.norm(x - x_ref) <= 1e-7 * np.linalg.norm(x_ref)
    true = np.linalg.norm(s.rhs() - s.full_matrix() @ x) / np.linalg.norm(s.rhs())
    assert true <= 1e-8


def test_slab_bounds_errors():
    with pytest.raises(ValueError):
        parallel.slab_bounds(4, 5)
    assert parallel.slab_bounds(8, 3) == [(0, 2), (2, 5), (5, 8)]


@pytest.mark.parametrize("parts,n,nz", [(2, 5, 10), (3, 6, 12), (4, 4, 16)])
def test_slab_layout_from_sub_box_equals_global_layout(parts, n, nz):
    """A rank that assembles only its own sub-box (configs.slab_case) gets the
    same owned rows, halo lists, send lists and local blocks as the layout
    cut from the global system (entries matched by global ids).  Patterns
    are exact; values agree to 1e-13 (numpy's batched element kernels round
    differently in the last bit for a different number of cells; the device
    assembly is per cell and bit-identical)."""

    def same(a, b):
        return (a.shape == b.shape and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
                and np.abs(a.data - b.data).max(initial=0.0) <= 1e-13 * np.abs(b.data).max(initial=1.0))
    s = configs.config2(n=n, nz=nz).system
    halo = parallel.halo_layers("static", "A")
    glays = parallel.build_layouts(s, parts, halo=halo)
    gkey_f, _ = parallel._sub_face_keys(n, n, nz, 0, nz)
    free_key = gkey_f[s.free_faces]
    for r in range(parts):
        k0, k1 = parallel.slab_bounds(nz, parts)[r]
        s0, s1 = max(0, k0 - halo - 1), min(nz, k1 + halo + 1)
        sub = configs.slab_case(2, n, s0, s1, nz=nz).system
        lay = parallel.build_slab_layout(sub, s0, nz, parts, r, halo)
        g = glays[r]
        assert np.array_equal(lay.face_keys[lay.own_faces], free_key[g.own_faces])
        assert np.array_equal(lay.cell_keys[lay.own_cells], g.own_cells)
        assert np.array_equal(lay.face_keys[lay.halo_faces], free_key[g.halo_faces])
        assert np.array_equal(lay.cell_keys[lay.halo_cells], g.halo_cells)
        assert lay.recv_faces == g.recv_faces and lay.recv_cells == g.recv_cells
        assert lay.send_faces.keys() == g.send_faces.keys() and lay.send_cells.keys() == g.send_cells.keys()
        for q in g.send_faces:
            assert np.array_equal(lay.send_faces[q], g.send_faces[q])
        for q in g.send_cells:
            assert np.array_equal(lay.send_cells[q], g.send_cells[q])
        for name in ("A_loc", "A_cf_loc", "A_fc_loc", "A_ff_own", "A_cc_own"):
            assert same(lay.blocks[name], g.blocks[name]), name
        for name in ("A_ff", "A_fc", "A_cf", "A_cc"):
            assert same(lay.blocks["ext"][name], g.blocks["ext"][name]), name
        for a, b in zip(lay.blocks["ext_topology"], g.blocks["ext_topology"]):
            assert np.array_equal(a, b)
        rb = g.blocks["rhs"]
        assert np.abs(lay.blocks["rhs"] - rb).max() <= 1e-13 * max(np.abs(rb).max(), 1.0)
