#!/usr/bin/env python
"""EDFA setup + GMRES(50) solve throughput on B200 (BASELINE.json metric).

One step = the hot path over one system: system creation from the resident
blocks (merged A, SELL copies, grid topology), restriction patterns, stage 1
(restricted row solves, G~/F~, H~ = G~ A_ff F~, IC(0) of -A_ff), stage 2
(S~ = A_cc - H~, ILU(0)) and right-preconditioned GMRES(50) to rtol 1e-8 from
x0 = 0 (hx/driver.py:108-142's stage timers: t_stage1, t_stage2, t_solve).

Workload at N = 1: BASELINE config 5 -- 256^3 hex grid (16.8M cells, 67.2M
DOF), config-2 lognormal anisotropic K, static prototype A, IC(0)/ILU(0) --
the largest single-GPU configuration, assembled on the device from seeded
synthetic inputs (SPE10 is not in this container).  ``value`` = N_dof *
steps / device time with the blocks, rhs and grid index arrays resident in
HBM; ``e2e`` = the same through the drop-in API from page-locked host scipy
blocks (H2D of the blocks, rhs and grid arrays, D2H of x inside the timed
region).  Config 2 (64^3) is measured too and reported under ``config2``.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl edfa|reference]
                    [--config C] [--n n] [--slabs P]

N > 1 (torchrun, one process per GPU): z-slab partitioned solve
(parallel.py), see run_slabs.  ``--impl reference`` times the CPU
restatement of the reference algorithm (oracle/, the reference is pure
Python and cannot travel to the GPU box): one full measured config-2 run
with the reference's stage timers, extrapolated per DOF to the bench config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "EDFA setup+GMRES solve throughput per system"
UNIT = "MDOF/s"
DEFAULT_N = {1: 16, 2: 64, 3: 128, 4: None, 5: 256}
# GMRES(50) iterations of config 5 at 256^3 on the GPU (profiles/r02n_bench.json);
# the CPU arm's extrapolation uses it (the MGS oracle matched the GPU count at 64^3: 84 = 84)
CONFIG5_ITERS = 382


def metric_of(k):
    return f"{METRIC} (config {k})"


def make_case(config, n, host=True):
    from paper_2009_13916_b200 import configs
    mk = configs.make if host else configs.inputs_only
    if config == 4:
        return mk(4) if n is None else mk(4, nx=n, ny=n, nz=n)
    return mk(config, n=n or DEFAULT_N[config])


INNER = {}   # --drop-tol / --fill override the config's inner-solve options


def inner_opts(case):
    p = case.precond
    o = dict(face_drop_tol=p.get("face_drop_tol", 0.0), schur_drop_tol=p.get("schur_drop_tol", 0.0),
             no_fill=p.get("no_fill", True))
    o.update(INNER)
    return o


def stage1_of(case, ds):
    """Stage 1 of a BASELINE config through the drop-in API."""
    from paper_2009_13916_b200.precond import DynamicConfig, build_stage1, patterns_for
    p, o = case.precond, inner_opts(case)
    if p["pattern"] == "dynamic":
        return build_stage1(ds, dynamic=DynamicConfig(p["n_add"], p["n_ent"]), face_drop_tol=o["face_drop_tol"],
                            no_fill=o["no_fill"])
    return build_stage1(ds, patterns=patterns_for(ds, p["pattern"], p.get("prototype", "A")),
                        face_drop_tol=o["face_drop_tol"], no_fill=o["no_fill"])


def precond_of(case, ds, s1):
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner
    o = inner_opts(case)
    pre = BlockLDUPreconditioner(ds, s1, settings=dict(tau_filt=0.0, filtration="none",
                                                       schur_drop_tol=o["schur_drop_tol"], no_fill=o["no_fill"]))
    pre.refresh(ds)
    return pre


def build_pre(case, ds):
    return precond_of(case, ds, stage1_of(case, ds))


def inner_tag(case):
    o = inner_opts(case)
    if o["no_fill"] and not o["face_drop_tol"] and not o["schur_drop_tol"]:
        return "IC0ILU0"
    return f"ICILU(tau={o['face_drop_tol']:g},{'nofill' if o['no_fill'] else 'fill'})"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="edfa", choices=["edfa", "reference"])
    ap.add_argument("--n", type=int, default=None, help="grid cells per side (default: the config's size)")
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config (5 = the headline: largest single-GPU workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config2", action="store_true", help="skip the extra config-2 leg")
    ap.add_argument("--drop-tol", type=float, default=0.0,
                    help="face_drop_tol = schur_drop_tol (evidence runs of the threshold inner solves)")
    ap.add_argument("--fill", action="store_true", help="no_fill=False (threshold factorisations with fill)")
    ap.add_argument("--single-system", action="store_true",
                    help="config 4: time one system instead of the 10-step sequence")
    ap.add_argument("--profile-json", default=None, help="write the per-kernel event profile here")
    ap.add_argument("--slabs", type=int, default=0,
                    help="z-slab partitioned solver with this many slabs per process (default: 1 slab per "
                         "GPU when N > 1, the single-device solver when N = 1)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong (one global grid cut into N slabs) or weak (n^3 per GPU, grown along z)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        if os.environ.get("EDFA_BENCH_NO_CLOCKS"):
            return self
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU baseline (oracle port)
def n_dof_config2(n, nz=None):
    """Free faces + cells of the config-2/5 generator on an n x n x nz box
    (x faces minus the two Dirichlet x planes, plus y and z faces)."""
    nz = nz or n
    return (n + 1) * n * nz - 2 * n * nz + n * (n + 1) * nz + n * n * (nz + 1) + n * n * nz


def oracle_run(n: int, max_it: int = 2000):
    """One full CPU run of the reference algorithm (oracle/ restatement, the
    reference is pure Python + scipy) on the config-2 generator at n^3 with
    hexflow's stage timers (hx/driver.py:110-140): stage 1 with n_workers=1
    (SURVEY.md §8(d)), stage 2, GMRES(50) to 1e-8.  Input generation is not
    timed."""
    from oracle import edfa_oracle as O
    from paper_2009_13916_b200 import configs
    s = configs.config2(n=n).system
    A = s.full_matrix()
    b = s.rhs()
    t0 = time.perf_counter()
    sets = O.static_sets(s.grid, s.face_index, "A")
    o1 = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, sets=sets, no_fill=True, n_workers=1)
    t1 = time.perf_counter()
    o2 = O.build_stage2(s.A_cc, o1, no_fill=True)
    t2 = time.perf_counter()
    _, rep = O.gmres(lambda v: A @ v, lambda r: O.apply(o1, o2, s.A_fc, s.A_cf, r), b, tol=1e-8, restart=50,
                     max_it=max_it)
    t3 = time.perf_counter()
    N = s.n_unknowns
    return dict(n=n, n_dof=N, t_stage1=t1 - t0, t_stage2=t2 - t1, t_solve=t3 - t2, iterations=rep.n_it,
                converged=bool(rep.converged), final_relres=rep.final_relres,
                mdof_s=N / (t3 - t0) / 1e6, setup_mdof_s=N / (t2 - t0) / 1e6, solve_mdof_s=N / (t3 - t2) / 1e6)


def extrapolate(run, N_full, iters_full):
    """Per-DOF setup cost and per-DOF-per-iteration solve cost of a measured
    run, scaled to N_full DOF and iters_full GMRES iterations (stage-1 rows
    are independent, the factorisation and the Krylov work are linear in N)."""
    per_dof_setup = (run["t_stage1"] + run["t_stage2"]) / run["n_dof"]
    per_dof_iter = run["t_solve"] / max(run["iterations"], 1) / run["n_dof"]
    t = N_full * per_dof_setup + iters_full * N_full * per_dof_iter
    return N_full / t / 1e6


def cpu_baseline(N_full, iters_full, n_sample=32):
    """The GPU line's cpu_baseline: a bounded (~15 s) full oracle run on the
    same generator at n_sample^3, one core, extrapolated to the workload."""
    run = oracle_run(n_sample)
    return {"value": extrapolate(run, N_full, iters_full), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle port (CPU restatement of hexflow's EDFA + GMRES(50)) on the config-2 generator at "
                       f"{n_sample}^3 (N={run['n_dof']}): stage 1 (n_workers=1) {run['t_stage1']:.2f} s, "
                       f"stage 2 {run['t_stage2']:.2f} s, GMRES {run['iterations']} it {run['t_solve']:.2f} s "
                       f"(measured); extrapolated per DOF to N={N_full} with {iters_full} iterations"),
            "measured_sample": run}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU algorithm on the box's host cores (no GPU).  The
    headline ``value`` extrapolates one full, measured config-2 run (64^3,
    stage timers, n_workers=1 as SURVEY.md §8(d)) per DOF to the bench config
    (config 5: 67.2M DOF, CONFIG5_ITERS iterations) -- a 256^3 CPU run would
    take ~10 hours; ``measured_config2`` is that run itself.  The W + K steps
    are bounded 24^3 samples (~5 s each) whose extrapolations show the spread."""
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    cfg = args.config
    n = args.n or DEFAULT_N[cfg]
    if cfg in (2, 5):
        N_full = n_dof_config2(n)
        iters = CONFIG5_ITERS if (cfg == 5 and n == 256) else None
    else:
        raise SystemExit("--impl reference covers the config-2/5 generator")
    full = oracle_run(64)
    if iters is None:
        iters = full["iterations"] if n == 64 else int(round(full["iterations"] * n / 64))
    samples = []
    for k in range(max(args.warmup, 0) + args.steps):
        r = oracle_run(24)
        if k >= args.warmup:
            samples.append(extrapolate(r, N_full, iters))
    v = extrapolate(full, N_full, iters) if not (cfg == 2 and n == 64) else full["mdof_s"]
    workload = f"config{cfg}-{n}^3-staticA-IC0ILU0-gmres50"
    line = {
        "impl": "reference", "metric": metric_of(cfg), "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N_full / (v * 1e6) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded config-{cfg} generator)",
        "config": {"workload": workload, "n_dof": N_full, "rtol": 1e-8, "restart": 50,
                   "gmres_iterations_assumed": iters, "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": (f"full measured oracle run on the config-2 generator at 64^3 (N={full['n_dof']}, "
                                    f"stage timers, n_workers=1, {full['iterations']} GMRES iterations), "
                                    + ("the bench workload itself" if (cfg == 2 and n == 64) else
                                       f"extrapolated per DOF to N={N_full} with {iters} iterations"))},
        "measured_config2": full,
        "step_samples_extrapolated": samples,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kernel_groups(prof):
    """Profile records by kernel: the forward and backward ILU solves are one
    kernel (k_wf / k_tile_flow run in the two directions), every other record
    is one kernel."""
    out = {}
    for k, v in prof.items():
        g = "trsv_ilu" if k.startswith("trsv_ilu") else k
        o = out.setdefault(g, {"ms": 0.0, "bytes": 0.0, "launches": 0})
        o["ms"] += v["ms"]
        o["bytes"] += v["bytes"]
        o["launches"] += v["launches"]
    return out


# ---------------------------------------------------------------- algorithmic bytes
def csr_b(nnz, rows):
    return 12.0 * nnz + 4.0 * (rows + 1)


def spmv_b(nnz, rows, cols):
    return csr_b(nnz, rows) + 8.0 * cols + 8.0 * rows


def trsv_b(nnz, n):
    return csr_b(nnz, n) + 16.0 * n


def algorithmic_bytes(ds, pre, n_it, m):
    """Setup bytes and total solve bytes of one step."""
    i1, i2 = pre.stage1.info, pre.stage2.info
    nf, ne = ds.n_free_faces, ds.n_cells
    N = nf + ne
    nnz = {k: getattr(ds, k).nnz for k in ("A_ff", "A_fc", "A_cf", "A_cc")}
    q = 4.0 * i1.nnz_Q + 4.0 * (ne + 1)
    setup = (csr_b(nnz["A_ff"], nf) + csr_b(nnz["A_cf"], ne) + csr_b(nnz["A_fc"], ne) + csr_b(nnz["A_cc"], ne) + q
             + csr_b(i1.nnz_G, ne) + csr_b(i1.nnz_FT, ne) + csr_b(i1.nnz_H, ne) + csr_b(i1.nnz_L, nf)
             + csr_b(i1.nnz_H, ne) + csr_b(i2.nnz_S, ne) + csr_b(i2.nnz_L, ne) + csr_b(i2.nnz_U, ne))
    nnz_A = sum(nnz.values())
    apply_b = (2 * (2 * trsv_b(i1.nnz_L, nf)) + spmv_b(nnz["A_cf"], ne, nf) + spmv_b(nnz["A_fc"], nf, ne)
               + trsv_b(i2.nnz_L, ne) + trsv_b(i2.nnz_U, ne) + 8.0 * (3 * nf + 2 * ne))
    spmv_A = spmv_b(nnz_A, N, N)
    solve = 0.0
    done, cycles = 0, 0
    while done < n_it:
        k = min(m, n_it - done)
        solve += sum(spmv_A + apply_b + 8.0 * N * (2 * j + 5) for j in range(k))
        solve += apply_b + 8.0 * N * (m + 2) + spmv_A + 16.0 * N     # restart: update + true residual
        done += k
        cycles += 1
    return setup, solve


def peak_hbm():
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        peaks = {}
    if peaks.get("hbm_gbs"):
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"


# ---------------------------------------------------------------- EDFA arm
def profile_report(lib, c, reset=1):
    import ctypes
    n = lib.edfa_ctx_profile_report(c, None, 0, 0)
    buf = ctypes.create_string_buffer(int(n))
    lib.edfa_ctx_profile_report(c, buf, n, reset)
    return json.loads(buf.value.decode())


def device_inputs(case):
    """Assemble the config on the device (device_assembly.assemble_device,
    hx/assembly.py:186-333) -- the resident inputs of the timed region."""
    import torch

    from paper_2009_13916_b200 import device_assembly as DA
    t = time.perf_counter()
    dsys = DA.assemble_device(*case.meta["inputs"], element_ops=False)
    torch.cuda.synchronize()
    return dsys, time.perf_counter() - t


def timed_steps(case, dsys, steps, warmup, lib, c, flush, clk=None):
    """W untimed + K timed steps on the resident blocks; per-phase CUDA events
    (stage 1, stage 2, solve) inside each step.  Returns per-step records and
    the last step's objects."""
    import torch

    from paper_2009_13916_b200.device import DeviceSystem, system_operator
    from paper_2009_13916_b200.krylov import gmres
    g = case.meta["inputs"][0]
    base = dsys.system
    blocks = (base.A_ff, base.A_fc, base.A_cf, base.A_cc)
    b = base.rhs()

    def step():
        ds = DeviceSystem(*blocks, rhs=b, topology_src=dsys.topology_inputs)
        ds.set_grid(g.nx, g.ny, g.nz)
        s1 = stage1_of(case, ds)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        pre = precond_of(case, ds, s1)
        e2 = torch.cuda.Event(enable_timing=True)
        e2.record()
        x, rep = gmres(system_operator(ds), pre, b, tol=case.rtol, restart=case.restart, max_it=case.max_it)
        return ds, pre, x, rep, e1, e2

    recs, last = [], None
    ds = pre = x = rep = None
    for w in range(warmup + steps):
        timed = w >= warmup
        if timed:
            flush.fill_(1.0)                        # evict L2 between steps
        torch.cuda.synchronize()
        e0, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        last = ds = pre = x = rep = None             # one preconditioner alive at a time (256^3 memory)
        e0.record()
        ds, pre, x, rep, e1, e2 = step()
        e3.record()
        torch.cuda.synchronize()
        if timed:
            recs.append(dict(ms=e0.elapsed_time(e3), stage1_ms=e0.elapsed_time(e1), stage2_ms=e1.elapsed_time(e2),
                             solve_ms=e2.elapsed_time(e3), n_it=rep.n_it, relres=rep.final_relres,
                             converged=rep.converged))
        last = (ds, pre, x, rep)
    return recs, last


def run_edfa(args):
    import ctypes

    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2009_13916_b200 import _lib
    from paper_2009_13916_b200.device import DeviceSystem, ctx, pinned_copy, system_operator, to_host_vector
    from paper_2009_13916_b200.krylov import gmres

    lib = _lib.lib()
    cfg = args.config
    n = args.n or DEFAULT_N[cfg]
    case = make_case(cfg, n, host=False)
    dsys, t_asm = device_inputs(case)
    N = dsys.n_unknowns
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    c = ctx()

    # ---- profile of one (untimed) warm-up step: kernel shares, dominant kernel
    lib.edfa_ctx_profile_filter(c, b"")
    lib.edfa_ctx_profile(c, 1)
    profile_report(lib, c)
    _, last = timed_steps(case, dsys, 0, 1, lib, c, flush)
    prof_full = profile_report(lib, c)
    lib.edfa_ctx_profile(c, 0)
    last = None
    dom_name = max(kernel_groups(prof_full).items(), key=lambda kv: kv[1]["ms"])[0] if prof_full else ""

    # ---- device-resident timed region; CUDA events bracket every launch of
    # the dominant kernel only (cheap enough not to perturb the step)
    lib.edfa_ctx_profile_filter(c, dom_name.encode())
    lib.edfa_ctx_profile(c, 1)
    profile_report(lib, c)
    launches0 = lib.edfa_ctx_launch_count(c)
    with ClockSampler(local) as clk:
        recs, last = timed_steps(case, dsys, args.steps, max(args.warmup - 1, 0), lib, c, flush)
    launches = lib.edfa_ctx_launch_count(c) - launches0
    prof = profile_report(lib, c)
    lib.edfa_ctx_profile(c, 0)
    lib.edfa_ctx_profile_filter(c, b"")
    clocks = clk.summary()
    t_total_ms = sum(r["ms"] for r in recs)
    value = N * args.steps / (t_total_ms / 1e3) / 1e6
    ds, pre, x, rep = last
    setup_b, solve_b = algorithmic_bytes(ds, pre, rep.n_it, case.restart)
    peak, peak_src = peak_hbm()
    med = {k: statistics.median(r[k] for r in recs) for k in ("ms", "stage1_ms", "stage2_ms", "solve_ms")}
    setup_ms = med["stage1_ms"] + med["stage2_ms"]
    phases = {
        "stage1_ms": med["stage1_ms"], "stage2_ms": med["stage2_ms"], "solve_ms": med["solve_ms"],
        "setup_mdof_s": N / (setup_ms / 1e3) / 1e6, "solve_mdof_s": N / (med["solve_ms"] / 1e3) / 1e6,
        "ms_per_iteration": med["solve_ms"] / max(rep.n_it, 1),
        "setup_algorithmic_bytes": setup_b, "solve_algorithmic_bytes": solve_b,
        "setup_hbm_frac": setup_b / (setup_ms / 1e3) / 1e9 / peak,
        "solve_hbm_frac": solve_b / (med["solve_ms"] / 1e3) / 1e9 / peak,
        "note": "phase fractions = SURVEY.md 8(d) algorithmic bytes / phase time / HBM peak; the setup phase "
                "includes system creation (merged A, SELL copies, topology) in stage 1",
    }
    del pre, x, ds
    last = None
    lib.edfa_ctx_trim(c)                     # hand the library's cached blocks back before the e2e leg

    # ---- end-to-end through the public API from host scipy blocks
    s_host = dsys.to_host()
    s_pin = pinned_copy(s_host)              # the host application's page-locked staging of the inputs
    h2d = sum(getattr(s_host, k).data.nbytes + getattr(s_host, k).indices.nbytes + getattr(s_host, k).indptr.nbytes
              for k in ("A_ff", "A_fc", "A_cf", "A_cc")) + s_host.rhs().nbytes
    h2d += 4 * (12 * s_host.n_cells + s_host.face_index.size)      # cell->face map, neighbours, face index
    d2h = N * 8
    e2e_times = []
    x_h = None
    n_e2e = max(1, min(args.steps, 3))
    e2e_stages = {}
    for it in range(1 + n_e2e):                                # one untimed pass first (allocator, page faults)
        x_h = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ds_h = DeviceSystem.from_host(s_pin)                  # H2D of the four blocks, rhs_f / rhs_c, topology
        if it == 0:                                            # stage walls of the untimed pass only (extra syncs)
            torch.cuda.synchronize()
            e2e_stages["upload_s"] = time.perf_counter() - t0
        pre_h = build_pre(case, ds_h)                          # patterns from the device topology
        if it == 0:
            torch.cuda.synchronize()
            e2e_stages["setup_s"] = time.perf_counter() - t0 - e2e_stages["upload_s"]
            t1 = time.perf_counter()
        x_d, rep_h = gmres(system_operator(ds_h), pre_h, ds_h.rhs(), tol=case.rtol, restart=case.restart,
                           max_it=case.max_it)
        if it == 0:
            torch.cuda.synchronize()
            e2e_stages["solve_s"] = time.perf_counter() - t1
            t1 = time.perf_counter()
        x_h = to_host_vector(x_d)                              # the solution read back (D2H)
        if it == 0:
            e2e_stages["readback_s"] = time.perf_counter() - t1
        del x_d
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
        del ds_h, pre_h
    e2e_val = N / statistics.median(e2e_times) / 1e6
    A_h = s_host.full_matrix()
    relres_host = float(np.linalg.norm(s_host.rhs() - A_h @ x_h) / np.linalg.norm(s_host.rhs()))
    del A_h, s_pin

    # ---- roofline of the dominant kernel (live CUDA events over the timed region)
    dname, d = max(kernel_groups(prof).items(), key=lambda kv: kv[1]["ms"]) if prof else (
        "none", {"ms": 0, "bytes": 0, "launches": 1})
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    try:
        traffic = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).get(f"config{cfg}", {}).get(dname)
    except Exception:
        pass
    tot_full = max(sum(p["ms"] for p in prof_full.values()), 1e-9)
    shares = {k: round(v["ms"] / tot_full, 4) for k, v in sorted(prof_full.items(), key=lambda kv: -kv[1]["ms"])[:10]}
    # the same figures for the six largest kernels of the step (warm-up step's events)
    top = [{"kernel": k, "ms_per_step": round(v["ms"], 3), "launches": v["launches"],
            "achieved": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else 0.0,
            "frac": round(v["bytes"] / (v["ms"] / 1e3) / 1e9 / peak, 4) if v["ms"] > 0 else 0.0}
           for k, v in sorted(kernel_groups(prof_full).items(), key=lambda kv: -kv[1]["ms"])[:6]]
    g = case.meta["inputs"][0]
    line = {
        "metric": metric_of(cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator of BASELINE config {cfg}: {case.name}), assembled on the device",
        "config": {"workload": f"{case.name}-{inner_tag(case)}-gmres50", "grid": [g.nx, g.ny, g.nz], "n_dof": N,
                   "n_free_faces": dsys.n_free_faces, "n_cells": dsys.n_cells, "rtol": case.rtol,
                   "restart": case.restart, "gmres_iterations": rep.n_it, "final_true_relres": rep.final_relres,
                   "host_check_relres": relres_host, "parallelism": "single",
                   "step_ms": [round(r["ms"], 3) for r in recs],
                   "step_phase_ms": [[round(r[k], 1) for k in ("stage1_ms", "stage2_ms", "solve_ms")] for r in recs],
                   "median_step_ms": round(med["ms"], 3),
                   "l2": "inputs larger than L2 and a 256 MiB L2 flush between steps",
                   "input_assembly_s": t_asm},
        "phases": phases,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "seconds_per_step": statistics.median(e2e_times),
                "passes": len(e2e_times),
                "untimed_first_pass_stages": e2e_stages,
                "note": "host blocks page-locked once before the timed region (pinned_copy); the copies are timed; "
                        "median of the timed passes after one untimed pass"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "launches_per_step": d["launches"] / args.steps,
                     "step_share_of_kernel_time": shares, "kernel_ms_per_step": tot_full,
                     "shares_from": "per-kernel CUDA events of one untimed warm-up step (same workload)"},
        "roofline_top": top,
        "clocks": clocks,
    }
    if args.profile_json:
        pathlib.Path(args.profile_json).write_text(json.dumps({"timed_region": prof, "warmup_step": prof_full},
                                                              indent=1))
    lib.edfa_ctx_trim(c)
    line["assembly"] = assembly_leg(case, c, lib, N)
    if cfg != 2 and not args.no_config2:
        line["config2"] = config2_leg(lib, c, flush)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(N, rep.n_it)
    print(json.dumps(line), flush=True)


def config2_leg(lib, c, flush, steps=5, warmup=2):
    """BASELINE config 2 (64^3) on the same path: the previous headline, kept
    for comparison across rounds."""
    case = make_case(2, 64, host=False)
    dsys, _ = device_inputs(case)
    recs, last = timed_steps(case, dsys, steps, warmup, lib, c, flush)
    N = dsys.n_unknowns
    t = sum(r["ms"] for r in recs)
    return {"workload": f"{case.name}-{inner_tag(case)}-gmres50", "value": N * steps / (t / 1e3) / 1e6,
            "unit": UNIT, "ms_per_step": t / steps, "gmres_iterations": last[3].n_it,
            "final_true_relres": last[3].final_relres,
            "stage1_ms": statistics.median(r["stage1_ms"] for r in recs),
            "stage2_ms": statistics.median(r["stage2_ms"] for r in recs),
            "solve_ms": statistics.median(r["solve_ms"] for r in recs)}


def assembly_leg(case, c, lib, N):
    """The device assembly of the same system (the
    producer of the path's blocks): hexflow's assemble through
    device_assembly.assemble_device -- grid arrays and tensors uploaded from
    host numpy, blocks left in HBM -- against the host numpy assembly."""
    import torch

    from paper_2009_13916_b200 import device_assembly as DA
    g, fld, props, bc, dt, p0 = case.meta["inputs"]
    DA.assemble_device(g, fld, props, bc, dt, p0)
    torch.cuda.synchronize()
    lib.edfa_ctx_profile_filter(c, b"asm_")
    lib.edfa_ctx_profile(c, 1)
    profile_report(lib, c)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = DA.assemble_device(g, fld, props, bc, dt, p0)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del d
    prof = profile_report(lib, c)
    lib.edfa_ctx_profile(c, 0)
    lib.edfa_ctx_profile_filter(c, b"")
    kms = sum(v["ms"] for v in prof.values()) / 3
    kbytes = sum(v["bytes"] for v in prof.values()) / 3
    t = statistics.median(ts)
    host = case.meta.get("host_assembly_s")
    return {"seconds": t, "mdof_s": N / t / 1e6, "kernel_ms": kms,
            "kernel_gbs": kbytes / (kms / 1e3) / 1e9 if kms > 0 else None,
            "kernels": {k: round(v["ms"] / 3, 4) for k, v in prof.items()},
            "host_numpy_seconds": host, "speedup_vs_host_numpy": host / t if host else None,
            "scope": "assemble_device: H2D of grid/tensor arrays + element operators + block rows + "
                     "Dirichlet elimination + accumulation (hx/assembly.py:186-333)"}


# ---------------------------------------------------------------- slab-partitioned arm (N > 1)
def slab_layouts_local(cfg, n, nz, parts, mine, halo):
    """Every slab this process holds, built from its own sub-box only
    (configs.slab_case assembled on the device, parallel.build_slab_layout):
    no process ever holds the global system (host memory O(slab))."""
    import torch

    from paper_2009_13916_b200 import configs, parallel
    from paper_2009_13916_b200 import device_assembly as DA
    lays = []
    for r in mine:
        k0, k1 = parallel.slab_bounds(nz, parts)[r]
        s0, s1 = max(0, k0 - halo - 1), min(nz, k1 + halo + 1)
        case = configs.slab_case(cfg, n, s0, s1, nz=nz, host=False)
        dsys = DA.assemble_device(*case.meta["inputs"], element_ops=False)
        sub = dsys.to_host()
        del dsys
        torch.cuda.synchronize()
        lays.append(parallel.build_slab_layout(sub, s0, nz, parts, r, halo))
    return lays


def run_slabs(args):
    """z-slab partitioned solve: one slab per GPU (or
    ``--slabs P`` slabs in one process), block-Jacobi inner factors per slab,
    halo exchanges over NCCL P2P, one all-reduce per Arnoldi step.
    --scaling strong: BASELINE config 5's 256^3 grid cut into N slabs;
    --scaling weak: n^3 per GPU (default 128^3) stacked along z."""
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    per_proc = max(args.slabs, 1)
    parts = world * per_proc
    from paper_2009_13916_b200 import _lib, parallel
    from paper_2009_13916_b200.device import ctx
    lib = _lib.lib()
    cfg = args.config if args.config in (1, 2, 5) else 5
    if args.scaling == "weak":
        n = args.n or 128
        nz = n * parts
    else:
        n = args.n or DEFAULT_N[cfg]
        nz = n
    rtol, restart, max_it = 1e-8, 50, 2000
    mine = [rank * per_proc + k for k in range(per_proc)]
    halo = parallel.halo_layers("static" if cfg != 1 else "base", "A")
    t0 = time.perf_counter()
    my_lays = slab_layouts_local(cfg, n, nz, parts, mine, halo)
    t_layout = time.perf_counter() - t0
    # global N from the per-slab owned counts
    n_own = torch.tensor([float(sum(l.n_own for l in my_lays))], device=dev, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(n_own)
    N = int(n_own.item())
    comm = (parallel.TorchComm([q // per_proc for q in range(parts)]) if world > 1
            else parallel.LocalComm(parts))
    kind = "base" if cfg == 1 else "static"
    solver = parallel.SlabSolver(my_lays, comm, kind=kind, prototype="A")
    if world > 1:
        t = torch.zeros(1, device=dev)
        torch.distributed.all_reduce(t)                # communicator up before the first P2P
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        solver.build()
        return solver.solve(tol=rtol, restart=restart, max_it=max_it)

    c = ctx()
    prof_full = {}
    for w in range(args.warmup):
        last = w == args.warmup - 1
        if last:
            lib.edfa_ctx_profile_filter(c, b"")
            lib.edfa_ctx_profile(c, 1)
            profile_report(lib, c)
        xs, rep = step()
        if last:
            prof_full = profile_report(lib, c)
            lib.edfa_ctx_profile(c, 0)
    torch.cuda.synchronize()
    dom_name = max(kernel_groups(prof_full).items(), key=lambda kv: kv[1]["ms"])[0] if prof_full else ""
    lib.edfa_ctx_profile_filter(c, dom_name.encode())
    lib.edfa_ctx_profile(c, 1)
    profile_report(lib, c)
    launches0 = lib.edfa_ctx_launch_count(c)
    times, reps = [], []
    solver.op.timer.enabled = True
    solver.op.timer.collect()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            xs, rep = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            reps.append(rep)
    comm_ms = solver.op.timer.collect()
    solver.op.timer.enabled = False
    launches = lib.edfa_ctx_launch_count(c) - launches0
    prof = profile_report(lib, c)
    lib.edfa_ctx_profile(c, 0)
    lib.edfa_ctx_profile_filter(c, b"")
    clocks = clk.summary()
    t_total_ms = sum(times)
    comm_share = (comm_ms["halo"] + comm_ms["allreduce"]) / max(t_total_ms, 1e-9)
    if world > 1:
        tt = torch.tensor([t_total_ms, comm_share], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_total_ms, comm_share = float(tt[0].item()), float(tt[1].item())
    value = N * args.steps / (t_total_ms / 1e3) / 1e6

    # ---- end to end from host blocks: H2D of the slab's local blocks, build, solve, D2H of x
    e2e_times = []
    h2d = 0
    for lay in my_lays:
        b = lay.blocks
        mats = [b["A_loc"], b["A_cf_loc"], b["A_fc_loc"], b["A_ff_own"], b["A_cc_own"]] + list(b["ext"].values())
        h2d += sum(m.data.nbytes + m.indices.nbytes + m.indptr.nbytes for m in mats) + b["rhs"].nbytes
        h2d += sum(a.nbytes for a in b["ext_topology"])
    d2h = sum(l.n_own for l in my_lays) * 8
    del solver
    for _ in range(max(1, min(args.steps, 2))):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        sv = parallel.SlabSolver(my_lays, comm, kind=kind, prototype="A")
        sv.build()
        xs_h, _ = sv.solve(tol=rtol, restart=restart, max_it=max_it)
        _ = [x.cpu().numpy() for x in xs_h]
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_times.append(dt)
        del sv
    e2e_val = N / statistics.median(e2e_times) / 1e6

    peak, peak_src = peak_hbm()
    dname, d = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else ("none", {"ms": 0, "bytes": 0,
                                                                                  "launches": 1})
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    tot_full = max(sum(p["ms"] for p in prof_full.values()), 1e-9)
    shares = {k: round(v["ms"] / tot_full, 4) for k, v in sorted(prof_full.items(), key=lambda kv: -kv[1]["ms"])[:8]}
    scaling = "weak" if args.scaling == "weak" else "strong"
    line = {
        "metric": metric_of(cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total_ms / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded config-{cfg} generator, {n}x{n}x{nz}); every rank assembles only its own "
                f"extended slab on the device",
        "config": {"workload": f"config{cfg}-{n}x{n}x{nz}-zslab{parts}-staticA-IC0ILU0-gmres50",
                   "n_dof": N, "slabs": parts, "slabs_per_gpu": per_proc, "halo_layers": halo,
                   "gmres_iterations": reps[-1].n_it, "final_true_relres": reps[-1].final_relres,
                   "parallelism": f"zslab{parts}", "layout_build_s": t_layout,
                   "inner_factors": "block-Jacobi per slab (IC(0) of -A_ff, ILU(0) of S~)",
                   "l2": "inputs larger than L2 and a 256 MiB L2 flush between steps"},
        "comm": {"halo_ms_per_step": comm_ms["halo"] / args.steps,
                 "allreduce_ms_per_step": comm_ms["allreduce"] / args.steps,
                 "share_of_step": comm_share,
                 "calls_per_step": (comm_ms["halo_calls"] + comm_ms["allreduce_calls"]) / args.steps,
                 "note": "CUDA events around the NCCL halo exchanges and all-reduces (max over ranks)"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "seconds_per_step": statistics.median(e2e_times)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "step_share_of_kernel_time": shares},
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------- config 4: time-step sequence
CONFIG4_DEFAULT = (20, 73, 28)   # the largest size at which the reference-native options converge (DESIGN 5.1)


def run_config4(args):
    """BASELINE config 4: a sequence of 10 backward-Euler systems on the
    channelised reservoir that reuse the restriction patterns -- stage 1 is
    built once, every step updates A_cc (update_accumulation,
    hx/assembly.py:314-333), refreshes stage 2 and solves (hx/driver.py:169-230).
    One bench step = the whole sequence; the line reports the setup
    amortisation and the per-system solve time.  The BASELINE size
    (60x220x85) stalls above rtol under every reference-native option, on the
    CPU oracle too (tests/test_gpu_configs.py), so the default
    is the largest size at which the sequence converges; --n scales it."""
    import numpy as np
    import torch

    from paper_2009_13916_b200 import _lib, configs
    from paper_2009_13916_b200 import device_assembly as DA
    from paper_2009_13916_b200.device import ctx, system_operator
    from paper_2009_13916_b200.krylov import gmres
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner, DynamicConfig, patterns_for

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.lib()
    c = ctx()
    if args.n:
        nx = args.n
        ny, nz = max(2, round(nx * 220 / 60)), max(2, round(nx * 85 / 60))
    else:
        nx, ny, nz = CONFIG4_DEFAULT
    case = configs.inputs_only(4, nx=nx, ny=ny, nz=nz)
    grid, field, props, bc, dt0, _p0 = case.meta["inputs"]
    meta = case.meta
    n_sys = 1 if args.single_system else int(meta["n_steps"])
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    opts = dict(case.precond)
    kind, proto = opts.pop("pattern"), opts.pop("prototype", "A")
    n_add, n_ent = opts.pop("n_add", 1), opts.pop("n_ent", 4)
    opts.update(INNER)
    p_init = torch.full((grid.n_elems,), float(meta["p_init"]), dtype=torch.float64, device=dev)
    base = DA.assemble_device(grid, field, props, bc, dt0, p_init)       # resident inputs
    N = base.n_unknowns

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def sequence(b=None, d2h=False):
        b = base if b is None else b
        p = p_init
        t0 = ev()
        if kind == "dynamic":
            pre = BlockLDUPreconditioner.build(b.system, dynamic=DynamicConfig(n_add, n_ent), **opts)
        else:
            pre = BlockLDUPreconditioner.build(b.system, patterns=patterns_for(b.system, kind, proto), **opts)
        marks, recs, dt, x = [t0, ev()], [], float(dt0), None
        for step in range(n_sys):
            s = b if step == 0 else DA.update_accumulation_device(b, dt, p)
            if step:
                pre.refresh(s.system)
            m1 = ev()
            x, rep = gmres(system_operator(s.system), pre, s.rhs(), tol=case.rtol, restart=case.restart,
                           max_it=case.max_it)
            m2 = ev()
            p_new = x[s.n_free_faces:]
            q = DA.recover_face_fluxes_device(s, x)
            _, chi_max, dp_max = DA.cfl_device(s, q, dt, p_new, p)
            if d2h:
                x.cpu()
            marks += [m1, m2, ev()]
            recs.append(dict(dt=dt, n_it=rep.n_it, converged=bool(rep.converged), relres=rep.final_relres))
            dt = DA.next_dt(dt, meta["dt_max"], meta["dt_mult"], meta["dp_target"], dp_max)
            p = p_new
        torch.cuda.synchronize()
        out = dict(stage_build_ms=marks[0].elapsed_time(marks[1]), systems=[])
        prev = marks[1]
        for k, r in enumerate(recs):
            m1, m2, m3 = marks[2 + 3 * k:5 + 3 * k]
            out["systems"].append(dict(r, refresh_ms=prev.elapsed_time(m1), solve_ms=m1.elapsed_time(m2),
                                       post_ms=m2.elapsed_time(m3)))
            prev = m3
        out["ms"] = marks[0].elapsed_time(prev)
        return out, x

    lib.edfa_ctx_profile_filter(c, b"")
    lib.edfa_ctx_profile(c, 1)
    profile_report(lib, c)
    sequence()
    prof_full = profile_report(lib, c)
    lib.edfa_ctx_profile(c, 0)
    for _ in range(max(args.warmup - 1, 0)):
        sequence()
    launches0 = lib.edfa_ctx_launch_count(c)
    seqs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            seqs.append(sequence()[0])
    launches = lib.edfa_ctx_launch_count(c) - launches0
    clocks = clk.summary()
    t_ms = sum(q["ms"] for q in seqs)
    value = N * n_sys * args.steps / (t_ms / 1e3) / 1e6
    last = seqs[-1]
    solve_ms = [y["solve_ms"] for y in last["systems"]]
    refresh_ms = [y["refresh_ms"] for y in last["systems"]]
    # end to end: host grid/field arrays -> device assembly -> sequence -> x of every step back on the host
    host_arrays = [v for obj in (grid, field) for v in vars(obj).values() if isinstance(v, np.ndarray)]
    h2d = int(sum(a.nbytes for a in host_arrays))
    e2e_t = []
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b2 = DA.assemble_device(grid, field, props, bc, dt0, p_init)
        sequence(b2, d2h=True)
        if it:
            e2e_t.append(time.perf_counter() - t0)
        del b2
    e2e_val = N * n_sys / statistics.median(e2e_t) / 1e6
    peak, peak_src = peak_hbm()
    groups = kernel_groups(prof_full)
    dname, d = max(groups.items(), key=lambda kv: kv[1]["ms"])
    achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
    tot_full = max(sum(v["ms"] for v in prof_full.values()), 1e-9)
    line = {
        "metric": metric_of(4), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator of BASELINE config 4: {case.name}), assembled on the device",
        "config": {"workload": f"{case.name}-{inner_tag(case)}-gmres50-{n_sys}systems", "grid": [nx, ny, nz],
                   "n_dof": N, "systems_per_step": n_sys, "rtol": case.rtol, "restart": case.restart,
                   "size_note": "BASELINE size 60x220x85 stalls above rtol under every reference-native option "
                                "(CPU oracle too): the default is the largest converging size; --n scales it",
                   "l2": "256 MiB L2 flush between sequences"},
        "sequence": {"stage_build_ms": last["stage_build_ms"],
                     "note": "stage_build = stage 1 (patterns, G~/F~, H~, IC) + the first stage 2; every later system "
                             "pays update_accumulation + stage-2 refresh only",
                     "refresh_ms": refresh_ms, "solve_ms": solve_ms,
                     "iterations": [y["n_it"] for y in last["systems"]],
                     "relres": [y["relres"] for y in last["systems"]],
                     "converged": [y["converged"] for y in last["systems"]],
                     "dt": [y["dt"] for y in last["systems"]],
                     "setup_share_first_system": last["stage_build_ms"] / max(last["stage_build_ms"] + solve_ms[0], 1e-9),
                     "setup_share_of_sequence": (last["stage_build_ms"] + sum(refresh_ms)) / max(last["ms"], 1e-9),
                     "ms_per_system_amortised": last["ms"] / n_sys},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(8 * N * n_sys),
                "seconds_per_step": statistics.median(e2e_t),
                "note": "host grid/field arrays -> assemble_device -> sequence, x of every system copied back"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                     "step_share_of_kernel_time": {k: round(v["ms"] / tot_full, 4) for k, v in
                                                   sorted(prof_full.items(), key=lambda kv: -kv[1]["ms"])[:10]},
                     "shares_from": "per-kernel CUDA events of one untimed warm-up sequence"},
        "clocks": clocks,
        "cpu_baseline": None,
    }
    if args.profile_json:
        pathlib.Path(args.profile_json).write_text(json.dumps({"warmup_step": prof_full}, indent=1))
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.drop_tol > 0 or args.fill:
        INNER.update(face_drop_tol=args.drop_tol, schur_drop_tol=args.drop_tol, no_fill=not args.fill)
    _, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
    elif world > 1 or args.slabs > 0:
        run_slabs(args)
    elif args.config == 4:
        run_config4(args)
    else:
        run_edfa(args)


if __name__ == "__main__":
    main()
