#!/usr/bin/env python
"""EDFA setup + GMRES(50) solve throughput on B200 (BASELINE.json metric).

One step = the hot path over one system: static-pattern generation, stage 1
(restricted row solves, G~/F~, H~ = G~ A_ff F~, IC(0) of -A_ff), stage 2
(S~ = A_cc - H~, ILU(0)) and right-preconditioned GMRES(50) to rtol 1e-8 from
x0 = 0.  Workload: BASELINE config 2 (64^3 hex grid, lognormal anisotropic K,
static prototype A, IC(0)/ILU(0)), synthetic seeded inputs (SPE10 is not in
this container).  ``value`` = N_dof * steps / device time with the blocks, rhs
and grid index arrays resident in HBM (the step derives everything else:
merged A, SELL copies, topology, patterns, stage 1/2, GMRES); ``e2e`` = the
same through the drop-in API from page-locked host scipy blocks (H2D of the
blocks, rhs and grid arrays, D2H of x inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl edfa|reference] [--slabs P]

N = 1: the single-device solver on config 2.  N > 1 (torchrun, one process
per GPU): weak scaling over z-slabs -- an n x n x (n N) grid of the config-2
generator, one n^3 slab per GPU, block-Jacobi inner factors per slab, halo
exchange and Krylov allreduces over NCCL (parallel.py).  ``--slabs P`` on one
GPU runs P slabs in one process (the same per-slab device work, local halos).

``--impl reference`` times the CPU restatement of the reference algorithm
(oracle/, the reference is pure Python and cannot travel to the GPU box) on a
bounded sample of the same workload and prints the same JSON line.
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
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "EDFA setup+GMRES solve throughput per system (config 2)"
METRIC_OF = lambda k: METRIC.replace("config 2", f"config {k}")  # noqa: E731
UNIT = "MDOF/s"


DEFAULT_N = {1: 16, 2: 64, 3: 128, 4: None, 5: 256}


def make_case(args):
    from paper_2009_13916_b200 import configs
    if args.config == 4:
        return configs.config4() if args.n is None else configs.config4(nx=args.n, ny=args.n, nz=args.n)
    return configs.make(args.config, n=args.n or DEFAULT_N[args.config])


INNER = {}   # --drop-tol / --fill override the config's inner-solve options


def inner_opts(case):
    p = case.precond
    o = dict(face_drop_tol=p.get("face_drop_tol", 0.0), schur_drop_tol=p.get("schur_drop_tol", 0.0),
             no_fill=p.get("no_fill", True))
    o.update(INNER)
    return o


def build_pre(case, ds):
    """Preconditioner of a BASELINE config through the drop-in API."""
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner, DynamicConfig, patterns_for
    p = case.precond
    if p["pattern"] == "dynamic":
        return BlockLDUPreconditioner.build(ds, dynamic=DynamicConfig(p["n_add"], p["n_ent"]), **inner_opts(case))
    pats = patterns_for(ds, p["pattern"], p.get("prototype", "A"))
    return BlockLDUPreconditioner.build(ds, patterns=pats, **inner_opts(case))


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
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config (2 = the headline workload; others for evidence runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--drop-tol", type=float, default=0.0,
                    help="face_drop_tol = schur_drop_tol (evidence runs of the threshold inner solves)")
    ap.add_argument("--fill", action="store_true", help="no_fill=False (threshold factorisations with fill)")
    ap.add_argument("--single-system", action="store_true",
                    help="config 4: time one system instead of the 10-step sequence")
    ap.add_argument("--profile-json", default=None, help="write the per-kernel event profile here")
    ap.add_argument("--slabs", type=int, default=0,
                    help="z-slab partitioned solver with this many slabs per process (default: 1 slab per "
                         "GPU when N > 1, the single-device solver when N = 1)")
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
def cpu_baseline(n_full: int, n_iters_full: int, sample_n: int = 20, gmres_iters: int = 8):
    """Time the oracle restatement of the reference on a bounded sample and
    extrapolate to the full workload: stage 1 and stage 2 are
    per-row independent work -> per-DOF rates from a sample_n^3 instance of the
    same generator; GMRES -> per-iteration-per-DOF rate from ``gmres_iters``
    iterations on that instance, scaled by the GPU's iteration count."""
    import numpy as np

    from oracle import edfa_oracle as O
    from paper_2009_13916_b200 import configs
    case = configs.config2(n=sample_n)
    s = case.system
    N = s.n_unknowns
    A = s.full_matrix()
    workers = max(1, os.cpu_count() or 1)
    t0 = time.perf_counter()
    sets = O.static_sets(s.grid, s.face_index, "A")
    o1 = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, sets=sets, no_fill=True, n_workers=workers)
    t1 = time.perf_counter()
    o2 = O.build_stage2(s.A_cc, o1, no_fill=True)
    t2 = time.perf_counter()
    O.gmres(lambda v: A @ v, lambda r: O.apply(o1, o2, s.A_fc, s.A_cf, r), s.rhs(), tol=1e-30,
            restart=50, max_it=1)                   # one-time scipy solver initialisation
    t2g = time.perf_counter()
    _, rep = O.gmres(lambda v: A @ v, lambda r: O.apply(o1, o2, s.A_fc, s.A_cf, r), s.rhs(), tol=1e-30,
                     restart=50, max_it=gmres_iters)
    t3 = time.perf_counter()
    it_time = (t3 - t2g) / max(rep.n_it, 1)
    N_full = None
    per_dof_setup = (t2 - t0) / N
    per_dof_iter = it_time / N
    return dict(per_dof_setup=per_dof_setup, per_dof_iter=per_dof_iter, sample_N=N,
                sample=f"oracle port on the config-2 generator at {sample_n}^3 (N={N}): full stage 1 (per-cell "
                       f"loop over {workers} processes, as the reference's n_workers fan-out) + stage 2 and "
                       f"{rep.n_it} GMRES(50) iterations (scipy, single-threaded); extrapolated per DOF to "
                       f"{n_full}^3 with {n_iters_full} iterations",
                cores=workers,
                t_stage1=t1 - t0, t_stage2=t2 - t1, t_iter=it_time, _np=np)


def extrapolate(cb, N_full, iters):
    t = N_full * cb["per_dof_setup"] + iters * N_full * cb["per_dof_iter"]
    return N_full / t / 1e6


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    from paper_2009_13916_b200 import configs  # noqa: F401
    n_full = args.n or 64
    # iteration count of the full workload: the oracle's own GMRES count is
    # not affordable at 64^3 per step; use the survey-measured 87 (SURVEY.md
    # §6.2, oracle restatement, config-2 shape) unless a smaller grid is asked
    iters = 87
    N_full = free_faces_config2(n_full) + n_full ** 3
    vals = []
    cb = None
    for k in range(max(args.warmup, 0) + args.steps):
        cb = cpu_baseline(n_full, iters, sample_n=16, gmres_iters=5)
        if k >= args.warmup:
            vals.append(extrapolate(cb, N_full, iters))
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N_full / (v * 1e6) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-2 generator)",
        "config": {"workload": f"config2-{n_full}^3-staticA-IC0ILU0-gmres50", "n_dof": N_full,
                   "rtol": 1e-8, "restart": 50, "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": "port", "sample": cb["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def free_faces_config2(n):
    # x-faces minus the two Dirichlet x-planes, plus y and z faces
    return (n + 1) * n * n - 2 * n * n + 2 * n * (n + 1) * n


# ---------------------------------------------------------------- EDFA arm
def run_edfa(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2009_13916_b200 import _lib, configs
    from paper_2009_13916_b200.device import DeviceSystem, ctx, system_operator
    from paper_2009_13916_b200.krylov import gmres
    from paper_2009_13916_b200.precond import BlockLDUPreconditioner, patterns_for

    lib = _lib.lib()
    diag = []
    if os.environ.get("EDFA_BENCH_DIAG"):      # slow-call tracer (diagnostics only)
        for _name in _lib._SIGS:
            _fn = getattr(lib, _name)

            def _w(*a, _fn=_fn, _name=_name):
                t = time.perf_counter()
                r = _fn(*a)
                dt = time.perf_counter() - t
                if dt > 0.03:
                    diag.append((_name, round(dt * 1e3, 1)))
                return r
            setattr(lib, _name, _w)
    case = make_case(args)
    if args.n is None:
        args.n = DEFAULT_N[args.config] or 0
    s = case.system
    N = s.n_unknowns
    # resident inputs: the four blocks, the rhs and the grid's index arrays;
    # every step derives everything else on the device (merged A, SELL
    # copies, topology, patterns, stage 1/2, GMRES)
    from paper_2009_13916_b200.device import DeviceCsr
    blocks = tuple(DeviceCsr.from_scipy(getattr(s, n)) for n in ("A_ff", "A_fc", "A_cf", "A_cc"))
    topo_src = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                     for a in (s.grid.elem_to_faces, s.grid.face_to_elems, s.face_index))
    b_dev = torch.from_numpy(s.rhs()).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    import ctypes

    from paper_2009_13916_b200 import _lib
    c = ctx()

    def step(_unused, b):
        system_dev = DeviceSystem(*blocks, rhs=b, host=s, topology_src=topo_src)
        pre = build_pre(case, system_dev)
        x, rep = gmres(system_operator(system_dev), pre, b, tol=case.rtol, restart=case.restart,
                       max_it=case.max_it)
        return x, rep, pre

    n_systems = 1
    if args.config == 4 and not args.single_system:
        # BASELINE config 4: one step = the 10-system time-step sequence -- stage 1
        # once, then per time step update_accumulation (A_cc + diag(acc/dt), rhs_c)
        # on the device, stage-2 refresh and GMRES from the previous pressure
        from paper_2009_13916_b200.device import DeviceCsr
        from paper_2009_13916_b200.device_assembly import next_dt
        m = case.meta
        n_systems = int(m["n_steps"])
        acc_d = torch.from_numpy(np.ascontiguousarray(s.accumulation)).to(dev)
        rcb_d = torch.from_numpy(np.ascontiguousarray(s.rhs_c_base)).to(dev)
        rhs_f_d = torch.from_numpy(np.ascontiguousarray(s.rhs_f)).to(dev)
        Acc_steady = DeviceCsr.from_scipy(s.A_cc_steady)
        nf = s.n_free_faces

        def step(_unused, b):
            system_dev = DeviceSystem(*blocks, rhs=b, host=s, topology_src=topo_src)
            pre = build_pre(case, system_dev)         # stage 1 + stage 2 of the first system
            dt, x, reps_seq = float(m["dt0"]), None, []
            p_prev = torch.full((s.n_cells,), float(m["p_init"]), dtype=torch.float64, device=dev)
            for k in range(n_systems):
                if k == 0:
                    sk = system_dev
                else:
                    rhs_c = torch.empty_like(rcb_d)
                    h = ctypes.c_void_p()
                    _lib.check(lib.edfa_update_accumulation(c, Acc_steady.handle, acc_d.data_ptr(),
                                                            rcb_d.data_ptr(), p_prev.data_ptr(), dt,
                                                            ctypes.byref(h), rhs_c.data_ptr()))
                    sk = DeviceSystem(blocks[0], blocks[1], blocks[2], DeviceCsr(h),
                                      rhs=torch.cat([rhs_f_d, rhs_c]), host=s, topology_src=topo_src)
                    pre.refresh(sk)                   # stage 2 only; stage 1 reused
                x, rep = gmres(system_operator(sk), pre, sk.rhs(), tol=case.rtol, restart=case.restart,
                               max_it=case.max_it)
                reps_seq.append(rep)
                # TimestepController (hx/driver.py:50-53): dt * min(mult, dp_target / dp_max), capped
                dp_max = float((x[nf:] - p_prev).abs().max())
                dt = next_dt(dt, float(m["dt_max"]), float(m["dt_mult"]), float(m["dp_target"]), dp_max)
                p_prev = x[nf:]
            rep.seq_iterations = [r.n_it for r in reps_seq]
            rep.seq_relres = max(r.final_relres for r in reps_seq)
            return x, rep, pre

    def report(c, reset=1):
        n = lib.edfa_ctx_profile_report(c, None, 0, 0)
        buf = ctypes.create_string_buffer(int(n))
        lib.edfa_ctx_profile_report(c, buf, n, reset)
        return json.loads(buf.value.decode())

    c = ctx()
    for w in range(args.warmup):
        last = w == args.warmup - 1
        if last:   # full per-kernel event profile of one (untimed) step: shares + dominant kernel
            lib.edfa_ctx_profile_filter(c, b"")
            lib.edfa_ctx_profile(c, 1)
            report(c)
        x = rep = pre = None              # one preconditioner alive at a time (256^3 memory)
        x, rep, pre = step(None, b_dev)
        if last:
            prof_full = report(c)
            lib.edfa_ctx_profile(c, 0)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    dom_name = max(prof_full.items(), key=lambda kv: kv[1]["ms"])[0] if prof_full else ""

    # ---- device-resident timed region; CUDA events bracket every launch of
    # the dominant kernel only (cheap enough not to perturb the step)
    lib.edfa_ctx_profile_filter(c, dom_name.encode())
    lib.edfa_ctx_profile(c, 1)
    report(c)
    launches0 = lib.edfa_ctx_launch_count(c)
    times = []
    reps = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)                        # evict L2 between steps
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x = rep = pre = None
            e0.record()
            x, rep, pre = step(None, b_dev)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            reps.append(rep)
            if diag:
                print("diag step", len(times), times[-1], diag, file=sys.stderr, flush=True)
                diag.clear()
    launches = lib.edfa_ctx_launch_count(c) - launches0
    prof = report(c)
    lib.edfa_ctx_profile(c, 0)
    lib.edfa_ctx_profile_filter(c, b"")
    clocks = clk.summary()
    t_total_ms = sum(times)
    if world > 1:
        tt = torch.tensor([t_total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_total_ms = float(tt.item())
    value = world * N * n_systems * args.steps / (t_total_ms / 1e3) / 1e6

    n_it_last, relres_last = reps[-1].n_it, reps[-1].final_relres
    seq_its = getattr(reps[-1], "seq_iterations", None)
    seq_rel = getattr(reps[-1], "seq_relres", None)
    del x, rep, pre, reps                 # release the timed step's preconditioner before the e2e leg

    # ---- end-to-end through the public API from host scipy blocks
    e2e_times = []
    from paper_2009_13916_b200.device import pinned_copy
    s_pin = pinned_copy(s)              # the host application's page-locked staging of the inputs
    h2d = sum(getattr(s, n).data.nbytes + getattr(s, n).indices.nbytes + getattr(s, n).indptr.nbytes
              for n in ("A_ff", "A_fc", "A_cf", "A_cc")) + s.rhs().nbytes
    h2d += 4 * (12 * s.n_cells + s.face_index.size)      # cell->face map, neighbours, face index
    d2h = N * 8
    for k in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ds_h = DeviceSystem.from_host(s_pin)                  # H2D of the four blocks, rhs, topology
        pre_h = build_pre(case, ds_h)                          # patterns from the device topology
        x_h, rep_h = gmres(system_operator(ds_h), pre_h, s_pin.rhs(), tol=case.rtol, restart=case.restart,
                           max_it=case.max_it)                # x returned to host (D2H)
        s_k = s_pin
        if n_systems > 1:   # the time-step sequence as a host application drives it
            from paper_2009_13916_b200 import assembly as host_asm
            from paper_2009_13916_b200.device_assembly import next_dt
            m = case.meta
            dt, p_prev_h = float(m["dt0"]), np.full(s.n_cells, float(m["p_init"]))
            for q in range(1, n_systems):
                p_new_h = x_h[s.n_free_faces:]
                dt = next_dt(dt, float(m["dt_max"]), float(m["dt_mult"]), float(m["dp_target"]),
                             float(np.abs(p_new_h - p_prev_h).max()))
                p_prev_h = p_new_h
                s_k = host_asm.update_accumulation(s_pin, dt, p_new_h)                # host A_cc, rhs_c
                pre_h.refresh(s_k)                                                   # H2D of A_cc
                x_h, rep_h = gmres(system_operator(pre_h.device_system), pre_h, s_k.rhs(), tol=case.rtol,
                                   restart=case.restart, max_it=case.max_it)
        e2e_times.append(time.perf_counter() - t0)
        del ds_h, pre_h
    if n_systems > 1:
        h2d += (n_systems - 1) * (12 * s.A_cc.nnz + 4 * (s.n_cells + 1) + 8 * N)
        d2h *= n_systems
    e2e_val = world * N * n_systems / statistics.median(e2e_times) / 1e6
    relres_host = float(np.linalg.norm(s_k.rhs() - s_k.full_matrix() @ x_h) / np.linalg.norm(s_k.rhs()))

    # ---- roofline of the dominant kernel
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs, burst)" if peak else "fallback 6650 GB/s (B200_PROFILING.md)"
    peak = peak or 6650.0
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else ("none", {"ms": 0, "bytes": 0, "launches": 1})
    dname, d = dom
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    try:
        nc = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        traffic = nc.get(dname)
    except Exception:
        pass
    step_ms = t_total_ms / args.steps
    tot_full = max(sum(p["ms"] for p in prof_full.values()), 1e-9)
    shares = {k: round(v["ms"] / tot_full, 4) for k, v in sorted(prof_full.items(), key=lambda kv: -kv[1]["ms"])[:8]}
    kernel_ms_per_step = tot_full

    line = {
        "metric": METRIC_OF(args.config), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded config-2 generator: 64^3, lnK~N(0,2), kz/kx=0.1)" if args.config == 2
                 else f"synthetic (seeded generator of BASELINE config {args.config}: {case.name})"),
        "config": {"workload": (f"config2-{args.n}^3-staticA-{inner_tag(case)}-gmres50" if args.config == 2
                                else f"{case.name}-{inner_tag(case)}-gmres50"), "n_dof": N,
                   "n_free_faces": s.n_free_faces, "n_cells": s.n_cells, "rtol": case.rtol,
                   "restart": case.restart, "gmres_iterations": n_it_last,
                   "final_true_relres": relres_last, "host_check_relres": relres_host,
                   **({"systems_per_step": n_systems, "sequence_iterations": seq_its,
                       "sequence_max_relres": seq_rel} if n_systems > 1 else {}),
                   "parallelism": "single", "step_ms": [round(t, 3) for t in times],
                   "l2": "inputs larger than L2 and a 256 MiB L2 flush between steps"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "seconds_per_step": statistics.median(e2e_times)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "launches_per_step": d["launches"] / args.steps,
                     "step_share_of_kernel_time": shares, "kernel_ms_per_step": kernel_ms_per_step,
                     "shares_from": "per-kernel CUDA events of the last warm-up step (same workload)"},
        "clocks": clocks,
    }
    if rank == 0 and "inputs" in case.meta:
        line["assembly"] = assembly_leg(case, c, lib, report, N)
    if args.profile_json and rank == 0:
        pathlib.Path(args.profile_json).write_text(json.dumps({"timed_region": prof, "warmup_step": prof_full},
                                                              indent=1))
    if rank == 0 and not args.no_cpu_baseline and args.config == 2:
        cb = cpu_baseline(args.n, n_it_last)
        v = extrapolate(cb, N, n_it_last)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": "port",
                                "sample": cb["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def assembly_leg(case, c, lib, report, N):
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
    report(c)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = DA.assemble_device(g, fld, props, bc, dt, p0)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del d
    prof = report(c)
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
def run_slabs(args):
    """Weak scaling over z-slabs (BASELINE config 5 method):
    the global grid is n x n x (n * slabs), one n^3 slab per GPU, block-Jacobi
    inner factors per slab, halo exchange + allreduce over NCCL."""
    import ctypes

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
    from paper_2009_13916_b200 import _lib, configs, parallel
    from paper_2009_13916_b200.device import ctx
    lib = _lib.lib()
    diag = []
    args.n = args.n or 64
    case = configs.config2(n=args.n, nz=args.n * parts)
    s = case.system
    N = s.n_unknowns
    mine = [rank * per_proc + k for k in range(per_proc)]
    halo = parallel.halo_layers("static", "A")
    lays = parallel.build_layouts(s, parts, halo=halo, ranks=mine)
    comm = (parallel.TorchComm([q // per_proc for q in range(parts)]) if world > 1
            else parallel.LocalComm(parts))
    my_lays = [lays[q] for q in mine]
    solver = parallel.SlabSolver(my_lays, comm, kind="static", prototype="A")
    if world > 1:
        t = torch.zeros(1, device=dev)
        torch.distributed.all_reduce(t)                # communicator up before the first P2P
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        solver.build()
        return solver.solve(tol=case.rtol, restart=case.restart, max_it=case.max_it)

    def report(c, reset=1):
        n = lib.edfa_ctx_profile_report(c, None, 0, 0)
        buf = ctypes.create_string_buffer(int(n))
        lib.edfa_ctx_profile_report(c, buf, n, reset)
        return json.loads(buf.value.decode())

    c = ctx()
    prof_full = {}
    for w in range(args.warmup):
        last = w == args.warmup - 1
        if last:
            lib.edfa_ctx_profile_filter(c, b"")
            lib.edfa_ctx_profile(c, 1)
            report(c)
        xs, rep = step()
        if last:
            prof_full = report(c)
            lib.edfa_ctx_profile(c, 0)
    torch.cuda.synchronize()
    dom_name = max(prof_full.items(), key=lambda kv: kv[1]["ms"])[0] if prof_full else ""
    lib.edfa_ctx_profile_filter(c, dom_name.encode())
    lib.edfa_ctx_profile(c, 1)
    report(c)
    launches0 = lib.edfa_ctx_launch_count(c)
    times, reps = [], []
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
            if diag:
                print("diag step", len(times), times[-1], diag, file=sys.stderr, flush=True)
                diag.clear()
    launches = lib.edfa_ctx_launch_count(c) - launches0
    prof = report(c)
    lib.edfa_ctx_profile(c, 0)
    lib.edfa_ctx_profile_filter(c, b"")
    clocks = clk.summary()
    t_total_ms = sum(times)
    if world > 1:
        tt = torch.tensor([t_total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_total_ms = float(tt.item())
    value = N * args.steps / (t_total_ms / 1e3) / 1e6
    # true residual of the assembled global solution on the host (rank 0 gathers)
    x_loc = [x.cpu().numpy() for x in xs]
    relres_host = None
    if world > 1:
        gathered = [None] * world
        torch.distributed.all_gather_object(gathered, x_loc)
        x_all = [v for g in gathered for v in g]
    else:
        x_all = x_loc
    if rank == 0:
        x = parallel.scatter_solution(lays, x_all, s.n_free_faces, s.n_cells)
        relres_host = float(np.linalg.norm(s.rhs() - s.full_matrix() @ x) / np.linalg.norm(s.rhs()))

    # ---- end to end from host blocks: H2D of the slab's local blocks, build, solve, D2H of x
    e2e_times = []
    h2d = 0
    for lay in my_lays:
        b = lay.blocks
        mats = [b["A_loc"], b["A_cf_loc"], b["A_fc_loc"], b["A_ff_own"], b["A_cc_own"]] + list(b["ext"].values())
        h2d += sum(m.data.nbytes + m.indices.nbytes + m.indptr.nbytes for m in mats) + b["rhs"].nbytes
        h2d += sum(a.nbytes for a in b["ext_topology"])
    d2h = sum(l.n_own for l in my_lays) * 8
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        sv = parallel.SlabSolver(my_lays, comm, kind="static", prototype="A")
        sv.build()
        xs_h, _ = sv.solve(tol=case.rtol, restart=case.restart, max_it=case.max_it)
        _ = [x.cpu().numpy() for x in xs_h]
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_times.append(dt)
        del sv
    e2e_val = N / statistics.median(e2e_times) / 1e6

    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = peaks.get("hbm_gbs") or 6650.0
    dname, d = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else ("none", {"ms": 0, "bytes": 0,
                                                                                    "launches": 1})
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    tot_full = max(sum(p["ms"] for p in prof_full.values()), 1e-9)
    shares = {k: round(v["ms"] / tot_full, 4) for k, v in sorted(prof_full.items(), key=lambda kv: -kv[1]["ms"])[:8]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded config-2 generator stacked along z: {args.n}x{args.n}x{args.n * parts})",
        "config": {"workload": f"config2-{args.n}^3-per-slab-z{parts}-staticA-IC0ILU0-gmres50",
                   "n_dof": N, "slabs": parts, "slabs_per_gpu": per_proc, "halo_layers": halo,
                   "gmres_iterations": reps[-1].n_it, "final_true_relres": reps[-1].final_relres,
                   "host_check_relres": relres_host, "parallelism": f"zslab{parts}",
                   "inner_factors": "block-Jacobi per slab (IC(0) of -A_ff, ILU(0) of S~)",
                   "l2": "inputs larger than L2 and a 256 MiB L2 flush between steps"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "seconds_per_step": statistics.median(e2e_times)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs, burst)",
                     "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "step_share_of_kernel_time": shares},
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.drop_tol > 0 or args.fill:
        INNER.update(face_drop_tol=args.drop_tol, schur_drop_tol=args.drop_tol, no_fill=not args.fill)
    _, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
    elif world > 1 or args.slabs > 0:
        run_slabs(args)
    else:
        run_edfa(args)


if __name__ == "__main__":
    main()
