#!/usr/bin/env python
"""Benchmark of the B200 wedge/tet DG time-stepping path (BASELINE.json metric).

Metric: DOF-updates/s = total_dofs x LSERK45 steps / device time (one step = 5
fused stage launches).  Workload = BASELINE.json configs[1]: "order sweep
N=1..7 on an extruded layered wedge mesh, ~1e6 elements per GPU" -- stack_layers
on the structured n=100 surface (20,000 triangles) with three flat layers
z=-1..-0.4 (15 sublayers), -0.4..0.2 (15), 0.2..1 (20): 1,000,000 wedges, media
kappa = 1, 4, 2.25 and rho = 1, Gaussian pulse initial state,
FP64, upwind flux, exact stored-lift mass.  The headline line is degree
--degree (default 5); --degrees 1,2,...,7 adds the sweep under "sweep".

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize and
CUDA events on the library's stream; value = total DOF-updates over all ranks
/ max-over-ranks time.  Inputs (>= 0.1 GB state, 4 GB at N=5) are far larger
than the 126 MB L2, so no flush is needed.  e2e = the same steps through the
C ABI with host buffers: per step H2D of the state from pinned memory,
pdg_step_lserk, D2H of the state.

--impl reference: the reference's CPU algorithm (the oracle port in oracle/,
because the reference itself cannot be built here: Eigen3 is absent) on the
box's host cores, on a bounded sample (same surface, fewer sublayers).  That
process never loads the product library: the oracle carries its own copy of
the host setup code and is rebuilt on the box with the reference's
-O3 -march=native (proj/CMakeLists.txt:10).

--gpus N without torchrun: bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU; it refuses to run when fewer
than N GPUs are visible).  --scaling weak (default, config 5 weak: 1e6 owned
wedges per GPU) or strong (config 5 strong: the n=200 x 50-sublayer mesh,
4e6 wedges, split over the N GPUs).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "DOF-updates/sec (1/2/4/8 B200, N=1..7); per-kernel HBM GB/s vs roofline"
UNIT = "DOF-updates/s"


def layered_workload(surface_n, sublayers):
    import paper_1607_03399_b200 as pdg
    return pdg.layered_mesh(surface_n, [-1.0, -0.4, 0.2, 1.0], sublayers, [(1.0, 1.0), (1.0, 4.0), (1.0, 2.25)])


def load_traffic(kind, degree):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of one stage
    kernel from the committed ncu capture of the same workload (profiles/ncu_traffic.json,
    made by scripts/make_traffic_json.py), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            tab = json.load(fh)
        return float(tab[kind][str(degree)]["bytes_per_launch"])
    except Exception:
        return None


DMMA_PEAK_TFLOPS = 37.0  # measured FP64 tensor-core throughput on this B200 pool (scripts/micro/dmma_bench.cu)
DFMA_PEAK_TFLOPS = 33.0  # measured FP64 FMA (CUDA-core) throughput, same microbenchmark


def wadg_flops_per_wedge_stage(N):
    """algorithmic FP64 flops of the WADG stage kernel per wedge:
    Ltilde formation, K-folded gradients, vertical terms, quad-face lifts, Ltilde B."""
    nq, nt, nc = N + 1, (N + 1) * (N + 2) // 2, (N + 2) ** 2
    return (2 * nt * nc * nt + 2 * 4 * nt * nt * nq + 4 * 2 * nt * nq * nq + 3 * 2 * 2 * nt * nq * nq
            + 2 * nt * nt * 4 * nq)


def tet_flops_per_stage(N):
    """algorithmic FP64 flops of the tet stage kernel per tet: gradients
    D_a P and divergence sum_a D_a W_a (6 NP x NP products), the W_a columns, and the
    four face lifts of the p and u fluxes (8 NP x NT products)."""
    np_, nt = (N + 1) * (N + 2) * (N + 3) // 6, (N + 1) * (N + 2) // 2
    return 12 * np_ * np_ + 3 * 5 * np_ + 16 * np_ * nt


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def native_oracle(timeout_s=300):
    """Build the oracle with the reference's -O3 -march=native on THIS host
    (oracle/build_native); fall back to the portable prebuilt oracle."""
    jobs = str(os.cpu_count() or 1)
    cmd = ["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j", jobs, "OUT=build_native", "HOST_ARCH=-march=native",
           "build_native/liboracle.so"]
    try:
        r = subprocess.run(cmd, capture_output=True, timeout=timeout_s)
        lib = os.path.join(ROOT, "oracle", "build_native", "liboracle.so")
        if r.returncode == 0 and os.path.exists(lib):
            return lib, "-O3 -march=native -fopenmp (built on this host)"
    except Exception:
        pass
    return os.path.join(ROOT, "oracle", "build", "liboracle.so"), "-O3 -march=x86-64-v3 -fopenmp (prebuilt, portable)"


def cpu_sample(degree, threads, steps, warmup=1, surface_n=100, sublayers=(1, 1, 1), oracle_lib=None):
    """The reference's CPU algorithm (oracle port, solver.cpp:536-557) on a bounded
    sample of the workload, timed per LSERK45 step in both update variants:
    'faithful' = the reference's serial update loop (solver.cpp:546-549),
    'parallel' = OpenMP on the update as well (a fair best-effort CPU).
    Loads only liboracle.so (its own mesh/discretization build), never the product."""
    if oracle_lib:
        os.environ["PDG_ORACLE_LIB"] = oracle_lib
    import oracle_binding as ob
    t0 = time.perf_counter()
    d = ob.layered_disc(surface_n, [-1.0, -0.4, 0.2, 1.0], list(sublayers), [(1.0, 1.0), (1.0, 4.0), (1.0, 2.25)],
                        degree, threads=threads)
    u0 = d.gaussian(0.25)
    dt = d.estimate_dt(0.5)
    setup = time.perf_counter() - t0
    rates = {"faithful": [], "parallel": []}
    u = u0
    for it in range(warmup + steps):
        for kind in ("parallel", "faithful"):
            t1 = time.perf_counter()
            u = ob.lserk(d, u, dt, 1, threads, kind == "parallel")
            el = time.perf_counter() - t1
            if it >= warmup:
                rates[kind].append(d.total_dofs / el)
    med = {k: (sorted(v)[len(v) // 2] if v else 0.0) for k, v in rates.items()}
    sample = (f"oracle port of solver.cpp:536-557 on {d.num_wedges} wedges (surface n={surface_n}, sublayers "
              f"{list(sublayers)}; the GPU arm runs 1e6), N={degree}, {d.total_dofs} DOFs, median of {steps} timed "
              f"LSERK45 steps per variant after {warmup} warm-up, {threads} OpenMP threads, setup {setup:.1f}s")
    return med, sample, d.total_dofs


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    lib, build = native_oracle()
    med, sample, _ = cpu_sample(args.degree, threads, steps=args.steps, warmup=args.warmup, oracle_lib=lib)
    value = med["parallel"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(ws, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (gaussian pulse on generated layered wedge mesh)",
        "config": {"workload": "configs[1] layered wedges (n=100 surface), bounded CPU sample of 3 sublayers",
                   "degree": args.degree, "same_config": False,
                   "why_not_same": "one reference LSERK step on the 1e6-wedge mesh takes ~13 s on 16 cores; the "
                                   "per-DOF rate of the 60k-wedge sample (state 0.24 GB at N=5, far beyond the "
                                   "CPU caches) is the same algorithm on the same element types"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "variant": "parallel update (value); faithful serial update below",
                         "faithful_serial_update": med["faithful"], "build": build, "cpu": cpu_model()},
        "variants": {"parallel_update": med["parallel"], "faithful_serial_update": med["faithful"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_degree(args, degree, ws, rank, local, peaks, with_e2e=True):
    import numpy as np
    import torch
    import paper_1607_03399_b200 as pdg

    t_setup = time.perf_counter()
    if getattr(args, "workload", "layered") == "hybrid":
        # configs[2]: structured_hybrid_box(64,64,32,32) = 262,144 wedges + 786,432 tets
        mesh = pdg.structured_hybrid_box(args.hybrid_n, args.hybrid_n, args.hybrid_n // 2, args.hybrid_n // 2,
                                         (1.0, 1.0), (1.0, 4.0))
    else:
        mesh = layered_workload(args.surface_n, args.sublayers)
    mass = getattr(args, "mass", "exact")
    d = pdg.build_discretization(mesh, degree, threads=os.cpu_count() or 1, mass=mass,
                                 host_lifts=(mass != "wadg"))
    s = pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0])
    dt = pdg.estimate_dt(d, 0.5)
    ctx = pdg.DeviceContext(d, device=local, flags=pdg.capi.CTX_TIMING)
    ctx.set_state(s.u)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    # warm-up
    ctx.step(dt, args.warmup)
    ctx.synchronize()
    ctx.kernel_times(reset=True)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(stream)
        ctx.step(dt, args.steps)
        stop.record(stream)
        stop.synchronize()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    kt = ctx.kernel_times(reset=True)
    wbytes, tbytes = ctx.stage_bytes()
    assert ctx.check_finite() == -1, "non-finite state after the timed steps"
    dofs = d.total_dofs
    value = dofs * args.steps * ws / (ms / 1e3)
    wedge_avg_ms = kt["wedge_ms"] / max(1, kt["wedge_launches"])
    achieved = wbytes / (wedge_avg_ms / 1e3) / 1e9 if wedge_avg_ms > 0 else 0.0
    tet_avg_ms = kt["tet_ms"] / max(1, kt["tet_launches"])
    res = {
        "degree": degree, "value": value, "ms_per_step": ms / args.steps, "total_dofs": dofs,
        "wedges": mesh.num_wedges(), "setup_s": round(setup_s, 1),
        "wedge_kernel_avg_ms": wedge_avg_ms, "wedge_stage_bytes": wbytes,
        "wedge_kernel_share": kt["wedge_ms"] / ms if ms > 0 else None,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks[0], "unit": "GB/s",
                     "frac": achieved / peaks[0], "peak_source": peaks[1],
                     "traffic": load_traffic(("wadg" if mass == "wadg" else "exact") if mesh.num_tets() == 0
                                             else "hybrid_wedge", degree),
                     "traffic_unit": "bytes/launch (ncu, profiles/ncu_traffic.json)",
                     "algorithmic_bytes": wbytes},
        "gpu_launches": int(kt["wedge_launches"] + kt["tet_launches"]),
        "tets": mesh.num_tets(),
        "clocks": clk.summary(),
    }
    if mass == "wadg" and mesh.num_tets() == 0:
        # WADG trades the streamed operators for FP64 tensor work: report
        # the FP64 DMMA pipe roofline beside the HBM one (algorithmic flops, DESIGN 3.3)
        fl = wadg_flops_per_wedge_stage(degree) * mesh.num_wedges()
        simt = degree <= 3  # the low-order WADG kernel runs on the FP64 CUDA cores
        pk = DFMA_PEAK_TFLOPS if simt else DMMA_PEAK_TFLOPS
        res["tensor_roofline"] = {"bound": "fp64" if simt else "tensor", "achieved": fl / (wedge_avg_ms / 1e3) / 1e12,
                                  "peak": pk, "unit": "TFLOP/s", "frac": fl / (wedge_avg_ms / 1e3) / 1e12 / pk,
                                  "peak_source": ("FP64 FMA" if simt else "FP64 mma.sync m8n8k4 (DMMA)") +
                                                 ", scripts/micro/dmma_bench.cu on this pool",
                                  "flops_per_launch": fl}
    if mesh.num_tets() > 0:
        t_ach = tbytes / (tet_avg_ms / 1e3) / 1e9
        res["tet_kernel_avg_ms"] = tet_avg_ms
        res["tet_kernel_share"] = kt["tet_ms"] / ms if ms > 0 else None
        res["tet_roofline"] = {"bound": "hbm", "achieved": t_ach, "peak": peaks[0], "unit": "GB/s",
                               "frac": t_ach / peaks[0], "peak_source": peaks[1],
                               "traffic": load_traffic("tet", degree), "algorithmic_bytes": tbytes}
        # at high N the tet stage is FP64 tensor work (dense NP x NP operators): its
        # roofline against the DMMA peak (N = 8, 9 run on the FP64 CUDA cores)
        tfl = tet_flops_per_stage(degree) * mesh.num_tets()
        tsimt = degree >= 8
        tpk = DFMA_PEAK_TFLOPS if tsimt else DMMA_PEAK_TFLOPS
        res["tet_tensor_roofline"] = {"bound": "fp64" if tsimt else "tensor",
                                      "achieved": tfl / (tet_avg_ms / 1e3) / 1e12, "peak": tpk, "unit": "TFLOP/s",
                                      "frac": tfl / (tet_avg_ms / 1e3) / 1e12 / tpk,
                                      "peak_source": ("FP64 FMA" if tsimt else "FP64 mma.sync m8n8k4 (DMMA)") +
                                                     ", scripts/micro/dmma_bench.cu on this pool",
                                      "flops_per_launch": tfl}
    if with_e2e:
        # e2e through the C ABI: pinned host state in, one step, state out, every step
        host = torch.empty(dofs, dtype=torch.float64, pin_memory=True)
        host.numpy()[:] = s.u
        hptr = C.c_void_p(host.data_ptr())
        lib = pdg.capi.lib()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            pdg.capi.check(lib.pdg_set_state(ctx.handle, hptr, 0))
            pdg.capi.check(lib.pdg_step_lserk(ctx.handle, dt, 1, None))
            pdg.capi.check(lib.pdg_get_state(ctx.handle, hptr, 0))
        el = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([el], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        res["e2e"] = {"value": dofs * e2e_steps * ws / el, "unit": UNIT, "h2d_bytes_per_step": dofs * 8,
                      "d2h_bytes_per_step": dofs * 8, "steps": e2e_steps,
                      "call": "per step: pdg_set_state (H2D) + pdg_step_lserk + pdg_get_state (D2H), i.e. the "
                              "reference's step(disc, state, dt, stepper) with a host SolutionState"}
        if ws == 1:
            # informational: the production call, run_simulation (solver.cpp:591-666), K steps per call:
            # state H2D once, energy (time, E) pair read back every step, state D2H once
            k = args.steps
            opts = pdg.capi.RunOptions(0.0, 0.5, dt, 0.0, 50, 10.0, 0, 0.0, pdg.capi.SNAPSHOT_CB(), None)
            rr = pdg.capi.RunResult()
            log = np.zeros(2 * (k + 2))
            tt = C.c_double(0.0)
            opts.final_time = k * dt
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pdg.capi.check(lib.pdg_run_simulation(ctx.handle, C.cast(hptr, pdg.capi.DP), C.byref(tt), C.byref(opts),
                                                  C.byref(rr),
                                                  log.ctypes.data_as(pdg.capi.DP), k + 2))
            el = time.perf_counter() - t0
            res["e2e_run_simulation"] = {
                "value": dofs * rr.steps / el, "unit": UNIT, "steps": int(rr.steps),
                "h2d_bytes_per_step": dofs * 8 / max(1, rr.steps),
                "d2h_bytes_per_step": dofs * 8 / max(1, rr.steps) + 16,
                "call": "pdg_run_simulation over the K timed steps: state in and out once, energy logged and read "
                        "back every step, watchdog every 50 steps (informational; e2e above is the per-step call)"}
    ctx.close()
    del d, mesh
    return res


def measure_degree_dist(args, degree, ws, rank, local, peaks):
    """N > 1 (config 5).  Weak: rank r owns the r-th slab of 1e6 wedges (stack of
    ws copies of the config-2 slab).  Strong: the n=200 x 50-sublayer mesh (4e6
    wedges) with its sublayers split over the ranks.  Ghosts are one sublayer
    above and below; their face traces are refreshed with NCCL point-to-point
    before every LSERK stage, overlapped with the interior elements."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1607_03399_b200 as pdg
    from paper_1607_03399_b200 import partition as P
    from paper_1607_03399_b200.distributed import DistributedLSERK

    t_setup = time.perf_counter()
    media = [(1.0, 1.0), (1.0, 4.0), (1.0, 2.25)]
    if args.scaling == "strong":
        part = P.layered_strong(args.strong_n, [-1.0, -0.4, 0.2, 1.0], args.sublayers, media, ws, rank)
    else:
        part = P.layered_slab(args.surface_n, [-1.0, -0.4, 0.2, 1.0], args.sublayers, media, ws, rank)
    # host setup threads split between the ranks of this node (no oversubscription)
    threads = max(1, (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", ws))))
    solver = DistributedLSERK(part, degree, device=local, threads=threads, flags=pdg.capi.CTX_TIMING)
    d = solver.disc
    s = pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0])
    dt = pdg.estimate_dt(d, 0.5)
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    dt = float(t.item())
    solver.set_state(s.u)
    setup_s = time.perf_counter() - t_setup
    solver.step(dt, args.warmup)
    solver.synchronize()
    solver.kernel_times(reset=True)
    dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(solver.stream)
        solver.step(dt, args.steps)
        stop.record(solver.stream)
        stop.synchronize()
    ms = start.elapsed_time(stop)
    tt = torch.tensor([ms], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    owned_dofs = 4 * d.info.np_wedge * part.n_owned
    tot = torch.tensor([owned_dofs], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot)
    value = float(tot.item()) * args.steps / (ms / 1e3)
    total_wedges = torch.tensor([part.n_owned], dtype=torch.float64, device="cuda")
    dist.all_reduce(total_wedges)
    # roofline of this rank's wedge stage kernel: a stage is an interior and a boundary
    # launch over disjoint owned elements, so per-stage time = summed launch time / stages
    kt = solver.kernel_times(reset=True)
    wbytes, _ = solver.stage_bytes()
    stages = 5 * args.steps
    stage_ms = kt["wedge_ms"] / stages if stages else 0.0
    achieved = wbytes / (stage_ms / 1e3) / 1e9 if stage_ms > 0 else 0.0
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks[0], "unit": "GB/s", "frac": achieved / peaks[0],
            "peak_source": peaks[1], "traffic": None, "algorithmic_bytes": wbytes,
            "note": "rank 0; per stage = interior + boundary launch time"}
    # e2e through the public API on every rank: pinned host state in, one step, state out
    host = torch.empty(d.total_dofs, dtype=torch.float64, pin_memory=True)
    hnp = host.numpy()
    hnp[:] = s.u
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        solver.set_state(hnp)
        solver.step(dt, 1)
        solver.get_state(hnp)
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    e2e = {"value": float(tot.item()) * e2e_steps / float(el.item()), "unit": UNIT,
           "h2d_bytes_per_step": d.total_dofs * 8, "d2h_bytes_per_step": d.total_dofs * 8, "steps": e2e_steps,
           "per_rank": True}
    cnt = (C.c_int64 * 6)()
    pdg.capi.check(pdg.capi.lib().pdg_partition_counts(solver.ctx, cnt))
    interior, owned = cnt[4] + cnt[5], cnt[0] + cnt[1]
    parts_nonempty = int(interior > 0) + int(owned - interior > 0)
    solver.close()
    return {"degree": degree, "value": value, "ms_per_step": ms / args.steps, "total_dofs": owned_dofs,
            "total_wedges": int(total_wedges.item()),
            "wedges": part.n_owned, "setup_s": round(setup_s, 1), "clocks": clk.summary(),
            "roofline": roof, "e2e": e2e, "wedge_kernel_avg_ms": stage_ms,
            # per stage: the non-empty interior / boundary stage launches, one trace gather
            # and one trace scatter per peer
            "gpu_launches": args.steps * 5 * (parts_nonempty + 2 * len(solver.peers)),
            "exchange_bytes_per_stage": solver.exchange_bytes}


def relaunch(args):
    """--gpus N outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run with the same arguments; refuse when fewer than N
    GPUs are visible (NCCL cannot put two ranks on one device)."""
    import socket
    if args.impl == "ours" and not args.launch_check:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}; "
                  f"refusing to report a {have}-GPU number as {args.gpus}", file=sys.stderr, flush=True)
            return 3
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    # torchrun would pin every rank to one OpenMP thread; the host setup of a
    # 1e6-wedge partition wants the node's cores split between the ranks
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // args.gpus)))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--degree", type=int, default=5)
    ap.add_argument("--degrees", default="1,2,3,4,6,7",
                    help="comma list for the order sweep reported under 'sweep' ('' = headline degree only)")
    ap.add_argument("--surface-n", type=int, default=100)
    ap.add_argument("--strong-n", type=int, default=200, help="surface n of the strong-scaling mesh (x 50 sublayers)")
    ap.add_argument("--sublayers", default="15,15,20")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-steps", type=int, default=3, help="timed CPU-baseline LSERK steps per update variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="layered", choices=["layered", "hybrid"],
                    help="layered = configs[1] (1e6 wedges); hybrid = configs[2] (wedge layers over a tet cap)")
    ap.add_argument("--hybrid-n", type=int, default=64)
    ap.add_argument("--partitioned", action="store_true",
                    help="run the multi-GPU path (slab partition, DistributedLSERK, NCCL group) even at one GPU")
    ap.add_argument("--mass", default="exact", choices=["exact", "wadg"],
                    help="exact stored-lift mass (reference parity mode) or weight-adjusted (north-star WADG)")
    ap.add_argument("--launch-check", action="store_true",
                    help="test hook: relaunch as for --gpus N, then every rank reports its rank and exits")
    args = ap.parse_args()
    args.sublayers = [int(x) for x in args.sublayers.split(",")]
    args.warmup = max(3, args.warmup)

    ws, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return relaunch(args)
    if "WORLD_SIZE" in os.environ and ws != args.gpus and args.gpus > 1:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        return 3
    if args.launch_check:
        print(json.dumps({"rank": rank, "world_size": ws, "local_rank": local,
                          "master": os.environ.get("MASTER_ADDR")}), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    torch.cuda.set_device(local)
    use_dist = ws > 1 or args.partitioned or args.scaling == "strong"
    if use_dist:
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29561")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        # communicator setup lines (rank count, NVLS / P2P transport) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = load_peaks()
    if use_dist:
        head = measure_degree_dist(args, args.degree, ws, rank, local, peaks)
        if rank == 0:
            if args.scaling == "strong":
                wl = (f"configs[4] strong: layered wedge mesh n={args.strong_n} surface x {sum(args.sublayers)} "
                      f"sublayers ({head['total_wedges']} wedges in total, fixed), sublayers split over {ws} GPU(s)")
            else:
                wl = ("configs[4] weak: layered wedge slabs, 1e6 owned wedges per GPU stacked in z")
            line = {
                "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (gaussian pulse on generated layered wedge mesh)",
                "config": {"workload": wl + ", face traces of the one-sublayer ghost layer exchanged per LSERK "
                                            "stage (NCCL p2p) on a side stream, overlapped with the interior elements",
                           "degree": args.degree, "wedges_per_gpu": head["wedges"],
                           "total_wedges": head["total_wedges"],
                           "parallelism": f"mesh partition x{ws}", "l2": "inputs larger than L2, no flush",
                           "exchange_bytes_per_stage_per_rank": head["exchange_bytes_per_stage"]},
                "roofline": head["roofline"], "cpu_baseline": None, "e2e": head["e2e"],
                "wedge_kernel_avg_ms": head["wedge_kernel_avg_ms"],
                "gpu_launches": head["gpu_launches"], "clocks": head["clocks"], "setup_s": head["setup_s"],
            }
            print(json.dumps(line), flush=True)
        torch.distributed.destroy_process_group()
        return 0
    head = measure_degree(args, args.degree, ws, rank, local, peaks)
    sweep = []
    for deg in [int(x) for x in args.degrees.split(",") if x.strip()]:
        if deg == args.degree:
            continue
        r = measure_degree(args, deg, ws, rank, local, peaks, with_e2e=False)
        sweep.append({k: r[k] for k in ("degree", "value", "ms_per_step", "wedge_kernel_avg_ms", "roofline",
                                        "total_dofs", "setup_s", "gpu_launches", "tensor_roofline",
                                        "tet_kernel_avg_ms", "tet_roofline", "tet_tensor_roofline") if k in r})
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        med, sample, _ = cpu_sample(args.degree, threads, steps=args.cpu_steps, warmup=1)
        cpu = {"value": med["parallel"], "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
               "variant": "parallel update (value)", "faithful_serial_update": med["faithful"],
               "build": "-O3 -march=x86-64-v3 -fopenmp (prebuilt oracle; bench.py --impl reference rebuilds it "
                        "with -march=native)", "cpu": cpu_model()}
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gaussian pulse on generated layered wedge mesh, random-free)",
            "config": {"workload": (f"configs[2]: structured_hybrid_box({args.hybrid_n},{args.hybrid_n},"
                                    f"{args.hybrid_n // 2},{args.hybrid_n // 2}), {head['wedges']} wedges + "
                                    f"{head['tets']} tets, " if args.workload == "hybrid" else
                                    "configs[1]: layered wedge mesh, stack_layers n=100 surface x 50 sublayers "
                                   "(1e6 wedges/GPU), ") + ("exact stored-lift mass" if args.mass == "exact" else
                                   "weight-adjusted (WADG) mass, no per-wedge operator storage") + ", upwind",
                       "mass": args.mass,
                       "degree": args.degree, "wedges_per_gpu": head["wedges"], "total_dofs_per_gpu": head["total_dofs"],
                       "parallelism": "single GPU",
                       "l2": "inputs larger than L2 (state >> 126 MB), no flush"},
            "roofline": head["roofline"], "cpu_baseline": cpu, "e2e": head.get("e2e"),
            **({"e2e_run_simulation": head["e2e_run_simulation"]} if "e2e_run_simulation" in head else {}),
            "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "wedge_kernel_avg_ms": head["wedge_kernel_avg_ms"], "wedge_kernel_share": head["wedge_kernel_share"],
            **({k: head[k] for k in ("tet_kernel_avg_ms", "tet_kernel_share", "tet_roofline", "tet_tensor_roofline",
                                       "tensor_roofline")
                if k in head}),
            "setup_s": head["setup_s"],
        }
        if sweep:
            line["sweep"] = sweep
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
