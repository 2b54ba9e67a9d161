#!/usr/bin/env python3
"""Throughput of the B200 TLSPH hot path on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp32|fp64]
                    [--impl ours|reference] [--config C4]

Workload (default C4, BASELINE.json configs[3]): the 3D Kalthoff-Winkler
phase-field fracture block, SVK + spectral split, nbsrange = 1 (26
neighbours), notch through the thickness, ramp velocity BC, Verlet with
adaptive dt -- 15,863,256 particles on one B200.  The
initial state is the seeded "synthetic block" perturbation of SURVEY.md 8(d)
(u ~ N(0, (2e-5 dp/1e-3)^2), v ~ N(0,1), s ~ U(0.3,1)) so every kernel
branch does real work.  A step = one device-clock Verlet step (dt, pass A,
pass B, commit).  value = particle-steps/s over the timed steps (CUDA
events, max over ranks).  --gpus N (torchrun) partitions the same 15.9 M
particles into N slabs with halo exchange (strong scaling, SURVEY.md
8(e)).  The ~9 GB per-step working set is far larger than the 126 MB L2, so
no flush is needed between steps.

Extra keys: roofline (dominant kernel vs measured HBM copy bandwidth,
SURVEY.md 8(d) algorithmic bytes), cpu_baseline (the CPU oracle port, a
bounded sample of the same case on this host's cores), e2e (the public API
with host buffers: push_state() of the page-locked host state, run() with the
case's output cadence and the OutputManager's energy / measure rows, then
pull_host() of every field), fp64 (the same workload in the reference's
precision), clocks, passes.

--impl reference times the reference algorithm on the host CPU (the oracle
port of solidsph's numba/numpy backends, oracle/; the reference itself is a
Python package that cannot travel to the GPU box) on a bounded sample of the
same workload and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/s, 3D phase-field fracture, 1/2/4/8 B200; % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")

# canonical algorithmic bytes per particle-step, per pass
# (w = bytes per Real).  3D: pass A reads X(24) + L(9w) + u(3w)
# [+ s, sdot, H (3w)] [+ Cp, epbar (7w)] and writes P(9w) + Avis(9w)
# [+ H, sddot (2w)] [+ Cp, epbar (7w)]; pass B reads X(24) + L, P, Avis (27w)
# + v, u (6w) [+ s, sdot, sddot (3w)] and writes v, u (6w) [+ s, sdot (2w)];
# each + 8 + 4k (indptr, int32 neighbour indices).  2D: X 16 B, tensors 4w,
# vectors 2w.  3D fracture FP32: 172 + 4k and 208 + 4k (C4: 585 B per step).
def pass_bytes(w, k, dim=3, fracture=True, j2=False):
    t, v, x = (9, 3, 24) if dim == 3 else (4, 2, 16)
    fa = 3 * w if fracture else 0
    fw = 2 * w if fracture else 0
    jr = (t - 3 + 1) * w if j2 else 0          # Cp (symmetric) + epbar
    a = x + t * w + v * w + fa + jr + t * w + t * w + fw + jr + 8 + 4 * k
    b = x + 3 * t * w + 2 * v * w + fa + 2 * v * w + fw + 8 + 4 * k
    return a, b


def peak_hbm():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _mix64(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _uniform(gid, stream, seed):
    """Counter-based U(0, 1) per global particle id: every rank draws the
    same numbers for the same particle, whatever part of the body it holds."""
    with np.errstate(over="ignore"):
        x = _mix64(gid.astype(np.uint64) * np.uint64(64) + np.uint64(stream)
                   + np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15))
    return ((x >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def _normal(gid, stream, seed):
    u1, u2 = _uniform(gid, 2 * stream, seed), _uniform(gid, 2 * stream + 1, seed)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def perturb(cfg, seed=0):
    """SURVEY.md 8(d) synthetic block state (mirrors backend_bench.py:29-34):
    u ~ N(0, (2e-5 dp/1e-3)^2), v ~ N(0, 1), s ~ U(0.3, 1), drawn per global
    particle id so a slab-local rank (cases.make_case(slab=...)) holds the
    same state as the whole-body build."""
    for b in cfg.bodies:
        st = b.state
        n = st.X.shape[0]
        slab = getattr(b, "slab", None)
        gid = slab.gid if slab is not None else np.arange(n, dtype=np.int64)
        scale = 2e-5 * b.dp_body / 1e-3
        for c in range(3):
            st.u[:, c] = scale * _normal(gid, c, seed)
            st.v[:, c] = _normal(gid, 3 + c, seed)
        if b.fracture:
            st.s[:] = 0.3 + 0.7 * _uniform(gid, 20, seed)
        if b.dim == 2:
            st.u[:, 1] = 0.0
            st.v[:, 1] = 0.0


# ---------------------------------------------------------------------------
# CPU reference arm / baseline (oracle port; test infrastructure)
# ---------------------------------------------------------------------------

CPU_SAMPLE = {"C4": dict(spec="kalthoff3d", dp_scale=0.918 * 4, mapfac=5),
              "P1": dict(spec="fourpoint3d", dp_scale=1.26 * 2, mapfac=None)}
WORKLOAD_NAMES = {
    "C1": "C1: 2D elastic cantilever plate (beam2d), SVK, radial, Verlet, adaptive dt",
    "C2": "C2: 3D elastic column (column3d), Neo-Hookean, radial (k~160), adaptive dt",
    "C3": "C3: 3D Taylor bar impact (taylor3d), J2 finite-strain plasticity, radial, adaptive dt",
    "C4": "C4: 3D Kalthoff-Winkler phase-field fracture, SVK+spectral split, nbsrange=1, "
          "Verlet, adaptive dt",
    "C5": "C5: 2D crack-branching plate (branch2d), SVK+PF AT2, nbsrange=1, adaptive dt",
    "P1": "P1 (paper anchor, PAPER.md:1605-1611): four-point bending beam (fourpoint3d), "
          "3D SVK+PF, radial (k~170), notch, restrictphi, 1M particles, adaptive dt"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# Port vs the reference's own numba backend, measured in the build container
# (the reference cannot travel to the GPU box): tools/cpu_calibrate.py
CALIB = os.path.join(ROOT, "profiles", "cpu_calibration.json")


def cpu_reference(config, steps, warmup, budget_s=25.0, threads=None):
    """Time the oracle (C/OpenMP restatement of the reference's numba
    kernels + numpy stepper) on a bounded sample of the workload."""
    from oracle import oracle as O
    from paper_2602_15149_b200 import cases
    O.build()
    threads = threads or os.cpu_count() or 1
    O.set_threads(threads)
    smp = CPU_SAMPLE[config]
    cfg = cases.make_case(smp["spec"], dp_scale=smp["dp_scale"], mapfac=smp["mapfac"],
                          build_adjacency=False)
    perturb(cfg)
    t0 = time.perf_counter()
    for b in cfg.bodies:
        b.adjacency = O.build_adjacency(b.state.X, b.state.V0, b.h, b.dim, int(cfg.kernel),
                                        nbsrange=b.nbsrange, dp_body=b.dp_body,
                                        notches=b.notches, correction=b.kernel_correction)
    setup = time.perf_counter() - t0
    n = sum(b.state.X.shape[0] for b in cfg.bodies)
    sim = O.OracleSimulation(cfg)
    sim.initialize()
    for _ in range(max(warmup, 1)):
        sim.step(sim.pick_dt())
    done, t0 = 0, time.perf_counter()
    while done < steps:
        sim.step(sim.pick_dt())
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    k = float(np.mean(np.diff(cfg.bodies[0].adjacency.indptr)))
    return {"value": n * done / el, "unit": "particle-steps/s", "cores": threads,
            "kind": "port",
            "sample": (f"{smp['spec']} dp_scale={smp['dp_scale']:.4g} mapfac={smp['mapfac']}: "
                       f"N={n}, k={k:.1f}, {done} timed Verlet steps after {max(warmup, 1)} "
                       f"warm-up, FP64, oracle/liboracle.so OpenMP x{threads} "
                       f"(adjacency setup {setup:.1f}s untimed)"),
            "steps": done, "seconds": el, "n": n, "cpu_model": cpu_model()}


def cpu_baseline_full(config):
    """All host threads (the reported baseline), a 1-thread figure on a
    shorter budget, the CPU model, and the port-vs-numba calibration."""
    ref = cpu_reference(config, 10, 1)
    one = cpu_reference(config, 3, 1, budget_s=8.0, threads=1)
    out = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
    out["value_1thread"] = one["value"]
    try:
        with open(CALIB) as f:
            out["calibration"] = json.load(f)
    except Exception:
        out["calibration"] = None
    return out


# ---------------------------------------------------------------------------

def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one
    process per GPU, the driver's own torchrun command line) and pass their
    output through; rank 0 prints the JSON line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5", "P1"],
                    help="BASELINE.json configs: C4 is the headline; the others are extra "
                         "measurements (no CPU baseline sample)")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true",
                    help="skip the FP64 (parity mode) sub-measurement of an FP32 run")
    ap.add_argument("--dp-scale", type=float, default=1.0,
                    help="multiply the config's particle spacing (profiling at reduced size)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share one GPU (halo buffers staged through the host; "
                         "a plumbing check, not a throughput number)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference(args.config, args.steps, args.warmup)
        line = {"metric": METRIC, "value": ref["value"], "unit": "particle-steps/s",
                "n_gpus": args.gpus, "steps": ref["steps"], "warmup": args.warmup,
                "ms_per_step": 1e3 * ref["seconds"] / max(ref["steps"], 1),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded perturbed lattice state)",
                "config": {"workload": WORKLOAD_NAMES[args.config],
                           "cpu_sample": ref["sample"], "precision": "fp64"},
                "impl": "reference",
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": "particle-steps/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    from paper_2602_15149_b200 import cases

    ndev = torch.cuda.device_count()
    if world > 1 and args.dist_backend == "nccl" and world > ndev:
        raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, {ndev} visible")
    torch.cuda.set_device(local % max(ndev, 1))
    if world > 1:
        if args.dist_backend == "nccl":
            # communicator init lines (rank count, NVLink/NVLS transport) to
            # stderr, so the JSON line on stdout stays the last line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", init_method="env://",
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo", init_method="env://")

    base_scale = cases.WORKLOADS[args.config][1].get("dp_scale", 1.0)

    def make_cfg():
        t0 = time.perf_counter()
        # N > 1: each rank builds only its slab of the lattice on the host
        cfg = cases.make_case(args.config, lean=True, build_adjacency=False,
                              lenient_targets=args.config == "C5",
                              dp_scale=base_scale * args.dp_scale,
                              slab=(rank, world) if world > 1 else None)
        perturb(cfg, seed=0)      # one global state; ranks own slabs of it
        return cfg, time.perf_counter() - t0

    cfg, t_case = make_cfg()
    res = measure(args, cfg, args.precision, world, local, clocks_on=True)
    sim = res.pop("sim")
    n, n_total = res["n"], res["n_total"]
    value = res["value"]

    # end to end through the public API: the host state goes up, run() steps
    # with the case's output cadence (energies + measure rows through the
    # device reductions output.install routes the reference's OutputManager
    # to), and the final state comes back to the host
    e2e = e2e_run(sim, args.e2e_steps, n_total) if args.e2e_steps > 0 else None
    del sim
    torch.cuda.empty_cache()

    # the reference's own precision beside the headline (FP64 parity mode)
    fp64 = None
    if args.precision == "fp32" and not args.no_fp64:
        cfg64, _ = make_cfg()
        r64 = measure(args, cfg64, "fp64", world, local, clocks_on=False, e2e=False)
        del r64["sim"]
        fp64 = {k: r64[k] for k in ("value", "ms_per_step", "roofline", "passes",
                                    "device_bytes_per_particle")}
        fp64["unit"] = "particle-steps/s"
        del cfg64
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in CPU_SAMPLE:
        try:
            cpu = cpu_baseline_full(args.config)
        except Exception as exc:  # the baseline must not kill the GPU line
            cpu = {"value": None, "error": repr(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "particle-steps/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32" if args.precision == "fp32" else "f64",
                "data": "synthetic (seeded perturbed lattice state, SURVEY.md 8(d))",
                "config": {"workload": WORKLOAD_NAMES[args.config],
                           "particles_per_gpu": n, "particles": int(n_total),
                           "pairs_per_particle": res["k_mean"],
                           "parallelism": (f"slab{world} (halo exchange over "
                                           f"{args.dist_backend})" if world > 1 else "single"),
                           "l2": "per-step working set >> 126 MB L2, no flush",
                           "precision": args.precision,
                           "bond_classes": res["bond_classes"],
                           "device_bytes_per_particle": res["device_bytes_per_particle"],
                           "cuda_graphs": res["graphs"],
                           "setup_s": {"case": t_case, "device_build": res["t_setup"]}},
                "roofline": res["roofline"], "passes": res["passes"], "fp64": fp64,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": res["launches"],
                "clocks": res["clocks"]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def measure(args, cfg, precision, world, local, clocks_on, e2e=True):
    """Device throughput of `args.steps` timed steps (inputs resident in HBM),
    max over ranks, plus per-pass kernel times for the roofline."""
    import torch
    import torch.distributed as dist
    from paper_2602_15149_b200.simulation import DeviceSimulation
    t0 = time.perf_counter()
    # host-layout FP64 mirrors (F, S, psi) only when the e2e outputs need them
    sim = DeviceSimulation(cfg, precision=precision, mirrors=e2e and args.e2e_steps > 0)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    n = sum(db.n for db in sim.dbodies)
    nnz = sum(int(db.layout.indptr[-1].item()) for db in sim.dbodies)   # owned rows
    k_mean = nnz / n
    sim.initialize()
    sim.advance(args.warmup)
    sim.finish_advance()
    sim.prepare_graphs()              # capture the step graphs outside the timed regions
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    pass_ev = []
    sampler = ClockSampler(local) if clocks_on else None
    if sampler:
        sampler.__enter__()
    try:
        torch.cuda.nvtx.range_push("timed")      # ncu --nvtx --nvtx-include timed/
        ev0.record(sim.stream)
        sim.advance(args.steps)
        ev1.record(sim.stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    finally:
        if sampler:
            sampler.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    sim.finish_advance()
    # per-pass kernel times for the roofline: a further short run with events
    # around each pass (eager launches)
    sim.advance(min(args.steps, 20), pass_events=pass_ev)
    torch.cuda.synchronize()
    sim.finish_advance()
    ta = [e[0].elapsed_time(e[1]) for e in pass_ev]
    tb = [e[2].elapsed_time(e[3]) for e in pass_ev]
    if world > 1:
        cdev = "cuda" if args.dist_backend == "nccl" else "cpu"
        tt = torch.tensor([ms], device=cdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        nt = torch.tensor([n], device=cdev, dtype=torch.float64)
        dist.all_reduce(nt)
        n_total = float(nt.item())
    else:
        n_total = float(n)
    value = n_total * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (per-launch algorithmic bytes / event time)
    w = 4 if precision == "fp32" else 8
    b0 = cfg.bodies[0]
    ba, bb = pass_bytes(w, k_mean, dim=int(b0.dim), fracture=bool(b0.fracture),
                        j2=int(b0.material.model) == 3)
    ma, mb = float(np.mean(ta)), float(np.mean(tb))
    peak, peak_kind = peak_hbm()
    dom = ("pass_b_force", bb, mb) if mb >= ma else ("pass_a_phase_field", ba, ma)
    achieved = dom[1] * n / (dom[2] / 1e3) / 1e9
    traffic = None
    try:
        with open(TRAFFIC) as f:
            tr = json.load(f)
        traffic = tr.get(f"{args.config}.{precision}.{dom[0]}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                "bytes_per_particle": dom[1],
                "step_frac": (ba + bb) * value / max(world, 1) / 1e9 / peak}
    passes = {"pass_a_ms": ma, "pass_b_ms": mb, "bytes_a": ba, "bytes_b": bb,
              "frac_a": ba * n / (ma / 1e3) / 1e9 / peak,
              "frac_b": bb * n / (mb / 1e3) / 1e9 / peak,
              "samples_ms": {"a": [round(x, 4) for x in ta], "b": [round(x, 4) for x in tb]}}
    # our kernels per timed step: clock begin + commit, and per body pass A and
    # pass B (+ the plastic-work reduction for J2 bodies); the dt-maxima reset
    # is a memset
    per_step = 2 + sum(2 + (int(db.body.material.model) == 3) for db in sim.dbodies)
    mem = torch.cuda.max_memory_allocated()
    return {"sim": sim, "n": n, "n_total": n_total, "k_mean": k_mean, "value": value,
            "device_bytes_per_particle": mem / max(n, 1),
            "ms_per_step": ms / args.steps, "roofline": roofline, "passes": passes,
            "t_setup": t_setup, "bond_classes": [int(db.desc.ncls) for db in sim.dbodies],
            "graphs": bool(sim.use_graphs), "launches": int(args.steps * per_step),
            "clocks": sampler.summary() if sampler else None}


def _state_bytes(sim, pull):
    """Bytes one push_state (pull=False) or full pull_state (True) moves."""
    tot = 0
    for db in sim.dbodies:
        names = ["us", "v", "sdot", "sddot", "Hh", "epbar"] + (["a"] if not pull else [])
        if int(db.body.material.model) == 3:
            names.append("Cpd")
        rows = db.n if pull else db.n_all
        for k in names:
            t = getattr(db, k)
            tot += t.element_size() * t.numel() * rows // max(db.n_all, 1)
        if pull and db.mirrors:
            tot += 8 * db.n * (3 + 9 + 9 + 1 + 1)     # a, F, S, psi_e, psi_plus (FP64)
    return tot


def e2e_run(sim, steps, n_total):
    """run() through the public API with host buffers: push the host state,
    step with outputs at the case's TimeOut (energies + measure rows, the
    reference OutputManager's CSV rows, through paper_2602_15149_b200.output),
    then pull the final state into body.state."""
    import torch
    from paper_2602_15149_b200 import output
    rows = []

    def on_output(s):
        for body in s.bodies:
            rows.append(output.compute_energies(body))
            for idx in getattr(body, "measure_sets", []) or []:
                rows.append(output.measure_row(body, idx, s.t))

    for db in sim.dbodies:           # the reference's full ParticleArrays (lean cases skip F, S)
        st = db.host
        nb = st.X.shape[0]
        for k, shape in (("F", (nb, 3, 3)), ("S", (nb, 3, 3))):
            if getattr(st, k) is None:
                setattr(st, k, np.zeros(shape))
    sim.pull_host()                  # the host state a user of the API holds
    sim.pin_host_state()             # page-locked once, as a user's repeated runs would
    on_output(sim)                   # output kernels loaded once (lazy module loading), untimed
    rows.clear()
    torch.cuda.synchronize()
    t_out = float(sim.config.time_out)
    # a fresh run from t = 0 (the reference's run() puts its first output
    # boundary at time_out, so it restarts the clock like a new Simulation)
    sim.t, sim.step_index = 0.0, 0
    start = sim.step_index
    t0 = time.perf_counter()
    sim.push_state()                                           # host -> device
    sim.run(time_max=float(sim.config.time_max), time_out=t_out, on_output=on_output,
            max_steps=start + steps)
    sim.pull_host()                                            # device -> host
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    done = sim.step_index - start
    h2d = _state_bytes(sim, pull=False)
    d2h = _state_bytes(sim, pull=True)
    n_out = len(rows)
    # the same run with the VTK snapshot fields of every output copied to the
    # host asynchronously (output.snapshot_async), overlapping the next steps
    snaps = []

    def on_output_vtk(s):
        on_output(s)
        snaps.append(output.snapshot_async(s))

    output.snapshot_async(sim).wait()   # page-locked snapshot buffers allocated once, untimed
    sim.t, sim.step_index = 0.0, 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.push_state()
    sim.run(time_max=float(sim.config.time_max), time_out=t_out, on_output=on_output_vtk,
            max_steps=steps)
    for sn in snaps:
        sn.wait()
    sim.pull_host()
    torch.cuda.synchronize()
    el_v = time.perf_counter() - t0
    done_v = sim.step_index
    snap_bytes = sum(sn.nbytes for sn in snaps)
    return {"value": n_total * done / el, "unit": "particle-steps/s", "steps": done,
            "with_vtk_snapshots": {"value": n_total * done_v / el_v, "snapshots": len(snaps),
                                   "d2h_bytes_per_step": (d2h + snap_bytes) / max(done_v, 1)},
            "h2d_bytes_per_step": h2d / max(done, 1),
            "d2h_bytes_per_step": (d2h + 8 * 64 * n_out) / max(done, 1),
            "outputs": n_out, "time_out": t_out,
            "api": "push_state(); DeviceSimulation.run(time_out=case TimeOut, on_output=energies "
                   "+ measure rows via output.install's device reductions, max_steps); "
                   "pull_host() -- the reference's Simulation.run + OutputManager CSV rows "
                   "(VTK writer out of scope)"}


if __name__ == "__main__":
    main()
