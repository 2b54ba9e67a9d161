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
bounded sample of the same case on this host's cores), e2e (the public
Simulation.run() API: device-clock batches of 64 steps, one host round trip
per batch; per_step_api = pick_dt() + step() with a round trip per step),
clocks, passes.

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


def perturb(cfg, seed=0):
    """SURVEY.md 8(d) synthetic block state (mirrors backend_bench.py:29-34)."""
    rng = np.random.default_rng(seed)
    for b in cfg.bodies:
        st = b.state
        n = st.X.shape[0]
        st.u[:] = rng.normal(scale=2e-5 * b.dp_body / 1e-3, size=(n, 3))
        st.v[:] = rng.normal(scale=1.0, size=(n, 3))
        if b.fracture:
            st.s[:] = rng.uniform(0.3, 1.0, n)
        if b.dim == 2:
            st.u[:, 1] = 0.0
            st.v[:, 1] = 0.0


# ---------------------------------------------------------------------------
# CPU reference arm / baseline (oracle port; test infrastructure)
# ---------------------------------------------------------------------------

CPU_SAMPLE = {"C4": dict(spec="kalthoff3d", dp_scale=0.918 * 4, mapfac=5)}
WORKLOAD_NAMES = {
    "C1": "C1: 2D elastic cantilever plate (beam2d), SVK, radial, Verlet, adaptive dt",
    "C2": "C2: 3D elastic column (column3d), Neo-Hookean, radial (k~160), adaptive dt",
    "C3": "C3: 3D Taylor bar impact (taylor3d), J2 finite-strain plasticity, radial, adaptive dt",
    "C4": "C4: 3D Kalthoff-Winkler phase-field fracture, SVK+spectral split, nbsrange=1, "
          "Verlet, adaptive dt",
    "C5": "C5: 2D crack-branching plate (branch2d), SVK+PF AT2, nbsrange=1, adaptive dt"}


def cpu_reference(config, steps, warmup, budget_s=25.0):
    """Time the oracle (C/OpenMP restatement of the reference's numba
    kernels + numpy stepper) on a bounded sample of the workload."""
    from oracle import oracle as O
    from paper_2602_15149_b200 import cases
    O.build()
    threads = os.cpu_count() or 1
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
            "steps": done, "seconds": el, "n": n}


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
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"],
                    help="BASELINE.json configs: C4 is the headline; the others are extra "
                         "measurements (no CPU baseline sample)")
    ap.add_argument("--e2e-steps", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
                "config": {"workload": f"{args.config} CPU sample", "sample": ref["sample"]},
                "impl": "reference",
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": "particle-steps/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation

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

    t0 = time.perf_counter()
    base_scale = cases.WORKLOADS[args.config][1].get("dp_scale", 1.0)
    cfg = cases.make_case(args.config, lean=True, build_adjacency=False,
                          lenient_targets=args.config == "C5",
                          dp_scale=base_scale * args.dp_scale)
    perturb(cfg, seed=0)      # one global state; ranks own slabs of it
    t_case = time.perf_counter() - t0
    t0 = time.perf_counter()
    sim = DeviceSimulation(cfg, precision=args.precision, mirrors=False)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    n = sum(db.n for db in sim.dbodies)
    nnz = sum(int(db.layout.indptr[-1].item()) for db in sim.dbodies)   # owned rows
    k_mean = nnz / n
    sim.initialize()
    sim.advance(args.warmup)
    sim.finish_advance()
    torch.cuda.synchronize()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    pass_ev = []
    with ClockSampler(local) as clocks:
        torch.cuda.nvtx.range_push("timed")      # ncu --nvtx --nvtx-include timed/
        ev0.record(sim.stream)
        sim.advance(args.steps)
        ev1.record(sim.stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    sim.finish_advance()
    # per-pass kernel times for the roofline: a further short run with events
    # around each pass (which launches the passes back to back, without the
    # single-GPU pass overlap of the timed steps)
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
    ms_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (per-launch algorithmic bytes / event time)
    w = 4 if args.precision == "fp32" else 8
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
        traffic = tr.get(f"{args.config}.{args.precision}.{dom[0]}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                "bytes_per_particle": dom[1],
                "step_frac": (ba + bb) * value / max(world, 1) / 1e9 / peak}
    passes = {"pass_a_ms": ma, "pass_b_ms": mb, "bytes_a": ba, "bytes_b": bb,
              "frac_a": ba * n / (ma / 1e3) / 1e9 / peak,
              "frac_b": bb * n / (mb / 1e3) / 1e9 / peak}

    # end to end through the public API (stepper.Simulation's): run() -- the
    # throughput entry point, device-clock batches of 64 steps with one host
    # round trip per batch -- and pick_dt() + step() with a round trip per step
    e2e = None
    if args.e2e_steps > 0:
        import math as _m
        nb = len(sim.dbodies)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.run(time_max=1e30, time_out=1e30, max_steps=sim.step_index + args.e2e_steps)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        batches = _m.ceil(args.e2e_steps / 64)
        e2e = {"value": n_total * args.e2e_steps / el, "unit": "particle-steps/s",
               # per batch: clock struct in; clock, error counters, plastic work out
               "h2d_bytes_per_step": 80 * batches / args.e2e_steps,
               "d2h_bytes_per_step": (80 + 72 * nb) * batches / args.e2e_steps,
               "steps": args.e2e_steps,
               "api": "DeviceSimulation.run(max_steps=...) (the reference's Simulation.run); "
                      "host state arrays refresh lazily on access (DeviceState)"}
        k = min(args.e2e_steps, 32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            sim.step(sim.pick_dt())
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        e2e["per_step_api"] = {"value": n_total * k / el, "steps": k,
                               "api": "pick_dt() + step(dt), one host round trip per step",
                               "h2d_bytes_per_step": 80,
                               "d2h_bytes_per_step": 16 * nb + 64 * nb + 8 * nb}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in CPU_SAMPLE:
        try:
            ref = cpu_reference(args.config, 10, 1)
            cpu = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # the baseline must not kill the GPU line
            cpu = {"value": None, "error": repr(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "particle-steps/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32" if args.precision == "fp32" else "f64",
                "data": "synthetic (seeded perturbed lattice state, SURVEY.md 8(d))",
                "config": {"workload": WORKLOAD_NAMES[args.config],
                           "particles_per_gpu": n, "particles": int(n_total),
                           "pairs_per_particle": k_mean,
                           "parallelism": (f"slab{world} (halo exchange over "
                                           f"{args.dist_backend})" if world > 1 else "single"),
                           "l2": "per-step working set >> 126 MB L2, no flush",
                           "precision": args.precision,
                           "bond_classes": [int(db.desc.ncls) for db in sim.dbodies],
                           "setup_s": {"case": t_case, "device_build": t_setup}},
                "roofline": roofline, "passes": passes, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(args.steps * (2 + 2 * len(sim.dbodies))),
                "clocks": clocks.summary()}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
