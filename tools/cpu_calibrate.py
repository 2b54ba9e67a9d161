"""Port-vs-reference calibration of the CPU baseline (build container only:
needs /root/reference, which cannot travel to the GPU box).

Times the reference's own numba backend (SOLIDSPH_BACKEND=numba,
stepper.Simulation.step with its adaptive dt) and the oracle port
(oracle/liboracle.so, the arm bench.py runs on the GPU box) on the same
bounded C4 sample bench.py uses, with all threads and with one, and writes
profiles/cpu_calibration.json.  bench.py attaches that file to its
cpu_baseline so the port's speed relative to the reference is on the line.

    python tools/cpu_calibrate.py
"""
import json
import os
import sys
import time

os.environ["SOLIDSPH_BACKEND"] = "numba"
REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from solidsph import backends, caseio, stepper  # noqa: E402

assert backends.active().NAME == "numba", backends.active().NAME
CASES = os.path.join(REF, "cases")


def _kalthoff3d_raw():
    """kalthoff2d.xml extruded to 3D with the notch through the thickness
    (as oracle/gen_golden.py, which pins the numpy backend
    and so is not imported here)."""
    raw = caseio.parse_case(os.path.join(CASES, "kalthoff2d.xml"))
    raw.dim = 3
    for q in raw.bodies[0].notches:
        q.points[2, 1] = 11e-3
        q.points[3, 1] = 11e-3
    return raw


def time_reference(threads, steps, budget):
    smp = bench.CPU_SAMPLE["C4"]
    backends.set_threads(threads)
    cfg = caseio.build_case(_kalthoff3d_raw(), dp_scale=smp["dp_scale"], mapfac=smp["mapfac"])
    bench.perturb(cfg, seed=0)
    sim = stepper.Simulation(cfg)
    sim.initialize()
    for _ in range(2):                       # warm-up (numba JIT)
        sim.step(sim.pick_dt())
    done, t0 = 0, time.perf_counter()
    while done < steps and time.perf_counter() - t0 < budget:
        sim.step(sim.pick_dt())
        done += 1
    el = time.perf_counter() - t0
    n = sum(b.state.X.shape[0] for b in cfg.bodies)
    return {"value": n * done / el, "steps": done, "n": n, "threads": threads}


def main():
    cores = os.cpu_count() or 1
    out = {"cores": cores, "cpu_model": bench.cpu_model(),
           "sample": "C4 CPU sample of bench.py (kalthoff3d dp_scale=3.672 mapfac=5, seeded "
                     "perturbed state), adaptive-dt Verlet steps after warm-up, FP64"}
    out["reference_numba"] = time_reference(cores, 20, 40.0)
    out["reference_numba_1thread"] = time_reference(1, 4, 40.0)
    p = bench.cpu_reference("C4", 20, 1, budget_s=40.0)
    p1 = bench.cpu_reference("C4", 4, 1, budget_s=40.0, threads=1)
    out["port"] = {"value": p["value"], "steps": p["steps"], "n": p["n"], "threads": cores}
    out["port_1thread"] = {"value": p1["value"], "steps": p1["steps"], "n": p1["n"], "threads": 1}
    out["numba_over_port"] = out["reference_numba"]["value"] / out["port"]["value"]
    out["numba_over_port_1thread"] = (out["reference_numba_1thread"]["value"]
                                      / out["port_1thread"]["value"])
    path = os.path.join(ROOT, "profiles", "cpu_calibration.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
