"""Phase timings of bench.e2e_run on one config (default C4): the same
sequence as the bench's e2e (push_state, run() with the case's outputs,
pull_host), run three times in a row, with the time spent in push, in the
on_output callbacks, in run() outside them, and in pull.

    python tools/diag_e2e.py [C4] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_15149_b200 import cases, output  # noqa: E402
from paper_2602_15149_b200.simulation import DeviceSimulation  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = cases.make_case(cfgname, lean=True, build_adjacency=False,
                      lenient_targets=cfgname == "C5",
                      dp_scale=cases.WORKLOADS[cfgname][1].get("dp_scale", 1.0))
bench.perturb(cfg, seed=0)
sim = DeviceSimulation(cfg, precision="fp32", mirrors=True)
sim.initialize()
sim.advance(10)
sim.finish_advance()
sim.prepare_graphs()
for db in sim.dbodies:
    st = db.host
    nb = st.X.shape[0]
    for k in ("F", "S"):
        if getattr(st, k) is None:
            setattr(st, k, np.zeros((nb, 3, 3)))
sim.pull_host()
sim.pin_host_state()
torch.cuda.synchronize()
n_total = sum(db.n for db in sim.dbodies)

for rep in range(3):
    t_cb = [0.0]
    rows = []

    def on_output(s):
        t0 = time.perf_counter()
        for body in s.bodies:
            rows.append(output.compute_energies(body))
            for idx in getattr(body, "measure_sets", []) or []:
                rows.append(output.measure_row(body, idx, s.t))
        t_cb[0] += time.perf_counter() - t0

    sim.t, sim.step_index = 0.0, 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.push_state()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sim.run(time_max=float(sim.config.time_max), time_out=float(sim.config.time_out),
            on_output=on_output, max_steps=steps)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    sim.pull_host()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    done = sim.step_index
    print(f"rep {rep}: {n_total * done / (t3 - t0) / 1e9:.3f} G particle-steps/s; "
          f"push {1e3 * (t1 - t0):.1f} ms, run {1e3 * (t2 - t1):.1f} ms "
          f"(outputs {1e3 * t_cb[0]:.1f} ms, {len(rows)} rows), pull {1e3 * (t3 - t2):.1f} ms, "
          f"{done} steps", flush=True)

t0 = time.perf_counter()
sim.advance(steps)
sim.finish_advance()
torch.cuda.synchronize()
print(f"advance {steps}: {1e3 * (time.perf_counter() - t0):.1f} ms")
