"""Time the host-side pieces of the e2e path on C4 (push_state, pull_host,
compute_energies, one run() batch)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2602_15149_b200 import cases, output
from paper_2602_15149_b200.simulation import DeviceSimulation

cfg = cases.make_case("C4", lean=True, build_adjacency=False, dp_scale=0.918)
bench.perturb(cfg)
for b in cfg.bodies:
    n = b.state.X.shape[0]
    b.state.F = np.zeros((n, 3, 3)); b.state.S = np.zeros((n, 3, 3))
sim = DeviceSimulation(cfg, precision="fp32", mirrors=True)
sim.initialize(); sim.advance(10); sim.finish_advance()
def T(name, f, k=3):
    for i in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        print(f"{name}: {1e3*(time.perf_counter()-t0):.1f} ms")
T("pull_host (pageable)", sim.pull_host)
T("push_state (pageable)", sim.push_state)
t0 = time.perf_counter(); sim.pin_host_state(); print(f"pin: {1e3*(time.perf_counter()-t0):.1f} ms")
T("pull_host (pinned)", sim.pull_host)
T("push_state (pinned)", sim.push_state)
T("compute_energies", lambda: output.compute_energies(cfg.bodies[0]))
sim.t, sim.step_index = 0.0, 0
T("run 128 steps", lambda: sim.run(time_max=cfg.time_max, time_out=cfg.time_out, max_steps=sim.step_index + 128), k=2)
T("advance 128", lambda: (sim.advance(128), sim.finish_advance()), k=2)
