"""A/B check of one environment switch on a bench config: device state after
the same steps with the switch on and off (max abs difference of u, v, s),
graph-replay and eager step times.

    python tools/diag_mode.py C5 TLSPH_CLS_CONST [steps] [dp_scale]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfgname, var = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 64
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0

CHILD = r'''
import os, sys, time, numpy as np, torch
sys.path.insert(0, ROOT)
import bench
from paper_2602_15149_b200 import cases
from paper_2602_15149_b200.simulation import DeviceSimulation
cfg = cases.make_case(CFG, lean=True, build_adjacency=False, lenient_targets=CFG == "C5",
                      dp_scale=cases.WORKLOADS[CFG][1].get("dp_scale", 1.0) * SCALE)
bench.perturb(cfg, seed=0)
sim = DeviceSimulation(cfg, precision="fp32")
sim.initialize()
torch.cuda.synchronize()
t0 = time.perf_counter(); sim.advance(STEPS); sim.finish_advance(); torch.cuda.synchronize()
tg = (time.perf_counter() - t0) / STEPS
ev = []
sim.advance(8, pass_events=ev); sim.finish_advance(); torch.cuda.synchronize()
ta = np.mean([e[0].elapsed_time(e[1]) for e in ev]); tb = np.mean([e[2].elapsed_time(e[3]) for e in ev])
st = cfg.bodies[0].state
np.savez(OUT, u=np.array(st.u), v=np.array(st.v), s=np.array(st.s), t=sim.t, step=sim.step_index)
print(f"{os.environ.get(VAR)}: graph {1e3*tg:.3f} ms/step, eager pass A {ta:.3f} B {tb:.3f} ms, t {sim.t:.6g} step {sim.step_index}")
'''
outs = []
for val in ("1", "0"):
    out = f"/tmp/diag_mode_{val}.npz"
    env = dict(os.environ, **{var: val})
    code = (CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfgname))
            .replace("SCALE", repr(scale)).replace("STEPS", str(steps)).replace("OUT", repr(out))
            .replace("VAR", repr(var)))
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
    outs.append(out)
import numpy as np  # noqa: E402
a, b = np.load(outs[0]), np.load(outs[1])
for k in ("u", "v", "s"):
    d = np.abs(a[k] - b[k]).max()
    print(f"{k}: max|on - off| {d:.3e}, max|off| {np.abs(b[k]).max():.3e}, finite {np.isfinite(a[k]).all()}")
print("t", float(a["t"]), float(b["t"]), "steps", int(a["step"]), int(b["step"]))
