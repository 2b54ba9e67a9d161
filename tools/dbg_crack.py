import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from conftest import golden, run_case
from paper_2602_15149_b200.simulation import DeviceSimulation
G = golden("crack_kalthoff2d")
for prec in ("fp64", "fp32"):
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision=prec)
    t_end = float(G["end.t"][0])
    sim.run(time_max=t_end, time_out=t_end)
    st = cfg.bodies[0].state
    ds = np.abs(st.s - G["end.s"])
    du = np.abs(st.u - G["end.u"]).max() / np.abs(G["end.u"]).max()
    print(prec, "steps", sim.step_index, "max|ds|", ds.max(), "rel du", du, "n(ds>1e-3)", (ds > 1e-3).sum())
    b = cfg.bodies[0]
    quad = b.notches[0].points
    tip = quad[int(np.argmax(quad[:, 0]))]
    mine = set(np.flatnonzero((st.s < 0.5) & (st.X[:, 0] > tip[0] + 2.0 * b.dp_body)).tolist())
    ref = set(G["damaged"].tolist())
    for q in sorted(mine ^ ref):
        print("   differ", q, "dev s", st.s[q], "ref s", G["end.s"][q])
