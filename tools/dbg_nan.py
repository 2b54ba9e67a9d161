import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from conftest import golden, run_case
from paper_2602_15149_b200.simulation import DeviceSimulation
G = golden("crack_kalthoff2d")
for prec in ("fp32", "fp64"):
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision=prec)
    sim.initialize()
    b = cfg.bodies[0]
    for k in range(30):
        dt = G["dts"][k]
        try:
            sim.step(dt)
        except Exception as e:
            print(prec, "step", k + 1, "error", e)
            break
        st = b.state
        bad = ~np.isfinite(st.a).all(axis=1) | ~np.isfinite(st.S.reshape(-1, 9)).all(axis=1)
        if k >= 20 or bad.any():
            q = 1313
            print(prec, k + 1, "nbad", bad.sum(), "u", st.u[q], "v", st.v[q], "a", st.a[q], "s", st.s[q], "sdot", st.sdot[q], "H", st.Hhist[q], "psi", st.psi_e[q], "S", st.S[q].ravel()[[0,2,8]], "F-I", (st.F[q]-np.eye(3)).ravel()[[0,2,6,8]])
