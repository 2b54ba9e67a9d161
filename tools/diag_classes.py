import os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden, run_case, relerr
from paper_2602_15149_b200.simulation import DeviceSimulation
for tag in ["beam2d", "kalthoff2d_p", "branch2d", "kalthoff3d", "fourpoint3d"]:
    G = golden(f"run_{tag}")
    for tb in ["1", "0"]:
        for mode in ["1", "0"]:
            os.environ["TLSPH_TILE_B"] = tb; os.environ["TLSPH_BOND_CLASS"] = mode
            cfg = run_case(G); sim = DeviceSimulation(cfg, precision="fp32")
            sim.initialize(); sim.step(G["dts"][0])
            st = cfg.bodies[0].state
            e = {k: relerr(getattr(st, k) - (np.eye(3) if k == "F" else 0), G[f"s1.b0.{k}"] - (np.eye(3) if k == "F" else 0)) for k in ("F", "S", "a", "v")}
            print(tag, "tile_b", tb, "cls", mode, sim.dbodies[0].desc.ncls, {k: f"{v:.2e}" for k, v in e.items()})
