"""Small device runs for compute-sanitizer (memcheck / racecheck / synccheck):
the tiled bond-class path (kalthoff3d), the brick path (column3d forced),
2D tiles + L2 gather (kalthoff2d_p), J2 (taylor3d), FP32 and FP64."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden, run_case  # noqa: E402
from paper_2602_15149_b200.simulation import DeviceSimulation  # noqa: E402

for tag, prec, env in [("kalthoff3d", "fp32", {}), ("kalthoff3d", "fp64", {}),
                       ("column3d", "fp32", {"TLSPH_BRICK": "force"}),
                       ("taylor3d", "fp64", {"TLSPH_BRICK": "force"}),
                       ("kalthoff2d_p", "fp32", {})]:
    for k, v in env.items():
        os.environ[k] = v
    G = golden(f"run_{tag}")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision=prec)
    sim.initialize()
    for s in range(2):
        sim.step(G["dts"][s])
    sim.advance(3)
    sim.finish_advance()
    for k in env:
        del os.environ[k]
    print(tag, prec, "ok")
