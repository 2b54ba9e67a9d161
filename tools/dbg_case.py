"""Run a workload a few steps and report the first error (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation
    name, prec, ds = sys.argv[1], sys.argv[2], float(sys.argv[3])
    cfg = cases.make_case(name, dp_scale=ds, lean=True, build_adjacency=False,
                          lenient_targets=True)
    if len(sys.argv) > 4 and sys.argv[4] == "perturb":
        bench.perturb(cfg)
    sim = DeviceSimulation(cfg, precision=prec, mirrors=False)
    print(name, prec, "n", sum(db.n for db in sim.dbodies), "tile", sim.dbodies[0].layout.tile)
    sim.initialize()
    for k in range(20):
        try:
            dt = sim.pick_dt()
            sim.step(dt)
        except Exception as e:
            print("step", k + 1, "error:", e)
            return
        st = cfg.bodies[0].state
        print(k + 1, "dt", dt, "vmax", float(abs(st.v).max()), "umax", float(abs(st.u).max()))


if __name__ == "__main__":
    main()
