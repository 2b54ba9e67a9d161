"""Tile halo statistics of the C4 device layout (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation
    cfg = cases.make_case(sys.argv[1] if len(sys.argv) > 1 else "C4", lean=True,
                          build_adjacency=False)
    sim = DeviceSimulation(cfg, precision="fp32", mirrors=False)
    lay = sim.dbodies[0].layout
    hoff = lay.hoff.cpu().numpy()
    H = np.diff(hoff)
    hs = lay.hslot.cpu().numpy().astype(np.int64) & 0xffff
    ext = np.array([hs[hoff[t]:hoff[t + 1]].max() - lay.tile + 1 if hoff[t + 1] > hoff[t] else 0
                    for t in range(len(H))])
    print("tiles", len(H), "T", lay.tile, "hmax", lay.hmax)
    for name, a in (("H", H), ("extent", ext)):
        print(name, "mean %.1f" % a.mean(), "pct50/90/99/99.9/max",
              np.percentile(a, [50, 90, 99, 99.9]).round(1), a.max())
    big = np.argsort(-H)[:5]
    print("fattest tiles", big, H[big])


if __name__ == "__main__":
    main()
