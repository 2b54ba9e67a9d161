"""Compare FP32 pass B with and without the 4-way row split (TLSPH_BSPLIT) on
one golden case: per-particle accelerations after initialize()."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from conftest import golden, run_case  # noqa: E402


def accel(tag, split, tile):
    os.environ["TLSPH_BSPLIT"] = str(split)
    os.environ["TLSPH_TILE"] = str(tile)
    from paper_2602_15149_b200.simulation import DeviceSimulation
    G = golden(f"run_{tag}")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision="fp32")
    for db in sim.dbodies:
        print(tag, "split", db.bsplit, "tile", db.layout.tile, "tile_b", db.tile_b, "n", db.n,
              "hmax", db.layout.hmax, "slmax", db.layout.slmax, "uniform", db.uniform,
              "k", int(db.layout.indptr[-1]) / db.n, "nbc", db.desc.nbc, "whole", db.desc.bc_whole,
              "visc", db.desc.visc)
    try:
        sim.initialize()
    except Exception as e:  # noqa: BLE001
        print("  init error:", e)
    return np.concatenate([np.array(b.state.a, dtype=np.float64) for b in cfg.bodies])


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "twisting3d"
    tile = sys.argv[2] if len(sys.argv) > 2 else "160"
    a1 = accel(tag, 1, tile)
    a4 = accel(tag, 4, tile)
    bad = ~np.isfinite(a4).all(axis=1)
    d = np.abs(a4 - a1).max(axis=1) / (np.abs(a1).max() + 1e-30)
    print("nonfinite", int(bad.sum()), "maxrel", float(np.nanmax(d)))
    idx = np.argsort(-np.nan_to_num(d, nan=1e30))[:10]
    print("worst", idx.tolist(), d[idx].tolist())
