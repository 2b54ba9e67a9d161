"""Test infrastructure: how far apart chaotic crack runs of the reference
algorithm end when their initial state differs at rounding level.

Runs the oracle (the CPU restatement of the reference, oracle.py) on a crack
golden's case K times, the initial u of run k > 0 offset per particle by 1e-22 m x N(0, 1) (seed k), through
the reference's run loop to the golden's end time, and prints the spread of
the metrics tests/test_gpu_output.py holds the device run to (damaged count,
centroid and crack-tip column of the damaged set against the golden's, u,
energies).  Used to set CRACK3D_TOL; the 2D tolerances (CRACK_TOL) came from
the same procedure.

    python oracle/crack_ensemble.py crack_kalthoff3d [K]
"""
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _crack(X, s, tip, dp):
    damaged = np.flatnonzero((s < 0.5) & (X[:, 0] > tip[0] + 2.0 * dp))
    pts = X[damaged][:, [0, 2]]
    _, _, vt = np.linalg.svd(pts - pts.mean(axis=0), full_matrices=False)
    return damaged, math.degrees(math.atan2(abs(vt[0][1]), abs(vt[0][0])))


def one(args):
    name, k = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from conftest import golden, run_case
    from oracle import oracle as O
    G = golden(name)
    cfg = run_case(G)
    b = cfg.bodies[0]
    b.adjacency = O.build_adjacency(b.state.X, b.state.V0, b.h, b.dim, int(cfg.kernel),
                                    nbsrange=b.nbsrange, dp_body=b.dp_body, notches=b.notches)
    if k:   # a per-particle offset (a uniform one is a rigid translation: no strain)
        b.state.u[:, 0] += 1e-22 * np.random.default_rng(k).standard_normal(b.state.u.shape[0])
    sim = O.OracleSimulation(cfg)
    t_end = float(G["end.t"][0])
    sim.run(time_max=t_end, time_out=t_end)
    st = b.state
    quad = b.notches[0].points
    tip = quad[int(np.argmax(quad[:, 0]))]
    dam, ang = _crack(st.X, st.s, tip, b.dp_body)
    ref = G["damaged"]
    dp = b.dp_body
    cen = np.linalg.norm(st.X[dam][:, [0, 2]].mean(axis=0) - st.X[ref][:, [0, 2]].mean(axis=0)) / dp
    tipd = abs(st.X[dam, 0].max() - st.X[ref, 0].max()) / dp
    uerr = float(np.abs(st.u - G["end.u"]).max() / np.abs(G["end.u"]).max())
    en = None
    ref_src = "/root/reference/pkg/src"          # the reference's own energies, when present
    if os.path.isdir(ref_src):
        sys.path.insert(0, ref_src)
        from solidsph import output as rout
        from solidsph.backends import reference as rbe
        e = np.array(rout.compute_energies(b, rbe))
        en = (e[:3] - G["end.energies"][:3]) / np.abs(G["end.energies"][:3])
    return k, dam.size, ang, cen, tipd, uerr, en


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "crack_kalthoff3d"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    with ProcessPoolExecutor(max_workers=min(K, os.cpu_count() or 1)) as ex:
        for k, n, ang, cen, tipd, uerr, en in ex.map(one, [(name, k) for k in range(K)]):
            print(f"run {k}: damaged {n}, kink {ang:.2f} deg, centroid {cen:.2f} dp, "
                  f"tip {tipd:.2f} dp, u {uerr:.2e}, energies (strain, kinetic, fracture) "
                  f"{'' if en is None else np.array2string(en, precision=4)}", flush=True)


if __name__ == "__main__":
    main()
