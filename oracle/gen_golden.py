"""Generate golden vectors by running the REFERENCE itself (numpy backend).

Run in the build container only (needs /root/reference):

    python oracle/gen_golden.py            # writes tests/golden/*.npz

Every fixture is produced through the reference's public API:
kernel_geom.build_adjacency / build_pairs, backends.reference.*,
caseio.load_case / parse_case + build_case, stepper.Simulation, and
expr.parse + expr.eval_field.  Inputs are seeded (numpy default_rng, whose
streams are stable across numpy versions) or are the reference's own case
files with scale overrides.  The fixtures pin both the oracle
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_*.py) on boxes
where the reference is absent.
"""

from __future__ import annotations

import os
import sys

os.environ["SOLIDSPH_BACKEND"] = "numpy"
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from solidsph import caseio, kernel_geom as kg, stepper  # noqa: E402
from solidsph import expr as rex  # noqa: E402
from solidsph.backends import reference as ref  # noqa: E402
from solidsph.core import KernelKind, Quad  # noqa: E402
from conftest import lattice_2d, lattice_3d  # noqa: E402

from paper_2602_15149_b200.cases import case_to_dict  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
CASES = os.path.join(REF, "cases")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{path}: {os.path.getsize(path) / 1e3:.1f} kB")


# ---------------------------------------------------------------------------
def gen_adjacency():
    out = {}

    def add(tag, pos, dp, dim, kind, nbsrange=None, notches=(), correction=True,
            h=None, full=True):
        V0 = np.full(pos.shape[0], dp ** dim)
        h = kg.smoothing_length(dp, 1.0, dim) if h is None else h
        adj = kg.build_adjacency(pos, V0, h, dim, kind, nbsrange=nbsrange, dp_body=dp,
                                 notches=[Quad(points=q) for q in notches],
                                 correction=correction)
        out[f"{tag}.X"] = pos
        out[f"{tag}.V0"] = V0
        out[f"{tag}.params"] = np.array([dp, dim, int(kind), -1 if nbsrange is None else nbsrange,
                                         int(correction), h], dtype=np.float64)
        out[f"{tag}.notches"] = np.asarray(notches, dtype=np.float64).reshape(-1, 4, 3)
        out[f"{tag}.indptr"] = adj.indptr
        out[f"{tag}.indices"] = adj.indices
        out[f"{tag}.fallbacks"] = np.array([adj.correction_fallbacks])
        if full:
            out[f"{tag}.grad0"] = adj.grad0
            out[f"{tag}.grad0r"] = adj.grad0r
            out[f"{tag}.r0norm"] = adj.r0norm
            out[f"{tag}.w0"] = adj.w0

    W, C = KernelKind.WENDLAND, KernelKind.CUBIC_SPLINE
    add("l2w", lattice_2d(12, 8, 1e-3), 1e-3, 2, W)
    add("l2c", lattice_2d(12, 8, 1e-3), 1e-3, 2, C)
    add("l3w", lattice_3d(7, 6, 5, 1e-3), 1e-3, 3, W)
    add("l3c", lattice_3d(6, 5, 4, 1.0), 1.0, 3, C)
    add("l3n", lattice_3d(7, 6, 5, 1e-3), 1e-3, 3, W, nbsrange=1)
    add("l2n", lattice_2d(12, 8, 1e-3), 1e-3, 2, W, nbsrange=1)
    add("l2n2", lattice_2d(9, 7, 1e-3), 1e-3, 2, W, nbsrange=2)
    add("nocorr", lattice_2d(12, 8, 1e-3), 1e-3, 2, W, correction=False)
    add("two", np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]]), 1.0, 3, W, h=1.0)
    # tie-heavy 3D lattice at dp=1e-3 (16% of candidate pairs sit on 2h)
    add("tie3", lattice_3d(12, 10, 9, 1e-3), 1e-3, 3, W, full=False)
    add("tie2", lattice_2d(40, 30, 1e-3), 1e-3, 2, W, full=False)
    # notches: between rows (full), partial extent, 3D through-thickness
    zc = 3.0
    add("notch_rows", lattice_2d(6, 6, 1.0), 1.0, 2, W,
        notches=[[[-1, -1, zc], [7, -1, zc], [7, 1, zc], [-1, 1, zc]]])
    add("notch_part", lattice_2d(8, 6, 1.0), 1.0, 2, W,
        notches=[[[-1, -1, zc], [3.2, -1, zc], [3.2, 1, zc], [-1, 1, zc]]])
    add("notch3d", lattice_3d(10, 4, 10, 1e-3), 1e-3, 3, W, nbsrange=1,
        notches=[[[0, -1e-3, 4.6e-3], [5e-3, -1e-3, 4.6e-3], [5e-3, 5e-3, 4.6e-3], [0, 5e-3, 4.6e-3]]])
    add("notch3dr", lattice_3d(8, 4, 8, 1e-3), 1e-3, 3, W,
        notches=[[[0, -1e-3, 4.0e-3], [5e-3, -1e-3, 4.0e-3], [5e-3, 5e-3, 4.0e-3], [0, 5e-3, 4.0e-3]]])
    # random points (test_kernel_geom.py:98-118 input)
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 1, size=(300, 3))
    pos[:, 1] = 0.0
    rows, cols = kg.build_pairs(pos, 0.08)
    out["rnd.X"] = pos
    out["rnd.rows"] = rows
    out["rnd.cols"] = cols
    rng = np.random.default_rng(11)
    pos = rng.uniform(0, 1, size=(400, 3))
    rows, cols = kg.build_pairs(pos, 0.1, nbsrange=1, dp_body=0.07)
    out["rndn.X"] = pos
    out["rndn.rows"] = rows
    out["rndn.cols"] = cols
    save("adjacency", **out)


# ---------------------------------------------------------------------------
def _setup(dim, n1=10, n2=8, dp=1e-3, seed=0):
    # mirrors test_backends.py:15-25
    pos = lattice_2d(n1, n2, dp) if dim == 2 else lattice_3d(n1, n2, 5, dp)
    V0 = np.full(pos.shape[0], dp ** dim)
    h = kg.smoothing_length(dp, 1.0, dim)
    adj = kg.build_adjacency(pos, V0, h, dim, KernelKind.WENDLAND)
    rng = np.random.default_rng(seed)
    n = pos.shape[0]
    u = rng.normal(scale=2e-5, size=(n, 3))
    v = rng.normal(scale=1.0, size=(n, 3))
    if dim == 2:
        u[:, 1] = 0.0
        v[:, 1] = 0.0
    return pos, V0, h, adj, u, v


def gen_kernels():
    out = {}
    for dim in (2, 3):
        pos, V0, h, adj, u, v = _setup(dim)
        n = pos.shape[0]
        s = np.random.default_rng(1).uniform(0.0, 1.0, n)
        F = np.zeros((n, 3, 3))
        ref.deformation_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0, u, V0, s, 0.1,
                                 True, F)
        f = np.ascontiguousarray(pos[:, 0] ** 2 + 0.3 * pos[:, 2])
        lap = np.zeros(n)
        ref.sph_laplacian(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.r0, adj.r0norm, V0,
                          f, lap)
        g = np.zeros((n, 3))
        ref.sph_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0, V0, f, g)
        p = f"d{dim}."
        out.update({p + "X": pos, p + "u": u, p + "v": v, p + "s": s, p + "F": F, p + "f": f,
                    p + "lap": lap, p + "grad": g})
        rng = np.random.default_rng(2)
        Fm = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
        Fm += rng.normal(scale=0.01, size=(n, 3, 3))
        S = rng.normal(scale=1e5, size=(n, 3, 3))
        S = 0.5 * (S + np.swapaxes(S, 1, 2))
        P = np.matmul(Fm, S)
        out[p + "Fm"] = Fm
        out[p + "P"] = P
        for tag, (b1, b2) in (("mom0", (0.0, 0.0)), ("mom1", (0.2, 0.1))):
            a = np.zeros((n, 3))
            nb = ref.momentum(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.grad0r, adj.r0,
                              adj.r0norm, P, 1000.0 * V0, 1000.0, v, h, 64.8, b1, b2, Fm, a)
            out[p + tag] = a
            out[p + tag + ".nbad"] = np.array([nb])
    # constitutive batches (test_backends.py:82-149 inputs)
    rng = np.random.default_rng(3)
    n = 300
    F = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    F += rng.normal(scale=0.08, size=(n, 3, 3))
    s = rng.uniform(0, 1, n)
    out["svk.F"], out["svk.s"] = F, s
    for fr in (0, 1):
        S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
        ref.svk_batch(F, 2.7733e6, 0.715e6, s, bool(fr), S, psi, psip)
        out[f"svk{fr}.S"], out[f"svk{fr}.psi"], out[f"svk{fr}.psip"] = S, psi, psip
    rng = np.random.default_rng(4)
    F = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    F += rng.normal(scale=0.1, size=(n, 3, 3))
    F[0] *= 1e-3
    s = rng.uniform(0, 1, n)
    out["nh.F"], out["nh.s"] = F, s
    for fr in (0, 1):
        S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
        nb = ref.nh_batch(F, 3.25e6, 0.715e6, s, bool(fr), S, psi, psip)
        out[f"nh{fr}.S"], out[f"nh{fr}.psi"], out[f"nh{fr}.psip"] = S, psi, psip
        out[f"nh{fr}.nbad"] = np.array([nb])
    rng = np.random.default_rng(5)
    n = 400
    F = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    F += rng.normal(scale=0.015, size=(n, 3, 3))
    F[7] *= 1e-3   # a degenerate lane
    Cp = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    ep = np.zeros(n)
    S, psi, dwp = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
    nb, fb = ref.j2_batch(F, Cp, ep, 43.333e9, 130e9, 4e8, 1e8, S, psi, dwp)
    out.update({"j2.F": F, "j2.Cp": Cp, "j2.ep": ep, "j2.S": S, "j2.psi": psi, "j2.dwp": dwp,
                "j2.ret": np.array([nb, fb])})
    # second J2 call from the updated state (history path)
    F2 = F + rng.normal(scale=0.004, size=(n, 3, 3))
    Cp2, ep2 = Cp.copy(), ep.copy()
    S, psi, dwp = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
    nb, fb = ref.j2_batch(F2, Cp2, ep2, 43.333e9, 130e9, 4e8, 1e8, S, psi, dwp)
    out.update({"j2b.F": F2, "j2b.Cp": Cp2, "j2b.ep": ep2, "j2b.S": S, "j2b.psi": psi,
                "j2b.dwp": dwp, "j2b.ret": np.array([nb, fb])})
    # contact (test_backends.py:152-174)
    rng = np.random.default_rng(6)
    na, nbb = 40, 50
    xa = rng.uniform(0, 0.05, (na, 3))
    xb = rng.uniform(0.01, 0.06, (nbb, 3))
    va = rng.normal(scale=10, size=(na, 3))
    vb = rng.normal(scale=10, size=(nbb, 3))
    pairs = np.array([(i, j) for i in range(na) for j in range(nbb)], dtype=np.int64)
    aa, ab = np.zeros((na, 3)), np.zeros((nbb, 3))
    w = ref.contact_pair_accumulate(xa, va, np.full(na, 0.3), xb, vb, np.full(nbb, 0.4), pairs,
                                    0.012, 1e7, 30.0, 0.3, aa, ab)
    out.update({"ct.xa": xa, "ct.xb": xb, "ct.va": va, "ct.vb": vb, "ct.aa": aa, "ct.ab": ab,
                "ct.warn": np.array([w])})
    # symmetric eigen problems for the Jacobi solver
    rng = np.random.default_rng(7)
    A = rng.normal(size=(200, 3, 3))
    A = 0.5 * (A + np.swapaxes(A, 1, 2))
    out["eig.A"] = A
    out["eig.w"] = np.linalg.eigvalsh(A)
    save("kernels", **out)


# ---------------------------------------------------------------------------
def _outputs(sim):
    """The reference's own output rows (output.py:25-71) at this step."""
    from solidsph import output as rout
    d = {}
    for bi, b in enumerate(sim.bodies):
        d[f"b{bi}.energies"] = np.array(rout.compute_energies(b, ref))
        for k, idx in enumerate(b.measure_sets):
            d[f"b{bi}.measure{k}"] = np.array(rout.measure_row(b, idx, sim.t)[1:], dtype=np.float64)
    return d


def _state(sim, full=True):
    d = {}
    keys = ("u", "v", "a", "s", "sdot", "sddot", "Hhist", "epbar", "psi_e", "F", "S", "Cp")
    for bi, b in enumerate(sim.bodies):
        st = b.state
        for k in keys if full else ("u", "v", "a", "s", "sdot"):
            d[f"b{bi}.{k}"] = getattr(st, k).copy()
        d[f"b{bi}.plastic_work"] = np.array([b.plastic_work])
        d[f"b{bi}.degenerate"] = np.array([b.degenerate_warnings])
    d["t"] = np.array([sim.t])
    return d


def _kalthoff3d_raw():
    raw = caseio.parse_case(os.path.join(CASES, "kalthoff2d.xml"))
    raw.dim = 3
    for q in raw.bodies[0].notches:
        q.points[2, 1] = 11e-3
        q.points[3, 1] = 11e-3
    return raw


def _perturb(cfg, seed):
    """Seeded non-trivial initial state (step-1 parity on a
    u=0 state is vacuous).  Mirrors backend_bench.py:29-34 scaling."""
    rng = np.random.default_rng(seed)
    for b in cfg.bodies:
        st = b.state
        n = st.X.shape[0]
        st.u[:] = rng.normal(scale=2e-5 * b.dp_body / 1e-3, size=(n, 3))
        st.v[:] = rng.normal(scale=1.0, size=(n, 3))
        if b.fracture:
            st.s[:] = rng.uniform(0.3, 1.0, n)
        if b.dim == 2:
            st.u[:, 1] = 0.0
            st.v[:, 1] = 0.0
    return cfg


def gen_runs():
    L = caseio.load_case
    C = lambda f: os.path.join(CASES, f)  # noqa: E731
    runs = [
        # tag, config builder, perturbation seed (None = as loaded), steps, checkpoints
        ("kalthoff2d", lambda: L(C("kalthoff2d.xml"), dp_scale=2, mapfac=1), None, 40, (1, 2, 10, 40)),
        ("kalthoff2d_p", lambda: L(C("kalthoff2d.xml"), dp_scale=2, mapfac=1), 31, 20, (1, 2, 20)),
        ("kalthoff2d_sym", lambda: _with_algo(L(C("kalthoff2d.xml"), dp_scale=2, mapfac=1), 2),
         32, 20, (1, 2, 20)),
        ("beam2d", lambda: L(C("beam2d.xml"), dp_scale=2, mapfac=2), None, 30, (1, 2, 30)),
        ("taylor3d", lambda: L(C("taylor3d.xml"), dp_scale=4), 33, 20, (1, 2, 20)),
        ("column3d", lambda: L(C("column3d.xml"), dp_scale=2, mapfac=1), 34, 20, (1, 2, 20)),
        ("branch2d", lambda: L(C("branch2d.xml"), dp_scale=8, mapfac=1), 35, 20, (1, 2, 20)),
        ("kalthoff3d", lambda: caseio.build_case(_kalthoff3d_raw(), dp_scale=6, mapfac=2), 36,
         10, (1, 2, 10)),
        ("twisting3d", lambda: L(C("twisting3d.xml"), dp_scale=4), 37, 10, (1, 10)),
        # two J2 bodies, penalty contact from step 1 (_touching)
        ("flyer2d", lambda: _touching(L(C("flyer2d.xml"), dp_scale=2)), None, 30, (1, 2, 30)),
        # the paper's benchmark case: 3D SVK + phase field on the radial stencil,
        # notch, restrictphi with compound `and` expressions (fourpoint3d.xml:49-59)
        ("fourpoint3d", lambda: L(C("fourpoint3d.xml"), dp_scale=6), 38, 10, (1, 2, 10)),
        # 3D SVK cantilever plate, artificial viscosity, cosh/sinh IC expression
        ("plate3d", lambda: L(C("plate3d.xml"), dp_scale=6), 39, 10, (1, 2, 10)),
    ]
    only = os.environ.get("GOLDEN_RUNS")
    if only:
        runs = [r for r in runs if r[0] in only.split(",")]
    for tag, make, seed, steps, checks in runs:
        cfg = make()
        if seed is not None:
            _perturb(cfg, seed)
        out = dict(case_to_dict(cfg))
        for bi, b in enumerate(cfg.bodies):
            out[f"adj{bi}.indptr"] = b.adjacency.indptr
            out[f"adj{bi}.indices"] = b.adjacency.indices
            out[f"adj{bi}.fallbacks"] = np.array([b.adjacency.correction_fallbacks])
            for k in ("u", "v", "s"):
                out[f"init.b{bi}.{k}"] = getattr(b.state, k).copy()
        sim = stepper.Simulation(cfg)
        sim.initialize()
        for k, v in _state(sim).items():
            out[f"s0.{k}"] = v
        dts = []
        for step in range(1, steps + 1):
            dt = sim.pick_dt()
            dts.append(dt)
            sim.step(dt)
            if step in checks:
                full = step in (checks[0], checks[-1])
                for k, v in _state(sim, full).items():
                    out[f"s{step}.{k}"] = v
                for k, v in _outputs(sim).items():
                    out[f"s{step}.{k}"] = v
        out["dts"] = np.array(dts)
        out["checkpoints"] = np.array(checks)
        save(f"run_{tag}", **out)


CRACK_T = 2.0e-4   # past the case's TimeMax (1.2e-4): the crack is well grown


def gen_crack():
    """2D Kalthoff-Winkler run to t = 2e-4 s (adaptive steps at dp_scale=2,
    the reference's run loop: the crack leaves the notch tip), with the reference's own
    crack metric (bench.py:237-260): the kink angle of the s < 0.5 set ahead
    of the tip.  The device run must reproduce the crack path."""
    import math
    cfg = caseio.load_case(os.path.join(CASES, "kalthoff2d.xml"), dp_scale=2, mapfac=1)
    out = dict(case_to_dict(cfg))
    b = cfg.bodies[0]
    out["adj0.indptr"] = b.adjacency.indptr
    out["adj0.indices"] = b.adjacency.indices
    sim = stepper.Simulation(cfg)
    dts = []
    orig_step = sim.step

    def step(dt):
        dts.append(dt)
        orig_step(dt)

    sim.step = step
    # the reference's own run loop (stepper.py:237-263): adaptive dt clipped
    # to the output grid, one output at TimeMax
    sim.run(time_max=CRACK_T, time_out=CRACK_T)
    st = b.state
    quad = b.notches[0].points
    tip = quad[int(np.argmax(quad[:, 0]))]
    damaged = np.flatnonzero((st.s < 0.5) & (st.X[:, 0] > tip[0] + 2.0 * b.dp_body))
    pts = st.X[damaged][:, [0, 2]]
    _, _, vt = np.linalg.svd(pts - pts.mean(axis=0), full_matrices=False)
    angle = math.degrees(math.atan2(abs(vt[0][1]), abs(vt[0][0])))
    print(f"crack: {len(dts)} steps, t={sim.t:.6g}, {damaged.size} damaged ahead of the tip, "
          f"kink {angle:.2f} deg")
    for k in ("u", "v", "s", "sdot", "Hhist"):
        out[f"end.{k}"] = getattr(st, k).copy()
    out["end.t"] = np.array([sim.t])
    out["end.energies"] = _outputs(sim)["b0.energies"]
    out["dts"] = np.array(dts)
    out["kink_angle_deg"] = np.array([angle])
    out["damaged"] = damaged
    save("crack_kalthoff2d", **out)


def gen_crack3d():
    """3D Kalthoff-Winkler (C4's body: the 2D case promoted to 3D with the
    notch through the thickness, dp_scale=3, 3,267 particles) run to t = 2e-4 s
    through the reference's run loop: the crack leaves the notch tip at about
    75 deg in the x-z plane.  Same metric as gen_crack (bench.py:237-260)."""
    import math
    cfg = caseio.build_case(_kalthoff3d_raw(), dp_scale=3, mapfac=1)
    out = dict(case_to_dict(cfg))
    b = cfg.bodies[0]
    out["adj0.indptr"] = b.adjacency.indptr
    out["adj0.indices"] = b.adjacency.indices
    sim = stepper.Simulation(cfg)
    dts = []
    orig_step = sim.step

    def step(dt):
        dts.append(dt)
        orig_step(dt)

    sim.step = step
    sim.run(time_max=CRACK_T, time_out=CRACK_T)
    st = b.state
    quad = b.notches[0].points
    tip = quad[int(np.argmax(quad[:, 0]))]
    damaged = np.flatnonzero((st.s < 0.5) & (st.X[:, 0] > tip[0] + 2.0 * b.dp_body))
    pts = st.X[damaged][:, [0, 2]]
    _, _, vt = np.linalg.svd(pts - pts.mean(axis=0), full_matrices=False)
    angle = math.degrees(math.atan2(abs(vt[0][1]), abs(vt[0][0])))
    print(f"crack3d: {len(dts)} steps, t={sim.t:.6g}, {damaged.size} damaged ahead of the tip, "
          f"kink {angle:.2f} deg")
    for k in ("u", "v", "s", "sdot", "Hhist"):
        out[f"end.{k}"] = getattr(st, k).copy()
    out["end.t"] = np.array([sim.t])
    out["end.energies"] = _outputs(sim)["b0.energies"]
    out["dts"] = np.array(dts)
    out["kink_angle_deg"] = np.array([angle])
    out["damaged"] = damaged
    save("crack_kalthoff3d", **out)


def _touching(cfg):
    """flyer2d with the upper body displaced (u, a rigid shift) so its lowest
    layer sits 0.6 dp_contact above the plate: contact acts from step 1."""
    up, low = cfg.bodies[0], cfg.bodies[1]
    if up.state.X[:, 2].min() < low.state.X[:, 2].min():
        up, low = low, up
    dpc = 0.5 * (up.dp_body + low.dp_body)
    shift = (up.state.X[:, 2].min() - low.state.X[:, 2].max()) - 0.6 * dpc
    up.state.u[:, 2] = -shift
    return cfg


def _with_algo(cfg, algo):
    from solidsph.core import StepAlgorithm
    cfg.step_algorithm = StepAlgorithm(algo)
    return cfg


LONG_STEPS = 2000


def gen_long():
    """beam2d (SVK, radial, IC expression) for 2,000 adaptive FP64 steps
    through the reference's step loop (<= 1e-10 after
    2,000 steps on a non-chaotic case).  End state only."""
    cfg = caseio.load_case(os.path.join(CASES, "beam2d.xml"), dp_scale=2, mapfac=2)
    out = dict(case_to_dict(cfg))
    b = cfg.bodies[0]
    out["adj0.indptr"] = b.adjacency.indptr
    out["adj0.indices"] = b.adjacency.indices
    sim = stepper.Simulation(cfg)
    sim.initialize()
    dts = []
    for _ in range(LONG_STEPS):
        dt = sim.pick_dt()
        dts.append(dt)
        sim.step(dt)
    for k, v in _state(sim).items():
        out[f"end.{k}"] = v
    out["end.energies"] = _outputs(sim)["b0.energies"]
    out["dts"] = np.array(dts)
    save("long_beam2d", **out)


def gen_branch():
    """Dynamic crack branching (branch2d) with the reference's own benchmark
    (bench.py:194-235 bench_branch; acceptance criterion 3 runs it at
    scale 4, test_acceptance.py:149-159): initiation time near the notch
    tip, the branched flag, FE monotone after initiation, SE decreasing, and
    the final damage field."""
    from solidsph import bench as rbench
    cfg = rbench._load("branch2d", 4.0, None, None, None, None, False)
    out = dict(case_to_dict(cfg))
    b = cfg.bodies[0]
    out["adj0.indptr"] = b.adjacency.indptr
    out["adj0.indices"] = b.adjacency.indices
    rep = rbench.bench_branch("branch2d", cfg, None, None)
    rows = {m: v for m, v, _, _ in rep.rows}
    print("branch2d:", rows)
    ser = rep.extras["series"]
    out["series.t"] = np.array(ser["t"])
    out["series.se"] = np.array(ser["se"])
    out["series.fe"] = np.array(ser["fe"])
    for m in ("initiation_time_s", "branched", "fe_monotone", "se_decreases"):
        out[f"metric.{m}"] = np.array([rows[m]])
    out["final_s"] = rep.extras["final_s"]
    out["end.t"] = np.array([ser["t"][-1]])
    save("branch_branch2d", **out)


# ---------------------------------------------------------------------------
# error paths: the reference's exceptions raised inside the step
# ---------------------------------------------------------------------------

def _err_case(tag, make, seed, edits=(), steps=None, run=None, dt_override=None,
              extra_exprs=(), extra_bcs=(), restrict=None, material=None, cp=None):
    """Run one error scenario through the reference (numpy backend) and
    record the case, the edits applied after initialize() and the exception.

    edits: (field, particle, axis, value) applied to body.state after
    initialize(); steps: number of step(dt) calls (dt from pick_dt); run:
    (time_max, time_out) for Simulation.run; extra_exprs: (id, src, locals);
    extra_bcs: BoundaryCondition kwargs; restrict: restrictphi expression id;
    material: MaterialParams overrides; cp: (particle, 3x3) plastic metric."""
    from solidsph import expr as rex2
    from solidsph.core import BoundaryCondition
    cfg = make()
    if dt_override is not None:
        cfg.dt_override = dt_override
    if seed is not None:
        _perturb(cfg, seed)
    b = cfg.bodies[0]
    for eid, src, loc in extra_exprs:
        cfg.expressions[eid] = rex2.parse(src, loc)
    for kw in extra_bcs:
        b.bcs.append(BoundaryCondition(**kw))
    if restrict is not None:
        b.restrictphi_expr = restrict
    for k, v in (material or {}).items():
        setattr(b.material, k, v)
    if cp is not None:
        b.state.Cp[cp[0]] = np.asarray(cp[1])
    out = {f"{tag}.{k}": v for k, v in case_to_dict(cfg).items()}
    for k in ("u", "v", "s"):
        out[f"{tag}.init.{k}"] = getattr(b.state, k).copy()
    if cp is not None:
        out[f"{tag}.init.Cp"] = b.state.Cp.copy()
    out[f"{tag}.edits"] = np.array([(float(i), float(a), float(v)) for _, i, a, v in edits]
                                   ).reshape(-1, 3)
    out[f"{tag}.edit_fields"] = np.frombuffer(",".join(f for f, _, _, _ in edits).encode(),
                                              dtype=np.uint8)
    sim = stepper.Simulation(cfg)
    exc = None
    nsteps = 0
    try:
        sim.initialize()
        for f, i, a, v in edits:
            getattr(b.state, f)[int(i), int(a)] = v
        if run is not None:
            sim.run(time_max=run[0], time_out=run[1])
        else:
            for _ in range(steps):
                sim.step(sim.pick_dt())
                nsteps += 1
    except Exception as e:  # the point: record what the reference raises
        exc = e
    assert exc is not None, f"{tag}: the reference raised nothing"
    print(f"{tag}: {type(exc).__name__}: {exc} (after {nsteps} steps, t={sim.t!r})")
    out[f"{tag}.driver"] = np.array([-1 if steps is None else steps,
                                     -1.0 if run is None else run[0],
                                     -1.0 if run is None else run[1]])
    out[f"{tag}.exc"] = np.frombuffer(f"{type(exc).__name__}\n{exc}".encode(), dtype=np.uint8)
    out[f"{tag}.steps_done"] = np.array([nsteps])
    out[f"{tag}.t"] = np.array([sim.t])
    return out


def gen_errors():
    L = caseio.load_case
    C = lambda f: os.path.join(CASES, f)  # noqa: E731
    beam = lambda: L(C("beam2d.xml"), dp_scale=2, mapfac=2)  # noqa: E731
    kal = lambda: L(C("kalthoff2d.xml"), dp_scale=2, mapfac=1)  # noqa: E731
    out = {}
    # stepper.py:96-100 -- NaN velocity of one particle: its neighbours'
    # accelerations go non-finite in the next force evaluation
    out.update(_err_case("acc", beam, 41, edits=[("v", 1234, 0, float("nan"))], steps=3))
    # stepper.py:203-209 -- a velocity BC drives one particle's v to inf at the
    # end of step 64; the state check at the 64th commit raises
    dt = 2.0e-6
    out.update(_err_case(
        "state64", beam, 42, steps=70, dt_override=dt,
        extra_exprs=[(99, f"if(t>{63.5 * dt!r},cosh(1000),skip)", "")],
        extra_bcs=[dict(kind="vel", expr=(99, None, None), target=np.array([777]))]))
    # stepper.py:254-255 -- an overflowing |v|^2 (no viscosity, so the
    # acceleration stays finite) makes the adaptive dt zero inside run()
    out.update(_err_case("dtcollapse", beam, 43, edits=[("v", 321, 0, 1e200)],
                         run=(1e-3, 1e-4), material=dict(beta1=0.0, beta2=0.0)))
    # expr.py:513-515 -- a velocity BC expression dividing by zero
    out.update(_err_case(
        "div0", beam, 44, steps=2,
        extra_exprs=[(98, "if(x0>0.05,1/(t-t),skip)", "")],
        extra_bcs=[dict(kind="vel", expr=(None, None, 98))]))
    # fracture.py:59-63 -- a time-dependent restrictphi leaving [0, 1]
    out.update(_err_case(
        "restrict", kal, 45, steps=5,
        extra_exprs=[(97, "if(t>1.0e-12,1.5,skip)", "")], restrict=97))
    # constitutive.py:191-194 -- a plastic metric whose radial return leaves
    # the SPD cone (one negative eigen-direction): the first bad particle
    T = lambda: L(C("taylor3d.xml"), dp_scale=4)  # noqa: E731
    out.update(_err_case("nonspd", T, None, steps=2,
                         cp=(517, np.diag([1e-4, 1e-4, 1e8]))))
    # fast.py:254-256 -- SVK spectral split: Jacobi fails to converge on a
    # matrix mixing NaN and finite entries (numba backend, plugin level)
    from solidsph.backends import fast
    rng = np.random.default_rng(46)
    n = 64
    F = np.broadcast_to(np.eye(3), (n, 3, 3)).copy() + rng.normal(scale=0.05, size=(n, 3, 3))
    F[5, 0, 1] = np.nan
    F[40, 2, 1] = np.nan
    S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
    s = rng.uniform(0.2, 1.0, n)
    nc = fast.svk_batch(F, 2.7733e6, 0.715e6, s, True, S, psi, psip)
    print("noconv:", nc)
    out.update({"noconv.F": F, "noconv.s": s, "noconv.n": np.array([nc])})
    save("errors", **out)


# ---------------------------------------------------------------------------
EXPRS = [
    ("if(t>ramt,maxv,t/ramt*maxv)", "maxv=16.5; ramt=1.0e-6"),
    ("if(x0<=0.0,0.0,skip)", ""),
    ("if(x0>xtip,if(t<=Tmax,t/Tmax,1.0)*Fmax,skip)", "Fmax=-1.75e9; Tmax=1.0; xtip=0.099;"),
    ("if(z<1.0e-12,0.0,if(t<=0.0,Vinit,skip))", "Vinit=-227;"),
    ("sin(x)*cos(y0) + tan(0.3*z) - cot(1+ux) + sinh(uy) - cosh(0.1*uz)", ""),
    ("tanh(x0*10) + coth(2+y) + sqrt(abs(z)) + log(2+x) + ln(3+t)", ""),
    ("pow(2, x0) + 2^3^0.5 - -x*-y + (x0 < 0.5 and y0 >= 0.2) + (z0 == 0 or t != 1)", ""),
    ("if(x0 < 0.3, if(y0 < 0.5, skip, x0*dx), -dt*3 + t)", ""),
    ("-2^2 + 3*-x0/(1+y0) - (z0 <= 0.5) * (x > 0.1)", ""),
    ("x0 - 2*(x0 > 0.5)*x0 + if(abs(y0-0.5) < 0.25, 1, 0)", ""),
]


def gen_expr():
    rng = np.random.default_rng(21)
    n = 257
    ctx = {"x0": rng.uniform(0, 1, n), "y0": rng.uniform(0, 1, n), "z0": rng.uniform(0, 1, n),
           "ux": rng.normal(scale=1e-3, size=n), "uy": rng.normal(scale=1e-3, size=n),
           "uz": rng.normal(scale=1e-3, size=n), "t": 2.5e-6, "dt": 1e-7, "dx": 0.002}
    ctx["x"] = ctx["x0"] + ctx["ux"]
    ctx["y"] = ctx["y0"] + ctx["uy"]
    ctx["z"] = ctx["z0"] + ctx["uz"]
    out = {k: np.asarray(v) for k, v in ctx.items()}
    for k, (src, loc) in enumerate(EXPRS):
        ast = rex.parse(src, loc)
        vals, skip = rex.eval_field(ast, ctx, n)
        out[f"e{k}.vals"] = vals
        out[f"e{k}.skip"] = skip
        out[f"e{k}.pretty"] = np.frombuffer(rex.pretty(ast).encode(), dtype=np.uint8)
    out["sources"] = np.frombuffer("\n".join(f"{s}\t{l}" for s, l in EXPRS).encode(),
                                   dtype=np.uint8)
    save("expr", **out)


def gen_targets():
    """BC target sets resolved by the reference's loader for the C1-C5
    geometries at reduced size (checks cases.make_case)."""
    out = {}
    specs = [("kalthoff2d", "kalthoff2d.xml", dict(dp_scale=2, mapfac=1)),
             ("branch2d", "branch2d.xml", dict(dp_scale=8, mapfac=1)),
             ("beam2d", "beam2d.xml", dict(dp_scale=2, mapfac=2)),
             ("taylor3d", "taylor3d.xml", dict(dp_scale=4)),
             ("column3d", "column3d.xml", dict(dp_scale=2, mapfac=1))]
    for tag, f, kw in specs:
        cfg = caseio.load_case(os.path.join(CASES, f), **kw)
        b = cfg.bodies[0]
        out[f"{tag}.X"] = b.state.X
        out[f"{tag}.kw"] = np.array([kw.get("dp_scale", 1.0), kw.get("mapfac", 0)])
        for ci, bc in enumerate(b.bcs):
            if bc.target is not None:
                out[f"{tag}.bc{ci}"] = bc.target
    cfg = caseio.build_case(_kalthoff3d_raw(), dp_scale=6, mapfac=2)
    out["kalthoff3d.X"] = cfg.bodies[0].state.X
    out["kalthoff3d.kw"] = np.array([6.0, 2])
    for ci, bc in enumerate(cfg.bodies[0].bcs):
        if bc.target is not None:
            out[f"kalthoff3d.bc{ci}"] = bc.target
    save("targets", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["adjacency", "kernels", "runs", "expr", "targets", "crack", "crack3d",
                             "long", "branch", "errors"]
    for w in which:
        globals()[f"gen_{w}"]()
