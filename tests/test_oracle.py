"""Pin the CPU oracle to golden vectors produced by the reference itself
(oracle/gen_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden, relerr, run_case
from paper_2602_15149_b200 import cases, expr as ex


@pytest.fixture(scope="module")
def G():
    return golden("adjacency")


ADJ_TAGS = ["l2w", "l2c", "l3w", "l3c", "l3n", "l2n", "l2n2", "nocorr", "two", "tie3", "tie2",
            "notch_rows", "notch_part", "notch3d", "notch3dr"]


def _adj_args(G, tag):
    dp, dim, kind, nbs, corr, h = G[f"{tag}.params"]
    nbs = None if nbs < 0 else int(nbs)
    return dict(positions=G[f"{tag}.X"], V0=G[f"{tag}.V0"], h=h, dim=int(dim), kind=int(kind),
                nbsrange=nbs, dp_body=dp, notches=list(G[f"{tag}.notches"]),
                correction=bool(corr))


@pytest.mark.parametrize("tag", ADJ_TAGS)
def test_oracle_adjacency_matches_reference(G, tag, oracle_mod):
    adj = oracle_mod.build_adjacency(**_adj_args(G, tag))
    assert np.array_equal(adj.indptr, G[f"{tag}.indptr"])
    assert np.array_equal(adj.indices, G[f"{tag}.indices"])
    assert adj.correction_fallbacks == int(G[f"{tag}.fallbacks"][0])
    if f"{tag}.grad0" in G:
        assert relerr(adj.grad0, G[f"{tag}.grad0"]) <= 1e-14
        assert relerr(adj.grad0r, G[f"{tag}.grad0r"]) <= 1e-14
        assert relerr(adj.r0norm, G[f"{tag}.r0norm"]) <= 1e-15
        assert relerr(adj.w0, G[f"{tag}.w0"]) <= 1e-14


@pytest.mark.parametrize("tag,kw", [("rnd", dict(h=0.08)),
                                    ("rndn", dict(h=0.1, nbsrange=1, dp_body=0.07))])
def test_oracle_pairs_random(G, tag, kw, oracle_mod):
    rows, cols = oracle_mod.build_pairs(G[f"{tag}.X"], **kw)
    assert np.array_equal(rows, G[f"{tag}.rows"])
    assert np.array_equal(cols, G[f"{tag}.cols"])


@pytest.fixture(scope="module")
def K():
    return golden("kernels")


def _adj_for(K, dim, oracle_mod):
    X = K[f"d{dim}.X"]
    V0 = np.full(X.shape[0], 1e-3 ** dim)
    h = 1e-3 * np.sqrt(dim)
    return X, V0, h, oracle_mod.build_adjacency(X, V0, h, dim, 2)


@pytest.mark.parametrize("dim", [2, 3])
def test_oracle_pair_kernels(K, dim, oracle_mod):
    B = oracle_mod.backend
    X, V0, h, adj = _adj_for(K, dim, oracle_mod)
    n = X.shape[0]
    p = f"d{dim}."
    F = np.zeros((n, 3, 3))
    B.deformation_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0, K[p + "u"], V0,
                           K[p + "s"], 0.1, True, F)
    assert relerr(F - np.eye(3), K[p + "F"] - np.eye(3)) <= 1e-13
    lap = np.zeros(n)
    B.sph_laplacian(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.r0, adj.r0norm, V0,
                    K[p + "f"], lap)
    assert relerr(lap, K[p + "lap"]) <= 1e-13
    g = np.zeros((n, 3))
    B.sph_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0, V0, K[p + "f"], g)
    assert relerr(g, K[p + "grad"]) <= 1e-13
    for tag, (b1, b2) in (("mom0", (0.0, 0.0)), ("mom1", (0.2, 0.1))):
        a = np.zeros((n, 3))
        nb = B.momentum(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.grad0r, adj.r0,
                        adj.r0norm, K[p + "P"], 1000.0 * V0, 1000.0, K[p + "v"], h, 64.8, b1, b2,
                        K[p + "Fm"], a)
        assert nb == int(K[p + tag + ".nbad"][0])
        assert relerr(a, K[p + tag]) <= 1e-12


def test_oracle_constitutive(K, oracle_mod):
    B = oracle_mod.backend
    n = K["svk.F"].shape[0]
    for fr in (0, 1):
        S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
        assert B.svk_batch(K["svk.F"], 2.7733e6, 0.715e6, K["svk.s"], bool(fr), S, psi, psip) == 0
        assert relerr(S, K[f"svk{fr}.S"]) <= 1e-12
        assert relerr(psi, K[f"svk{fr}.psi"]) <= 1e-12
        assert relerr(psip, K[f"svk{fr}.psip"]) <= 1e-12
        S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
        nb = B.nh_batch(K["nh.F"], 3.25e6, 0.715e6, K["nh.s"], bool(fr), S, psi, psip)
        assert nb == int(K[f"nh{fr}.nbad"][0])
        assert relerr(S, K[f"nh{fr}.S"]) <= 1e-12
        assert relerr(psi, K[f"nh{fr}.psi"]) <= 1e-12
    for tag, Fk, Cp0, ep0 in (("j2", "j2.F", None, None), ("j2b", "j2b.F", "j2.Cp", "j2.ep")):
        F = K[Fk]
        n = F.shape[0]
        Cp = np.tile(np.eye(3), (n, 1, 1)) if Cp0 is None else K[Cp0].copy()
        ep = np.zeros(n) if ep0 is None else K[ep0].copy()
        S, psi, dwp = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
        nb, fb = B.j2_batch(F, Cp, ep, 43.333e9, 130e9, 4e8, 1e8, S, psi, dwp)
        assert [nb, fb] == list(K[f"{tag}.ret"])
        assert relerr(S, K[f"{tag}.S"]) <= 1e-12
        assert relerr(Cp - np.eye(3), K[f"{tag}.Cp"] - np.eye(3)) <= 1e-12
        assert relerr(ep, K[f"{tag}.ep"]) <= 1e-12
        # psi / dwp carry O(eps/strain) cancellation in the reference itself
        assert relerr(psi, K[f"{tag}.psi"]) <= 1e-9
        assert relerr(dwp, K[f"{tag}.dwp"]) <= 1e-9


def test_oracle_contact_and_eigen(K, oracle_mod):
    B = oracle_mod.backend
    xa, xb = K["ct.xa"], K["ct.xb"]
    pairs = np.array([(i, j) for i in range(40) for j in range(50)], dtype=np.int64)
    aa, ab = np.zeros((40, 3)), np.zeros((50, 3))
    w = B.contact_pair_accumulate(xa, K["ct.va"], np.full(40, 0.3), xb, K["ct.vb"],
                                  np.full(50, 0.4), pairs, 0.012, 1e7, 30.0, 0.3, aa, ab)
    assert w == int(K["ct.warn"][0])
    assert relerr(aa, K["ct.aa"]) <= 1e-12 and relerr(ab, K["ct.ab"]) <= 1e-12
    for A, wref in zip(K["eig.A"], K["eig.w"]):
        w, Q = np.zeros(3), np.zeros((3, 3))
        assert B.eig3_jacobi(A, w, Q) < 64
        assert np.all(np.diff(w) <= 0)
        assert np.abs(np.sort(w) - wref).max() <= 1e-12
        assert np.abs((Q * w) @ Q.T - A).max() <= 1e-12 * max(1.0, np.abs(A).max())


RUNS = ["kalthoff2d", "kalthoff2d_p", "kalthoff2d_sym", "beam2d", "taylor3d", "column3d",
        "branch2d", "kalthoff3d", "twisting3d"]

# FP64 multi-step tolerances: the reference's own numba-vs-numpy spread after
# 2000 steps is <= 2e-12; these runs are <= 40 steps.
TOL = {"u": 1e-10, "v": 1e-10, "a": 1e-9, "s": 1e-10, "sdot": 1e-9, "Hhist": 1e-9,
       "epbar": 1e-10, "F": 1e-11, "S": 1e-9, "Cp": 1e-11}


def check_state(got, G, step, bi=0):
    errs = {}
    for k, tol in TOL.items():
        if f"s{step}.b{bi}.{k}" not in G:
            continue
        ref = G[f"s{step}.b{bi}.{k}"]
        x = got[k]
        if k in ("F", "Cp"):
            x, ref = x - np.eye(3), ref - np.eye(3)
        if k == "s":
            err = np.abs(x - ref).max()
        else:
            err = relerr(x, ref)
        errs[k] = err
        assert err <= tol, (step, k, err)
    return errs


@pytest.mark.parametrize("tag", RUNS)
def test_oracle_run_matches_reference(tag, oracle_mod):
    G = golden(f"run_{tag}")
    cfg = run_case(G)
    for bi, b in enumerate(cfg.bodies):
        b.adjacency = oracle_mod.build_adjacency(
            b.state.X, b.state.V0, b.h, b.dim, int(cfg.kernel), nbsrange=b.nbsrange,
            dp_body=b.dp_body, notches=b.notches, correction=b.kernel_correction)
        assert np.array_equal(b.adjacency.indptr, G[f"adj{bi}.indptr"])
        assert np.array_equal(b.adjacency.indices, G[f"adj{bi}.indices"])
    sim = oracle_mod.OracleSimulation(cfg)
    sim.initialize()
    checks = set(int(c) for c in G["checkpoints"])
    dts = G["dts"]
    for step in range(1, len(dts) + 1):
        dt = sim.pick_dt()
        assert abs(dt - dts[step - 1]) <= 1e-12 * dts[step - 1]
        sim.step(dts[step - 1])
        if step in checks:
            for bi, b in enumerate(cfg.bodies):
                st = b.state
                check_state({k: getattr(st, k) for k in TOL}, G, step, bi)
    assert sim.t == pytest.approx(float(G[f"s{max(checks)}.t"][0]), rel=1e-14)


def test_oracle_crack3d_matches_reference(oracle_mod):
    """The oracle through the reference's run loop on the 3D Kalthoff crack
    golden (1,094 adaptive steps, generated by the reference itself): the
    same adjacency, dt sequence, crack and end state (u at 1e-12)."""
    G = golden("crack_kalthoff3d")
    cfg = run_case(G)
    b = cfg.bodies[0]
    b.adjacency = oracle_mod.build_adjacency(
        b.state.X, b.state.V0, b.h, b.dim, int(cfg.kernel), nbsrange=b.nbsrange,
        dp_body=b.dp_body, notches=b.notches, correction=b.kernel_correction)
    assert np.array_equal(b.adjacency.indices, G["adj0.indices"])
    sim = oracle_mod.OracleSimulation(cfg)
    dts = []
    orig = sim.step

    def step(dt):
        dts.append(dt)
        orig(dt)

    sim.step = step
    t_end = float(G["end.t"][0])
    sim.run(time_max=t_end, time_out=t_end)
    assert len(dts) == len(G["dts"])
    assert np.abs(np.array(dts) - G["dts"]).max() <= 1e-12 * G["dts"].max()
    st = b.state
    assert relerr(st.u, G["end.u"]) <= 1e-12
    assert np.abs(st.s - G["end.s"]).max() <= 1e-10
    quad = b.notches[0].points
    tip = quad[int(np.argmax(quad[:, 0]))]
    damaged = np.flatnonzero((st.s < 0.5) & (st.X[:, 0] > tip[0] + 2.0 * b.dp_body))
    assert np.array_equal(damaged, G["damaged"])


def test_oracle_expressions():
    G = golden("expr")
    srcs = bytes(G["sources"]).decode().split("\n")
    ctx = {k: (G[k] if G[k].ndim else float(G[k])) for k in
           ("x0", "y0", "z0", "x", "y", "z", "ux", "uy", "uz")}
    ctx.update(t=float(G["t"]), dt=float(G["dt"]), dx=float(G["dx"]))
    from oracle import oracle as O
    for k, line in enumerate(srcs):
        src, loc = line.split("\t")
        ast = ex.parse(src, loc)
        assert ex.pretty(ast) == bytes(G[f"e{k}.pretty"]).decode()
        vals, skip = O.eval_field(ast, ctx, G["x0"].shape[0])
        assert np.array_equal(skip, G[f"e{k}.skip"])
        m = ~skip
        assert np.array_equal(vals[m], G[f"e{k}.vals"][m])


@pytest.mark.parametrize("tag,spec", [("kalthoff2d", "kalthoff2d"), ("branch2d", "branch2d"),
                                      ("beam2d", "beam2d"), ("taylor3d", "taylor3d"),
                                      ("column3d", "column3d"), ("kalthoff3d", "kalthoff3d")])
def test_case_builder_matches_reference_loader(tag, spec):
    G = golden("targets")
    dps, mf = G[f"{tag}.kw"]
    cfg = cases.make_case(spec, dp_scale=float(dps), mapfac=int(mf) if mf > 0 else None,
                          build_adjacency=False)
    b = cfg.bodies[0]
    assert np.array_equal(b.state.X, G[f"{tag}.X"])
    for ci, bc in enumerate(b.bcs):
        key = f"{tag}.bc{ci}"
        if key in G:
            assert np.array_equal(bc.target, G[key]), key
        else:
            assert bc.target is None
