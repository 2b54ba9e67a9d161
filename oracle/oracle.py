"""CPU oracle for the TLSPH hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this module.  The product package
(paper_2602_15149_b200/) never imports it and has no CPU fallback.

What it restates (all citations into /root/reference/pkg/src/solidsph/):
  * the 8 backend-plugin kernels -> liboracle.so (tlsph_oracle.c), wrapped
    here with the plugin signatures of backends/reference.py:18-244;
  * reference-configuration geometry: kernel_eval (kernel_geom.py:30-62),
    build_pairs (:65-97, exact test in C), notch severing (:100-166),
    correction + CSR + reverse map (:169-261);
  * the stepper: Simulation phases, Verlet and symplectic steps, pick_dt and
    the run loop (stepper.py:19-263), with force / velocity BCs
    (dynamics.py:159-217), phase-field update and clamps (fracture.py:12-83)
    and stress dispatch (constitutive.py:168-199);
  * the masked vectorised expression evaluator (expr.py:419-551) over the
    tuple ASTs both packages produce.

Pinning: tests/test_oracle.py checks every function here against the golden
vectors in tests/golden/ that oracle/gen_golden.py produced by running the
reference itself (numpy backend) in the build container.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
J_MIN = 1.0e-6
COND_LIMIT = 1.0e8

_lib = None


def build():
    """Compile liboracle.so (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _lib = ctypes.CDLL(path)
        _declare(_lib)
    return _lib


_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


def _declare(L):
    sig = {
        "orc_deformation_gradient": (None, [_I, _P, _P, _P, _P, _P, _P, _D, _INT, _P]),
        "orc_sph_laplacian": (None, [_I, _P, _P, _P, _P, _P, _P, _P, _P]),
        "orc_sph_gradient": (None, [_I, _P, _P, _P, _P, _P, _P]),
        "orc_momentum": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _D, _D,
                              _D, _D, _P, _P]),
        "orc_svk_batch": (_I, [_I, _P, _D, _D, _P, _INT, _P, _P, _P]),
        "orc_nh_batch": (_I, [_I, _P, _D, _D, _P, _INT, _P, _P, _P]),
        "orc_j2_batch": (_I, [_I, _P, _P, _P, _D, _D, _D, _D, _P, _P, _P, _P]),
        "orc_contact_pair_accumulate": (_I, [_P, _P, _P, _P, _P, _P, _I, _P, _D, _D,
                                             _D, _D, _P, _P]),
        "orc_eig3_jacobi": (_INT, [_P, _P, _P]),
        "orc_build_pairs": (_INT, [_I, _P, _INT, _D, _D, _P, _P, _P]),
        "orc_correction": (_I, [_I, _P, _P, _P, _P, _P, _INT, _P, _P]),
        "orc_num_threads": (_INT, []),
        "orc_set_threads": (None, [_INT]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def set_threads(n):
    lib().orc_set_threads(int(n))


def num_threads():
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------------------
# backend plugin (same names / signatures as backends/reference.py)
# ---------------------------------------------------------------------------

class _Backend:
    NAME = "oracle"

    @staticmethod
    def deformation_gradient(indptr, rows, indices, grad0, u, V0, s, s_l,
                             gated, out):
        assert out.flags.c_contiguous and out.dtype == np.float64
        n = out.shape[0]
        lib().orc_deformation_gradient(n, _p(_i64(indptr)), _p(_i64(indices)),
                                       _p(_f64(grad0)), _p(_f64(u)), _p(_f64(V0)),
                                       _p(_f64(s)), float(s_l), int(bool(gated)), _p(out))
        return out

    @staticmethod
    def sph_laplacian(indptr, rows, indices, grad0, r0, r0norm, V0, f, out):
        lib().orc_sph_laplacian(out.shape[0], _p(_i64(indptr)), _p(_i64(indices)),
                                _p(_f64(grad0)), _p(_f64(r0)), _p(_f64(r0norm)),
                                _p(_f64(V0)), _p(_f64(f)), _p(out))
        return out

    @staticmethod
    def sph_gradient(indptr, rows, indices, grad0, V0, f, out):
        lib().orc_sph_gradient(out.shape[0], _p(_i64(indptr)), _p(_i64(indices)),
                               _p(_f64(grad0)), _p(_f64(V0)), _p(_f64(f)), _p(out))
        return out

    @staticmethod
    def momentum(indptr, rows, indices, grad0, grad0r, r0, r0norm, P, m0, rho0,
                 v, h, c0, beta1, beta2, F, out):
        return int(lib().orc_momentum(
            out.shape[0], _p(_i64(indptr)), _p(_i64(indices)), _p(_f64(grad0)),
            _p(_f64(grad0r)), _p(_f64(r0)), _p(_f64(r0norm)), _p(_f64(P)),
            _p(_f64(m0)), float(rho0), _p(_f64(v)), float(h), float(c0),
            float(beta1), float(beta2), _p(_f64(F)), _p(out)))

    @staticmethod
    def svk_batch(F, lam, mu, s, fracture, out_S, out_psi, out_psip):
        return int(lib().orc_svk_batch(F.shape[0], _p(_f64(F)), float(lam), float(mu),
                                       _p(_f64(s)), int(bool(fracture)), _p(out_S),
                                       _p(out_psi), _p(out_psip)))

    @staticmethod
    def nh_batch(F, kappa, mu, s, fracture, out_S, out_psi, out_psip):
        return int(lib().orc_nh_batch(F.shape[0], _p(_f64(F)), float(kappa), float(mu),
                                      _p(_f64(s)), int(bool(fracture)), _p(out_S),
                                      _p(out_psi), _p(out_psip)))

    @staticmethod
    def j2_batch(F, Cp, epbar, mu, kappa, sigma_y0, H_hard, out_S, out_psi,
                 out_dwp):
        assert Cp.flags.c_contiguous and epbar.flags.c_contiguous
        fb = ctypes.c_int64(-1)
        nb = lib().orc_j2_batch(F.shape[0], _p(_f64(F)), _p(Cp), _p(epbar), float(mu),
                                float(kappa), float(sigma_y0), float(H_hard), _p(out_S),
                                _p(out_psi), _p(out_dwp), ctypes.byref(fb))
        return int(nb), int(fb.value)

    @staticmethod
    def contact_pair_accumulate(xa, va, ma, xb, vb, mb, pairs, dp_contact, k_n,
                                c_n, kfric, out_aa, out_ab):
        pairs = _i64(pairs).reshape(-1, 2)
        return int(lib().orc_contact_pair_accumulate(
            _p(_f64(xa)), _p(_f64(va)), _p(_f64(ma)), _p(_f64(xb)), _p(_f64(vb)),
            _p(_f64(mb)), pairs.shape[0], _p(pairs), float(dp_contact), float(k_n),
            float(c_n), float(kfric), _p(out_aa), _p(out_ab)))

    @staticmethod
    def eig3_jacobi(A, w, Q):
        return int(lib().orc_eig3_jacobi(_p(_f64(A)), _p(w), _p(Q)))


backend = _Backend()


# ---------------------------------------------------------------------------
# reference-configuration geometry (kernel_geom.py)
# ---------------------------------------------------------------------------

def smoothing_length(dp, coefh, dim):
    return coefh * dp * math.sqrt(dim)


def kernel_eval(q, h, dim, kind):
    """(W, dW/dr) for kind 1 = cubic spline, 2 = Wendland C2; support 2h."""
    q = np.asarray(q, dtype=np.float64)
    if dim == 2:
        ac, aw = 10.0 / (7.0 * math.pi * h * h), 7.0 / (4.0 * math.pi * h * h)
    else:
        ac, aw = 1.0 / (math.pi * h ** 3), 21.0 / (16.0 * math.pi * h ** 3)
    if int(kind) == 1:
        w = np.where(q < 1.0, 1.0 - 1.5 * q * q + 0.75 * q ** 3,
                     np.where(q < 2.0, 0.25 * (2.0 - q) ** 3, 0.0))
        dw = np.where(q < 1.0, -3.0 * q + 2.25 * q * q,
                      np.where(q < 2.0, -0.75 * (2.0 - q) ** 2, 0.0))
        return ac * w, ac * dw / h
    t = np.where(q < 2.0, 1.0 - 0.5 * q, 0.0)
    return aw * (t ** 4 * (2.0 * q + 1.0)), aw * (-5.0 * q * t ** 3) / h


class CaseErrorOracle(Exception):
    pass


def build_pairs(positions, h, nbsrange=None, dp_body=None):
    X = _f64(positions)
    n = X.shape[0]
    if n < 2:
        raise CaseErrorOracle("need at least 2 particles to build neighbors")
    nbs = nbsrange is not None
    win = nbsrange * dp_body * (1.0 + 1e-9) if nbs else 0.0
    counts = np.zeros(n, dtype=np.int64)
    lib().orc_build_pairs(n, _p(X), int(nbs), float(h), float(win), _p(counts), None, None)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    if indptr[-1] == 0:
        raise CaseErrorOracle("no neighbor pairs found")
    cols = np.zeros(indptr[-1], dtype=np.int64)
    lib().orc_build_pairs(n, _p(X), int(nbs), float(h), float(win), _p(counts), _p(indptr),
                          _p(cols))
    rows = np.repeat(np.arange(n, dtype=np.int64), counts)
    return rows, cols


def quad_frame(points, scale):
    p = np.asarray(points, dtype=np.float64).reshape(4, 3)
    e1 = p[1] - p[0]
    nv = np.cross(e1, p[2] - p[0])
    nn = np.linalg.norm(nv)
    if nn <= 1e-14 * max(scale, 1e-300) ** 2:
        raise CaseErrorOracle("degenerate quad (zero area)")
    nh = nv / nn
    diag = np.linalg.norm(p.max(axis=0) - p.min(axis=0))
    if abs((p[3] - p[0]) @ nh) > 1e-6 * diag:
        raise CaseErrorOracle("quad points are not coplanar")
    e1h = e1 / np.linalg.norm(e1)
    e2h = np.cross(nh, e1h)
    poly = (p - p[0]) @ np.stack([e1h, e2h], axis=1)
    return p[0], nh, e1h, e2h, poly


def _in_poly(pts, poly):
    tol = 1e-12 * max(1.0, np.abs(poly).max())
    pos = np.ones(pts.shape[0], dtype=bool)
    neg = np.ones(pts.shape[0], dtype=bool)
    for k in range(poly.shape[0]):
        a, b = poly[k], poly[(k + 1) % poly.shape[0]]
        cr = (b[0] - a[0]) * (pts[:, 1] - a[1]) - (b[1] - a[1]) * (pts[:, 0] - a[0])
        pos &= cr >= -tol
        neg &= cr <= tol
    return pos | neg


def segments_cross_quad(Xa, Xb, points):
    Xa, Xb = np.atleast_2d(Xa), np.atleast_2d(Xb)
    pts = np.asarray(points, dtype=np.float64).reshape(4, 3)
    scale = max(np.abs(pts).max(), 1.0)
    o, nh, e1h, e2h, poly = quad_frame(pts, scale)
    da = (Xa - o) @ nh
    db = (Xb - o) @ nh
    tol = 1e-12 * scale
    cand = (((da < -tol) & (db > tol)) | ((da > tol) & (db < -tol))
            | ((np.abs(da) <= tol) & (np.abs(db) > tol))
            | ((np.abs(db) <= tol) & (np.abs(da) > tol)))
    out = np.zeros(Xa.shape[0], dtype=bool)
    if cand.any():
        den = da[cand] - db[cand]
        den = np.where(np.abs(den) < 1e-300, 1e-300, den)
        t = np.clip(da[cand] / den, 0.0, 1.0)
        hit = Xa[cand] + t[:, None] * (Xb[cand] - Xa[cand])
        out[cand] = _in_poly((hit - o) @ np.stack([e1h, e2h], axis=1), poly)
    return out


def build_adjacency(positions, V0, h, dim, kind, nbsrange=None, dp_body=None,
                    notches=(), correction=True):
    X = _f64(positions)
    V0 = _f64(V0)
    n = X.shape[0]
    rows, cols = build_pairs(X, h, nbsrange=nbsrange, dp_body=dp_body)
    for q in notches:
        pts = q.points if hasattr(q, "points") else q
        keep = ~segments_cross_quad(X[rows], X[cols], pts)
        rows, cols = rows[keep], cols[keep]
    counts = np.bincount(rows, minlength=n)
    if (counts == 0).any():
        raise CaseErrorOracle(
            f"particle {int(np.flatnonzero(counts == 0)[0])} has no neighbors after notch severing")
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    r0 = X[rows] - X[cols]
    r0norm = np.linalg.norm(r0, axis=1)
    w0, dwdr = kernel_eval(r0norm / h, h, dim, kind)
    with np.errstate(invalid="ignore", divide="ignore"):
        gb = (dwdr / r0norm)[:, None] * r0
    gb[r0norm == 0.0] = 0.0
    gb = np.ascontiguousarray(gb)
    fallbacks = 0
    L = np.tile(np.eye(3), (n, 1, 1))
    if correction:
        A = np.zeros((n, 3, 3))
        fallbacks = int(lib().orc_correction(n, _p(indptr), _p(_i64(cols)), _p(X), _p(V0),
                                             _p(gb), int(dim), _p(A), _p(L)))
        grad = np.einsum("kab,kb->ka", L[rows], gb)
    else:
        grad = gb
    keys = rows * n + cols
    rev = np.searchsorted(keys, cols * n + rows)
    return SimpleNamespace(indptr=indptr, rows=rows, indices=cols,
                           grad0=np.ascontiguousarray(grad),
                           grad0r=np.ascontiguousarray(grad[rev]),
                           r0=np.ascontiguousarray(r0), r0norm=r0norm, w0=w0,
                           correction_fallbacks=fallbacks, L=L,
                           nnz=int(cols.shape[0]))


# ---------------------------------------------------------------------------
# masked vectorised expression evaluation (expr.py:419-551)
# ---------------------------------------------------------------------------

class OracleExprError(ValueError):
    pass


def _field_call(name, args, act):
    a = args[0]
    if name in ("log", "ln", "sqrt"):
        ok = a > 0.0 if name != "sqrt" else a >= 0.0
        if np.any(act & ~ok):
            raise OracleExprError(f"{name} domain")
        a = np.where(act, a, 1.0)
        return {"log": np.log10, "ln": np.log, "sqrt": np.sqrt}[name](a)
    if name == "cot":
        return np.cos(a) / np.sin(np.where(act, a, 1.0))
    if name == "coth":
        c = np.where(act, np.clip(a, -700, 700), 1.0)
        return np.cosh(c) / np.sinh(c)
    if name == "pow":
        with np.errstate(invalid="ignore", over="ignore"):
            out = np.power(np.where(act, a, 1.0), np.where(act, args[1], 1.0))
        if np.any(act & ~np.isfinite(out)):
            raise OracleExprError("pow domain")
        return out
    fn = {"sin": np.sin, "cos": np.cos, "tan": np.tan, "sinh": np.sinh,
          "cosh": np.cosh, "tanh": np.tanh, "abs": np.abs}[name]
    with np.errstate(over="ignore"):
        return fn(np.where(act, a, 0.0))


def _field_bin(op, a, b, act):
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op == "/":
        if np.any(act & (b == 0.0)):
            raise OracleExprError("division by zero")
        return a / np.where(act, b, 1.0)
    if op == "^":
        with np.errstate(invalid="ignore", over="ignore"):
            out = np.power(np.where(act, a, 1.0), np.where(act, b, 1.0))
        if np.any(act & ~np.isfinite(out)):
            raise OracleExprError("^ domain")
        return out
    cmp = {"<": np.less, ">": np.greater, "<=": np.less_equal,
           ">=": np.greater_equal, "==": np.equal, "!=": np.not_equal}
    if op in cmp:
        return cmp[op](a, b).astype(np.float64)
    if op == "and":
        return ((a != 0.0) & (b != 0.0)).astype(np.float64)
    return ((a != 0.0) | (b != 0.0)).astype(np.float64)


def _field(node, ctx, act):
    n = act.shape[0]
    tag = node[0]
    if tag == "num":
        return np.full(n, node[1]), np.zeros(n, bool)
    if tag == "skip":
        return np.zeros(n), np.ones(n, bool)
    if tag == "var":
        val = ctx[node[1]]
        if np.isscalar(val):
            return np.full(n, float(val)), np.zeros(n, bool)
        return np.asarray(val, dtype=np.float64), np.zeros(n, bool)
    if tag == "un":
        v, s = _field(node[2], ctx, act)
        return -v, s
    if tag == "if":
        c, _ = _field(node[1], ctx, act)
        tm, fm = act & (c != 0.0), act & (c == 0.0)
        vals, skip = np.zeros(n), np.zeros(n, bool)
        if tm.any():
            tv, ts = _field(node[2], ctx, tm)
            vals[tm], skip[tm] = tv[tm], ts[tm]
        if fm.any():
            fv, fs = _field(node[3], ctx, fm)
            vals[fm], skip[fm] = fv[fm], fs[fm]
        return vals, skip
    if tag == "call":
        parts = [_field(a, ctx, act)[0] for a in node[2]]
        return _field_call(node[1], parts, act), np.zeros(n, bool)
    av, _ = _field(node[2], ctx, act)
    bv, _ = _field(node[3], ctx, act)
    return _field_bin(node[1], av, bv, act), np.zeros(n, bool)


def eval_field(ast, ctx, n):
    root = ast.root if hasattr(ast, "root") else ast
    return _field(root, ctx, np.ones(n, bool))


def field_context(body, t, dt, idx=None):
    st = body.state
    sel = (lambda a: a) if idx is None else (lambda a: a[idx])
    x = st.X + st.u
    return {"t": float(t), "dt": float(dt), "dx": float(body.dp_body),
            "x0": sel(st.X[:, 0]), "y0": sel(st.X[:, 1]), "z0": sel(st.X[:, 2]),
            "x": sel(x[:, 0]), "y": sel(x[:, 1]), "z": sel(x[:, 2]),
            "ux": sel(st.u[:, 0]), "uy": sel(st.u[:, 1]), "uz": sel(st.u[:, 2])}


# ---------------------------------------------------------------------------
# stepper restatement (stepper.py, dynamics.py, fracture.py, constitutive.py)
# ---------------------------------------------------------------------------

class OracleSimulationError(RuntimeError):
    pass


def _axis_values(bc, axis, exprs, ctx, count):
    c = bc.const[axis]
    if c is not None:
        return np.full(count, c), np.ones(count, bool)
    eid = bc.expr[axis]
    if eid is None:
        return None
    vals, skip = eval_field(exprs[eid], ctx, count)
    return vals, ~skip


def _bc_active(bc, t):
    return bc.tst <= t <= bc.tend


class OracleSimulation:
    """Restates solidsph.stepper.Simulation on the oracle kernels.

    ``config`` is any object with the CaseConfig attributes (this package's
    or the reference's); the per-body state arrays are advanced in place."""

    def __init__(self, config, be=None):
        self.config = config
        self.bodies = config.bodies
        self.expressions = config.expressions
        self.be = be or backend
        self.t = 0.0
        self.step_index = 0
        self._init = False
        self.ws = []
        for b in self.bodies:
            n = b.state.X.shape[0]
            self.ws.append(SimpleNamespace(P=np.zeros((n, 3, 3)), a_int=np.zeros((n, 3)),
                                           lap=np.zeros(n), dwp=np.zeros(n)))
        self._static = {}

    # internal phase -------------------------------------------------------
    def _stress(self, body, ws):
        st, mat = body.state, body.material
        m = int(mat.model)
        if m == 1:
            nc = self.be.svk_batch(st.F, mat.lam, mat.mu, st.s, body.fracture, st.S,
                                   st.psi_e, st.psi_plus)
            if nc:
                raise OracleSimulationError("eigensolver failed to converge")
        elif m == 2:
            body.degenerate_warnings += self.be.nh_batch(
                st.F, mat.kappa, mat.mu, st.s, body.fracture, st.S, st.psi_e, st.psi_plus)
        else:
            nb, fb = self.be.j2_batch(st.F, st.Cp, st.epbar, mat.mu, mat.kappa,
                                      mat.sigma_y0, mat.H_hard, st.S, st.psi_e, ws.dwp)
            if fb >= 0:
                raise OracleSimulationError(f"non-SPD plastic metric at particle {fb}")
            body.degenerate_warnings += nb
            body.plastic_work += float(ws.dwp @ st.V0)
            st.psi_plus[:] = 0.0

    def _internal(self, t, dt):
        for body, ws in zip(self.bodies, self.ws):
            st, adj, mat = body.state, body.adjacency, body.material
            self.be.deformation_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0,
                                         st.u, st.V0, st.s, mat.s_l, body.fracture, st.F)
            self._stress(body, ws)
            if body.fracture:
                st.Hhist[:] = np.maximum(st.psi_plus, st.Hhist)
                self.be.sph_laplacian(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.r0,
                                      adj.r0norm, st.V0, st.s, ws.lap)
                ratio = st.Hhist / mat.Gc
                c = mat.c0
                damp = 2.0 * np.sqrt(4.0 * mat.eps0 * ratio + 1.0) / c
                st.sddot[:] = (c * c / (2.0 * mat.eps0)) * (
                    2.0 * mat.eps0 * ws.lap + (1.0 - st.s) / (2.0 * mat.eps0)
                    - damp * st.sdot - 2.0 * st.s * ratio)
            np.matmul(st.F, st.S, out=ws.P)
            body.degenerate_warnings += self.be.momentum(
                adj.indptr, adj.rows, adj.indices, adj.grad0, adj.grad0r, adj.r0,
                adj.r0norm, ws.P, st.m0, mat.rho0, st.v, body.h, mat.c0, mat.beta1,
                mat.beta2, st.F, ws.a_int)
            st.a[:] = ws.a_int
            st.a += body.f0
            for bc in body.bcs:
                if bc.kind == "force":
                    self._force_bc(body, bc, t, dt)
            if body.dim == 2:
                st.a[:, 1] = 0.0
            if not np.isfinite(st.a).all():
                bad = int(np.flatnonzero(~np.isfinite(st.a).all(axis=1))[0])
                raise OracleSimulationError(f"non-finite acceleration at particle {bad}")

    def _force_bc(self, body, bc, t, dt):
        if not _bc_active(bc, t):
            return
        st = body.state
        idx = bc.target
        count = st.X.shape[0] if idx is None else idx.shape[0]
        if count == 0:
            return
        ctx = field_context(body, t, dt, idx)
        m0 = st.m0 if idx is None else st.m0[idx]
        if bc.ftype == 1:
            scale = 1.0 / m0
        elif bc.ftype == 2:
            scale = body.dp_body ** (body.dim - 1) / m0
        else:
            scale = np.ones(count)
        for axis in range(3):
            got = _axis_values(bc, axis, self.expressions, ctx, count)
            if got is None:
                continue
            vals, mask = got
            add = np.where(mask, vals * scale, 0.0)
            if idx is None:
                st.a[:, axis] += add
            else:
                st.a[idx, axis] += add

    def _vel_bcs(self, t, dt):
        for body in self.bodies:
            st = body.state
            for bc in body.bcs:
                if bc.kind != "vel" or not _bc_active(bc, t):
                    continue
                idx = bc.target
                count = st.X.shape[0] if idx is None else idx.shape[0]
                if count == 0:
                    continue
                ctx = field_context(body, t, dt, idx)
                for axis in range(3):
                    got = _axis_values(bc, axis, self.expressions, ctx, count)
                    if got is None:
                        continue
                    vals, mask = got
                    if idx is None:
                        st.v[mask, axis] = vals[mask]
                    else:
                        st.v[idx[mask], axis] = vals[mask]
            if body.dim == 2:
                st.v[:, 1] = 0.0

    def _restrict(self, body, t, dt):
        eid = body.restrictphi_expr
        if eid is None:
            return None
        ast = self.expressions[eid]
        vals, skip = eval_field(ast, field_context(body, t, dt), body.state.X.shape[0])
        return vals, ~skip

    def _advance_pf(self, body, dts, dtr, t, dt):
        st = body.state
        st.sdot += dtr * st.sddot
        st.s += dts * st.sdot
        lo, hi = st.s < 0.0, st.s > 1.0
        st.s[lo] = 0.0
        st.sdot[lo] = 0.0
        st.s[hi] = 1.0
        st.sdot[hi] = 0.0
        r = self._restrict(body, t, dt)
        if r is not None:
            vals, applied = r
            eng = applied & (st.s < vals)
            st.s[eng] = vals[eng]
            st.sdot[eng] = 0.0

    # public API -------------------------------------------------------------
    def initialize(self):
        self._internal(0.0, 0.0)
        self._vel_bcs(0.0, 0.0)
        self._init = True

    def step(self, dt):
        if not self._init:
            self.initialize()
        if int(self.config.step_algorithm) == 2:
            self._symplectic(dt)
        else:
            self._verlet(dt)

    def _verlet(self, dt):
        t = self.t
        self._internal(t, dt)
        self._vel_bcs(t, dt)
        tn = t + dt
        for b in self.bodies:
            b.state.v += dt * b.state.a
        self._vel_bcs(tn, dt)
        for b in self.bodies:
            b.state.u += dt * b.state.v
            if b.dim == 2:
                b.state.u[:, 1] = 0.0
            if b.fracture:
                self._advance_pf(b, dt, dt, tn, dt)
        self._commit(dt)

    def _symplectic(self, dt):
        t = self.t
        th, tn = t + 0.5 * dt, t + dt
        for b in self.bodies:
            b.state.v += 0.5 * dt * b.state.a
        self._vel_bcs(th, dt)
        for b in self.bodies:
            b.state.u += 0.5 * dt * b.state.v
            if b.dim == 2:
                b.state.u[:, 1] = 0.0
            if b.fracture:
                self._advance_pf(b, 0.5 * dt, 0.5 * dt, th, dt)
        self._internal(th, dt)
        self._vel_bcs(th, dt)
        for b in self.bodies:
            b.state.v += 0.5 * dt * b.state.a
        self._vel_bcs(tn, dt)
        for b in self.bodies:
            b.state.u += 0.5 * dt * b.state.v
            if b.dim == 2:
                b.state.u[:, 1] = 0.0
            if b.fracture:
                self._advance_pf(b, 0.5 * dt, 0.5 * dt, tn, dt)
        self._commit(dt)

    def _commit(self, dt):
        self.t += dt
        self.step_index += 1

    def pick_dt(self):
        if self.config.dt_override is not None:
            return self.config.dt_override
        dt = math.inf
        for b in self.bodies:
            st = b.state
            vmax = float(np.sqrt(np.max(np.einsum("nd,nd->n", st.v, st.v))))
            amax = float(np.sqrt(np.max(np.einsum("nd,nd->n", st.a, st.a))))
            dtv = b.h / (b.material.c0 + vmax)
            cand = self.config.cfl * (min(dtv, math.sqrt(b.h / amax)) if amax > 0.0 else dtv)
            dt = min(dt, cand)
        return dt

    def run(self, time_max=None, time_out=None, on_output=None, max_steps=None):
        cfg = self.config
        t_max = cfg.time_max if time_max is None else time_max
        t_out = cfg.time_out if time_out is None else time_out
        if not self._init:
            self.initialize()
        if on_output is not None:
            on_output(self)
        if t_max <= 0.0:
            return
        nxt = t_out if t_out > 0.0 else t_max
        eps = 1e-12 * max(t_max, 1.0)
        while self.t < t_max - eps:
            dt = min(self.pick_dt(), nxt - self.t, t_max - self.t)
            if dt <= 0.0:
                raise OracleSimulationError(f"timestep collapsed to {dt!r}")
            self.step(dt)
            if self.t >= nxt - eps:
                if on_output is not None:
                    on_output(self)
                nxt = min(nxt + t_out, t_max) if t_out > 0.0 else t_max
            if max_steps is not None and self.step_index >= max_steps:
                break
