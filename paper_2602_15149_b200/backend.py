"""Kernel-level drop-in for the reference backend plugin.

A module with ``NAME`` and the same kernels, signatures and return
conventions as ``solidsph.backends.reference`` / ``.fast``
(/root/reference/pkg/src/solidsph/backends/reference.py:18-244): host numpy
FP64 arrays in, outputs written in place, counts returned, never raises on
numerical events.  Each call copies its inputs to the B200, runs the
libtlsph kernel and copies the result back, so

    sim = solidsph.stepper.Simulation(cfg)
    sim.be = paper_2602_15149_b200.backend

reruns the reference's own step on the GPU kernel by kernel (SURVEY.md 8(b):
``Simulation.__init__`` snapshots ``backends.active()`` into ``sim.be``).
Adjacency arrays are constant for a body's lifetime (total Lagrangian), so
their device copies are cached per host array.  The throughput path is
``simulation.DeviceSimulation``, which keeps all state resident.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _lib

NAME = "b200"

_cache: dict = {}


def _dev(a, dtype=None, cache=False):
    import torch
    a = np.asarray(a)
    if dtype is not None and a.dtype != dtype:
        a = a.astype(dtype)
    a = np.ascontiguousarray(a)
    if cache:
        key = (id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str)
        hit = _cache.get(key)
        if hit is not None and hit[0]() is a:
            return hit[1]
        t = torch.from_numpy(a).cuda()
        try:
            ref = weakref.ref(a, lambda _r, k=key: _cache.pop(k, None))
            _cache[key] = (ref, t)
        except TypeError:
            pass
        return t
    return torch.from_numpy(a).cuda()


def _out(out):
    import torch
    return torch.empty(out.shape, dtype=torch.float64, device="cuda")


def _back(t, out):
    out[...] = t.cpu().numpy().reshape(out.shape)


def _counter(n=1, fill=0):
    import torch
    return torch.full((n,), fill, dtype=torch.int64, device="cuda")


_keep: list = []


def _call(name, *args):
    """Launch and only then release the argument tensors: a device temporary
    dropped before the launch would hand its memory to the next argument."""
    L = _lib.lib()
    try:
        _lib.check(getattr(L, name)(_lib.stream_ptr(), *args), name)
    finally:
        _keep.clear()


def P(t):
    if t is not None:
        _keep.append(t)
    return _lib.ptr(t)


def deformation_gradient(indptr, rows, indices, grad0, u, V0, s, s_l, gated, out):
    n = out.shape[0]
    o = _out(out)
    _call("tl_deformation_gradient", n, P(_dev(indptr, np.int64, True)),
          P(_dev(indices, np.int64, True)), P(_dev(grad0, np.float64, True)),
          P(_dev(u, np.float64)), P(_dev(V0, np.float64, True)), P(_dev(s, np.float64)),
          float(s_l), int(bool(gated)), P(o))
    _back(o, out)
    return out


def sph_laplacian(indptr, rows, indices, grad0, r0, r0norm, V0, f, out):
    o = _out(out)
    _call("tl_sph_laplacian", out.shape[0], P(_dev(indptr, np.int64, True)),
          P(_dev(indices, np.int64, True)), P(_dev(grad0, np.float64, True)),
          P(_dev(r0, np.float64, True)), P(_dev(r0norm, np.float64, True)),
          P(_dev(V0, np.float64, True)), P(_dev(f, np.float64)), P(o))
    _back(o, out)
    return out


def sph_gradient(indptr, rows, indices, grad0, V0, f, out):
    o = _out(out)
    _call("tl_sph_gradient", out.shape[0], P(_dev(indptr, np.int64, True)),
          P(_dev(indices, np.int64, True)), P(_dev(grad0, np.float64, True)),
          P(_dev(V0, np.float64, True)), P(_dev(f, np.float64)), P(o))
    _back(o, out)
    return out


def momentum(indptr, rows, indices, grad0, grad0r, r0, r0norm, P_, m0, rho0, v, h, c0, beta1,
             beta2, F, out):
    o = _out(out)
    nb = _counter()
    _call("tl_momentum", out.shape[0], P(_dev(indptr, np.int64, True)),
          P(_dev(indices, np.int64, True)), P(_dev(grad0, np.float64, True)),
          P(_dev(grad0r, np.float64, True)), P(_dev(r0, np.float64, True)),
          P(_dev(r0norm, np.float64, True)), P(_dev(P_, np.float64)),
          P(_dev(m0, np.float64, True)), float(rho0), P(_dev(v, np.float64)), float(h),
          float(c0), float(beta1), float(beta2), P(_dev(F, np.float64)), P(o), P(nb))
    _back(o, out)
    return int(nb.item())


def svk_batch(F, lam, mu, s, fracture, out_S, out_psi, out_psip):
    n = F.shape[0]
    S, psi, psip, nc = _out(out_S), _out(out_psi), _out(out_psip), _counter()
    _call("tl_svk_batch", n, P(_dev(F, np.float64)), float(lam), float(mu),
          P(_dev(s, np.float64)), int(bool(fracture)), P(S), P(psi), P(psip), P(nc))
    _back(S, out_S)
    _back(psi, out_psi)
    _back(psip, out_psip)
    return int(nc.item())


def nh_batch(F, kappa, mu, s, fracture, out_S, out_psi, out_psip):
    n = F.shape[0]
    S, psi, psip, nb = _out(out_S), _out(out_psi), _out(out_psip), _counter()
    _call("tl_nh_batch", n, P(_dev(F, np.float64)), float(kappa), float(mu),
          P(_dev(s, np.float64)), int(bool(fracture)), P(S), P(psi), P(psip), P(nb))
    _back(S, out_S)
    _back(psi, out_psi)
    _back(psip, out_psip)
    return int(nb.item())


def j2_batch(F, Cp, epbar, mu, kappa, sigma_y0, H_hard, out_S, out_psi, out_dwp):
    import torch
    n = F.shape[0]
    Cpd = _dev(Cp, np.float64).clone()
    epd = _dev(epbar, np.float64).clone()
    S, psi, dwp = _out(out_S), _out(out_psi), _out(out_dwp)
    cnt = torch.tensor([0, np.iinfo(np.int64).max], dtype=torch.int64, device="cuda")
    _call("tl_j2_batch", n, P(_dev(F, np.float64)), P(Cpd), P(epd), float(mu), float(kappa),
          float(sigma_y0), float(H_hard), P(S), P(psi), P(dwp), P(cnt), None)
    c = cnt.cpu().numpy()
    if c[1] != np.iinfo(np.int64).max:
        return int(c[0]), int(c[1])
    _back(S, out_S)
    _back(psi, out_psi)
    _back(dwp, out_dwp)
    Cp[...] = Cpd.cpu().numpy()
    epbar[...] = epd.cpu().numpy()
    return int(c[0]), -1


def contact_pair_accumulate(xa, va, ma, xb, vb, mb, pairs, dp_contact, k_n, c_n, kfric,
                            out_aa, out_ab):
    import torch
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    npairs = pairs.shape[0]
    aa = _dev(out_aa, np.float64).clone()
    ab = _dev(out_ab, np.float64).clone()
    warn = _counter()
    scratch = torch.empty(max(3 * npairs, 1), dtype=torch.float64, device="cuda")
    _call("tl_contact_pair_accumulate", P(_dev(xa, np.float64)), P(_dev(va, np.float64)),
          P(_dev(ma, np.float64)), P(_dev(xb, np.float64)), P(_dev(vb, np.float64)),
          P(_dev(mb, np.float64)), npairs, P(_dev(pairs, np.int64)), float(dp_contact),
          float(k_n), float(c_n), float(kfric), P(aa), P(ab), P(warn), P(scratch))
    _back(aa, out_aa)
    _back(ab, out_ab)
    return int(warn.item())


def _eig3_jacobi(A, w, Q):
    """Single-matrix eigen solve (fast._eig3_jacobi signature)."""
    import torch
    Ad = _dev(np.asarray(A, dtype=np.float64).reshape(1, 3, 3))
    wd = torch.empty((1, 3), dtype=torch.float64, device="cuda")
    Qd = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
    sw = torch.empty(1, dtype=torch.int32, device="cuda")
    _call("tl_eig3_jacobi", 1, P(Ad), P(wd), P(Qd), P(sw))
    w[...] = wd.cpu().numpy().reshape(3)
    Q[...] = Qd.cpu().numpy().reshape(3, 3)
    return int(sw.item())


def eig3_jacobi_batch(A):
    """Batched Jacobi: (w (n,3) descending, Q (n,3,3), sweeps (n,))."""
    import torch
    A = np.ascontiguousarray(A, dtype=np.float64).reshape(-1, 3, 3)
    n = A.shape[0]
    wd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    Qd = torch.empty((n, 3, 3), dtype=torch.float64, device="cuda")
    sw = torch.empty(n, dtype=torch.int32, device="cuda")
    _call("tl_eig3_jacobi", n, P(_dev(A)), P(wd), P(Qd), P(sw))
    return wd.cpu().numpy(), Qd.cpu().numpy(), sw.cpu().numpy()
