"""Reference-configuration geometry on the device: the neighbour build,
correction matrices and the Adjacency the reference's loader expects.

Drop-in for ``solidsph.kernel_geom`` (/root/reference/pkg/src/solidsph/
kernel_geom.py): same function names, arguments, return types and CaseError
messages.  ``build_adjacency`` is the hook the reference's case loader calls
as a module attribute (caseio.py:562), so

    import solidsph.kernel_geom, paper_2602_15149_b200.kernel_geom as kg
    solidsph.kernel_geom.build_adjacency = kg.build_adjacency

moves the one-time O(N k) build onto the GPU.  The returned ``Adjacency``
keeps the device structure (``adj.device``) that ``DeviceSimulation`` reuses;
its per-pair host arrays (grad0, r0, ...; ~104 B/pair) are produced lazily,
only if host code reads them.
"""

from __future__ import annotations

import math

import os

import numpy as np

from . import _lib
from .core import Adjacency, CaseError, KernelKind

COND_LIMIT = 1.0e8


def smoothing_length(dp, coefh, dim):
    """h = coefh * dp * sqrt(dim) (kernel_geom.py:21-27)."""
    if dp <= 0.0 or coefh <= 0.0:
        raise CaseError("dp and coefh must be positive")
    if dim not in (2, 3):
        raise CaseError(f"dim must be 2 or 3, got {dim}")
    return coefh * dp * math.sqrt(dim)


def kernel_alpha(h, dim, kind):
    """Normalisation of the cubic spline (1) / Wendland C2 (2) kernel."""
    if dim not in (2, 3):
        raise CaseError(f"dim must be 2 or 3, got {dim}")
    if int(kind) == int(KernelKind.CUBIC_SPLINE):
        return 10.0 / (7.0 * math.pi * h * h) if dim == 2 else 1.0 / (math.pi * h ** 3)
    if int(kind) == int(KernelKind.WENDLAND):
        return 7.0 / (4.0 * math.pi * h * h) if dim == 2 else 21.0 / (16.0 * math.pi * h ** 3)
    raise CaseError(f"unknown kernel kind {kind!r}")


def kernel_eval(q, h, dim, kind):
    """(W, dW/dr) at q = r/h, support 2h (kernel_geom.py:30-62).  Host-side
    helper for diagnostics; the step kernels evaluate dW/dr inline."""
    q = np.asarray(q, dtype=np.float64)
    a = kernel_alpha(h, dim, kind)
    if int(kind) == int(KernelKind.CUBIC_SPLINE):
        tm = 2.0 - q
        w = np.where(q < 1.0, 1.0 - 1.5 * q * q + 0.75 * q ** 3, np.where(q < 2.0, 0.25 * tm ** 3, 0.0))
        dw = np.where(q < 1.0, -3.0 * q + 2.25 * q * q, np.where(q < 2.0, -0.75 * tm ** 2, 0.0))
    else:
        t = np.where(q < 2.0, 1.0 - 0.5 * q, 0.0)
        w = t ** 4 * (2.0 * q + 1.0)
        dw = -5.0 * q * t ** 3
    return a * w, a * dw / h


# ---------------------------------------------------------------------------
# notch frames (kernel_geom.py:100-131), computed once on the host
# ---------------------------------------------------------------------------

def _quad_points(q):
    return np.asarray(q.points if hasattr(q, "points") else q, dtype=np.float64).reshape(4, 3)


def quad_frame(points, scale):
    p = _quad_points(points)
    e1 = p[1] - p[0]
    nvec = np.cross(e1, p[2] - p[0])
    nn = np.linalg.norm(nvec)
    if nn <= 1e-14 * max(scale, 1e-300) ** 2:
        raise CaseError("degenerate quad (zero area)")
    nhat = nvec / nn
    diag = np.linalg.norm(p.max(axis=0) - p.min(axis=0))
    if abs((p[3] - p[0]) @ nhat) > 1e-6 * diag:
        raise CaseError("quad points are not coplanar")
    e1h = e1 / np.linalg.norm(e1)
    e2h = np.cross(nhat, e1h)
    poly = (p - p[0]) @ np.stack([e1h, e2h], axis=1)
    return p[0], nhat, e1h, e2h, poly


def notch_struct(q):
    pts = _quad_points(q)
    scale = max(np.abs(pts).max(), 1.0)
    o, nh, e1, e2, poly = quad_frame(pts, scale)
    s = _lib.tl_notch()
    for k in range(3):
        s.origin[k], s.nhat[k], s.e1[k], s.e2[k] = o[k], nh[k], e1[k], e2[k]
    for k in range(4):
        s.poly[k][0], s.poly[k][1] = poly[k, 0], poly[k, 1]
    s.tol_plane = 1e-12 * scale
    s.tol_poly = 1e-12 * max(1.0, np.abs(poly).max())
    return s


# ---------------------------------------------------------------------------
# device structure
# ---------------------------------------------------------------------------

class DeviceAdjacency:
    """Fixed neighbour structure resident in HBM.

    indptr (n+1) int64, indices (nnz) int32 in ascending partner order per
    row (the reference CSR), L (n,9) FP64 correction matrices, and the
    lane-interleaved sliced-ELL copy (soff, sidx) the step kernels read."""

    def __init__(self, X, indptr, indices, L, fallbacks, h, dim, kind, correction):
        self.X = X
        self.indptr = indptr
        self.indices = indices
        self.L = L
        self.correction_fallbacks = int(fallbacks)
        self.h = h
        self.dim = dim
        self.kind = int(kind)
        self.correction = bool(correction)
        self.n = int(X.shape[0])
        self.nnz = int(indices.shape[0])
        self._sell = None

    def sell(self):
        """(soff int64[nw+1], sidx int32[32*sum slen]) built once on demand."""
        if self._sell is None:
            import torch
            L = _lib.lib()
            st = _lib.stream_ptr()
            nw = (self.n + 31) // 32
            slen = torch.empty(nw, dtype=torch.int32, device=self.X.device)
            _lib.check(L.tl_sell_lengths(st, self.n, _lib.ptr(self.indptr), _lib.ptr(slen)),
                       "tl_sell_lengths")
            soff = torch.zeros(nw + 1, dtype=torch.int64, device=self.X.device)
            torch.cumsum(slen.to(torch.int64) * 32, 0, out=soff[1:])
            total = int(soff[-1].item())
            sidx = torch.empty(max(total, 1), dtype=torch.int32, device=self.X.device)
            _lib.check(L.tl_sell_fill(st, self.n, _lib.ptr(self.indptr), _lib.ptr(self.indices),
                                      _lib.ptr(soff), _lib.ptr(sidx)), "tl_sell_fill")
            self._sell = (soff, sidx)
        return self._sell

    def expand(self, rows=True, r0=True, r0norm=True, w0=True, grad0=True, grad0r=True):
        """Per-pair FP64 arrays of the reference Adjacency, on the device."""
        import torch
        dev = self.X.device
        nnz = self.nnz
        out = {}

        def mk(flag, shape, dt=torch.float64):
            return torch.empty(shape, dtype=dt, device=dev) if flag else None

        out["rows"] = mk(rows, (nnz,), torch.int64)
        out["r0"] = mk(r0, (nnz, 3))
        out["r0norm"] = mk(r0norm, (nnz,))
        out["w0"] = mk(w0, (nnz,))
        out["grad0"] = mk(grad0, (nnz, 3))
        out["grad0r"] = mk(grad0r, (nnz, 3))
        alpha = kernel_alpha(self.h, self.dim, self.kind)
        L = _lib.lib()
        _lib.check(L.tl_adjacency_expand(
            _lib.stream_ptr(), self.n, _lib.ptr(self.indptr), _lib.ptr(self.indices),
            _lib.ptr(self.X), _lib.ptr(self.L), float(self.h), float(alpha), self.kind,
            *[_lib.ptr(out[k]) for k in ("rows", "r0", "r0norm", "w0", "grad0", "grad0r")]),
            "tl_adjacency_expand")
        return out


def class_geometry(q, dp, h, kind, precision):
    """(m, 8) table of bond classes with lattice offsets q (r0 = q dp = X_i -
    X_j): W = w(r) r0, kappa = 1/(w(r) (r^2 + 0.001 h^2)) (0 when w = 0),
    U = r0 / r^2, 0 -- evaluated in FP64 with the pair loops' kernel shape
    (step.cu kshape; the reference's kernel_geom.py:21-62 without the
    per-body constant)."""
    r0 = np.asarray(q, dtype=np.float64).reshape(-1, 3) * float(dp)
    r2 = np.einsum("ij,ij->i", r0, r0)
    r = np.sqrt(r2)
    inv_h = 1.0 / float(h)
    if int(kind) == 2:     # Wendland C2: t^3, t = max(1 - r/2h, 0)
        t = np.maximum(1.0 - r * (0.5 * inv_h), 0.0)
        w = t * t * t
    else:                  # cubic spline (step.cu kshape, KIND 1)
        qh = r * inv_h
        w = np.where(qh < 1.0, (-3.0 + 2.25 * qh) * inv_h,
                     np.where(qh < 2.0, -0.75 * (2.0 - qh) ** 2 / np.where(r > 0, r, 1.0), 0.0))
    table = np.zeros((r0.shape[0], 8), dtype=np.float64)
    table[:, 0:3] = w[:, None] * r0
    den = w * (r2 + 0.001 * float(h) * float(h))
    table[:, 3] = np.where(w != 0.0, 1.0 / np.where(w != 0.0, den, 1.0), 0.0)
    table[:, 4:7] = r0 / r2[:, None]
    # a pair a rounding error inside the support edge (r = 2h - 1e-16) has
    # w ~ 1e-48: W flushes to zero in FP32 while kappa overflows, so its
    # (negligible) terms are dropped outright rather than turned into 0 * inf
    tiny = np.abs(table[:, 3]) > (1e30 if precision == "fp32" else 1e300)
    table[tiny] = 0.0
    return table


class StepLayout:
    """Device particle order and neighbour tiles for the step kernels.

    perm[p] = original index of device position p (Morton order of cells of
    about one particle, so T consecutive particles form a compact brick);
    the CSR is renamed into that order with each row still in ascending
    original partner order (the reference's summation order), copied to a
    lane-interleaved sliced ELL (soff, sidx), and, when ``tile`` > 0, every
    CTA of ``tile`` particles gets the halo list of the neighbours it does not
    own plus uint16 shared-memory slots for each pair (tiles.cu)."""

    GROUP = 4   # TL_SELL_GROUP
    RESIDUE = int(os.environ.get("TLSPH_HALO_RESIDUE", "8"))   # 8 = bank-aligned halo slots

    def __init__(self, dadj, tile=256, rows=None, halo=None, precision="fp64", order=None):
        """rows: adjacency rows this device owns (default all); halo: adjacency
        ids of the off-rank particles those rows reference, in exchange order
        (multi-GPU, see dist.py).  Device positions: owned [0, n) in Morton
        order (or ``order``: device position -> index into rows, e.g. the
        brick-major order of BrickLayout), then the halo block [n, n_all) in
        the given order."""
        import torch
        L = _lib.lib()
        st = _lib.stream_ptr()
        dev = dadj.X.device
        if rows is None:
            rows = torch.arange(dadj.n, dtype=torch.int64, device=dev)
        rows = torch.as_tensor(rows, dtype=torch.int64, device=dev)
        halo = (torch.zeros(0, dtype=torch.int64, device=dev) if halo is None
                else torch.as_tensor(halo, dtype=torch.int64, device=dev))
        n = int(rows.shape[0])
        self.n = n
        self.n_all = n + int(halo.shape[0])
        Xh = dadj.X.index_select(0, rows).contiguous()
        lo = Xh.min(dim=0).values.cpu().numpy()
        hi = Xh.max(dim=0).values.cpu().numpy()
        ext = hi - lo
        active = ext > 0
        vol = float(np.prod(ext[active])) if active.any() else 1.0
        cell = (vol / n) ** (1.0 / max(int(active.sum()), 1)) if active.any() else 1.0
        cell = max(cell, 1e-300)
        if order is not None:
            pown = torch.as_tensor(order, device=dev).to(torch.int32)
        else:
            pown = torch.empty(n, dtype=torch.int32, device=dev)
            ipown = torch.empty(n, dtype=torch.int32, device=dev)
            lo_arr = (_lib.D * 3)(*lo)
            _lib.check(L.tl_reorder(st, n, _lib.ptr(Xh), lo_arr, float(cell), _lib.ptr(pown),
                                    _lib.ptr(ipown)), "tl_reorder")
        prow = rows.index_select(0, pown.long()).to(torch.int32)     # device pos -> adj row
        # adjacency id -> device position (owned, then halo); -1 = never referenced
        iperm = torch.full((dadj.n,), -1, dtype=torch.int32, device=dev)
        iperm[prow.long()] = torch.arange(n, dtype=torch.int32, device=dev)
        if halo.numel():
            iperm[halo] = torch.arange(n, self.n_all, dtype=torch.int32, device=dev)
        self.perm = torch.cat([prow, halo.to(torch.int32)])          # device pos -> adj id
        self.iperm = iperm
        counts = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(L.tl_csr_permute_counts(st, n, _lib.ptr(prow), _lib.ptr(dadj.indptr),
                                           _lib.ptr(counts)), "tl_csr_permute_counts")
        self.indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=self.indptr[1:])
        self.indices = torch.empty(int(self.indptr[-1].item()), dtype=torch.int32, device=dev)
        _lib.check(L.tl_csr_permute(st, n, _lib.ptr(prow), _lib.ptr(iperm),
                                    _lib.ptr(dadj.indptr), _lib.ptr(dadj.indices),
                                    _lib.ptr(self.indptr), _lib.ptr(self.indices)),
                   "tl_csr_permute")
        if int(self.indices.min().item()) < 0 if self.indices.numel() else False:
            raise ValueError("owned rows reference a particle that is neither owned nor halo")
        nw = (n + 31) // 32
        slen = torch.empty(nw, dtype=torch.int32, device=dev)
        _lib.check(L.tl_sell_lengths(st, n, _lib.ptr(self.indptr), _lib.ptr(slen)),
                   "tl_sell_lengths")
        # longest real row of every slice (the slice itself is padded to 4)
        rl = torch.zeros(nw * 32, dtype=torch.int32, device=dev)
        rl[:n] = (self.indptr[1:] - self.indptr[:-1]).to(torch.int32)
        self.wlen = rl.view(nw, 32).amax(dim=1).contiguous()
        self.soff = torch.zeros(nw + 1, dtype=torch.int64, device=dev)
        torch.cumsum(slen.to(torch.int64) * 32, 0, out=self.soff[1:])
        total = int(self.soff[-1].item())
        self.sidx = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        _lib.check(L.tl_sell_fill(st, n, _lib.ptr(self.indptr), _lib.ptr(self.indices),
                                  _lib.ptr(self.soff), _lib.ptr(self.sidx)), "tl_sell_fill")
        self.tile = 0
        self.hmax = 0
        self.slmax = 0
        self.hoff = self.halo = self.slots = self.hslot = self.toff = None
        # slots hold slot * 16 (16-byte units; FP64 records are two units)
        self.slot_shift = 4
        if tile and tile > 0:
            if tile % 32 or tile > 256:
                raise ValueError(f"tile size {tile}: a multiple of 32, at most 256")
            self._build_tiles(int(tile), total)

    def _build_tiles(self, T, total):
        import torch
        L = _lib.lib()
        st = _lib.stream_ptr()
        dev = self.indptr.device
        n = self.n
        nnz = int(self.indices.shape[0])
        ntile = (n + T - 1) // T
        halo = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        tcount = torch.zeros(ntile, dtype=torch.int64, device=dev)
        nh = _lib.I64(0)
        _lib.check(L.tl_tile_halo(st, n, T, _lib.ptr(self.indptr), _lib.ptr(self.indices), nnz,
                                  _lib.ptr(halo), _lib.ptr(tcount), _lib.C.byref(nh)),
                   "tl_tile_halo")
        self.halo = halo[: max(int(nh.value), 1)].clone()
        del halo
        self.hoff = torch.zeros(ntile + 1, dtype=torch.int64, device=dev)
        torch.cumsum(tcount, 0, out=self.hoff[1:])
        if T + 8 * int(tcount.max().item() if ntile else 0) > 65535:
            return   # slot indices are uint16: leave the body untiled
        # shared-memory slot of every halo entry (bank-conflict-free residues;
        # tiles that would outgrow the densest dense halo are packed densely)
        self.hslot = torch.empty(max(int(self.halo.shape[0]), 1), dtype=torch.int16, device=dev)
        extent = torch.zeros(max(ntile, 1), dtype=torch.int32, device=dev)
        hdense = int(tcount.max().item()) if ntile else 0
        cap = ((int(float(os.environ.get("TLSPH_HALO_CAP", "1.0")) * hdense) + 7) // 8) * 8
        _lib.check(L.tl_tile_hslots(st, ntile, T, self.RESIDUE, cap, _lib.ptr(self.hoff),
                                    _lib.ptr(self.halo), _lib.ptr(self.hslot), _lib.ptr(extent)),
                   "tl_tile_hslots")
        self.hmax = int(extent.max().item()) if ntile else 0
        # staged position records: tile t owns records [toff[t], toff[t+1])
        self.toff = torch.zeros(ntile + 1, dtype=torch.int64, device=dev)
        torch.cumsum(extent[:ntile].to(torch.int64) + T, 0, out=self.toff[1:])
        # slot-table entries of each tile (its warps' slices), staged per CTA
        nw = (n + 31) // 32
        wb = torch.arange(0, ntile + 1, device=dev, dtype=torch.int64) * (T // 32)
        wb.clamp_(max=nw)
        self.slmax = int((self.soff[wb[1:]] - self.soff[wb[:-1]]).max().item()) if ntile else 0
        self.slots = torch.empty(max(total, 4), dtype=torch.int16, device=dev)
        if (T + self.hmax) << self.slot_shift > 65535:
            self.hoff = self.halo = self.hslot = self.toff = None
            self.hmax = 0
            return   # slot byte offsets are uint16: leave the body untiled
        _lib.check(L.tl_tile_slots(st, n, T, self.GROUP, self.slot_shift, _lib.ptr(self.indptr),
                                   _lib.ptr(self.indices), _lib.ptr(self.hoff),
                                   _lib.ptr(self.halo), _lib.ptr(self.hslot), _lib.ptr(self.soff),
                                   _lib.ptr(self.slots)), "tl_tile_slots")
        self.tile = T


    KEY_R = 7              # tiles.cu kKeyR: lattice offsets |q| <= 7 per axis
    KEY_SELF, KEY_OFF = 0xFFFF, 0xFFFE
    MAX_CLASSES = 63       # 6 class bits above the 10 slot bits of a uint16 entry

    def bond_classes(self, Xs, dp, h, kind, precision="fp32"):
        """Bond-class slot table for lattice bodies (uniform V0 and m0).

        Every pair of a body cut from one lattice of spacing dp has a
        reference separation r0 = X_i - X_j = q dp with q an integer offset,
        so the pair geometry (kernel shape, r0, 1/r^2) takes one of a few
        values -- 26 for a 3D nbsrange = 1 stencil.  The slots are rewritten
        to (class << 10) | slot (tiles.cu k_class_slots) and the returned
        (ncls, 8) table (FP32 or FP64, the body's precision) holds, per class, W = w(r) r0, kappa =
        1/(w(r) (r^2 + 0.001 h^2)) and U = r0 / r^2, evaluated in FP64 with the
        pair loops' kernel shape (step.cu kshape; kernel_geom.py:21-62 of the
        reference).  Class 0 is the padding entry (j = i), all zero.  Returns
        None, leaving the slots unchanged, when some pair is off the lattice
        (|r0 - q dp| > 1e-6 dp), the tile has more than 1024 slots, or there
        are more than MAX_CLASSES classes."""
        import torch
        if not self.tile or not (dp > 0) or self.tile + self.hmax > 1024:
            return None
        L = _lib.lib()
        st = _lib.stream_ptr()
        P = _lib.ptr
        total = int(self.soff[-1].item())
        if total == 0:
            return None
        keys = torch.empty_like(self.slots)
        _lib.check(L.tl_tile_slots_keyed(st, self.n, self.tile, self.GROUP, self.slot_shift,
                                         P(self.indptr), P(self.indices), P(self.hoff),
                                         P(self.halo), P(self.hslot), P(self.soff),
                                         P(self.slots), P(Xs), self.n_all, float(dp), P(keys)),
                   "tl_tile_slots_keyed")
        seen = torch.zeros(1 << 16, dtype=torch.bool, device=keys.device)
        chunk = 1 << 26                     # bounded temporaries at 10^9 pairs (C5)
        for c0 in range(0, total, chunk):
            k = keys[c0:min(c0 + chunk, total)].to(torch.int32) & 0xFFFF
            seen[k.long()] = True
            del k
        ku = torch.nonzero(seen).flatten().cpu().numpy()
        if (ku == self.KEY_OFF).any():
            return None
        ku = ku[ku != self.KEY_SELF]
        if ku.size > self.MAX_CLASSES:
            return None
        side = 2 * self.KEY_R + 1
        cls_of_key = np.full(side ** 3, -1, dtype=np.int16)
        cls_of_key[ku] = np.arange(1, ku.size + 1, dtype=np.int16)
        q = np.stack([ku // (side * side), (ku // side) % side, ku % side], axis=1) - self.KEY_R
        table = np.zeros((ku.size + 1, 8), dtype=np.float64)
        table[1:] = class_geometry(q, dp, h, kind, precision)
        dev = self.slots.device
        _lib.check(L.tl_class_slots(st, total, self.slot_shift, P(keys),
                                    P(torch.from_numpy(cls_of_key).to(dev)), P(self.slots)),
                   "tl_class_slots")
        torch.cuda.current_stream().synchronize()
        del keys
        dt = np.float32 if precision == "fp32" else np.float64
        return torch.from_numpy(table.astype(dt)).to(dev).contiguous()

    def split_tiles(self):
        """Multi-GPU launch order: (tile list, number of interior tiles).
        Interior tiles read no halo row (device position >= n) and can run
        while the halo exchange is in flight; the rest follow it."""
        import torch
        if not self.tile or self.n_all == self.n:
            return None, 0
        ntile = int(self.hoff.shape[0]) - 1
        counts = self.hoff[1:] - self.hoff[:-1]
        owner = torch.repeat_interleave(torch.arange(ntile, device=counts.device), counts)
        hal = self.halo[: owner.shape[0]].long()
        boundary = torch.zeros(ntile, dtype=torch.bool, device=counts.device)
        boundary[owner[hal >= self.n]] = True
        interior = torch.nonzero(~boundary).flatten()
        border = torch.nonzero(boundary).flatten()
        tlist = torch.cat([interior, border]).to(torch.int32).contiguous()
        return tlist, int(interior.shape[0])

    def positions(self, Xs, weight=None, precision="fp32"):
        """Staged position records (x, y, z, w) of every tile slot
        (tl_tile_pos): Xs = 3 device FP64 planes of stride n_all in device
        order; weight = per-particle device FP64 (V0 or m0) or None."""
        import torch
        if not self.tile:
            return None
        R = torch.float32 if precision == "fp32" else torch.float64
        ntile = int(self.hoff.shape[0]) - 1
        out = torch.zeros((int(self.toff[-1].item()), 4), dtype=R, device=Xs.device)
        _lib.check(_lib.lib().tl_tile_pos(
            _lib.stream_ptr(), self.n, self.n_all, self.tile, ntile, _lib.ptr(self.hoff),
            _lib.ptr(self.halo), _lib.ptr(self.hslot), _lib.ptr(self.toff), _lib.ptr(Xs),
            _lib.ptr(weight) if weight is not None else None, 4 if precision == "fp32" else 8,
            _lib.ptr(out)), "tl_tile_pos")
        return out


class BrickLayout:
    """Lattice-brick mode of the step kernels (tl_body.brick; step.cu
    k_brick_a / k_brick_b) for 3D bodies cut from one lattice with wide
    (radial, k ~ 170) stencils.

    Every particle sits on a lattice cell c = round((X - X_min) / dp); a
    bond i -> j has class q = c_i - c_j (r0 = q dp).  The device order is
    brick-major (bricks of B cells, z fastest), a CTA per brick stages the
    records of the (B + 2 reach) box of cells around it by cell, and each
    particle's bonds are one mask bit per class -- exactly its CSR row, with
    the classes numbered in the reference's CSR summation order (the order of
    a complete row).  ``plan`` returns None when the body is not a single
    lattice (a position off the lattice by > 1e-6 dp, two particles in one
    cell, |q| > 7) or has more than MAX_CLASSES classes."""

    MAX_CLASSES = 256     # TL_BRICK_MAX_CLASSES
    KEY_R = 7
    SMEM = 226 * 1024
    CANDIDATES = [(16, 8, 8), (8, 16, 8), (8, 8, 16), (8, 8, 8), (16, 8, 4), (16, 4, 8),
                  (8, 16, 4), (4, 16, 8), (8, 4, 16), (4, 8, 16), (8, 8, 4), (8, 4, 8),
                  (4, 8, 8), (4, 4, 8), (4, 8, 4), (8, 4, 4), (4, 4, 4)]

    MAX_COLUMNS = 64       # TL_BRICK_MAX_COLUMNS

    @classmethod
    def _columns(cls, qk):
        """(qx, qy, qz_lo, qz_hi, first class) per stencil column when the
        class order (CSR order) runs each (qx, qy) column once with qz
        descending by one (split into two entries where it skips the
        particle itself) -- the condition of the register-blocked walk --
        else None."""
        cols, seen = [], set()
        c = 0
        while c < qk.shape[0]:
            qx, qy, qz = (int(v) for v in qk[c])
            # a column may resume right after a gap (the (0, 0) column around
            # the particle itself): a second entry, walked next
            if (qx, qy) in seen and not (cols and cols[-1][:2] == (qx, qy)):
                return None
            seen.add((qx, qy))
            e = c
            while (e + 1 < qk.shape[0] and int(qk[e + 1, 0]) == qx and int(qk[e + 1, 1]) == qy
                   and int(qk[e + 1, 2]) == int(qk[e, 2]) - 1):
                e += 1
            cols.append((qx, qy, int(qk[e, 2]), qz, c))
            c = e + 1
        return cols if len(cols) <= cls.MAX_COLUMNS else None

    @classmethod
    def plan(cls, dadj, dp, h, kind, precision):
        import torch
        X = dadj.X
        dev = X.device
        n = int(X.shape[0])
        if n == 0 or not (dp > 0):
            return None
        lo = X.min(dim=0).values
        cf = torch.round((X - lo) / dp)
        if float((X - (lo + cf * dp)).abs().max().item()) > 1e-6 * dp:
            return None
        c = cf.to(torch.int64)
        cells = (c.max(dim=0).values + 1).cpu().numpy().astype(np.int64)
        if int(np.prod(cells)) > (1 << 31) - 1:
            return None
        lin = (c[:, 0] * int(cells[1]) + c[:, 1]) * int(cells[2]) + c[:, 2]
        if int(torch.unique(lin).shape[0]) != n:
            return None                                   # two particles in one cell
        # classes (lattice offsets) of every bond, in chunks
        side = 2 * cls.KEY_R + 1
        seen = torch.zeros(side ** 3, dtype=torch.bool, device=dev)
        counts = dadj.indptr[1:] - dadj.indptr[:-1]
        nnz = int(dadj.indptr[-1].item())
        chunk = 1 << 25
        rows_all = torch.repeat_interleave(torch.arange(n, device=dev), counts)
        for a in range(0, nnz, chunk):
            rr = rows_all[a:a + chunk]
            jj = dadj.indices[a:a + chunk].long()
            q = c[rr] - c[jj]
            if int(q.abs().max().item()) > cls.KEY_R:
                return None
            key = ((q[:, 0] + cls.KEY_R) * side + q[:, 1] + cls.KEY_R) * side + q[:, 2] + cls.KEY_R
            seen[key] = True
        ku = torch.nonzero(seen).flatten().cpu().numpy()
        if ku.size == 0 or ku.size > cls.MAX_CLASSES:
            return None
        # class order: the CSR order of a longest (complete) row
        rmax = int(torch.argmax(counts).item())
        a0, a1 = int(dadj.indptr[rmax].item()), int(dadj.indptr[rmax + 1].item())
        q = (c[rmax][None, :] - c[dadj.indices[a0:a1].long()]).cpu().numpy()
        first = ((q[:, 0] + cls.KEY_R) * side + q[:, 1] + cls.KEY_R) * side + q[:, 2] + cls.KEY_R
        rest = np.setdiff1d(ku, first)
        keys = np.concatenate([first, rest]).astype(np.int64)
        qk = np.stack([keys // (side * side), (keys // side) % side, keys % side], 1) - cls.KEY_R
        if rest.size:
            # classes the longest row lacks (ties at r = 2h kept for some
            # particles only): order every class as the lattice's CSR order
            # does -- q descending, slowest index axis first (axis strides
            # from the longest row's unit-offset partners) -- if that order
            # agrees with the longest row
            jj = dadj.indices[a0:a1].long().cpu().numpy()
            stride = np.zeros(3)
            for ax in range(3):
                hit = np.flatnonzero((np.abs(q[:, ax]) == 1) & (np.abs(q).sum(axis=1) == 1))
                if hit.size:
                    stride[ax] = abs(int(jj[hit[0]]) - rmax)
            if (stride > 0).sum() == (np.ptp(qk, axis=0) > 0).sum():
                axo = np.argsort(-stride, kind="stable")
                order = np.lexsort(tuple(-qk[:, a] for a in axo[::-1]))
                pos = np.empty(keys.size, dtype=np.int64)
                pos[order] = np.arange(keys.size)
                if np.all(np.diff(pos[:first.size]) > 0):
                    keys, qk = keys[order], qk[order]
        reach = int(np.abs(qk).max())
        k_mean = nnz / n
        rsz = 16 if precision == "fp32" else 32
        cols = cls._columns(qk)
        best = None
        cands = cls.CANDIDATES
        env_dims = os.environ.get("TLSPH_BRICK_DIMS")     # "bx,by,bz": measurement override
        if env_dims:
            cands = [tuple(int(v) for v in env_dims.split(","))]
        for B in cands:
            # register blocking (2 cells per thread) measured slower on B200 --
            # C2 0.98 vs 1.50 G particle-steps/s: half the warps per SM for a
            # walk with data-dependent bounds -- so it is opt-in
            cpt = 2 if (cols is not None and B[2] % 2 == 0
                        and os.environ.get("TLSPH_BRICK_CPT", "1") == "2") else 1
            T = B[0] * B[1] * B[2] // cpt
            if T % 32 or T > 1024 // cpt:
                continue
            boxz = B[2] + 2 * reach
            if cpt == 2 and boxz % 2 == 0:
                boxz += 1          # odd z extent: a warp's records hit distinct bank groups
            S = (B[0] + 2 * reach) * (B[1] + 2 * reach) * boxz
            if S * 3 * rsz > cls.SMEM:
                continue
            nbv = [int(-(-int(cells[k]) // B[k])) for k in range(3)]
            bid = ((c[:, 0] // B[0]) * nbv[1] + c[:, 1] // B[1]) * nbv[2] + c[:, 2] // B[2]
            nbr = int(torch.unique(bid).shape[0])
            cost = nbr * (B[0] * B[1] * B[2] * k_mean + 8.0 * S)
            if best is None or cost < best[0]:
                best = (cost, B, nbv, cpt, boxz)
        if best is None:
            return None
        _, B, nbv, cpt, boxz = best
        bid = ((c[:, 0] // B[0]) * nbv[1] + c[:, 1] // B[1]) * nbv[2] + c[:, 2] // B[2]
        loc = ((c[:, 0] % B[0]) * B[1] + c[:, 1] % B[1]) * B[2] + c[:, 2] % B[2]
        order = torch.argsort(bid * (B[0] * B[1] * B[2]) + loc)
        self = cls()
        self.order = order                 # device position -> adjacency row
        self.c = c
        self.cells = cells
        self.brick = B
        self.nbrick = nbv
        self.reach = reach
        self.keys = keys
        self.q = qk
        self.cpt = cpt
        self.boxz = boxz
        # pass A on half-width bricks where the pass-B brick is 16 wide: two
        # 512-thread CTAs per SM instead of one of 1024 (TLSPH_BRICK_A_SPLIT)
        asp = int(os.environ.get("TLSPH_BRICK_A_SPLIT", "2"))
        self.a_split = asp if (asp > 1 and B[0] % asp == 0
                               and (B[0] // asp) * B[1] * B[2] // cpt >= 64) else 1
        self.cols = cols if cpt == 2 else None
        self.table = class_geometry(qk, dp, h, kind, precision)
        self.precision = precision
        return self

    def finish(self, lay):
        """Device structures for the layout's device order: cell map, bond
        masks, box offsets, class table."""
        import torch
        dev = lay.indptr.device
        n, n_all = lay.n, lay.n_all
        cd = self.c.index_select(0, lay.perm[:n].long())     # device order cells
        C1, C2 = int(self.cells[1]), int(self.cells[2])
        lin = (cd[:, 0] * C1 + cd[:, 1]) * C2 + cd[:, 2]
        self.cellmap = torch.full((int(np.prod(self.cells)),), -1, dtype=torch.int32, device=dev)
        self.cellmap[lin] = torch.arange(n, dtype=torch.int32, device=dev)
        side = 2 * self.KEY_R + 1
        cls_of_key = torch.full((side ** 3,), -1, dtype=torch.int64, device=dev)
        cls_of_key[torch.from_numpy(self.keys).to(dev)] = torch.arange(
            self.keys.size, dtype=torch.int64, device=dev)
        nmask = (self.keys.size + 31) // 32
        acc = torch.zeros((nmask, n_all), dtype=torch.int64, device=dev)
        counts = lay.indptr[1:] - lay.indptr[:-1]
        nnz = int(lay.indptr[-1].item())
        rows_all = torch.repeat_interleave(torch.arange(n, device=dev), counts)
        chunk = 1 << 25
        for a in range(0, nnz, chunk):
            rr = rows_all[a:a + chunk]
            jj = lay.indices[a:a + chunk].long()
            q = cd[rr] - cd[jj]
            key = ((q[:, 0] + self.KEY_R) * side + q[:, 1] + self.KEY_R) * side + q[:, 2] + self.KEY_R
            k = cls_of_key[key]
            # one distinct bit per (row, class): a sum is an OR
            acc.view(-1).index_add_(0, (k // 32) * n_all + rr, torch.bitwise_left_shift(
                torch.ones_like(k), k % 32))
        acc = torch.where(acc >= (1 << 31), acc - (1 << 32), acc)
        self.bmask = acc.to(torch.int32).contiguous()
        self.nmask = nmask
        SY = self.brick[1] + 2 * self.reach
        SZ = self.boxz
        delta = -((self.q[:, 0] * SY + self.q[:, 1]) * SZ + self.q[:, 2])
        if self.cols is not None:
            # (box offset of the column, qz_lo, qz_hi, class of qz_hi)
            self.col_table = np.array([[-(qx * SY + qy) * SZ, lo, hi, c0]
                                       for (qx, qy, lo, hi, c0) in self.cols], dtype=np.int32)
        self.bdelta = torch.from_numpy(delta.astype(np.int32)).to(dev)
        dt = torch.float32 if self.precision == "fp32" else torch.float64
        self.bbcls = torch.from_numpy(self.table).to(dev, dt).contiguous()
        self.nbricks = int(np.prod(self.nbrick))
        if self.a_split > 1:      # pass A's (more) CTAs write plastic-work partials too
            nba = -(-int(self.cells[0]) // (self.brick[0] // self.a_split))
            self.nbricks = max(self.nbricks, nba * int(self.nbrick[1]) * int(self.nbrick[2]))
        del self.c
        return self

    def fill(self, d):
        """Set the brick fields of a tl_body descriptor."""
        for k in range(3):
            d.brick[k] = int(self.brick[k])
            d.nbrick[k] = int(self.nbrick[k])
            d.cells[k] = int(self.cells[k])
        d.reach = int(self.reach)
        d.a_split = int(self.a_split)
        d.cpt = int(self.cpt)
        d.boxz = int(self.boxz)
        if self.cpt == 2:
            self._col_host = np.ascontiguousarray(self.col_table.reshape(-1))
            d.ncol = int(self.col_table.shape[0])
            d.bcol_host = self._col_host.ctypes.data
        d.nbcls = int(self.keys.size)
        d.nmask = int(self.nmask)
        d.cellmap = _lib.ptr(self.cellmap)
        d.bmask = _lib.ptr(self.bmask)
        d.bdelta = _lib.ptr(self.bdelta)
        d.bbcls = _lib.ptr(self.bbcls)
        # host copies for the launch's kernel-parameter class table
        self._delta_host = np.ascontiguousarray(self.bdelta.cpu().numpy())
        self._cls_host = np.ascontiguousarray(self.bbcls.cpu().numpy())
        d.bdelta_host = self._delta_host.ctypes.data
        d.bbcls_host = self._cls_host.ctypes.data


class LazyAdjacency(Adjacency):
    """core.Adjacency whose per-pair host arrays are fetched from the device
    on first access."""

    _PAIR = ("rows", "grad0", "grad0r", "r0", "r0norm", "w0")

    def __init__(self, dev: DeviceAdjacency):
        object.__setattr__(self, "device", dev)
        object.__setattr__(self, "_host", {})
        object.__setattr__(self, "correction_fallbacks", dev.correction_fallbacks)

    def __getattribute__(self, name):
        if name in LazyAdjacency._PAIR or name in ("indptr", "indices"):
            host = object.__getattribute__(self, "_host")
            if name not in host:
                dev = object.__getattribute__(self, "device")
                if name == "indptr":
                    host[name] = dev.indptr.cpu().numpy()
                elif name == "indices":
                    host[name] = dev.indices.to(dtype=__import__("torch").int64).cpu().numpy()
                else:
                    arrs = dev.expand()
                    for k in LazyAdjacency._PAIR:
                        host[k] = arrs[k].cpu().numpy()
            return host[name]
        return object.__getattribute__(self, name)

    def __setattr__(self, name, value):
        if name in LazyAdjacency._PAIR or name in ("indptr", "indices"):
            object.__getattribute__(self, "_host")[name] = value
        else:
            object.__setattr__(self, name, value)

    @property
    def nnz(self):
        return object.__getattribute__(self, "device").nnz

    def counts(self):
        return np.diff(self.indptr)


def _grid_params(X, reach):
    lo = X.min(axis=0)
    hi = X.max(axis=0)
    cell = reach * (1.0 + 1e-6)
    dims = (np.floor((hi - lo) / cell).astype(np.int64) + 1)
    return lo, cell, dims


def _device_pairs(Xd, Xh, h, nbsrange, dp_body, notches):
    """CSR (indptr int64, indices int32) on the device."""
    import torch
    L = _lib.lib()
    n = int(Xh.shape[0])
    if n < 2:
        raise CaseError("need at least 2 particles to build neighbors")
    mode = 0 if nbsrange is None else 1
    win = 0.0 if mode == 0 else nbsrange * dp_body * (1.0 + 1e-9)
    lo, cell, dims = _grid_params(Xh, 2.0 * h if mode == 0 else win)
    frames = [notch_struct(q) for q in notches]
    arr = (_lib.tl_notch * max(len(frames), 1))(*frames) if frames else None
    p = _lib.tl_nb_params(n=n, X=_lib.ptr(Xd), mode=mode, h=float(h), win=float(win),
                          lo=(_lib.D * 3)(*lo), cell=float(cell), dims=(_lib.I64 * 3)(*dims),
                          n_notch=len(frames),
                          notches=_lib.C.cast(arr, _lib.P) if frames else None)
    st = _lib.stream_ptr()
    plan = _lib.P()
    _lib.check(L.tl_nb_plan_create(st, _lib.C.byref(p), _lib.C.byref(plan)), "tl_nb_plan_create")
    try:
        counts = torch.empty(n, dtype=torch.int64, device=Xd.device)
        _lib.check(L.tl_nb_count(plan, _lib.ptr(counts)), "tl_nb_count")
        indptr = torch.zeros(n + 1, dtype=torch.int64, device=Xd.device)
        torch.cumsum(counts, 0, out=indptr[1:])
        nnz = int(indptr[-1].item())
        if nnz == 0:
            raise CaseError("no neighbor pairs found (body too sparse for the kernel support)")
        indices = torch.empty(nnz, dtype=torch.int32, device=Xd.device)
        _lib.check(L.tl_nb_fill(plan, _lib.ptr(indptr), _lib.ptr(indices)), "tl_nb_fill")
    finally:
        L.tl_nb_plan_destroy(plan)
    return indptr, indices, counts


def build_pairs(positions, h, nbsrange=None, dp_body=None):
    """Symmetric pair list (rows, cols) in lexsort((cols, rows)) order
    (kernel_geom.py:65-97), built on the device."""
    import torch
    Xh = np.ascontiguousarray(positions, dtype=np.float64)
    Xd = torch.from_numpy(Xh).cuda()
    indptr, indices, counts = _device_pairs(Xd, Xh, h, nbsrange, dp_body, ())
    rows = np.repeat(np.arange(Xh.shape[0], dtype=np.int64), counts.cpu().numpy())
    return rows, indices.to(torch.int64).cpu().numpy()


def build_device_adjacency(positions, V0, h, dim, kind, nbsrange=None, dp_body=None,
                           notches=(), correction=True, required=None):
    """The device half of build_adjacency: returns a DeviceAdjacency.
    ``required``: optional bool mask of the rows that must have neighbours
    (a rank's owned rows; halo-region rows at the subset edge may not)."""
    import torch
    Xh = np.ascontiguousarray(positions, dtype=np.float64)
    if Xh.shape[0] < 2:
        raise CaseError("need at least 2 particles to build neighbors")
    for q in notches:   # frame validation raises CaseError like the reference
        notch_struct(q)
    Xd = torch.from_numpy(Xh).cuda()
    indptr, indices, counts = _device_pairs(Xd, Xh, h, nbsrange, dp_body, notches)
    empty = counts == 0
    if required is not None:
        empty &= torch.as_tensor(np.asarray(required, dtype=bool), device=empty.device)
    lonely = torch.nonzero(empty)
    if lonely.numel():
        raise CaseError(f"particle {int(lonely[0, 0])} has no neighbors after notch severing")
    V0d = torch.from_numpy(np.ascontiguousarray(V0, dtype=np.float64)).cuda()
    n = Xh.shape[0]
    Ld = torch.empty((n, 9), dtype=torch.float64, device=Xd.device)
    fb = torch.zeros(1, dtype=torch.int64, device=Xd.device)
    alpha = kernel_alpha(h, dim, kind)
    L = _lib.lib()
    _lib.check(L.tl_correction(_lib.stream_ptr(), n, _lib.ptr(indptr), _lib.ptr(indices),
                               _lib.ptr(Xd), _lib.ptr(V0d), float(h), float(alpha), int(kind),
                               int(dim), int(bool(correction)), _lib.ptr(Ld), _lib.ptr(fb)),
               "tl_correction")
    return DeviceAdjacency(Xd, indptr, indices, Ld, int(fb.item()), h, dim, kind, correction)


def build_adjacency(positions, V0, h, dim, kind, nbsrange=None, dp_body=None, notches=(),
                    correction=True):
    """Drop-in for kernel_geom.build_adjacency (kernel_geom.py:220-261)."""
    dev = build_device_adjacency(positions, V0, h, dim, kind, nbsrange=nbsrange,
                                 dp_body=dp_body, notches=notches, correction=correction)
    return LazyAdjacency(dev)
