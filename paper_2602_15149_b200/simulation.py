"""Device-resident drop-in for ``solidsph.stepper.Simulation``.

Same public surface as the reference (/root/reference/pkg/src/solidsph/
stepper.py:49-263): ``DeviceSimulation(config, trace=None)`` with
``initialize() / step(dt) / pick_dt() / run(time_max, time_out, on_output,
max_steps)`` and attributes ``t, step_index, bodies, be, trace,
contact_warnings``.  ``config`` may be this package's ``CaseConfig`` or the
reference's (duck-typed).

What differs is where the state lives: every body's particle state sits in
HBM in the structure-of-arrays / gather-record layout of include/tlsph.h
and the whole step -- F, stress, phase field, momentum, boundary conditions,
integrator, dt -- runs in libtlsph kernels (pass A, pass B, device clock).
The host ``body.state`` arrays are mirrors: refreshed before every
``on_output`` callback, after ``step()`` and at the end of ``run()``
(``sync_host()``), and pushed back with ``push_state()`` after host edits.

Errors the reference raises inside the step (SimulationError for non-finite
acceleration, eigen non-convergence, non-SPD plastic metric; ExprError for
expression domain errors) are recorded on the device and raised at the next
sync point -- after every ``step()`` call, and at the end of each batch of
device-clock steps in ``run()`` -- with the reference's messages.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import _lib, backend, dist, kernel_geom
from . import expr as ex
from .core import CaseError, Model, SimulationError

INT64_MAX = np.iinfo(np.int64).max
N_COUNTERS = 8
# particles per CTA / shared-memory tile, one per thread (TLSPH_TILE overrides;
# a multiple of 32, at most 256)
# measured on B200 (C4, bond classes): FP32 256 particles per tile (6.90 -> 6.99
# G particle-steps/s against 160; pass B 1.31 -> 1.28 ms); FP64 (128 registers per
# thread) 128 (2.69 -> 2.91)
DEFAULT_TILE = {"fp32": 256, "fp64": 128}
TILE_SMEM_LIMIT = 200 * 1024  # bytes of shared memory a pass-B tile may take


def _torch():
    import torch
    return torch


def _mean_row(dadj, rows=None):
    """Mean neighbours per particle of a device adjacency, over ``rows``
    (a rank's owned rows; default all).  A slab's halo-region rows have
    truncated lists and must not steer the tile choice."""
    n = int(dadj.indptr.shape[0]) - 1
    if rows is None:
        return float(dadj.indptr[-1].item()) / max(n, 1)
    torch = _torch()
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dadj.indptr.device)
    cnt = (dadj.indptr[r + 1] - dadj.indptr[r]).sum()
    return float(cnt.item()) / max(int(r.shape[0]), 1)


class DeviceBody:
    """Device buffers and the tl_body descriptor of one body."""

    def __init__(self, body, config, precision, programs, mirrors=True, part=None):
        """part: this rank's share of the body (multi-GPU, see
        DeviceSimulation._partition); None = the whole body on this device."""
        torch = _torch()
        self.mirrors = mirrors
        self.body = body
        self.part = part
        st = body.state
        self.host = st           # the host arrays behind body.state (see DeviceState)
        self.dirty = False
        self.R = torch.float32 if precision == "fp32" else torch.float64
        dev = torch.device("cuda")
        self.dev = dev
        mat = body.material
        kind = int(config.kernel)
        corr = getattr(body, "kernel_correction", True)
        if part is not None:
            sub = part.host_rows
            dadj = kernel_geom.build_device_adjacency(
                st.X[sub], st.V0[sub], body.h, body.dim, kind, nbsrange=body.nbsrange,
                dp_body=body.dp_body, notches=body.notches, correction=corr,
                required=part.owned_mask)
        else:
            adj = body.adjacency
            dadj = getattr(adj, "device", None) if adj is not None else None
            if dadj is None:
                if adj is not None:
                    dadj = _upload_adjacency(adj, st, body, kind)
                else:
                    dadj = kernel_geom.build_device_adjacency(
                        st.X, st.V0, body.h, body.dim, kind, nbsrange=body.nbsrange,
                        dp_body=body.dp_body, notches=body.notches, correction=corr)
        self.adj = dadj
        # device particle order + neighbour tiles (kernel_geom.StepLayout)
        tile = DEFAULT_TILE[precision]
        if int(body.dim) == 2:
            tile = 128    # 2D stencils: thin 1-deep halos, measured best for pass A (C5)
        elif precision == "fp32" and _mean_row(
                dadj, part.owned_rows if part is not None else None) > 64.0:
            # radial 3D stencils: pass A gathers from L2 and pass B runs one CTA
            # per SM with split rows; the widest tile has the thinnest halo per
            # member (pass B, C2: 1.38 -> 1.17 ms, C3: 5.78 -> 4.76 ms)
            tile = 256
        tile = int(os.environ.get("TLSPH_TILE", str(tile)))
        # lattice-brick mode (kernel_geom.BrickLayout): single-device 3D lattice
        # bodies with wide stencils (> 64 neighbours per particle), uniform V0
        # and m0.  TLSPH_BRICK=0 disables it, =force ignores the stencil width.
        V0h = np.asarray(st.V0, dtype=np.float64)
        m0h = np.asarray(st.m0, dtype=np.float64)
        uniform = bool(np.all(V0h == V0h[0]) and np.all(m0h == m0h[0]))
        self.brick = None
        env_k = os.environ.get("TLSPH_BRICK", "1")
        if (part is None and int(body.dim) == 3 and uniform and env_k != "0"
                and (env_k == "force" or _mean_row(dadj) > 64.0)):
            self.brick = kernel_geom.BrickLayout.plan(dadj, float(body.dp_body), float(body.h),
                                                      kind, precision)
        if part is not None:
            part.complete(dadj)          # halo ids in exchange order (collective-free)
            lay = kernel_geom.StepLayout(dadj, tile=tile, rows=part.owned_rows,
                                         halo=part.halo_rows, precision=precision)
        elif self.brick is not None:
            lay = kernel_geom.StepLayout(dadj, tile=0, precision=precision,
                                         order=self.brick.order)
            self.brick.finish(lay)
        else:
            lay = kernel_geom.StepLayout(dadj, tile=tile, precision=precision)
        rec = 64 if precision == "fp32" else 128          # pass-B bytes per staged particle
        if lay.tile and (lay.tile + lay.hmax) * rec > TILE_SMEM_LIMIT:
            lay.tile = 0                                   # halo too fat: gather from L2
        if lay.tile and ((lay.tile + lay.hmax) * rec + 2 * lay.slmax > TILE_SMEM_LIMIT
                         or os.environ.get("TLSPH_SLOT_STAGE", "1") == "0"):
            lay.slmax = 0                                  # slot table read from global memory
        self.layout = lay
        n, n_all = lay.n, lay.n_all
        self.n, self.n_all = n, n_all
        self.perm = lay.perm                               # device pos -> adjacency id
        pl = lay.perm.long()
        adj_ids = lay.perm.cpu().numpy().astype(np.int64)
        # device position -> caller (global) particle index
        self.gid = part.sub[adj_ids] if part is not None else adj_ids
        # device position -> row of the host state arrays (== gid unless the
        # host holds only this rank's slab, cases.make_case(slab=...))
        self.hrow = part.host_rows[adj_ids] if part is not None else adj_ids
        self.perm_h = self.gid
        if part is not None:
            self.perm_global = torch.from_numpy(self.gid.astype(np.int32)).to(dev)
        else:
            self.perm_global = self.perm
        self.soff, self.sidx = lay.soff, lay.sidx
        R = self.R
        z = lambda *shape: torch.zeros(shape, dtype=R, device=dev)  # noqa: E731
        # all planes use stride n_all; halo rows of own-only fields stay unused
        self.Xs = dadj.X.index_select(0, pl).t().contiguous()                 # 3 planes
        self.L = dadj.L.index_select(0, pl).t().contiguous().to(R)             # 9 planes
        V0 = np.asarray(st.V0, dtype=np.float64)
        m0 = np.asarray(st.m0, dtype=np.float64)
        self.uniform = bool(np.all(V0 == V0[0]) and np.all(m0 == m0[0]))
        self.V0 = torch.from_numpy(V0[self.hrow]).to(dev)
        self.m0 = torch.from_numpy(m0[self.hrow]).to(dev)
        N = n_all
        self.us = z(N, 4)
        self.rb = z(N, 12)
        self.v = z(3, N)
        self.al = z(9, N)
        self.sdot = z(N)
        self.sddot = z(N)
        self.Hh = z(N)
        self.Cpd = z(6, N) if mat.model == Model.J2 else z(6, 1)
        self.epbar = z(N)
        self.a = z(3, N)
        f64 = lambda *shape: torch.zeros(shape, dtype=torch.float64, device=dev)  # noqa: E731
        # FP64 host-layout mirrors of F, S, psi (written only on output steps)
        self.F_out = f64(n, 3, 3) if mirrors else None
        self.S_out = f64(n, 3, 3) if mirrors else None
        self.psi_out = f64(n) if mirrors else None
        self.psip_out = f64(n) if mirrors else None
        # pass B tiling: with few neighbours per particle (2D stencils) an FP32
        # tile's short compute cannot hide its staging latency, and the
        # L2-gather pass B measured faster on B200 (C5: 8.96 vs 11.9 ms); FP64
        # 2D gathers twice the bytes per pair and the tiles win there (C5
        # FP64: 12.5 vs 16.4 ms).  Pass A keeps its tiles either way.
        # TLSPH_TILE_B=0/1 overrides.
        env_b = os.environ.get("TLSPH_TILE_B")
        self.tile_b = bool(lay.tile) and (int(env_b) != 0 if env_b is not None
                                          else (int(body.dim) == 3 or precision == "fp64"))
        # pass A tiling: radial 3D stencils (k ~ 165) on 160-particle tiles
        # (FP64) stage ~13 halo records per member and gather faster from L2
        # (measured in FP32: C2 0.60 vs 0.68 ms, C3 3.0 vs 3.55 ms); on the
        # FP32 256-particle tiles the tiled pass A wins (C2 0.38 vs 0.58 ms,
        # C3 2.55 vs 2.69 ms).  TLSPH_TILE_A overrides.
        env_a = os.environ.get("TLSPH_TILE_A")
        k_mean = float(lay.indptr[-1].item()) / max(n, 1)
        wide = precision == "fp32" and int(body.dim) == 3
        self.tile_a = bool(lay.tile) and (int(env_a) != 0 if env_a is not None
                                          else (k_mean <= 64.0 or wide))
        # radial 3D stencils, FP32: their tiled pass B runs one CTA per SM
        # (shared memory), so 4 threads per member split each row to give that
        # CTA 4x the warps (256-particle tiles, pass B: C2 1.48 -> 1.17 ms, C3
        # 5.53 -> 4.76 ms).  TLSPH_BSPLIT=1/4 overrides.
        env_s = os.environ.get("TLSPH_BSPLIT")
        split_ok = (self.tile_b and precision == "fp32" and int(body.dim) == 3
                    and 4 * int(lay.tile) <= 1024
                    and ((lay.tile + lay.hmax) * 64 + 2 * lay.slmax + 16 + 3 * 36 * lay.tile
                         <= TILE_SMEM_LIMIT))
        self.bsplit = (4 if split_ok and (int(env_s) == 4 if env_s is not None
                                          else k_mean > 64.0) else 1)
        # bond classes (lattice bodies, uniform V0 and m0): the tiled passes
        # take the pair geometry from a per-class table instead of staged
        # position records (kernel_geom.StepLayout.bond_classes).
        # TLSPH_BOND_CLASS=0 keeps the position path.
        self.bcls = None
        if (lay.tile and self.uniform and self.bsplit == 1
                and os.environ.get("TLSPH_BOND_CLASS", "1") != "0"):
            self.bcls = lay.bond_classes(self.Xs, float(body.dp_body), float(body.h), kind,
                                         precision)
        # staged tile positions with the pass-A (V0) and pass-B (m0) weights
        if lay.tile and self.bcls is None:
            self.tpos_a = lay.positions(self.Xs, None if self.uniform else self.V0, precision)
            self.tpos_b = (self.tpos_a if self.uniform
                           else lay.positions(self.Xs, self.m0, precision))
        else:
            self.tpos_a = self.tpos_b = None
        # multi-GPU: interior tiles first (they overlap the halo exchange)
        self.tlist, self.n_interior = lay.split_tiles() if part is not None else (None, 0)
        self.counters = torch.zeros(N_COUNTERS, dtype=torch.int64, device=dev)
        self.red = torch.zeros(2, dtype=torch.int64, device=dev)
        # one plastic-work partial per pass-A CTA: tiled launches use CTAs of
        # `tile` particles, untiled ones of 256 (tl_pass_blocks)
        self.nblocks = int(_lib.lib().tl_pass_blocks(n))
        if lay.tile:
            self.nblocks = max(self.nblocks, (n + lay.tile - 1) // lay.tile)
        if self.brick is not None:
            self.nblocks = max(self.nblocks, self.brick.nbricks)
        self.pw_partial = torch.zeros(max(self.nblocks, 1), dtype=torch.float64, device=dev)
        self.pw_acc = torch.zeros(1, dtype=torch.float64, device=dev)
        self.pw_base = float(getattr(body, "plastic_work", 0.0))
        self.deg_base = int(getattr(body, "degenerate_warnings", 0))
        self._reset_counters()
        self._setup_bcs(body, config, programs)
        self.push_state()
        self.desc = self._descriptor(mat, body, kind, precision)

    # -- boundary conditions -------------------------------------------------
    def _setup_bcs(self, body, config, programs):
        torch = _torch()
        bcs = list(getattr(body, "bcs", []))
        if len(bcs) > _lib_max_bc():
            raise CaseError(f"body {body.mk}: more than {_lib_max_bc()} boundary conditions")
        mask = np.zeros(self.host.X.shape[0], dtype=np.uint32)
        bit = 0
        X0 = np.asarray(self.host.X, dtype=np.float64)
        # static skip patterns (expr.nonskip_mask / nonskip_mask_after) become
        # targeted bits while bits remain for the explicit targets and
        # restrictphi.  Bodies whose pass B is a single wave (under ~38 k
        # particles) keep whole-body expressions whole: there the kernel is
        # latency-bound and warps mixing BC and BC-free particles run both
        # paths (C1: 32 -> 37 us); TLSPH_STATIC_SKIP=1 forces, =0 disables.
        # A targeted entry whose late-time value is one literal number on all
        # its particles (expr.late_constant: C1's clamped end is 0.0 after
        # t = 0) stores the constant and runs no expression at all, so small
        # bodies convert those too (C1 pass B 31 -> 24 us).
        n_explicit = sum(1 for bc in bcs if bc.target is not None)
        env_ss = os.environ.get("TLSPH_STATIC_SKIP", "auto")
        static_ok = env_ss == "1" or (env_ss != "0" and X0.shape[0] > 148 * 256)
        const_ok = static_ok or env_ss == "auto"
        # device entries in file order: (bc, bit, tst, tend, guard, late-time
        # constants); a whole-body BC whose pattern is static after a time T
        # becomes two time-disjoint entries, whole-body up to T and targeted
        # after it (the windows are inclusive on the device, so the second
        # starts at the next double)
        entries = []
        for k, bc in enumerate(bcs):
            if bc.kind == "force" and int(getattr(bc, "ftype", 0) or 0) not in (1, 2, 3):
                raise CaseError(f"unknown force BC type {bc.ftype}")
            tst = float(bc.tst)
            tend = float(bc.tend) if math.isfinite(bc.tend) else 1e308
            if bc.target is not None:
                if bit >= 32:
                    raise CaseError(f"body {body.mk}: more than 32 targeted boundary conditions")
                mask[np.asarray(bc.target, dtype=np.int64)] |= np.uint32(1 << bit)
                entries.append((bc, bit, tst, tend, None, None))
                bit += 1
                continue
            # a split adds one device entry: room for it and every BC still to come
            room = _lib_max_bc() - (len(entries) + len(bcs) - k)
            got = (self._static_targets(bc, config, X0)
                   if const_ok and bit + n_explicit < 31 and room >= 1 else None)
            lconst = self._late_constants(bc, config, X0) if got is not None else None
            if got is not None and not static_ok and lconst is None:
                got = None                 # small body: only constant-folded entries pay
            if got is None:
                entries.append((bc, -1, tst, tend, self._skip_guard(bc, config)
                                if static_ok else None, None))
                continue
            T, tgt = got
            if T >= tend:                  # static only after the BC has ended
                entries.append((bc, -1, tst, tend, None, None))
                continue
            if T >= tst:
                entries.append((bc, -1, tst, T, None, None))
                tst = float(np.nextafter(T, np.inf))
            mask[tgt] |= np.uint32(1 << bit)
            entries.append((bc, bit, tst, tend, None, lconst))
            bit += 1
        if len(entries) > _lib_max_bc():
            raise CaseError(f"body {body.mk}: more than {_lib_max_bc()} boundary conditions")
        arr = (_lib.tl_bc * max(len(entries), 1))()
        self.bc_whole = 0
        self.bcw_lo, self.bcw_hi = math.inf, -math.inf   # activity window of whole-body entries
        for k, (bc, bbit, tst, tend, guard, lconst) in enumerate(entries):
            d = arr[k]
            d.kind = 0 if bc.kind == "vel" else 1
            d.ftype = int(getattr(bc, "ftype", 0) or 0)
            d.bit = bbit
            d.gvar = -1
            if guard is not None:
                d.gt, d.gvar, d.gop, d.gc = guard
            if bbit < 0:
                self.bc_whole = 1
                self.bcw_lo = min(self.bcw_lo, tst)
                self.bcw_hi = max(self.bcw_hi, tend)
            for ax in range(3):
                c = bc.const[ax]
                e = bc.expr[ax]
                if lconst is not None and lconst[ax] is not None:
                    c, e = lconst[ax], None    # the expression's late-time literal
                d.has_const[ax] = int(c is not None)
                d.cval[ax] = float(c) if c is not None else 0.0
                if c is None and e is not None:
                    ast = config.expressions.get(e)
                    if ast is None:
                        raise CaseError(
                            f"boundary condition references unknown expression id {e}")
                    d.prog[ax] = programs.index_of(e, ast)
                else:
                    d.prog[ax] = -1
            d.tst = tst
            d.tend = tend
        self.nbc = len(entries)
        self._bc_arr = arr
        nbytes = C.sizeof(_lib.tl_bc) * max(len(entries), 1)
        self.bcs_dev = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        host = torch.frombuffer(bytearray(C.string_at(C.addressof(arr), nbytes)), dtype=torch.uint8)
        self.bcs_dev.copy_(host)
        rp = getattr(body, "restrictphi_expr", None)
        self.restrict_bit = -1
        if rp is not None:
            ast = config.expressions.get(rp)
            if ast is None:
                raise CaseError(f"restrictphi references unknown expression id {rp} "
                                f"(body {body.mk})")
            self.restrict_prog = programs.index_of(rp, ast)
            nz = ex.nonskip_mask(ast, X0) if (static_ok and bit < 32) else None
            if nz is not None:     # evaluate it only where it is not skip
                self.restrict_bit = bit
                mask[np.flatnonzero(nz)] |= np.uint32(1 << bit)
                bit += 1
        else:
            self.restrict_prog = -1
        self.bcmask = torch.from_numpy(mask[self.hrow].view(np.int32)).to(self.dev)

    @staticmethod
    def _skip_guard(bc, config):
        """(T, var, op, c) when every expression axis of a whole-body BC is
        skip for t > T wherever the same single comparison ``var op c`` is
        false (expr.skip_guard_after) and no axis is a constant; else None."""
        guard = None
        T = -math.inf
        for ax in range(3):
            c, e = bc.const[ax], bc.expr[ax]
            if c is not None:
                return None
            if e is None:
                continue
            ast = config.expressions.get(e)
            g = ex.skip_guard_after(ast) if ast is not None else None
            if g is None or (guard is not None and g[1:] != guard):
                return None
            guard = g[1:]
            T = max(T, g[0])
        return None if guard is None else (T,) + guard

    @staticmethod
    def _late_constants(bc, config, X0):
        """Per-axis literal (None for an axis without an expression) when every
        expression axis of the BC takes one literal number wherever it is not
        skip after its threshold (expr.late_constant); else None."""
        out = [None, None, None]
        sel = None
        for ax in range(3):
            e = bc.expr[ax]
            if bc.const[ax] is not None or e is None:
                continue
            ast = config.expressions.get(e)
            v = ex.late_constant(ast, X0) if ast is not None else None
            got = ex.nonskip_mask_after(ast, X0) if v is not None else None
            # the entry targets the union of the axes' non-skip sets: a
            # constant must not land where its own axis is skip
            if got is None or (sel is not None and not np.array_equal(sel, got[1])):
                return None
            sel = got[1]
            out[ax] = v
        return tuple(out) if sel is not None else None

    @staticmethod
    def _static_targets(bc, config, X0):
        """(T, particles) for a whole-body BC whose every expression axis has
        a skip pattern fixed by x0, y0, z0 for t > T (expr.nonskip_mask_after;
        T = -inf when it never depends on t) and no axis is a constant: the
        particles it can act on after T.  None otherwise (or when that is
        every particle)."""
        sel = np.zeros(X0.shape[0], dtype=bool)
        T = -math.inf
        any_expr = False
        for ax in range(3):
            c, e = bc.const[ax], bc.expr[ax]
            if c is not None:
                return None
            if e is None:
                continue
            ast = config.expressions.get(e)
            if ast is None:
                return None            # _setup_bcs raises the reference's error
            got = ex.nonskip_mask_after(ast, X0)
            if got is None:
                return None
            T = max(T, got[0])
            sel |= got[1]
            any_expr = True
        if not any_expr or sel.all():
            return None
        return T, np.flatnonzero(sel)

    def _descriptor(self, mat, body, kind, precision):
        b = _lib.tl_body()
        b.n = self.n
        b.n_all = self.n_all
        b.dim = int(body.dim)
        b.model = int(mat.model)
        b.fracture = int(bool(body.fracture))
        b.visc = int(mat.beta1 != 0.0 or mat.beta2 != 0.0)
        b.precision = 4 if precision == "fp32" else 8
        b.kind = kind
        b.uniform = int(self.uniform)
        b.write_out = 0
        b.store_a = 0
        b.nbc = self.nbc
        b.mk = int(body.mk)
        b.restrict_prog = self.restrict_prog
        b.restrict_bit = self.restrict_bit
        b.bc_whole = self.bc_whole
        b.bcw_lo, b.bcw_hi = float(self.bcw_lo), float(self.bcw_hi)
        h = float(body.h)
        b.h, b.inv_h = h, 1.0 / h
        b.alpha = kernel_geom.kernel_alpha(h, body.dim, kind)
        for k in ("rho0", "lam", "mu", "kappa", "beta1", "beta2", "Gc", "eps0", "s_l",
                  "sigma_y0", "H_hard"):
            setattr(b, k, float(getattr(mat, k)))
        b.c0 = float(mat.c0)
        b.inv_Gc = 1.0 / b.Gc if b.Gc else 0.0
        b.inv_eps0 = 1.0 / b.eps0 if b.eps0 else 0.0
        b.inv_c0 = 1.0 / b.c0 if b.c0 else 0.0
        b.V0c = float(self.body.state.V0[0])
        b.m0c = float(self.body.state.m0[0])
        b.dp_body = float(body.dp_body)
        b.jac_tol = 1e-30 if precision == "fp64" else 1e-12
        for k in range(3):
            b.f0[k] = float(body.f0[k])
        P = _lib.ptr
        b.soff, b.sidx, b.Xs, b.L = P(self.soff), P(self.sidx), P(self.Xs), P(self.L)
        b.wlen = P(self.layout.wlen)
        lay = self.layout
        b.tile, b.hmax, b.slmax = int(lay.tile), int(lay.hmax), int(lay.slmax)
        b.bsplit = int(getattr(self, "bsplit", 1))
        # L2-gather pass B on small FP32 bodies: up to 4 lanes per particle
        # while the grid stays one wave (148 SMs x 1024 threads) -- each lane's
        # chain of dependent gathers is 1/lpp as long (C1 pass B 24 -> 21 us;
        # 8 lanes measured slower: the epilogue runs on one lane in eight).
        # FP64, the parity mode, sums every row in CSR order (lpp 1).
        # TLSPH_LPP overrides.
        lpp = 1
        if precision == "fp32":
            while lpp < 4 and self.n * lpp * 2 <= 148 * 1024:
                lpp *= 2
        b.lpp = int(os.environ.get("TLSPH_LPP", str(lpp)))
        if lay.tile:
            b.hoff, b.halo, b.slots, b.hslot = (P(lay.hoff), P(lay.halo), P(lay.slots),
                                                P(lay.hslot))
            b.toff, b.tpos_a, b.tpos_b = P(lay.toff), P(self.tpos_a), P(self.tpos_b)
        if self.bcls is not None:
            b.ncls, b.bcls = int(self.bcls.shape[0]), P(self.bcls)
            # the tiled passes read the class geometry from the constant bank
            # (tl_body.bcls_host): C4 FP32 pass B 1.30 -> 1.26 ms, C5 FP32 pass A
            # 5.65 -> 5.58 ms, C5 FP64 pass B flat; FP64 3D keeps the shared-
            # memory table (C4 FP64 pass B 3.34 vs 3.43 ms).  TLSPH_CLS_CONST=0
            # keeps it everywhere.
            if (os.environ.get("TLSPH_CLS_CONST", "1") != "0"
                    and (precision == "fp32" or int(body.dim) == 2)):
                self._bcls_host = np.ascontiguousarray(self.bcls.cpu().numpy())
                b.bcls_host = self._bcls_host.ctypes.data
        if self.brick is not None:
            self.brick.fill(b)
        b.perm = P(self.perm_global)
        b.V0, b.m0 = P(self.V0), P(self.m0)
        for k in ("us", "rb", "v", "al", "sdot", "sddot", "Hh", "Cpd", "epbar", "a"):
            setattr(b, k, P(getattr(self, k)))
        b.F_out, b.S_out, b.psi_out, b.psip_out = (P(self.F_out), P(self.S_out),
                                                  P(self.psi_out), P(self.psip_out))
        b.bcmask, b.bcs = P(self.bcmask), P(self.bcs_dev)
        b.red, b.counters, b.pw_partial = P(self.red), P(self.counters), P(self.pw_partial)
        return b

    def _reset_counters(self):
        c = self.counters
        c.zero_()
        c[2] = INT64_MAX
        c[3] = INT64_MAX
        c[6] = INT64_MAX
        c[7] = INT64_MAX

    # -- host mirrors ------------------------------------------------------------
    def _gid_dev(self):
        """Device copy of gid (device row -> host row), and for a whole-body
        device its inverse over the owned rows."""
        if getattr(self, "_gidd", None) is None:
            torch = _torch()
            self._gidd = torch.from_numpy(np.asarray(self.hrow, dtype=np.int64)).to(self.dev)
            nh = int(self.host.X.shape[0])
            if self.n == nh:
                inv = torch.empty(nh, dtype=torch.int64, device=self.dev)
                inv[self._gidd[:self.n]] = torch.arange(self.n, dtype=torch.int64,
                                                        device=self.dev)
                self._invd = inv
            else:
                self._invd = None
        return self._gidd, self._invd

    def push_state(self):
        """Upload body.state (host, FP64, original order) into the device
        layout and order: each host array goes up as is (one contiguous copy,
        DMA when the host state is pinned, see pin_host) and is permuted on
        the device."""
        torch = _torch()
        st = self.host
        R, dev = self.R, self.dev
        g, _ = self._gid_dev()

        def up(arr):
            # asynchronous from page-locked arrays: the fields' copies run back
            # to back on the stream (DeviceSimulation.push_state syncs once)
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(
                dev, non_blocking=True)
            return t.index_select(0, g)

        self.us[:, :3].copy_(up(st.u))
        self.us[:, 3].copy_(up(st.s))
        self.v.copy_(up(st.v).t())
        self.a.copy_(up(st.a).t())
        for name, arr in (("sdot", st.sdot), ("sddot", st.sddot), ("Hh", st.Hhist),
                          ("epbar", st.epbar)):
            getattr(self, name).copy_(up(arr))
        if self.body.material.model == Model.J2 and st.Cp is not None:
            Cp = up(np.asarray(st.Cp, dtype=np.float64).reshape(-1, 9))
            cpd = torch.stack([Cp[:, 0] - 1.0, Cp[:, 4] - 1.0, Cp[:, 8] - 1.0,
                               Cp[:, 1], Cp[:, 2], Cp[:, 5]])
            self.Cpd.copy_(cpd)
        self.refresh_dt_maxima()
        torch.cuda.current_stream().synchronize()     # the host arrays are free again

    def pin_host(self):
        """Page-lock the host state arrays (cudaHostRegister) so push_state /
        pull_state move them by DMA.  Idempotent."""
        if getattr(self, "_pinned", False):
            return
        torch = _torch()
        st = self.host
        for k in ("u", "v", "a", "s", "sdot", "sddot", "Hhist", "epbar", "F", "S", "psi_e",
                  "psi_plus", "Cp"):
            arr = getattr(st, k, None)
            if isinstance(arr, np.ndarray) and arr.flags.c_contiguous and arr.nbytes:
                # a failure (e.g. pages shared with an already registered
                # array) leaves that array on the pageable path
                torch._C._cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
        self._pinned = True

    def pull_state(self, full=True):
        """Refresh body.state (host, original order) from the device.  A
        whole-body device permutes on the device and copies each field
        straight into the host array; a slab fills its owned rows."""
        torch = _torch()
        st = self.host
        n = self.n
        self.dirty = False
        _, inv = self._gid_dev()
        pm = self.hrow[:n]                             # owned device rows only

        def put(dst, val):
            """val: device (n_rows, ...) in device order, rows >= n ignored.
            A host field the case did not allocate (lean layouts) is skipped."""
            if dst is None:
                return
            val = val[:n].double()
            if inv is not None and dst.flags.c_contiguous and dst.dtype == np.float64:
                # asynchronous into page-locked arrays (DeviceSimulation.pull_host
                # syncs once after every field is queued)
                torch.from_numpy(dst).copy_(val.index_select(0, inv).reshape(dst.shape),
                                            non_blocking=True)
            else:
                dst[pm] = val.cpu().numpy().reshape((n,) + dst.shape[1:])

        put(st.u, self.us[:, :3])
        put(st.s, self.us[:, 3])
        put(st.v, self.v.t())
        put(st.sdot, self.sdot)
        put(st.sddot, self.sddot)
        put(st.Hhist, self.Hh)
        put(st.epbar, self.epbar)
        if full and self.mirrors:
            put(st.a, self.a.t())
            put(st.F, self.F_out)
            put(st.S, self.S_out)
            put(st.psi_e, self.psi_out)
            put(st.psi_plus, self.psip_out)
        if self.body.material.model == Model.J2 and st.Cp is not None:
            c = self.Cpd.double()[:, :n]
            Cp = torch.stack([1.0 + c[0], c[3], c[4], c[3], 1.0 + c[1], c[5],
                              c[4], c[5], 1.0 + c[2]], dim=1).reshape(n, 3, 3)
            put(st.Cp, Cp)
        torch.cuda.current_stream().synchronize()     # every queued copy has landed

    def refresh_dt_maxima(self):
        """max |v|^2 and max |a|^2 of the owned rows into ``red`` (what pass B
        leaves there), so pick_dt after a host edit sees the edited state like
        the reference's (stepper.py:221-233): FP64 squares in numpy's einsum
        order (x*x + z*z) + y*y of the mode's values; a NaN counts as 0 (pass B
        reports it through the error counters).  Not collective: the slab path
        all-reduces ``red`` in the next pass B."""
        torch = _torch()
        n = self.n
        out = []
        for pl in (self.v, self.a):
            d = pl[:, :n].double()
            sq = (d[0] * d[0] + d[2] * d[2]) + d[1] * d[1]
            sq = torch.where(torch.isnan(sq), torch.zeros_like(sq), sq)
            out.append(sq.max() if n else torch.zeros((), dtype=torch.float64, device=self.dev))
        self.red.copy_(torch.stack(out).view(torch.int64))

    def dtinfo(self):
        return _lib.tl_dtinfo(h=float(self.body.h), c0=float(self.body.material.c0),
                              red=_lib.ptr(self.red))


class DeviceState:
    """``body.state`` of a device-resident body.

    Attribute reads of the evolving fields copy the device state into the
    host arrays first if a step ran since the last copy, so host code (output
    writers, tests) sees the reference's ParticleArrays contract while the
    step loop never pays for a full-state device->host copy.  Writes go to
    the host arrays; call ``DeviceSimulation.push_state()`` after editing
    them in place."""

    _LIVE = frozenset(("u", "v", "a", "F", "S", "s", "sdot", "sddot", "Hhist", "Cp", "epbar",
                       "psi_e", "psi_plus", "x"))

    def __init__(self, host, dbody):
        object.__setattr__(self, "_host", host)
        object.__setattr__(self, "_db", dbody)

    def __getattr__(self, name):
        db = object.__getattribute__(self, "_db")
        if name in DeviceState._LIVE and db.dirty:
            db.pull_state()
        return getattr(object.__getattribute__(self, "_host"), name)

    def __setattr__(self, name, value):
        setattr(object.__getattribute__(self, "_host"), name, value)


def _lib_max_bc():
    return 32


def _upload_adjacency(adj, st, body, kind):
    """Device structure from a host (reference) Adjacency: its CSR is used
    as given; L_i is recomputed on the device from the positions."""
    torch = _torch()
    dev = torch.device("cuda")
    X = torch.from_numpy(np.ascontiguousarray(st.X, dtype=np.float64)).to(dev)
    indptr = torch.from_numpy(np.asarray(adj.indptr, dtype=np.int64)).to(dev)
    indices = torch.from_numpy(np.asarray(adj.indices, dtype=np.int64)).to(dev, torch.int32)
    n = X.shape[0]
    Ld = torch.empty((n, 9), dtype=torch.float64, device=dev)
    fb = torch.zeros(1, dtype=torch.int64, device=dev)
    corr = bool(getattr(body, "kernel_correction", True))
    alpha = kernel_geom.kernel_alpha(body.h, body.dim, kind)
    V0 = torch.from_numpy(np.asarray(st.V0, dtype=np.float64)).to(dev)
    _lib.check(_lib.lib().tl_correction(
        _lib.stream_ptr(), n, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(X), _lib.ptr(V0),
        float(body.h), float(alpha), int(kind), int(body.dim), int(corr), _lib.ptr(Ld),
        _lib.ptr(fb)), "tl_correction")
    return kernel_geom.DeviceAdjacency(X, indptr, indices, Ld, int(fb.item()), body.h,
                                       body.dim, kind, corr)


class ProgramTable:
    """All expressions of a case compiled once to device bytecode."""

    def __init__(self):
        self.ids = []
        self.progs = []

    def index_of(self, eid, ast):
        if eid in self.ids:
            return self.ids.index(eid)
        self.ids.append(eid)
        self.progs.append(ex.compile_program(ast))
        return len(self.ids) - 1

    def upload(self):
        torch = _torch()
        dev = torch.device("cuda")
        self.code = [torch.from_numpy(p.code.reshape(-1).copy()).to(dev) for p in self.progs]
        self.consts = [torch.from_numpy(p.consts.copy()).to(dev) for p in self.progs]
        arr = (_lib.tl_prog * max(len(self.progs), 1))()
        for k, p in enumerate(self.progs):
            arr[k].code = _lib.ptr(self.code[k])
            arr[k].consts = _lib.ptr(self.consts[k])
            arr[k].len = int(p.code.shape[0])
        nbytes = C.sizeof(_lib.tl_prog) * max(len(self.progs), 1)
        self.table = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.table.copy_(torch.frombuffer(bytearray(C.string_at(C.addressof(arr), nbytes)),
                                          dtype=torch.uint8))
        return self.table


class DeviceSimulation:
    """Drop-in for solidsph.stepper.Simulation running on one B200."""

    def __init__(self, config, trace=None, precision="fp64", stream=None, mirrors=True,
                 group=None, partition=None, hourglass=0.0):
        """partition: run the slab path (halo exchange, collectives) -- by
        default whenever a process group of more than one rank is initialised;
        True also with one rank (exercises the exchange plumbing).

        hourglass: alpha of the opt-in hourglass control (tl_hourglass,
        Ganzenmueller 2015; one GPU).  The reference has no such term, so there
        is nothing to check it against; 0 (the default) leaves the step the
        reference's."""
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        L = _lib.lib()  # fails loudly without the native library / GPU
        torch = _torch()
        self.config = config
        self.bodies = config.bodies
        self.expressions = config.expressions
        self.t = 0.0
        self.step_index = 0
        self.trace = trace
        self.be = backend
        self.precision = precision
        self.mirrors = mirrors
        self.contact_warnings = 0
        self._initialized = False
        self.stream = stream or torch.cuda.current_stream()
        self.group = group
        self.world = 1
        import torch.distributed as tdist
        if tdist.is_available() and tdist.is_initialized():
            self.world = tdist.get_world_size(group)
        self.partitioned = self.world > 1 if partition is None else bool(partition)
        self.peer = False
        if self.partitioned and not (tdist.is_available() and tdist.is_initialized()):
            raise ValueError("partition=True needs an initialised torch.distributed group")
        if len(self.bodies) > 1 and self.partitioned:
            raise NotImplementedError("multi-body (contact) cases run on one GPU")
        self.hourglass = float(hourglass)
        if self.hourglass < 0.0:
            raise ValueError("hourglass alpha must be >= 0")
        if self.hourglass and self.partitioned:
            raise NotImplementedError("hourglass control runs on one GPU (it reads F of "
                                      "halo partners, which the slab exchange does not carry)")
        parts = [self._partition(b) if self.partitioned else None for b in self.bodies]
        self.programs = ProgramTable()
        self.dbodies = [DeviceBody(b, config, precision, self.programs, mirrors, part)
                        for b, part in zip(self.bodies, parts)]
        for db in self.dbodies:
            db.exchange = None
            if db.part is not None:
                lay = db.layout
                pos = lay.iperm.index_select(
                    0, torch.from_numpy(db.part.owned_rows).to(lay.iperm.device)).cpu().numpy()
                plan = dist.build_halo_plan(db.part.owned_gid, pos, db.part.needed_gid,
                                            db.part.owner, group=group)
                assert plan.n_halo == db.n_all - db.n
                db.exchange = dist.HaloExchange(plan, "cuda", group=group)
                db.comm_stream = torch.cuda.Stream()
        # peer-memory halo (dist.PeerHalo, TLSPH_PEER=1; Verlet): the step
        # kernels store boundary records into the neighbours' halo rows
        self.peer = (self.partitioned and os.environ.get("TLSPH_PEER", "0") == "1"
                     and int(config.step_algorithm) != 2)
        if self.peer:
            halos = [dist.PeerHalo.build(db.exchange.plan, db.us, db.rb, group=group)
                     for db in self.dbodies]
            flag = torch.tensor([int(all(h is not None for h in halos))], dtype=torch.int64,
                                device="cuda")
            dist.allreduce(flag, "min", group)
            self.peer = bool(int(flag.item()))
            for db, h in zip(self.dbodies, halos):
                db.peer = h if self.peer else None
                if db.peer is not None:
                    db.peer.fill(db.desc)
            self._barrier_t = torch.zeros(1, dtype=torch.int64, device="cuda")
        for b, db in zip(self.bodies, self.dbodies):
            b.state = DeviceState(db.host, db)
        self._setup_contact(torch)
        if self.hourglass:
            from .core import youngs_from_lame
            for db in self.dbodies:
                db.Fh = torch.zeros((9, db.n_all), dtype=db.R, device=db.dev)
                if getattr(db, "ac", None) is None:
                    db.ac = torch.zeros((3, db.n_all), dtype=torch.float64, device=db.dev)
                mat = db.body.material
                E = youngs_from_lame(mat.lam, mat.mu)[0]
                db.desc.Fh = _lib.ptr(db.Fh)
                db.desc.ac = _lib.ptr(db.ac)
                db.desc.hg_coef = self.hourglass * E / (2.0 * mat.rho0)
        prog_table = self.programs.upload()
        self.clock_dev = torch.zeros(C.sizeof(_lib.tl_clock), dtype=torch.uint8,
                                     device="cuda")
        for db in self.dbodies:
            db.desc.progs = _lib.ptr(prog_table)
            db.desc.clock = _lib.ptr(self.clock_dev)
            db.desc.store_a = int(int(config.step_algorithm) == 2)
        self._lib = L
        self._dt_arr = (_lib.tl_dtinfo * len(self.dbodies))(*[db.dtinfo() for db in self.dbodies])
        self.workspaces = [None for _ in self.bodies]
        # CUDA graphs of fixed-length device-clock step batches (run / advance).
        # The descriptors are passed by value, so a graph stays valid while
        # they do; multi-GPU slabs keep eager launches (host-side exchange
        # scheduling).  TLSPH_GRAPHS=0 disables.
        self._graphs = {}
        self.use_graphs = (not self.partitioned and
                           os.environ.get("TLSPH_GRAPHS", "1") != "0")

    # -- penalty contact (dynamics.py:81-135) --------------------------------
    CONTACT_CELLS = 1 << 20      # cell-grid capacity of one body pair

    def _setup_contact(self, torch):
        """Per body pair, the reference's contact constants (dynamics.py:
        106-122) and a device workspace; per body, the contact-acceleration
        planes pass B adds before f0."""
        from .core import youngs_from_lame, damping_ratio
        self.contact_pairs = []
        self.contact_counters = None
        if len(self.dbodies) < 2:
            return
        contcoeff = float(getattr(self.config, "contcoeff", 1.0))
        for db in self.dbodies:
            db.ac = torch.zeros((3, db.n_all), dtype=torch.float64, device=db.dev)
            db.desc.ac = _lib.ptr(db.ac)
            s = _lib.tl_contact_side()
            s.n, s.n_all = db.n, db.n_all
            s.precision = 4 if db.R == torch.float32 else 8
            s.uniform, s.m0c = int(db.uniform), float(db.body.state.m0[0])
            s.Xs, s.us, s.v, s.m0, s.perm = (_lib.ptr(db.Xs), _lib.ptr(db.us), _lib.ptr(db.v),
                                             _lib.ptr(db.m0), _lib.ptr(db.perm_global))
            db.contact_side = s
        L = _lib.lib()
        for ia in range(len(self.dbodies)):
            for ib in range(ia + 1, len(self.dbodies)):
                a, b = self.bodies[ia], self.bodies[ib]
                dpc = 0.5 * (a.dp_body + b.dp_body)
                Ea = youngs_from_lame(a.material.lam, a.material.mu)[0]
                Eb = youngs_from_lame(b.material.lam, b.material.mu)[0]
                k_n = contcoeff * min(Ea, Eb) * dpc
                ma = float(np.mean(a.state.m0))
                mb = float(np.mean(b.state.m0))
                m_eff = ma * mb / (ma + mb)
                zeta = damping_ratio(min(a.material.restcoef, b.material.restcoef))
                c_n = 2.0 * zeta * math.sqrt(k_n * m_eff)
                kfric = 0.5 * (a.material.kfric + b.material.kfric)
                nbytes = _lib.I64(0)
                _lib.check(L.tl_contact_workspace_bytes(self.dbodies[ia].n, self.dbodies[ib].n,
                                                        self.CONTACT_CELLS, C.byref(nbytes)),
                           "tl_contact_workspace_bytes")
                work = torch.empty(int(nbytes.value), dtype=torch.uint8, device="cuda")
                self.contact_pairs.append((ia, ib, dpc, k_n, c_n, kfric, work))
        self.contact_counters = torch.zeros(2, dtype=torch.int64, device="cuda")

    def _contact(self):
        """Contact accelerations from x = X + u, v at the start of the force
        evaluation (pass A leaves u and v untouched)."""
        if not self.contact_pairs:
            return
        for db in self.dbodies:
            db.ac.zero_()
        dim = int(self.bodies[0].dim)
        for ia, ib, dpc, k_n, c_n, kfric, work in self.contact_pairs:
            A, B = self.dbodies[ia], self.dbodies[ib]
            _lib.check(self._lib.tl_contact_pair(
                self._st(), C.byref(A.contact_side), C.byref(B.contact_side), dim, dpc, k_n, c_n,
                kfric, self.CONTACT_CELLS, _lib.ptr(work), int(work.numel()), _lib.ptr(A.ac),
                _lib.ptr(B.ac), _lib.ptr(self.contact_counters)), "tl_contact_pair")

    def _between_passes(self):
        """Between pass A and pass B: penalty contact, then the opt-in
        hourglass control, both into the acceleration planes pass B adds."""
        self._contact()
        if not self.hourglass:
            return
        for db in self.dbodies:
            if not self.contact_pairs:
                db.ac.zero_()
            _lib.check(self._lib.tl_hourglass(self._st(), C.byref(db.desc)), "tl_hourglass")

    def _partition(self, body):
        """This rank's slab of ``body`` (dist.py): equal-count slabs along the
        longest axis; the halo region extends one interaction reach."""
        import torch.distributed as tdist
        slab = getattr(body, "slab", None)
        if slab is not None:
            if slab.nranks != self.world or slab.rank != tdist.get_rank(self.group):
                raise ValueError(f"body {body.mk} was built for slab {slab.rank} of "
                                 f"{slab.nranks}, not this rank of {self.world}")
            return dist.BodyPartition.from_slab(slab)
        X = body.state.X
        owner, axis = dist.slab_owner(X, self.world)
        reach = (body.nbsrange * body.dp_body * (1.0 + 1e-9) if body.nbsrange is not None
                 else 2.0 * body.h)
        return dist.BodyPartition(X, owner, tdist.get_rank(self.group), axis, reach)

    # -- plumbing ------------------------------------------------------------
    def _st(self):
        return C.c_void_p(self.stream.cuda_stream)

    def _mark(self, phase):
        if self.trace is not None:
            self.trace.append(phase)

    def _set_clock(self, **kw):
        c = _lib.tl_clock()
        c.t = self.t
        c.dt = 0.0
        c.next_out = math.inf
        c.t_max = math.inf
        c.eps = 0.0
        c.dt_override = -1.0
        c.cfl = float(self.config.cfl)
        c.step = self.step_index
        c.max_steps = -1
        c.halted = 0
        c.out_step = 0
        for k, v in kw.items():
            setattr(c, k, v)
        raw = bytearray(C.string_at(C.addressof(c), C.sizeof(c)))
        torch = _torch()
        self.clock_dev.copy_(torch.frombuffer(raw, dtype=torch.uint8), non_blocking=False)

    def _get_clock(self):
        raw = bytes(self.clock_dev.cpu().numpy().tobytes())
        c = _lib.tl_clock.from_buffer_copy(raw)
        return c

    def _exchange_and_launch(self, db, buf, launch):
        """Fill the halo rows of ``buf`` from their owners and run a pass.
        Tiled slabs overlap the two: the exchange runs on a side stream while
        the interior tiles (no halo reads) compute, then the boundary tiles
        run once the halo has landed."""
        if db.exchange is None:
            launch()
            return
        if db.tlist is None:
            db.exchange.exchange(buf)
            launch()
            return
        torch = _torch()
        ready = torch.cuda.Event()
        ready.record(self.stream)              # buf's owned rows are final
        side = db.comm_stream
        with torch.cuda.stream(side):
            side.wait_event(ready)
            db.exchange.exchange(buf)
            done = torch.cuda.Event()
            done.record(side)
        d = db.desc
        d.tlist = _lib.ptr(db.tlist)
        nt = int(db.tlist.shape[0])
        try:
            if db.n_interior:
                d.tbase, d.tcount = 0, db.n_interior
                launch()
            self.stream.wait_event(done)
            if nt > db.n_interior:
                d.tbase, d.tcount = db.n_interior, nt - db.n_interior
                launch()
        finally:
            d.tlist, d.tbase, d.tcount = None, 0, 0

    def _exchange_plain(self, db, buf, launch):
        if db.exchange is not None:
            db.exchange.exchange(buf)
        launch()

    def _pass_a(self, db):
        def launch():
            d = db.desc
            if db.tile_a:
                _lib.check(self._lib.tl_pass_a(self._st(), C.byref(d)), "tl_pass_a")
                return
            tile, tl = d.tile, d.tlist        # L2-gather pass A (see DeviceBody)
            d.tile, d.tlist = 0, None
            try:
                _lib.check(self._lib.tl_pass_a(self._st(), C.byref(d)), "tl_pass_a")
            finally:
                d.tile, d.tlist = tile, tl

        if self.peer:
            # the halo (u, s) rows were stored by the neighbours' pass B, ordered
            # by the dt all-reduce; after pass A, a barrier all-reduce orders
            # the pass-B records this pass A stored into the neighbours
            launch()
            dist.allreduce(self._barrier_t, "max", self.group)
        elif db.tile_a:
            self._exchange_and_launch(db, db.us, launch)   # halo (u, s) from the owners
        else:
            self._exchange_plain(db, db.us, launch)

    def _pass_b(self, db, mode, reset=True):
        # device-clock steps: k_clock_begin cleared the maxima after reading them
        if reset:
            _lib.check(self._lib.tl_reset_red(self._st(), _lib.ptr(db.red)), "tl_reset_red")

        def launch():
            d = db.desc
            if db.tile_b:
                _lib.check(self._lib.tl_pass_b(self._st(), C.byref(d), mode), "tl_pass_b")
                return
            tile, tl = d.tile, d.tlist        # L2-gather pass B (see DeviceBody)
            d.tile, d.tlist = 0, None
            try:
                _lib.check(self._lib.tl_pass_b(self._st(), C.byref(d), mode), "tl_pass_b")
            finally:
                d.tile, d.tlist = tile, tl

        if self.peer:
            launch()                                   # halo records stored by the neighbours
        elif db.tile_b:
            self._exchange_and_launch(db, db.rb, launch)   # halo (P L, v) from the owners
        else:
            self._exchange_plain(db, db.rb, launch)        # no tile split: exchange first
        if db.exchange is not None:
            dist.allreduce(db.red, "max", self.group)   # global dt maxima, exact
        if int(db.body.material.model) == int(Model.J2):
            _lib.check(self._lib.tl_reduce_partials(self._st(), _lib.ptr(db.pw_partial),
                                                    db.nblocks, _lib.ptr(db.pw_acc)),
                       "tl_reduce_partials")

    def _launch_step(self, mode_verlet, reset=True):
        """One step's launches; reset=False under the device clock (its
        k_clock_begin clears the dt maxima)."""
        if mode_verlet:
            for db in self.dbodies:
                self._pass_a(db)
            self._between_passes()
            for db in self.dbodies:
                self._pass_b(db, 1, reset)
        else:
            for db in self.dbodies:
                _lib.check(self._lib.tl_predict(self._st(), C.byref(db.desc)), "tl_predict")
            for db in self.dbodies:
                self._pass_a(db)
            self._between_passes()
            for db in self.dbodies:
                self._pass_b(db, 2, reset)

    def _check_errors(self, clock=None):
        """Raise the reference's exceptions for events recorded on the device.

        In-step errors first (stress, acceleration, expressions, restrictphi:
        the reference raises them inside the step, before the commit), then
        the non-finite state check of a 64-step commit (clock.halted == 6).
        Multi-GPU: every rank raises when any rank recorded an event."""
        if self.contact_counters is not None:
            cc = self.contact_counters.cpu().numpy()
            self.contact_warnings = int(cc[0])
            if cc[1]:
                raise SimulationError(f"contact: {int(cc[1])} candidate pairs over the per-particle "
                                      f"capacity (TL_CONTACT_CAP)")
        nf_halt = clock is not None and int(clock.halted) == 6
        if self.partitioned:
            flag = _torch().zeros(1, dtype=_torch().int64, device="cuda")
            for db in self.dbodies:
                c = db.counters
                flag |= ((c[1] != 0) | (c[4] != 0) | (c[5] != 0) | (c[2] != INT64_MAX)
                         | (c[3] != INT64_MAX)).to(flag.dtype).reshape(1)
            flag |= int(nf_halt)
            dist.allreduce(flag, "max", self.group)
            if int(flag.item()):
                local = nf_halt or any(int(db.counters[k]) != v for db in self.dbodies
                                       for k, v in ((1, 0), (4, 0), (5, 0), (2, INT64_MAX),
                                                    (3, INT64_MAX)))
                if not local:
                    raise SimulationError("numerical error reported by another rank")
        for db in self.dbodies:
            c = db.counters.cpu().numpy()
            mk = db.body.mk
            db.body.degenerate_warnings = db.deg_base + int(c[0])
            if c[4]:
                db._reset_counters()
                raise ex.ExprError(ex.ERRORS.get(int(c[4]), "expression error"))
            if c[5]:
                db._reset_counters()
                raise CaseError(f"restrictphi expression must evaluate within [0, 1] "
                                f"(body {mk})")
            if c[1]:
                db._reset_counters()
                raise SimulationError(
                    f"eigensolver failed to converge for {int(c[1])} particles (body {mk})")
            if c[2] != INT64_MAX:
                db._reset_counters()
                raise SimulationError(f"non-SPD plastic metric at particle {int(c[2])} "
                                      f"(body {mk})")
            if c[3] != INT64_MAX:
                step = int(c[6]) if c[6] != INT64_MAX else self.step_index
                db._reset_counters()
                raise SimulationError(f"non-finite acceleration at particle {int(c[3])} "
                                      f"(body {mk}, step {step})")
        if nf_halt:
            self._raise_nonfinite_state(int(clock.step))

    def _raise_nonfinite_state(self, step):
        """stepper.py:203-209: the first body whose u or v is non-finite."""
        for db in self.dbodies:
            if int(db.counters[7].item()) != INT64_MAX:
                db._reset_counters()
                raise SimulationError(f"non-finite state in body {db.body.mk} at step {step}")
        raise SimulationError(f"non-finite state at step {step} (another rank)")

    def sync_host(self, full=True):
        """Mark the host mirrors stale: the next read of a body.state field
        copies the device state (DeviceState); plastic work and warning
        counters are refreshed now."""
        for db in self.dbodies:
            db.dirty = True
            pw = db.pw_acc.clone()
            if self.partitioned:
                dist.allreduce(pw, "sum", self.group)
            db.body.plastic_work = db.pw_base + float(pw.item())

    def pull_host(self):
        """Copy the device state into every body.state now."""
        for db in self.dbodies:
            db.pull_state()

    def pin_host_state(self):
        """Page-lock every body's host state arrays (DMA for push/pull)."""
        for db in self.dbodies:
            db.pin_host()

    def push_state(self):
        """Upload host edits of body.state to the device."""
        for db in self.dbodies:
            db.dirty = False
            db.push_state()

    # -- reference API -----------------------------------------------------------
    def initialize(self):
        """One force evaluation at t=0 plus the initial velocity BCs
        (stepper.py:134-142)."""
        self._set_clock(t=0.0, dt=0.0)
        for db in self.dbodies:
            db.desc.write_out = 1
        self._mark("contact")
        self._mark("internal")
        for db in self.dbodies:
            self._pass_a(db)
        self._between_passes()
        for db in self.dbodies:
            self._pass_b(db, 0)
        for db in self.dbodies:
            db.desc.write_out = 0
        if self.trace is not None:
            del self.trace[:]
        self._initialized = True
        self.sync_host()
        self._check_errors()

    def step(self, dt):
        """One Verlet or symplectic step of size dt (stepper.py:211-217).
        An error the reference raises inside the step leaves t and
        step_index uncommitted, as there."""
        if not self._initialized:
            self.initialize()
        verlet = int(self.config.step_algorithm) != 2
        self._set_clock(t=self.t, dt=float(dt), out_step=int(self.mirrors),
                        step=self.step_index)
        if verlet:
            for ph in ("contact", "internal", "bc", "update", "commit"):
                self._mark(ph)
        else:
            for ph in ("predictor", "contact", "internal", "bc", "update", "commit"):
                self._mark(ph)
        self._launch_step(verlet)
        self.sync_host()
        c = self._get_clock()
        self._check_errors()
        self.t += dt
        self.step_index += 1
        # stepper.py:203-209: every 64th commit checks the state
        if self.step_index % 64 == 0:
            nf = int(c.nf_now)
            if self.partitioned:
                f = _torch().tensor([nf], dtype=_torch().int64, device="cuda")
                dist.allreduce(f, "max", self.group)
                nf = int(f.item())
            if nf:
                self._raise_nonfinite_state(self.step_index)

    def pick_dt(self):
        """Adaptive dt from the device maxima, bit-identical to the
        reference's FP64 formula (stepper.py:221-233)."""
        if self.config.dt_override is not None:
            return self.config.dt_override
        dt = math.inf
        for db in self.dbodies:
            red = db.red.cpu().numpy().view(np.float64)
            vmax = float(np.sqrt(red[0]))
            amax = float(np.sqrt(red[1]))
            h, c0, cfl = db.body.h, db.body.material.c0, self.config.cfl
            dtv = h / (c0 + vmax)
            cand = cfl * min(dtv, math.sqrt(h / amax)) if amax > 0.0 else cfl * dtv
            dt = min(dt, cand)
        return dt

    def _clock_steps(self, nsteps, verlet):
        """Launch nsteps device-clock steps (clock begin, passes, commit)."""
        for _ in range(nsteps):
            _lib.check(self._lib.tl_clock_begin(self._st(), _lib.ptr(self.clock_dev),
                                                 len(self.dbodies), self._dt_arr), "clock")
            self._launch_step(verlet, reset=False)
            _lib.check(self._lib.tl_clock_commit(self._st(), _lib.ptr(self.clock_dev)), "commit")

    def _launch_batch(self, nsteps, verlet):
        """nsteps device-clock steps, as one replay of a captured CUDA graph
        when graphs are on (captured on first use for each (nsteps, mode))."""
        if not self.use_graphs:
            self._clock_steps(nsteps, verlet)
            return
        torch = _torch()
        g = self._graph(nsteps, verlet)
        with torch.cuda.stream(self.stream):
            g.replay()

    def prepare_graphs(self, batch=64):
        """Capture the step graphs run() and advance() replay (power-of-two
        batch lengths up to ``batch``) ahead of time; otherwise each is
        captured on first use.  Launches nothing."""
        if not self.use_graphs:
            return
        if not self._initialized:
            self.initialize()
        verlet = int(self.config.step_algorithm) != 2
        p = 1
        while p <= batch:
            self._graph(p, verlet)
            p *= 2

    def _graph(self, nsteps, verlet):
        """The captured graph of nsteps device-clock steps (captured once)."""
        torch = _torch()
        key = (int(nsteps), bool(verlet))
        g = self._graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(self.stream)
            saved = self.stream
            self.stream = cap
            try:
                with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                    self._clock_steps(nsteps, verlet)
            finally:
                self.stream = saved
            self.stream.wait_stream(cap)
            self._upload_graph(g)
            self._graphs[key] = g
        return g

    def _upload_graph(self, g):
        """Upload the instantiated graph to the device now (cuGraphUpload), so
        its first replay inside run() does not pay for it (about 28 ms over
        the six batch lengths of a C4 run).  Best effort: without cuda-python
        the first replay uploads it, as before.  TLSPH_GRAPH_UPLOAD=0 skips."""
        if os.environ.get("TLSPH_GRAPH_UPLOAD", "1") == "0":
            return
        try:
            from cuda.bindings import driver as drv
        except ImportError:
            return
        ex = int(g.raw_cuda_graph_exec())
        (err,) = drv.cuGraphUpload(drv.CUgraphExec(ex), drv.CUstream(int(self.stream.cuda_stream)))
        if int(err) != 0:
            raise SimulationError(f"cuGraphUpload failed: {err}")

    def advance(self, nsteps, pass_events=None):
        """Launch exactly ``nsteps`` device-clock steps (adaptive dt, or the
        override) with no host synchronisation; the throughput entry point.
        ``pass_events``: optional list that receives (ev_a0, ev_a1, ev_b0, ev_b1)
        CUDA events around pass A and pass B of every step."""
        if not self._initialized:
            self.initialize()
        cfg = self.config
        verlet = int(cfg.step_algorithm) != 2
        dto = -1.0 if cfg.dt_override is None else float(cfg.dt_override)
        self._set_clock(t=self.t, next_out=math.inf, t_max=math.inf, eps=0.0, dt_override=dto)
        if pass_events is None:
            full, rest = divmod(nsteps, 64)
            for _ in range(full):
                self._launch_batch(64, verlet)
            self._clock_steps(rest, verlet)
        else:
            torch = _torch()
            for _ in range(nsteps):
                _lib.check(self._lib.tl_clock_begin(self._st(), _lib.ptr(self.clock_dev),
                                                     len(self.dbodies), self._dt_arr), "clock")
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                if not verlet:
                    for db in self.dbodies:
                        _lib.check(self._lib.tl_predict(self._st(), C.byref(db.desc)), "predict")
                ev[0].record(self.stream)
                for db in self.dbodies:
                    self._pass_a(db)
                self._between_passes()
                ev[1].record(self.stream)
                ev[2].record(self.stream)
                for db in self.dbodies:
                    self._pass_b(db, 1 if verlet else 2, reset=False)
                ev[3].record(self.stream)
                pass_events.append(ev)
                _lib.check(self._lib.tl_clock_commit(self._st(), _lib.ptr(self.clock_dev)),
                           "commit")
        self.step_index += nsteps
        for db in self.dbodies:
            db.dirty = True

    def finish_advance(self):
        """Sync point after advance(): read the clock back, raise errors."""
        c = self._get_clock()
        self.t = float(c.t)
        self.step_index = int(c.step)
        self._check_errors(c)
        if c.halted == 4:
            raise SimulationError(f"timestep collapsed to {c.dt!r}")

    def run(self, time_max=None, time_out=None, on_output=None, max_steps=None, batch=64):
        """Advance to time_max with on_output at t=0, every time_out boundary
        and the end (stepper.py:237-263).  Steps are launched in batches with
        dt, t and the output/stop decisions computed on the device clock."""
        cfg = self.config
        t_max = cfg.time_max if time_max is None else time_max
        t_out = cfg.time_out if time_out is None else time_out
        if not self._initialized:
            self.initialize()
        if on_output is not None:
            on_output(self)
        if t_max <= 0.0:
            return
        next_out = t_out if t_out > 0.0 else t_max
        eps = 1e-12 * max(t_max, 1.0)
        verlet = int(cfg.step_algorithm) != 2
        dto = -1.0 if cfg.dt_override is None else float(cfg.dt_override)
        dt_hint = None
        while self.t < t_max - eps:
            self._set_clock(t=self.t, next_out=next_out, t_max=t_max, eps=eps, dt_override=dto,
                            max_steps=-1 if max_steps is None else int(max_steps))
            # batch length: the steps to the next stop (output, t_max or
            # max_steps) at the last dt, so few launches run halted after the
            # device clock stops; powers of two replay cached graphs
            if dt_hint is None:
                dt_hint = self.pick_dt()
            n = batch
            if dt_hint > 0.0 and math.isfinite(dt_hint):
                n = min(n, int((min(next_out, t_max) - self.t) / dt_hint) + 1)
            if max_steps is not None:
                n = min(n, int(max_steps) - self.step_index)
            n = max(n, 1)
            p = batch
            while n > 0:
                while p > n:
                    p //= 2
                self._launch_batch(p, verlet)
                n -= p
            c = self._get_clock()
            if float(c.dt) > 0.0:
                dt_hint = float(c.dt)
            for db in self.dbodies:
                db.dirty = True           # host mirrors refresh on read (also after a raise)
            steps_done = int(c.step) - self.step_index
            if self.trace is not None:
                seq = ("contact", "internal", "bc", "update", "commit") if verlet else \
                      ("predictor", "contact", "internal", "bc", "update", "commit")
                self.trace.extend(seq * steps_done)
            self.t = float(c.t)
            self.step_index = int(c.step)
            self._check_errors(c)
            if c.halted == 4:
                raise SimulationError(f"timestep collapsed to {c.dt!r}")
            if c.halted == 2:
                self.sync_host()
                if on_output is not None:
                    on_output(self)
                next_out = min(next_out + t_out, t_max) if t_out > 0.0 else t_max
            if max_steps is not None and self.step_index >= max_steps:
                break
            if c.halted == 1:
                break
        self.sync_host()


# The reference name, for ``from paper_2602_15149_b200.simulation import Simulation``
Simulation = DeviceSimulation
