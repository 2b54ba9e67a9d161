"""Device-side output rows for device-resident bodies.

Drop-ins for the reference's ``solidsph.output.compute_energies`` and
``measure_row`` (/root/reference/pkg/src/solidsph/output.py:25-71) with the
same signatures and return values.  The reference evaluates them on the host
from the full particle state, which for a ``DeviceSimulation`` body would
copy every field (and, for the fracture energy, every per-pair gradient)
back from HBM at each output.  Here the sums run on the device
(``tl_energies`` / ``tl_measure``, csrc/output.cu) into per-block FP64
partials (folded on the device to at most 1024 chunk sums for large bodies)
that are added on the host with ``math.fsum``; only those cross the bus.

The summation order differs from numpy's, so the results agree with the
reference to rounding (tests/test_gpu_output.py states the tolerance), not
bit for bit.

``install(solidsph.output)`` points the reference's ``OutputManager`` at these
functions: it looks both names up as module globals at call time
(output.py:144-151)."""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .core import Model


def _dbody(body):
    from .simulation import DeviceState
    st = body.state
    if not isinstance(st, DeviceState):
        raise TypeError("device output rows need a DeviceSimulation body "
                        "(body.state is not device-resident)")
    return object.__getattribute__(st, "_db")


def _allreduce_sum(vals, db):
    """Sum a small vector over the ranks of a partitioned body."""
    if db.part is None:
        return vals
    import torch
    from . import dist
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    dist.allreduce(t, "sum")
    return t.cpu().tolist()


def compute_energies(body, be=None, grad_buf=None):
    """(strain, kinetic, fracture, plastic) energy of one device body, as
    output.py:25-49.  ``be`` and ``grad_buf`` are accepted for signature
    compatibility; the gradient of s is formed on the device."""
    import torch
    db = _dbody(body)
    if db.psi_out is None:
        raise ValueError("energies need the stress mirrors: construct the simulation "
                         "with mirrors=True")
    if (db.body.fracture and getattr(db, "exchange", None) is not None
            and getattr(db, "peer", None) is None):
        # the fracture energy's grad s reads halo s, last exchanged before pass A:
        # refresh the halo rows from their owners (collective)
        db.exchange.exchange(db.us)
    L = _lib.lib()
    nb = int(L.tl_energy_blocks(db.n))
    part = torch.empty((nb, 3), dtype=torch.float64, device=db.dev)
    _lib.check(L.tl_energies(_lib.stream_ptr(), _lib.C.byref(db.desc), _lib.ptr(part)),
               "tl_energies")
    if nb > 4096:
        # fold the block partials to 1024 FP64 chunk sums on the device (a
        # fixed-shape reduction: deterministic) so the exact host sum below
        # runs over 1024 rows, not one per block (C4: 62 k rows, ~6 ms)
        c = -(-nb // 1024)
        part = torch.nn.functional.pad(part, (0, 0, 0, c * 1024 - nb)).view(1024, c, 3).sum(1)
    p = part.cpu().numpy()
    se, ke, fe = (math.fsum(p[:, k]) for k in range(3))
    se, ke, fe = _allreduce_sum([se, ke, fe], db)
    if not body.fracture:
        fe = 0.0
    pe = float(body.plastic_work) if body.material.model == Model.J2 else 0.0
    return float(se), float(ke), float(fe), pe


def _positions(db, idx):
    """Device positions of the owned particles among global ids ``idx``."""
    import torch
    if getattr(db, "_pos_of", None) is None:
        rows = np.asarray(db.hrow[:db.n], dtype=np.int64)      # host rows of the owned particles
        pos_of = np.full(int(db.host.X.shape[0]), -1, dtype=np.int64)
        pos_of[rows] = np.arange(db.n)
        db._pos_of = pos_of
    pos = db._pos_of[np.asarray(idx, dtype=np.int64)]
    pos = pos[pos >= 0]
    return torch.from_numpy(pos.astype(np.int32)).to(db.dev)


def measure_row(body, idx, t):
    """(t, mean u, total m0 a, count) over a measure-plane particle set, as
    output.py:63-71."""
    import torch
    idx = np.asarray(idx)
    if idx.size == 0:
        return (t, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0)
    db = _dbody(body)
    pos = _positions(db, idx)
    m = int(pos.shape[0])
    L = _lib.lib()
    nb = max((m + 255) // 256, 1)
    part = torch.zeros((nb, 6), dtype=torch.float64, device=db.dev)
    if m:
        _lib.check(L.tl_measure(_lib.stream_ptr(), _lib.C.byref(db.desc), _lib.ptr(pos), m,
                                _lib.ptr(part)), "tl_measure")
    p = part.cpu().numpy()
    sums = [math.fsum(p[:, k]) for k in range(6)]
    sums = _allreduce_sum(sums, db)
    n = int(idx.size)
    return (t, sums[0] / n, sums[1] / n, sums[2] / n, sums[3], sums[4], sums[5], n)


def install(module):
    """Route a reference ``solidsph.output`` module's OutputManager through
    the device reductions (output.py:144-151 resolves both at call time)."""
    module.compute_energies = compute_energies
    module.measure_row = measure_row
    return module


class Snapshot:
    """Asynchronous VTK snapshot of every body (the fields output.py:84-127
    writes: position, displacement, velocity, phase field or equivalent
    plastic strain, Cauchy stress).  ``tl_snapshot`` packs them on the device
    into one (n, 16) FP64 buffer in the caller's order, and a side stream
    copies it into page-locked host memory while the next steps run.
    ``fields(bi)`` waits for body bi's copy and returns numpy views; they stay
    valid until the next snapshot of the simulation.  Needs the F/S mirrors
    (mirrors=True), written on output steps, so take it from ``on_output``."""

    LAYOUT = {"x": (0, 3), "u": (3, 6), "v": (6, 9), "scalar": (9, 10), "cauchy": (10, 16)}

    def __init__(self, sim):
        import torch
        self.parts = []
        L = _lib.lib()
        for db in sim.dbodies:
            if db.F_out is None:
                raise ValueError("snapshots need the stress mirrors: construct the simulation "
                                 "with mirrors=True")
            nh = int(db.host.X.shape[0])
            buf = getattr(db, "_snap", None)
            if buf is None:
                buf = {"dev": torch.zeros((nh, 16), dtype=torch.float64, device=db.dev),
                       "host": torch.zeros((nh, 16), dtype=torch.float64, pin_memory=True),
                       "stream": torch.cuda.Stream(), "done": None}
                db._snap = buf
            if buf["done"] is not None:      # the previous copy still reads these buffers
                buf["done"].synchronize()
            dst, _ = db._gid_dev()
            _lib.check(L.tl_snapshot(sim._st(), _lib.C.byref(db.desc), _lib.ptr(dst),
                                     _lib.ptr(buf["dev"])), "tl_snapshot")
            ready = torch.cuda.Event()
            ready.record(sim.stream)
            with torch.cuda.stream(buf["stream"]):
                buf["stream"].wait_event(ready)
                buf["host"].copy_(buf["dev"], non_blocking=True)
                done = torch.cuda.Event()
                done.record(buf["stream"])
            buf["done"] = done
            self.parts.append(buf)
        self.t = sim.t
        self.step = sim.step_index

    @property
    def nbytes(self):
        return sum(int(b["host"].numel()) * 8 for b in self.parts)

    def wait(self):
        for b in self.parts:
            b["done"].synchronize()
        return self

    def fields(self, bi=0):
        b = self.parts[bi]
        b["done"].synchronize()
        a = b["host"].numpy()
        return {k: a[:, lo:hi] if hi - lo > 1 else a[:, lo] for k, (lo, hi) in self.LAYOUT.items()}


def snapshot_async(sim):
    """Start an asynchronous snapshot of ``sim`` (see Snapshot)."""
    return Snapshot(sim)
