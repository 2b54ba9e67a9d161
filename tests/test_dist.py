"""Slab partition + fixed halo lists + halo exchange, world_size 2 on gloo
(CPU).  Each rank computes only its owned rows with the CPU oracle's kernels,
receiving (u, s) before the F/stress/phase-field pass and (P, v) before the
momentum pass through paper_2602_15149_b200.dist.HaloExchange; the result must
be bit-identical to the single-process oracle (same rows, same summation
order, same inputs)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, golden, run_case

NSTEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _reach(b):
    return b.nbsrange * b.dp_body * (1.0 + 1e-9) if b.nbsrange is not None else 2.0 * b.h


def _forces(O, adj, st, b, rows_only=None):
    """One force evaluation (stepper._internal_phase without BCs) on
    arrays of the (sub)domain; returns a and updates F, S, Hhist, sddot."""
    B = O.backend
    mat = b.material
    n = st["X"].shape[0]
    B.deformation_gradient(adj.indptr, adj.rows, adj.indices, adj.grad0, st["u"], st["V0"],
                           st["s"], mat.s_l, b.fracture, st["F"])
    S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
    B.svk_batch(st["F"], mat.lam, mat.mu, st["s"], b.fracture, S, psi, psip)
    st["H"][:] = np.maximum(psip, st["H"])
    lap = np.zeros(n)
    B.sph_laplacian(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.r0, adj.r0norm, st["V0"],
                    st["s"], lap)
    ratio = st["H"] / mat.Gc
    c = mat.c0
    st["sdd"][:] = (c * c / (2.0 * mat.eps0)) * (
        2.0 * mat.eps0 * lap + (1.0 - st["s"]) / (2.0 * mat.eps0)
        - 2.0 * np.sqrt(4.0 * mat.eps0 * ratio + 1.0) / c * st["sd"] - 2.0 * st["s"] * ratio)
    st["P"][:] = np.matmul(st["F"], S)


def _momentum(O, adj, st, b):
    mat = b.material
    a = np.zeros((st["X"].shape[0], 3))
    O.backend.momentum(adj.indptr, adj.rows, adj.indices, adj.grad0, adj.grad0r, adj.r0,
                       adj.r0norm, st["P"], st["m0"], mat.rho0, st["v"], b.h, mat.c0,
                       mat.beta1, mat.beta2, st["F"], a)
    return a


def _verlet(st, a, dt, rows):
    st["v"][rows] += dt * a[rows]
    st["u"][rows] += dt * st["v"][rows]
    st["sd"][rows] += dt * st["sdd"][rows]
    st["s"][rows] += dt * st["sd"][rows]
    np.clip(st["s"], 0.0, 1.0, out=st["s"])


def _state(b, idx=None):
    s = b.state
    sel = (lambda x: x.copy()) if idx is None else (lambda x: x[idx].copy())
    n = s.X.shape[0] if idx is None else len(idx)
    return {"X": sel(s.X), "V0": sel(s.V0), "m0": sel(s.m0), "u": sel(s.u), "v": sel(s.v),
            "s": sel(s.s), "sd": sel(s.sdot), "H": sel(s.Hhist), "sdd": np.zeros(n),
            "F": np.zeros((n, 3, 3)), "P": np.zeros((n, 3, 3))}


def _worker(rank, world, port, tag, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2602_15149_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = golden(f"run_{tag}")
    cfg = run_case(G)
    b = cfg.bodies[0]
    X = b.state.X
    owner, axis = D.slab_owner(X, world)
    # the oracle's momentum reads grad0r = -L_j gb, so halo rows need their
    # own complete neighbourhood: build on the slab +- 2 reaches (the device
    # path receives P L_j from the owner instead and needs only one reach)
    sub = D.subset_for_rank(X, owner, rank, axis, 2.0 * _reach(b))
    adj = O.build_adjacency(X[sub], b.state.V0[sub], b.h, b.dim, int(cfg.kernel),
                            nbsrange=b.nbsrange, dp_body=b.dp_body, notches=b.notches,
                            correction=b.kernel_correction)
    st = _state(b, sub)
    owned_sub = np.flatnonzero(owner[sub] == rank)          # subset rows this rank owns
    owned_gid = sub[owned_sub]
    # off-rank partners referenced by owned rows
    nbr = np.concatenate([adj.indices[adj.indptr[i]:adj.indptr[i + 1]] for i in owned_sub])
    needed = np.unique(sub[nbr])
    needed = needed[owner[needed] != rank]
    plan = D.build_halo_plan(owned_gid, np.arange(len(owned_gid)), needed, owner)
    ex = D.HaloExchange(plan, "cpu")
    pos_in_sub = {g: k for k, g in enumerate(sub.tolist())}
    halo_sub = np.array([pos_in_sub[g] for g in plan.halo_gid.tolist()], dtype=np.int64)
    local_rows = np.concatenate([owned_sub, halo_sub])

    def exchange(fields):
        # pack owned + halo rows of the subset arrays, exchange, scatter back
        cols = [st[f].reshape(len(sub), -1) for f in fields]
        buf = torch.from_numpy(np.concatenate([c[local_rows] for c in cols], axis=1).copy())
        ex.exchange(buf)
        out = buf.numpy()
        o = 0
        for f, c in zip(fields, cols):
            w = c.shape[1]
            c[halo_sub] = out[len(owned_sub):, o:o + w]
            st[f] = c.reshape(st[f].shape)
            o += w

    dts = G["dts"]
    for k in range(NSTEPS):
        exchange(["u", "s"])
        _forces(O, adj, st, b)
        exchange(["P", "v"])
        a = _momentum(O, adj, st, b)
        _verlet(st, a, dts[k], owned_sub)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), gid=owned_gid, u=st["u"][owned_sub],
             v=st["v"][owned_sub], s=st["s"][owned_sub], n_halo=plan.n_halo)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("tag,world", [("kalthoff2d_p", 2), ("kalthoff3d", 2), ("kalthoff3d", 3)])
def test_multi_rank_halo_exchange_bit_identical(tag, world, tmp_path, oracle_mod):
    G = golden(f"run_{tag}")
    mp.spawn(_worker, args=(world, _free_port(), tag, str(tmp_path)), nprocs=world, join=True)
    # single-process reference with the same helper functions
    O = oracle_mod
    cfg = run_case(G)
    b = cfg.bodies[0]
    adj = O.build_adjacency(b.state.X, b.state.V0, b.h, b.dim, int(cfg.kernel),
                            nbsrange=b.nbsrange, dp_body=b.dp_body, notches=b.notches,
                            correction=b.kernel_correction)
    st = _state(b)
    rows = np.arange(b.state.X.shape[0])
    for k in range(NSTEPS):
        _forces(O, adj, st, b)
        a = _momentum(O, adj, st, b)
        _verlet(st, a, G["dts"][k], rows)
    seen = np.zeros(len(rows), dtype=bool)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        g = d["gid"]
        assert d["n_halo"] > 0
        seen[g] = True
        assert np.array_equal(d["u"], st["u"][g])
        assert np.array_equal(d["v"], st["v"][g])
        assert np.array_equal(d["s"], st["s"][g])
    assert seen.all()


def test_slab_partition_properties():
    from paper_2602_15149_b200 import dist as D
    rng = np.random.default_rng(0)
    X = rng.uniform(0, 1, (1001, 3)) * np.array([3.0, 1.0, 2.0])
    for nr in (1, 2, 3, 8):
        owner, axis = D.slab_owner(X, nr)
        assert axis == 0
        cnt = np.bincount(owner, minlength=nr)
        assert cnt.max() - cnt.min() <= 1
        # slabs are contiguous along the axis
        for r in range(nr - 1):
            assert X[owner == r, 0].max() <= X[owner == r + 1, 0].min()


def test_slab_local_build_matches_whole_body():
    """cases.make_case(slab=(r, N)) builds only a rank's planes plus the
    interaction reach: positions, V0, BC targets and the bench's perturbed
    state equal the whole-body build restricted to those global ids; the
    plane owners cover every particle once; the partition's subset holds the
    reach around the owned planes."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_15149_b200 import cases, dist as D
    full = cases.make_case("kalthoff3d", dp_scale=6, mapfac=2, build_adjacency=False)
    bench.perturb(full)
    bf = full.bodies[0]
    n = bf.state.X.shape[0]
    seen = np.zeros(n, dtype=int)
    for world in (2, 3):
        seen[:] = 0
        for r in range(world):
            c = cases.make_case("kalthoff3d", dp_scale=6, mapfac=2, build_adjacency=False,
                                slab=(r, world))
            bench.perturb(c)
            b = c.bodies[0]
            g = b.slab.gid
            assert np.array_equal(b.state.X, bf.state.X[g])
            assert np.array_equal(b.state.V0, bf.state.V0[g])
            for k in ("u", "v", "s"):
                assert np.array_equal(getattr(b.state, k), getattr(bf.state, k)[g])
            for bl, bfull in zip(b.bcs, bf.bcs):
                gf = np.asarray(bfull.target)
                assert np.array_equal(np.sort(g[bl.target]), np.sort(gf[np.isin(gf, g)]))
            part = D.BodyPartition.from_slab(b.slab)
            assert np.array_equal(part.sub, g) and np.array_equal(part.host_rows, np.arange(g.size))
            seen[part.owned_gid] += 1
            # the held planes reach one interaction range beyond the owned ones
            xo = b.state.X[part.owned_rows, 0]
            reach = b.nbsrange * b.dp_body * (1.0 + 1e-9)
            need = (bf.state.X[:, 0] >= xo.min() - reach) & (bf.state.X[:, 0] <= xo.max() + reach)
            assert np.isin(np.flatnonzero(need), g).all()
        assert (seen == 1).all()
    own = D.PlaneOwner([0, 3, 7], 10)
    assert own[np.array([0, 29, 30, 69])].tolist() == [0, 0, 1, 1]
