"""Multi-rank device path (slabs + halo exchange) on the single available
B200: 2 and 3 ranks share cuda:0 over gloo (halo buffers staged through the
host).  FP64: owned rows must be bit-identical to the single-rank device run
-- same rows, same CSR summation order, same inputs.  FP32:
within 1e-5 (tile-relative coordinates round differently per tiling)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, golden, run_case

pytestmark = pytest.mark.gpu
NSTEPS = 4


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tag, precision, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_15149_b200.simulation import DeviceSimulation
    G = golden(f"run_{tag}")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision=precision)
    sim.initialize()
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
    db = sim.dbodies[0]
    st = cfg.bodies[0].state
    g = db.gid[:db.n]
    dt_next = sim.pick_dt()
    from paper_2602_15149_b200 import output
    energies = np.array(output.compute_energies(cfg.bodies[0], sim.be))   # collective
    idx = np.arange(0, st.X.shape[0], 5)
    mrow = np.array(output.measure_row(cfg.bodies[0], idx, sim.t)[1:7])  # collective
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), gid=g, u=st.u[g], v=st.v[g], s=st.s[g],
             S=st.S[g], n_halo=db.n_all - db.n, dt=dt_next, energies=energies, mrow=mrow,
             bsplit=db.bsplit, tile=db.layout.tile, peer=int(sim.peer))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("tag,world,precision", [("kalthoff3d", 2, "fp64"),
                                                 ("kalthoff2d_p", 3, "fp64"),
                                                 ("taylor3d", 2, "fp64"),
                                                 ("taylor3d", 2, "fp32")])
def test_multi_rank_device_bit_identical(tag, world, precision, tmp_path, monkeypatch):
    from paper_2602_15149_b200.simulation import DeviceSimulation
    mp.spawn(_worker, args=(world, _port(), tag, precision, str(tmp_path)), nprocs=world,
             join=True)
    G = golden(f"run_{tag}")
    if precision == "fp64":
        # slabs run the tiled kernels: the 1-GPU reference of the bit-identity
        # check runs them too (the brick kernels' sums round differently; the
        # brick path is held to the slabs at 1e-12 below)
        _brick_vs_slabs(tag, world, tmp_path, G)
        monkeypatch.setenv("TLSPH_BRICK", "0")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision=precision)
    sim.initialize()
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
    st = cfg.bodies[0].state
    dt_ref = sim.pick_dt()
    from paper_2602_15149_b200 import output
    e_ref = np.array(output.compute_energies(cfg.bodies[0], sim.be))
    m_ref = np.array(output.measure_row(cfg.bodies[0], np.arange(0, st.X.shape[0], 5),
                                        sim.t)[1:7])
    seen = np.zeros(st.X.shape[0], dtype=bool)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        g = d["gid"]
        assert d["n_halo"] > 0
        seen[g] = True
        for k in ("u", "v", "s", "S"):
            if precision == "fp64":
                assert np.array_equal(d[k], getattr(st, k)[g]), (r, k)
            else:
                # FP32 neighbour differences are formed relative to each tile's
                # origin, and tiles differ between the slab and the whole body:
                # identical up to FP32 rounding of the reference coordinates
                ref = getattr(st, k)
                err = np.abs(d[k] - ref[g]).max() / max(np.abs(ref).max(), 1e-300)
                assert err <= 1e-5, (r, k, err)
        if precision == "fp64":
            assert float(d["dt"]) == dt_ref
        else:
            assert abs(float(d["dt"]) - dt_ref) <= 1e-5 * dt_ref
        # output reductions over the slabs (per-rank fsum, then an all-reduce):
        # a different summation order than one GPU
        tol = 1e-12 if precision == "fp64" else 1e-5
        scale = max(np.abs(e_ref).max(), 1e-300)
        assert np.abs(d["energies"] - e_ref).max() <= tol * scale, (d["energies"], e_ref)
        mscale = max(np.abs(m_ref).max(), 1e-300)
        assert np.abs(d["mrow"] - m_ref).max() <= tol * mscale, (d["mrow"], m_ref)
    assert seen.all()


def _brick_vs_slabs(tag, world, tmp_path, G):
    """The default 1-GPU kernels (lattice bricks where they apply) against
    the slab runs, FP64, within 1e-12 of each field's scale."""
    from paper_2602_15149_b200.simulation import DeviceSimulation
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision="fp64")
    sim.initialize()
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
    st = cfg.bodies[0].state
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        g = d["gid"]
        for k in ("u", "v", "s", "S"):
            ref = getattr(st, k)
            err = np.abs(d[k] - ref[g]).max() / max(np.abs(ref).max(), 1e-300)
            assert err <= 1e-12, (r, k, err)


def test_multi_rank_split_rows(tmp_path, monkeypatch):
    """The 4-way row split of pass B (tl_body.bsplit) on slabs, whose tiled
    passes launch interior and boundary tile lists separately."""
    monkeypatch.setenv("TLSPH_BSPLIT", "4")   # inherited by the spawned ranks
    monkeypatch.setenv("TLSPH_BRICK", "0")    # the 1-GPU reference on tiles too
    from paper_2602_15149_b200.simulation import DeviceSimulation
    sim = DeviceSimulation(run_case(golden("run_taylor3d")), precision="fp32")
    assert sim.dbodies[0].bsplit == 4
    del sim
    test_multi_rank_device_bit_identical("taylor3d", 2, "fp32", tmp_path, monkeypatch)
    for r in range(2):   # every slab ran the split kernel, not a bsplit=1 fallback
        d = np.load(tmp_path / f"r{r}.npz")
        assert int(d["bsplit"]) == 4, (r, int(d["bsplit"]), int(d["tile"]))


def _nccl_worker(rank, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2602_15149_b200 import dist as D
    from paper_2602_15149_b200.simulation import DeviceSimulation
    # the collectives of the step on NCCL: MAX on FP64 bit patterns, MIN, SUM
    t = torch.tensor([3, -7, 11], dtype=torch.int64, device="cuda")
    red = [D.allreduce(t.clone(), op).cpu().numpy() for op in ("max", "min", "sum")]
    G = golden("run_kalthoff3d")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision="fp64", partition=True)
    assert sim.partitioned and sim.dbodies[0].exchange is not None
    sim.initialize()
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
    st = cfg.bodies[0].state
    np.savez(os.path.join(out_dir, "nccl.npz"), u=st.u, v=st.v, s=st.s, S=st.S,
             red=np.stack(red), backend=dist.get_backend())
    dist.destroy_process_group()


def test_nccl_world1_slab_path(tmp_path):
    """The NCCL branch of the slab path on a one-rank NCCL group: the halo
    plan's all_to_all, the (empty) exchanges and the all-reduces run through
    NCCL, and the state is bit-identical to the unpartitioned run."""
    mp.spawn(_nccl_worker, args=(_port(), str(tmp_path)), nprocs=1, join=True)
    d = np.load(tmp_path / "nccl.npz")
    assert str(d["backend"]) == "nccl"
    assert d["red"].tolist() == [[3, -7, 11]] * 3
    from paper_2602_15149_b200.simulation import DeviceSimulation
    G = golden("run_kalthoff3d")
    cfg = run_case(G)
    sim = DeviceSimulation(cfg, precision="fp64")
    sim.initialize()
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
    st = cfg.bodies[0].state
    for k in ("u", "v", "s", "S"):
        assert np.array_equal(d[k], getattr(st, k)), k


def _slab_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation
    cfg = cases.make_case("kalthoff3d", dp_scale=6, mapfac=2, build_adjacency=False,
                          slab=(rank, world))
    bench.perturb(cfg)
    b = cfg.bodies[0]
    assert b.slab is not None
    sim = DeviceSimulation(cfg, precision="fp64")
    sim.initialize()
    for _ in range(NSTEPS):
        sim.step(sim.pick_dt())
    db = sim.dbodies[0]
    st = b.state
    rows = db.hrow[:db.n]
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), gid=db.gid[:db.n], u=st.u[rows],
             v=st.v[rows], s=st.s[rows], S=st.S[rows], t=sim.t, n_host=st.X.shape[0])
    dist.barrier()
    dist.destroy_process_group()


def test_slab_local_ranks_bit_identical(tmp_path):
    """Ranks that build only their slab of the lattice on the host
    (cases.make_case(slab=...), bench.py at N > 1) reproduce the whole-body
    single-GPU run bit for bit (FP64, adaptive dt), with far less host state
    per rank."""
    import bench
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation
    world = 3
    mp.spawn(_slab_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    cfg = cases.make_case("kalthoff3d", dp_scale=6, mapfac=2, build_adjacency=False)
    bench.perturb(cfg)
    sim = DeviceSimulation(cfg, precision="fp64", partition=False)
    sim.initialize()
    for _ in range(NSTEPS):
        sim.step(sim.pick_dt())
    st = cfg.bodies[0].state
    n = st.X.shape[0]
    seen = np.zeros(n, dtype=bool)
    for r in range(world):
        d = np.load(tmp_path / f"s{r}.npz")
        g = d["gid"]
        seen[g] = True
        assert int(d["n_host"]) < n
        assert float(d["t"]) == sim.t
        for k in ("u", "v", "s", "S"):
            assert np.array_equal(d[k], getattr(st, k)[g]), (r, k)
    assert seen.all()


@pytest.mark.parametrize("tag,world", [("kalthoff3d", 2), ("kalthoff2d_p", 3), ("taylor3d", 2)])
def test_peer_memory_halo_bit_identical(tag, world, tmp_path, monkeypatch):
    """Peer-memory halo exchange (dist.PeerHalo, TLSPH_PEER=1): the step
    kernels store boundary records straight into the neighbours' halo rows
    (CUDA IPC mappings; ranks share the one GPU here, NVLink peers on a
    multi-GPU box), ordered by the per-step all-reduces.  FP64 owned rows stay
    bit-identical to one GPU."""
    monkeypatch.setenv("TLSPH_PEER", "1")          # inherited by the spawned ranks
    test_multi_rank_device_bit_identical(tag, world, "fp64", tmp_path, monkeypatch)
    for r in range(world):
        assert int(np.load(tmp_path / f"r{r}.npz")["peer"]) == 1, r
