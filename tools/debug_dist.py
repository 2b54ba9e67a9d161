"""Debug helper: per-step comparison of a multi-rank device run (gloo, one
GPU) against the single-rank device run, field by field (us, rb, v).

    python tools/debug_dist.py kalthoff3d 2 fp64
"""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
NSTEPS = 3


def snap(sim):
    db = sim.dbodies[0]
    g = db.gid
    lay = db.layout
    ip = lay.indptr.cpu().numpy()
    nb = g[lay.indices.cpu().numpy()]
    return dict(gid=g, n=db.n, ip=ip, nb=nb, L=db.L.double().cpu().numpy().T, us=db.us.double().cpu().numpy(), rb=db.rb.double().cpu().numpy(),
                v=db.v.double().cpu().numpy().T, al=db.al.double().cpu().numpy().T,
                sddot=db.sddot.double().cpu().numpy(), Hh=db.Hh.double().cpu().numpy())


def run(sim, G, out):
    import torch
    sim.initialize()
    torch.cuda.synchronize()
    out.append(snap(sim))
    for k in range(NSTEPS):
        sim.step(G["dts"][k])
        torch.cuda.synchronize()
        out.append(snap(sim))


def worker(rank, world, port, tag, precision, odir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import golden, run_case
    from paper_2602_15149_b200.simulation import DeviceSimulation
    G = golden(f"run_{tag}")
    sim = DeviceSimulation(run_case(G), precision=precision)
    out = []
    run(sim, G, out)
    np.save(os.path.join(odir, f"r{rank}.npy"), np.array(out, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    tag, world, precision = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    odir = "/tmp/dbg_dist"
    os.makedirs(odir, exist_ok=True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(world, port, tag, precision, odir), nprocs=world, join=True)
    from conftest import golden, run_case
    from paper_2602_15149_b200.simulation import DeviceSimulation
    G = golden(f"run_{tag}")
    sim = DeviceSimulation(run_case(G), precision=precision)
    ref = []
    run(sim, G, ref)
    for r in range(world):
        got = np.load(os.path.join(odir, f"r{r}.npy"), allow_pickle=True)
        for k, (d, e) in enumerate(zip(got, ref)):
            inv = np.empty_like(e["gid"])
            inv[e["gid"]] = np.arange(e["gid"].shape[0])
            if k == 0:
                nbad = 0
                for p in range(d["n"]):
                    q = inv[d["gid"][p]]
                    a = d["nb"][d["ip"][p]:d["ip"][p + 1]]
                    b = e["nb"][e["ip"][q]:e["ip"][q + 1]]
                    if not np.array_equal(a, b) or not np.array_equal(d["L"][p], e["L"][q]):
                        nbad += 1
                        if nbad < 4:
                            print("row", d["gid"][p], "nb", a, "ref", b, "L", d["L"][p], e["L"][q])
                print(f"rank {r}: {nbad} owned rows with different neighbours/L")
            for part, rows in (("own", slice(0, d["n"])), ("halo", slice(d["n"], None))):
                pos = inv[d["gid"][rows]]
                for f in ("us", "rb", "v", "al", "sddot", "Hh"):
                    a, b = d[f][rows], e[f][pos]
                    if f == "al" or f == "sddot" or f == "Hh":
                        if part == "halo":
                            continue
                    bad = np.flatnonzero(~np.all(a.reshape(a.shape[0], -1) == b.reshape(b.shape[0], -1), axis=1)) if a.size else []
                    if len(bad):
                        print(f"rank {r} snap {k} {part} {f}: {len(bad)}/{a.shape[0]} rows differ, "
                              f"first gid {d['gid'][rows][bad[:5]]} maxdiff {np.abs(a-b).max():.3e}")
    print("done")


if __name__ == "__main__":
    main()
