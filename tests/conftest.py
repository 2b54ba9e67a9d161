"""Shared test plumbing.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.  The oracle is test
infrastructure and is only imported from here and from bench.py.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def relerr(x, ref):
    """Normwise metric of the reference tests: max|x-ref| / max|ref|."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(x - ref).max() if ref.size else 0.0
    if den == 0.0:
        return num
    return num / den


def lattice_2d(nx, nz, dp, origin=(0.0, 0.0, 0.0)):
    xs = origin[0] + (np.arange(nx) + 0.5) * dp
    zs = origin[2] + (np.arange(nz) + 0.5) * dp
    gx, gz = np.meshgrid(xs, zs, indexing="ij")
    return np.column_stack([gx.ravel(), np.full(gx.size, origin[1]), gz.ravel()])


def lattice_3d(nx, ny, nz, dp, origin=(0.0, 0.0, 0.0)):
    xs = origin[0] + (np.arange(nx) + 0.5) * dp
    ys = origin[1] + (np.arange(ny) + 0.5) * dp
    zs = origin[2] + (np.arange(nz) + 0.5) * dp
    g = np.meshgrid(xs, ys, zs, indexing="ij")
    return np.column_stack([a.ravel() for a in g])


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    return O


def run_case(G):
    """CaseConfig of a golden run with its stored initial state applied."""
    from paper_2602_15149_b200 import cases
    cfg = cases.case_from_dict(G)
    for bi, b in enumerate(cfg.bodies):
        for k in ("u", "v", "s"):
            key = f"init.b{bi}.{k}"
            if key in G:
                getattr(b.state, k)[:] = G[key]
    return cfg
