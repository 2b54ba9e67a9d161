"""B200-native (sm_100a) TLSPH hot path for the SoliDualSPHysics solid solver
(arxiv 2602.15149), a drop-in behind the reference package ``solidsph``.

Public surface (mirrors the reference API):
  * ``backend``       -- the backend plugin (NAME + the 8 per-step kernels)
  * ``kernel_geom``   -- device neighbour build / correction (build_adjacency hook)
  * ``DeviceSimulation`` (alias ``Simulation``) -- device-resident stepper
  * ``core``, ``expr``, ``cases`` -- data model, expressions, case assembly
The compute runs in ``libtlsph.so`` (include/tlsph.h); there is no CPU path.
"""

__version__ = "0.1.0"

from . import core, expr  # noqa: F401


def __getattr__(name):
    if name in ("DeviceSimulation", "Simulation"):
        from .simulation import DeviceSimulation
        return DeviceSimulation
    if name in ("backend", "kernel_geom", "cases", "simulation", "build"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
