"""Error paths of the device step against the reference's own exceptions.

tests/golden/errors.npz holds, per scenario, a case, the state edits applied
after initialize() and the exception the REFERENCE raised (type and message,
oracle/gen_golden.py gen_errors, numpy backend):

  acc        non-finite acceleration, first bad particle and step
             (stepper.py:96-100)
  state64    non-finite state at the 64th commit (stepper.py:203-209)
  dtcollapse adaptive dt collapsing to 0 inside run() (stepper.py:254-255)
  div0       velocity-BC expression dividing by zero (expr.py:513-515)
  restrict   restrictphi expression outside [0, 1] (fracture.py:59-63)
  nonspd     J2 radial return leaving the SPD cone, first bad particle
             (constitutive.py:191-194)
  noconv     SVK split: Jacobi non-convergence count (fast.py:254-256)

The device records these in counters and clock flags and raises at the
next sync point with the reference's message; a step that raised is not
committed (t and step_index as the reference leaves them).
"""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def GE():
    return golden("errors")


def _expected(G, tag):
    name, msg = bytes(np.asarray(G[f"{tag}.exc"], dtype=np.uint8)).decode().split("\n", 1)
    return name, msg


def _build(G, tag, precision="fp64"):
    from paper_2602_15149_b200 import cases
    from paper_2602_15149_b200.simulation import DeviceSimulation
    cfg = cases.case_from_dict(G, prefix=f"{tag}.")
    st = cfg.bodies[0].state
    for k in ("u", "v", "s"):
        getattr(st, k)[:] = G[f"{tag}.init.{k}"]
    if f"{tag}.init.Cp" in G:
        st.Cp[:] = G[f"{tag}.init.Cp"]
    return cfg, DeviceSimulation(cfg, precision=precision)


def _drive(G, tag, sim, cfg, via_run=False):
    sim.initialize()
    fields = bytes(np.asarray(G[f"{tag}.edit_fields"], dtype=np.uint8)).decode()
    edits = G[f"{tag}.edits"]
    if len(edits):
        st = cfg.bodies[0].state
        for f, (i, a, v) in zip(fields.split(","), edits):
            getattr(st, f)[int(i), int(a)] = v
        sim.push_state()
    steps, t_max, t_out = G[f"{tag}.driver"]
    if t_max > 0:
        sim.run(time_max=float(t_max), time_out=float(t_out))
    elif via_run:
        sim.run(time_max=1.0, time_out=1.0, max_steps=int(steps), batch=16)
    else:
        for _ in range(int(steps)):
            sim.step(sim.pick_dt())


@pytest.mark.parametrize("via_run", [False, True])
@pytest.mark.parametrize("tag", ["acc", "state64", "dtcollapse", "div0", "restrict", "nonspd"])
def test_device_raises_like_reference(GE, tag, via_run):
    name, msg = _expected(GE, tag)
    cfg, sim = _build(GE, tag)
    with pytest.raises(Exception) as ei:
        _drive(GE, tag, sim, cfg, via_run)
    assert type(ei.value).__name__ == name
    assert str(ei.value) == msg
    # the step that raised is not committed (the reference raises before
    # _commit, except the state check, which follows it)
    assert sim.t == float(GE[f"{tag}.t"][0])
    assert sim.step_index == int(GE[f"{tag}.steps_done"][0]) + (1 if tag == "state64" else 0)


def test_fp32_acceleration_error(GE):
    """FP32 mode reports the same first non-finite particle and step."""
    name, msg = _expected(GE, "acc")
    cfg, sim = _build(GE, "acc", "fp32")
    with pytest.raises(Exception) as ei:
        _drive(GE, "acc", sim, cfg)
    assert (type(ei.value).__name__, str(ei.value)) == (name, msg)


def test_nonspd_skips_momentum(GE):
    """A stress error raises before momentum (constitutive.py:191-194): pass B
    does not run, so u and v keep their values from the start of the step."""
    cfg, sim = _build(GE, "nonspd")
    st = cfg.bodies[0].state
    u0, v0 = st.u.copy(), st.v.copy()
    with pytest.raises(Exception, match="non-SPD plastic metric at particle 517"):
        sim.initialize()
    assert np.array_equal(st.u, u0)
    assert np.array_equal(st.v, v0)


def test_plugin_svk_noconv_count(GE):
    """Jacobi non-convergence through the plugin (numba reference count)."""
    from paper_2602_15149_b200 import backend
    F = GE["noconv.F"]
    n = F.shape[0]
    S, psi, psip = np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n)
    nc = backend.svk_batch(F, 2.7733e6, 0.715e6, GE["noconv.s"], True, S, psi, psip)
    assert nc == int(GE["noconv.n"][0])


def test_noconv_message(GE):
    """The step path's eigen counter becomes the reference's message
    (constitutive.py:177-180) and the step is not committed."""
    cfg, sim = _build(GE, "restrict")
    sim.initialize()
    sim.dbodies[0].counters[1] = 3
    with pytest.raises(Exception) as ei:
        sim._check_errors()
    assert type(ei.value).__name__ == "SimulationError"
    assert str(ei.value) == "eigensolver failed to converge for 3 particles (body 1)"
