"""Lagrangian particle loop (Algorithm 1; SPEC.md:466-470,
acceptance criterion 11): the device step against a numpy restatement of the
same update driven by the oracle's find/eval, the analytic uniform-flow
trajectory, particle conservation under periodic wrapping."""
import numpy as np
import pytest
import torch

from oracle import oracle as O


def ab2_reference(x, v, u_of, tau, dt, steps, lo, hi):
    """numpy restatement of fpx_particles_advance + periodic wrap."""
    vp = np.zeros_like(v)
    ap = np.zeros_like(v)
    L = hi - lo
    for s in range(steps):
        u = u_of(x)
        a = (u - v) / tau
        if s == 0:
            xn, vn = x + dt * v, v + dt * a
        else:
            xn, vn = x + dt * (1.5 * v - 0.5 * vp), v + dt * (1.5 * a - 0.5 * ap)
        xn = lo + (xn - lo) - L * np.floor((xn - lo) / L)
        vp, ap, x, v = v, a, xn, vn
    return x, v


def test_ab2_reference_uniform_flow_converges():
    # host restatement alone: v -> u, x translates at speed 1
    x0 = np.array([[0.2, 0.3, 0.4]])
    x, v = ab2_reference(x0, np.zeros_like(x0), lambda x: np.array([[1.0, 0, 0]]), 0.01, 1e-3,
                         400, np.zeros(3), np.ones(3))
    assert abs(v[0, 0] - 1.0) < 1e-6 and abs(v[0, 1]) < 1e-12
    assert 0 <= x[0, 0] < 1


@pytest.mark.gpu
def test_uniform_flow_conservation_and_translation():
    from paper_2501_12349_b200 import engine, particles, toolkit
    mesh = toolkit.box_mesh(3, 6, 3)
    S = engine.setup(mesh)
    vel = toolkit.analytic_field("uniform_velocity", mesh, value=(1.0, 0.0, 0.0))
    x0 = toolkit.uniform_points(2000, 3, seed=3, lo=0.05, hi=0.95)
    out = particles.run_particles(S, vel, x0, tau=0.01, dt=1e-3, steps=300,
                                  box=((0, 0, 0), (1, 1, 1)))
    st = out["state"]
    assert out["particles"] == 2000 and out["removed"] == 0   # conservation
    v = st.v.cpu().numpy()
    assert np.max(np.abs(v[:, 0] - 1.0)) < 1e-6 and np.max(np.abs(v[:, 1:])) < 1e-12
    xr, vr = ab2_reference(x0, np.zeros_like(x0), lambda x: np.tile([1.0, 0, 0], (len(x), 1)),
                           0.01, 1e-3, 300, np.zeros(3), np.ones(3))
    assert np.max(np.abs(st.x.cpu().numpy() - xr)) < 1e-12
    assert set(out["phase_ms"]) == {"interpolate", "integrate", "find"}


@pytest.mark.gpu
def test_taylor_green_matches_oracle_loop():
    from paper_2501_12349_b200 import engine, particles, toolkit
    from paper_2501_12349_b200.basis import BasisConstants
    mesh = toolkit.box_mesh(3, 5, 4)
    S = engine.setup(mesh)
    vel = toolkit.analytic_field("taylor_green", mesh)
    bc = BasisConstants.of(S.basis, S.envelope)
    B = O.basis_from_arrays(bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta, bc.lo, bc.hi)
    OS = O.OracleSetup(mesh.nodes, 3, 3, 4, B=B, ncell=S.ncell)

    def u_of(x):
        rec = OS.find(x)
        return O.evaluate(B, 3, vel, rec["code"], rec["elem"], rec["r"])

    x0 = toolkit.uniform_points(500, 3, seed=4, lo=0.1, hi=0.9)
    v0 = np.zeros_like(x0)
    out = particles.run_particles(S, vel, x0, v=v0, tau=0.2, dt=2e-3, steps=25,
                                  box=((0, 0, 0), (1, 1, 1)))
    xr, vr = ab2_reference(x0, v0, u_of, 0.2, 2e-3, 25, np.zeros(3), np.ones(3))
    st = out["state"]
    assert out["particles"] == 500
    assert np.max(np.abs(st.x.cpu().numpy() - xr)) < 1e-11
    assert np.max(np.abs(st.v.cpu().numpy() - vr)) < 1e-10


@pytest.mark.gpu
def test_not_found_after_wrap_is_removed():
    # a non-periodic axis lets particles leave the mesh: they are dropped
    from paper_2501_12349_b200 import engine, particles, toolkit
    mesh = toolkit.box_mesh(3, 4, 2)
    S = engine.setup(mesh)
    vel = toolkit.analytic_field("uniform_velocity", mesh, value=(0.0, 0.0, 5.0))
    x0 = np.array([[0.5, 0.5, 0.98], [0.5, 0.5, 0.2]])
    out = particles.run_particles(S, vel, x0, tau=0.004, dt=2e-3, steps=20,
                                  box=((0, 0, 0), (1, 1, 1)), periodic=0b011)
    assert out["removed"] == 1 and out["particles"] == 1
