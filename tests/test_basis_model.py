"""The basis-function vehicle model: the reference's
BasisFunctionModel (proj/src/dynamics.cpp:83-157) as a second device model.

CPU: the reference's own eval_basis / step_basis_model pins
(proj/tests/test_dynamics.cpp:158-226) against the oracle restatement.
GPU: the device model against the oracle — fp64 per-sample costs and state
trajectories to rtol 1e-12, fp32 to the float restatement, the reference
pins through the device rollout, mpc_step and the closed loop.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1707_02342_b200 import workload


def test_basis_vanishes_at_origin():
    """test_dynamics.cpp:158-161."""
    assert np.max(np.abs(oracle.eval_basis([0, 0, 0, 0], [0, 0]))) == 0.0


def test_basis_identities_and_slow_speed_branch():
    """test_dynamics.cpp:163-174: v_x = 0.05 is below the 0.1 guard."""
    phi = oracle.eval_basis([0.1, 0.05, 0.4, -0.2], [0.3, -0.6])
    assert phi[0] == -0.6
    assert phi[8] == math.sin(0.3)
    assert phi[9] == 0.0
    assert phi[10] == math.tan(-0.3) / 1400.0
    assert phi[13] == 0.0
    assert phi[23] == pytest.approx(0.36)
    assert phi[24] == pytest.approx(-0.216)


def test_basis_slip_angles_above_guard():
    """test_dynamics.cpp:176-186."""
    phi = oracle.eval_basis([0.0, 2.0, 0.4, 1.0], [0.25, 0.0])
    af = math.atan(0.4 / 2.0 + 0.45 * 1.0 / 2.0 - 0.25)
    ar = math.atan(0.4 / 2.0 - 0.35 * 1.0 / 2.0)
    assert phi[10] == pytest.approx(math.tan(af) / 1400.0, rel=1e-15)
    assert phi[13] == pytest.approx(math.tan(ar) / 40.0, rel=1e-15)
    assert phi[9] == pytest.approx((0.4 / 2.0) / 40.0, rel=1e-15)
    assert phi[16] == pytest.approx(1.0 * 2.0 / 50.0, rel=1e-15)


def _x(theta=0.0, vx=0.0, vy=0.0, thd=0.0, roll=0.0, px=0.0, py=0.0):
    return np.array([px, py, theta, roll, vx, vy, thd])


def test_zero_theta_leaves_dynamic_block():
    """test_dynamics.cpp:188-202."""
    x = _x(theta=0.7, vx=4.0, vy=-0.5, thd=0.9, roll=0.02)
    n = oracle.step_basis(x, [0.2, 0.5], 0.025, np.zeros((25, 4)))
    assert n[3] == x[3] and n[4] == x[4] and n[5] == x[5] and n[6] == x[6]
    assert n[0] == pytest.approx((math.cos(0.7) * 4.0 - math.sin(0.7) * -0.5) * 0.025)
    assert n[2] == pytest.approx(0.7 + 0.9 * 0.025)


def test_heading_rotation():
    """test_dynamics.cpp:204-211."""
    n = oracle.step_basis(_x(theta=math.pi / 2, vx=1.0), [0, 0], 0.1, np.zeros((25, 4)))
    assert n[1] == pytest.approx(0.1, rel=1e-12)
    assert abs(n[0]) <= 1e-15


def test_basis_step_linear_in_theta():
    """test_dynamics.cpp:213-226."""
    th = np.zeros((25, 4))
    th[8, 1] = 2.0
    x = _x(vx=3.0)
    n = oracle.step_basis(x, [0.4, 0.1], 0.025, th)
    assert n[4] == pytest.approx(3.0 + 2.0 * math.sin(0.4) * 0.025, rel=1e-15)
    n2 = oracle.step_basis(x, [0.4, 0.1], 0.025, 2 * th)
    assert n2[4] - 3.0 == pytest.approx(2.0 * (n[4] - 3.0), rel=1e-12)


def test_basis_dt_must_be_positive():
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.step_basis(_x(vx=1.0), [0, 0], 0.0, np.zeros((25, 4)))


# ------------------------------------------------------------------ device
def _pair(w, prec, noise):
    from paper_1707_02342_b200.api import Controller
    g = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise=noise, system="vehicle_basis")
    o = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, precision=prec, noise=noise,
                                system="vehicle_basis")
    for c in (g, o):
        c.set_basis(w.theta)
        c.set_costmap(w.costmap)
    return g, o


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_device_basis_rollout_matches_oracle(prec):
    w = workload.make("ref10", samples=512)
    g, o = _pair(w, prec, "injected")
    eps, _ = oracle.sample_perturbations(512, w.params.horizon_steps, w.params.sigma_diag,
                                         w.params.explore_fraction, w.params.seed, 0)
    U = np.random.default_rng(5).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
    g.plan = U
    o.plan = U
    dc, oc = g.rollout_batch(w.x0[0], eps), o.rollout_batch(w.x0[0], eps, threads=8)
    if prec == "fp64":
        assert np.allclose(dc, oc, rtol=1e-12, atol=0)
        for k in (0, 200, 511):
            assert np.allclose(g.rollout_states(w.x0[0], k), o.rollout_states(w.x0[0], k), rtol=1e-12, atol=1e-12)
    else:
        rel = np.abs(dc - oc) / np.abs(oc)
        assert (rel <= 1e-5).mean() >= 0.99 and np.sum(np.abs(dc - oc) > 5000) <= 2


@pytest.mark.gpu
def test_device_basis_zero_theta_pin():
    """test_dynamics.cpp:188-202 through the device rollout: with Theta = 0 the
    dynamic block of every state along the trajectory stays at x0's."""
    from paper_1707_02342_b200.api import Controller
    w = workload.make("ref10", samples=1, horizon_steps=6)
    g = Controller(w.params, w.bounds, w.sg, w.cost, precision="fp64", noise="injected", system="vehicle_basis")
    g.set_basis(np.zeros((25, 4)))
    g.set_costmap(w.costmap)
    x0 = _x(theta=0.7, vx=4.0, vy=-0.5, thd=0.9, roll=0.02)
    g.rollout_batch(x0, np.zeros((1, 2, 6)))
    traj = g.rollout_states(x0, 0)
    assert np.all(traj[:, 3:] == x0[3:])
    assert traj[1, 0] == pytest.approx((math.cos(0.7) * 4.0 - math.sin(0.7) * -0.5) * w.params.dt)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_device_basis_mpc_step_and_closed_loop(prec):
    w = workload.make("ref10", samples=1024)
    g, o = _pair(w, prec, "ref_splitmix")
    x = w.x0[0].copy()
    for it in range(3):
        ud, uo = g.mpc_step(x), o.mpc_step(x, threads=8)
        tol = 1e-10 if prec == "fp64" else 1e-4
        assert np.max(np.abs(g.plan - o.plan)) <= tol, it
        assert np.max(np.abs(ud - uo)) <= tol
        g.plan = o.plan
        x = o.vehicle_step(x, uo)
    if prec == "fp64":  # the device plant is the basis model too
        c, _ = _pair(w, prec, "ref_splitmix")
        u, xt = c.closed_loop(w.x0[0], 3)
        for i in range(3):
            assert np.allclose(xt[i + 1, 0], o.vehicle_step(xt[i, 0], u[i, 0]), rtol=1e-12, atol=1e-12)
