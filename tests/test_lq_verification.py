"""The reference's LQ verification: the sampling optimizer converges to the
Riccati plan on a linear-quadratic instance (verification.cpp:44-108,
test_verification.cpp:130-222, acceptance.cpp:47-87).

CPU: the numpy restatement of riccati_plan / lqr_oracle (tests/oracle.py)
against the reference's own pins.  GPU: the device controller's
optimize_to_convergence on the reference's quadratic test system
(x' = x + v dt, running cost s |x|^2, terminal 0 — an LQ instance with
A = I, B = dt I, Q = s I, Q_f = 0) against that oracle, with the acceptance
criterion's bar (rms plan error <= 5 % of the oracle plan's rms).
"""
import numpy as np
import pytest

import oracle


def double_integrator(T, lam, sigma2):
    """test_verification.cpp:9-20."""
    return dict(A=np.array([[1.0, 0.05], [0.0, 1.0]]), B=np.array([[0.0], [0.05]]),
                Q=np.diag([1.0, 0.1]), Qf=np.diag([20.0, 2.0]), sigma_diag=[sigma2], lam=lam, T=T,
                x0=np.array([2.0, 0.0]))


def test_riccati_scalar_zero_costs_and_scale_invariance():
    """test_verification.cpp:130-162."""
    one = np.eye(1)
    plan = oracle.lqr_oracle(one, one, np.zeros((1, 1)), one, [1.0], 2.0, 1, np.ones(1))
    assert plan[0, 0] == pytest.approx(-0.5, rel=1e-14)

    zero = double_integrator(10, 0.5, 1.0)
    zero["Q"] = np.zeros((2, 2))
    zero["Qf"] = np.zeros((2, 2))
    assert np.abs(oracle.lqr_oracle(**zero)).max() == 0.0

    base = double_integrator(15, 0.5, 1.0)
    doubled = dict(base, Q=2.0 * base["Q"], Qf=2.0 * base["Qf"], lam=2.0 * base["lam"])  # doubles R too
    assert np.abs(oracle.lqr_oracle(**base) - oracle.lqr_oracle(**doubled)).max() <= 1e-12

    bad = dict(base, Q=np.array([[0.0, 5.0], [5.0, 0.0]]))  # indefinite
    with pytest.raises(ValueError):
        oracle.lqr_oracle(**bad)


def test_riccati_is_the_minimizer_on_a_short_horizon():
    """test_verification.cpp:164-199 (there by coordinate descent; here the
    exact minimizer of the same convex quadratic J(V))."""
    inst = double_integrator(3, 0.8, 0.5)
    A, B, Q, Qf, T, x0 = inst["A"], inst["B"], inst["Q"], inst["Qf"], inst["T"], inst["x0"]
    r = inst["lam"] / 2.0 / inst["sigma_diag"][0]
    # x_{t+1} = F_t x0 + G_t V; J = sum_t x_{t+1}' Q x_{t+1} + r |V|^2 + x_T' Qf x_T
    H = r * np.eye(T)
    g = np.zeros(T)
    F = np.eye(2)
    G = np.zeros((2, T))
    for t in range(T):
        F = A @ F
        G = A @ G
        G[:, t] = B[:, 0]
        W = Q + (Qf if t == T - 1 else 0.0)
        H += G.T @ W @ G
        g += G.T @ W @ (F @ x0)
    v = np.linalg.solve(H, -g)
    plan = oracle.lqr_oracle(**inst)
    assert np.allclose(plan[:, 0], v, rtol=1e-5, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_device_optimizer_converges_to_riccati(precision):
    """acceptance.cpp:47-87 on the reference's quadratic test system: gamma =
    lambda (alpha = 0, the oracle's objective), no exploration samples, no
    smoothing, unbounded controls, 100 optimize_to_convergence iterations of
    4096 samples; rms(plan - riccati) <= 5 % of rms(riccati)."""
    from paper_1707_02342_b200.api import ControlBounds, Controller, SamplingParams

    T, dt, s, lam, sig2 = 20, 0.05, 1.0, 0.02, 0.04
    x0 = np.array([2.0, -1.0])
    p = SamplingParams(samples=4096, horizon_steps=T, dt=dt, sigma_diag=(sig2, sig2), lambda_=lam, gamma=lam,
                       explore_fraction=0.0, seed=1)
    g = Controller(p, ControlBounds((-1e9, -1e9), (1e9, 1e9)), None, system="quadratic", precision=precision,
                   noise="philox", quad_cost_scale=s)
    plan = g.optimize_to_convergence(x0, 100)
    ref = oracle.lqr_oracle(np.eye(2), dt * np.eye(2), s * np.eye(2), np.zeros((2, 2)), [sig2, sig2], lam, T, x0)
    ratio = np.sqrt(np.mean((plan - ref) ** 2)) / np.sqrt(np.mean(ref ** 2))
    print(f"{precision}: rms(plan - riccati) / rms(riccati) = {ratio:.4f}")
    assert ratio <= 0.05
