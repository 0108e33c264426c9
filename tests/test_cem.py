"""The cross-entropy weight rule: cem_weights
(proj/src/weights.cpp:27-53) behind compute_weights (controller.cpp:111-116).

CPU: the reference's CEM pins (proj/tests/test_weights.cpp:64-102) against the
oracle.  GPU: the same pins through mppi_gpu_weights (device radix select with
index tie-breaking), and mpc_step with the CEM rule against the oracle.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1707_02342_b200.api import ControlBounds, SamplingParams

PINS_COSTS_1200 = np.array([math.cos(0.37 * k) * 50.0 + k % 7 for k in range(1200)])


def _check_pins(weights):
    w, rho, eta = weights(np.array([5.0, 1.0, 4.0, 2.0, 3.0]), 0.8)  # test_weights.cpp:64-73
    assert w[1] == 1.0 and w.sum() == 1.0 and all(w[k] == 0.0 for k in (0, 2, 3, 4))
    assert rho == 1.0 and eta == 1.0
    w, _, _ = weights(np.full(10, 3.5), 0.8)  # ties by ascending index, test_weights.cpp:75-81
    assert w[0] == 0.5 and w[1] == 0.5 and np.all(w[2:] == 0.0)
    w, _, _ = weights(PINS_COSTS_1200, 0.8)  # test_weights.cpp:83-95
    nz = w[w != 0.0]
    assert len(nz) == 240 and np.all(nz == 1.0 / 240.0)
    assert w.sum() == pytest.approx(1.0, abs=1e-12)


def test_cem_pins_oracle():
    _check_pins(oracle.cem_weights)


def test_cem_rejects_bad_delta_oracle():
    """test_weights.cpp:97-102."""
    for d in (0.999, 1.2, 0.0):
        with pytest.raises(oracle.OracleInvalidArgument):
            oracle.cem_weights(np.zeros(3), d)
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.cem_weights(np.array([0.0, np.nan, 1.0]), 0.5)


def _device_weights(costs, delta):
    from paper_1707_02342_b200.api import Controller
    p = SamplingParams(samples=len(costs), horizon_steps=4, lambda_=1.0)
    g = Controller(p, system="quadratic", precision="fp64", weight_rule="cem", cem_delta=delta)
    r = g.compute_weights(costs)
    return r.weights, r.rho, r.normalizer


@pytest.mark.gpu
def test_cem_pins_device():
    _check_pins(_device_weights)
    # a random permutation with heavy ties: the device selection equals the stable sort
    rng = np.random.default_rng(3)
    c = rng.integers(0, 50, 20000).astype(float)
    w, _, _ = _device_weights(c, 0.7)
    wo, _, _ = oracle.cem_weights(c, 0.7)
    assert np.array_equal(w, wo)


@pytest.mark.gpu
def test_cem_device_rejects_nonfinite():
    from paper_1707_02342_b200.api import Controller, InvalidArgument
    p = SamplingParams(samples=3, horizon_steps=4, lambda_=1.0)
    g = Controller(p, system="quadratic", precision="fp64", weight_rule="cem", cem_delta=0.5)
    with pytest.raises(InvalidArgument):
        g.compute_weights([0.0, np.nan, 1.0])
    with pytest.raises(InvalidArgument):
        Controller(p, system="quadratic", precision="fp64", weight_rule="cem", cem_delta=0.999)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_cem_mpc_step_matches_oracle(prec):
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller
    w = workload.make("c0")
    kw = dict(hidden=32, precision=prec, noise="ref_splitmix", weight_rule="cem", cem_delta=0.8)
    g = Controller(w.params, w.bounds, w.sg, w.cost, **kw)
    o = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, **kw)
    for c in (g, o):
        c.set_mlp(w.mlp)
        c.set_costmap(w.costmap)
    x = w.x0[0].copy()
    for it in range(3):
        g.mpc_step(x)
        uo = o.mpc_step(x, threads=8)
        # fp64 agrees to rounding.  In fp32 a sample whose cost sits at the
        # elite threshold can swap in or out (costs agree to ~5e-8 relative);
        # one swap moves the update by at most 2 max|eps| / elite ~ 8e-3 here.
        tol = 1e-10 if prec == "fp64" else 1e-2
        assert np.max(np.abs(g.plan - o.plan)) <= tol, (it, np.max(np.abs(g.plan - o.plan)))
        g.plan = o.plan
        x = o.vehicle_step(x, uo)
