"""The reference's controller pins (proj/tests/test_controller.cpp) on the
quadratic test system, run against both the oracle (CPU) and the device path
(through the C ABI, fp64).  Same inputs, same assertions as the reference.
"""
import math

import numpy as np
import pytest

from paper_1707_02342_b200.api import ControlBounds, SamplingParams, SGFilter

BACKENDS = [pytest.param("oracle", id="oracle"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


def small_params(K, T, seed):
    """test_controller.cpp:9-20."""
    return SamplingParams(samples=K, horizon_steps=T, dt=0.05, sigma_diag=(0.04, 0.09), lambda_=1.0, gamma=0.0,
                          explore_fraction=0.0, seed=seed)


def make(backend, params, sg=None, bounds=None, quad_cost_scale=1.0, noise="ref_splitmix"):
    """make_state (test_controller.cpp:39-42): bounds +-10, IT rule."""
    bounds = bounds or ControlBounds((-10.0, -10.0), (10.0, 10.0))
    kw = dict(system="quadratic", precision="fp64", noise=noise, quad_cost_scale=quad_cost_scale)
    if backend == "oracle":
        import oracle
        return oracle.OracleController(params, bounds, sg, None, **kw)
    from paper_1707_02342_b200.api import Controller
    return Controller(params, bounds, sg, **kw)


def batch(K, T, fill):
    """PerturbationBatch of constant T x 2 matrices, reference layout (K, 2, T)."""
    e = np.empty((K, 2, T))
    e[:] = np.asarray(fill, dtype=float).T if np.ndim(fill) == 2 else fill
    return e


@pytest.fixture(params=BACKENDS)
def backend(request):
    return request.param


def test_single_zero_noise_sample(backend):
    """test_controller.cpp:46-64."""
    p = small_params(1, 12, 3)
    cs = make(backend, p)
    U = np.zeros((12, 2))
    U[:, 0] = 0.5
    cs.plan = U
    costs = cs.rollout_batch(np.zeros(2), np.zeros((1, 2, 12)))
    x0, expect = 0.0, 0.0
    for _ in range(12):
        x0 += 0.5 * p.dt
        expect += x0 * x0
    assert costs[0] == pytest.approx(expect, rel=1e-15)


def test_duplicate_samples(backend):
    """test_controller.cpp:66-76."""
    p = small_params(4, 8, 7)
    cs = make(backend, p)
    costs = cs.rollout_batch(np.ones(2), batch(4, 8, 0.123))
    assert np.all(costs[1:] == costs[0])


def test_zero_mean_noop_at_zero_plan(backend):
    """test_controller.cpp:78-89 (flags {0,1} = trailing lround(0.5*2) = 1)."""
    p = small_params(2, 10, 11)
    p.explore_fraction = 0.5
    cs = make(backend, p)
    e = batch(2, 10, 0.2)
    costs, stored = cs.rollout_batch(np.zeros(2), e, return_batch=True)
    assert costs[0] == costs[1]
    assert np.array_equal(stored[1], e[1])


def test_flagged_samples_store_eps_minus_plan(backend):
    """test_controller.cpp:91-108."""
    p = small_params(2, 6, 13)
    p.explore_fraction = 0.5
    cs = make(backend, p)
    cs.plan = np.full((6, 2), 0.4)
    costs, stored = cs.rollout_batch(np.zeros(2), batch(2, 6, 0.25), return_batch=True)
    assert costs[1] < costs[0]
    assert np.max(np.abs(stored[1] - (0.25 - 0.4))) <= 1e-15
    assert np.max(np.abs(0.4 + stored[1] - 0.25)) <= 1e-15


def test_costs_independent_of_partitioning(backend):
    """test_controller.cpp:110-123: thread count (oracle) / launch shape (device) do not change costs."""
    p = small_params(37, 15, 17)
    cs = make(backend, p)
    cs.plan = np.full((15, 2), 0.1)
    c1 = cs.rollout_batch(np.ones(2))
    if backend == "oracle":
        assert np.array_equal(c1, cs.rollout_batch(np.ones(2), threads=4))
        assert np.array_equal(c1, cs.rollout_batch(np.ones(2), threads=8))
    else:
        assert np.array_equal(c1, cs.rollout_batch(np.ones(2)))


def test_one_hot_weight_adds_that_perturbation(backend):
    """test_controller.cpp:125-134."""
    p = small_params(3, 9, 19)
    cs = make(backend, p)
    _, stored = cs.rollout_batch(np.zeros(2), return_batch=True)
    w = np.zeros(3)
    w[2] = 1.0
    U = cs.update_plan(w)
    assert np.max(np.abs(U - stored[2].T)) <= 1e-15


def test_symmetric_pairs_cancel(backend):
    """test_controller.cpp:136-148."""
    p = small_params(2, 7, 23)
    cs = make(backend, p)
    cs.plan = np.full((7, 2), 0.3)
    e = np.random.default_rng(0).uniform(-1, 1, (2, 7))
    cs.rollout_batch(np.zeros(2), np.stack([e, -e]))
    U = cs.update_plan(np.array([0.5, 0.5]))
    assert np.max(np.abs(U - 0.3)) <= 1e-15


def test_uniform_weights_clt_envelope(backend):
    """test_controller.cpp:150-161."""
    p = small_params(10000, 5, 29)
    cs = make(backend, p)
    cs.rollout_batch(np.zeros(2))
    U = cs.update_plan(np.full(10000, 1e-4))
    for c in range(2):
        assert np.abs(U[:, c]).max() <= 4.0 * math.sqrt(p.sigma_diag[c]) / 100.0


def test_aggregation_matches_sequential_bitwise(backend):
    """test_controller.cpp:163-175: U' == sum_k w_k eps_k in ascending order, bitwise."""
    import oracle
    p = small_params(64, 10, 31)
    cs = make(backend, p)
    cs.iteration = 4
    _, stored = cs.rollout_batch(np.zeros(2), return_batch=True)
    costs = np.array([math.sin(0.2 * k) * 3.0 + k % 5 for k in range(64)])
    w, _, _ = oracle.it_weights(costs, p.lambda_)
    ref = np.zeros((10, 2))
    for k in range(64):
        ref = ref + w[k] * stored[k].T
    U = cs.update_plan(w)
    assert np.array_equal(U, ref)


def test_mpc_step_emits_clamped_first_input_then_shifts(backend):
    """test_controller.cpp:177-197."""
    p = small_params(128, 6, 37)
    p.sigma_diag = (2.0, 2.0)
    bounds = ControlBounds((-0.1, -0.1), (0.1, 0.1))
    probe = make(backend, p, bounds=bounds)
    costs = probe.rollout_batch(np.ones(2))
    import oracle
    w, _, _ = oracle.it_weights(costs, p.lambda_)
    updated = probe.update_plan(w)
    cs = make(backend, p, bounds=bounds)
    u0 = cs.mpc_step(np.ones(2))
    tol = 0 if backend == "oracle" else 1e-12  # device softmin merge order differs by rounding
    assert abs(u0[0] - np.clip(updated[0, 0], -0.1, 0.1)) <= tol
    assert abs(u0[1] - np.clip(updated[0, 1], -0.1, 0.1)) <= tol
    plan = cs.plan
    assert np.allclose(plan[:5], updated[1:], rtol=0, atol=tol)
    assert np.all(plan[5] == 0)
    assert cs.iteration == 1


def test_mpc_step_bit_identical_across_partitioning(backend):
    """test_controller.cpp:199-217."""
    p = small_params(96, 12, 41)
    runs = []
    for threads in (1, 4, 8):
        cs = make(backend, p, sg=SGFilter(5, 2))
        for _ in range(3):
            u = cs.mpc_step(np.ones(2), threads=threads) if backend == "oracle" else cs.mpc_step(np.ones(2))
        runs.append((cs.plan, u))
    for plan, u in runs[1:]:
        assert np.array_equal(plan, runs[0][0]) and np.array_equal(u, runs[0][1])


def test_zero_cost_landscape_pulls_plan_to_zero(backend):
    """test_controller.cpp:219-231."""
    p = small_params(256, 8, 43)
    p.gamma = p.lambda_
    cs = make(backend, p, quad_cost_scale=0.0)
    cs.plan = np.full((8, 2), 1.5)
    initial = np.linalg.norm(cs.plan)
    out = cs.optimize_to_convergence(np.zeros(2), 60)
    assert np.linalg.norm(out) < 0.25 * initial


def test_one_pass_equals_mpc_update_without_shift(backend):
    """test_controller.cpp:233-247."""
    import oracle
    p = small_params(32, 9, 47)
    a = make(backend, p)
    a.plan = np.full((9, 2), 0.2)
    b = make(backend, p)
    b.plan = np.full((9, 2), 0.2)
    converged = a.optimize_to_convergence(np.ones(2), 1)
    costs = b.rollout_batch(np.ones(2))
    w, _, _ = oracle.it_weights(costs, p.lambda_)
    expected = b.update_plan(w)
    if backend == "oracle":
        assert np.array_equal(converged, expected)
    else:  # fused chunk-partial softmin vs explicit weights: rounding-level difference
        assert np.allclose(converged, expected, rtol=0, atol=1e-13)


@pytest.mark.parametrize("f", [0.0, 0.05, 0.2])
def test_explore_fraction_does_not_bias(backend, f):
    """test_controller.cpp:249-270."""
    import oracle
    p = small_params(20000, 4, 53)
    p.explore_fraction = f
    cs = make(backend, p, quad_cost_scale=0.0)
    cs.plan = np.full((4, 2), 0.1)
    costs = cs.rollout_batch(np.zeros(2))
    w, _, _ = oracle.it_weights(costs, p.lambda_)
    U = cs.update_plan(w)
    for c in range(2):
        se = math.sqrt(p.sigma_diag[c] / p.samples)
        assert np.abs(U[:, c] - 0.1).max() <= 6.0 * se
