"""The bicycle truth model and the closed-loop driver.

* CPU: the reference's brush-tire and truth-model pins (test_dynamics.cpp:65-156)
  on the library's host plant (mppi_brush_tire_force / mppi_bicycle_step) and
  on the oracle restatement, and the two bit-identical to each other.
* GPU: the bicycle as the controller's own rollout model (fp64 rtol 1e-12
  and fp32 against the restatements), the model-agnostic trajectory-cost pins
  (test_costs.cpp:203-260: with gamma = 0 the plan only matters through the
  realised inputs; pre-clamped rollouts equal clamping inside the rollout) on
  the device path, and simulate_episode (simulator.cpp:102-177) with the
  reference's closed-loop properties (test_simulator.cpp:132-260): same seed
  identical / different seeds differ, noise-free traces replay bitwise through
  the truth model, disturbances change nothing before their time, the straight
  corridor over 20 seeds, and the trace file columns.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_1707_02342_b200 import api
from paper_1707_02342_b200.api import (BicycleParams, ControlBounds, Controller, CostMap, CostParams, Disturbance,
                                       DomainError, SamplingParams, SGFilter, SimConfig)

P = BicycleParams()
PV = np.array([getattr(P, f) for f in BicycleParams.__dataclass_fields__], dtype=np.float64)


def o_brush(alpha, u_F):
    out = np.zeros(1)
    code = oracle.load().oracle_brush_tire_force(alpha, u_F, oracle.p(PV), oracle.p(out))
    if code:
        raise DomainError(code, "domain")
    return float(out[0])


def o_step(x, v, dt):
    out = np.zeros(7)
    oracle.chk(oracle.load().oracle_step_bicycle(oracle.p(np.asarray(x, float)), oracle.p(np.asarray(v, float)), dt,
                                                oracle.p(PV), oracle.p(out)))
    return out


BRUSH = [("library", api.brush_tire_force), ("oracle", lambda a, u: o_brush(a, u))]


@pytest.mark.parametrize("name,brush", BRUSH)
def test_brush_tire_pins(name, brush, oracle):
    # vanishes at zero slip
    assert brush(0.0, 0.0) == 0.0
    # linearizes to -C alpha at small slip
    for alpha in (0.001, 0.005, 0.01, -0.01, -0.003):
        assert brush(alpha, 0.0) == pytest.approx(-P.stiffness * alpha, rel=0.01)
    # branches agree at the crossover; the saturated branch is taken exactly there
    for u_F in (0.0, 10.0, -25.0, 50.0):
        limit = P.mu * P.load
        xi = math.sqrt(limit * limit - u_F * u_F) / limit
        cross = math.atan(3.0 * xi * P.mu * P.load / P.stiffness)
        for sign in (1.0, -1.0):
            saturated = -P.mu * xi * P.load * sign
            ta, c, m = math.tan(sign * cross), P.stiffness, P.mu * xi * P.load
            cubic = -c * ta + c * c / (3.0 * m) * ta * abs(ta) - c ** 3 / (27.0 * m * m) * ta ** 3
            assert cubic == pytest.approx(saturated, rel=1e-9)
            assert brush(sign * cross, u_F) == saturated
    # saturates hard past the crossover, odd in alpha
    f = brush(1.2, 0.0)
    assert f == pytest.approx(-P.mu * P.load, rel=1e-12) and brush(-1.2, 0.0) == -f
    # outside the friction circle: std::domain_error
    with pytest.raises(DomainError):
        brush(0.1, 1.01 * P.mu * P.load)
    brush(0.1, 0.99 * P.mu * P.load)


STEP = [("library", lambda x, v, dt: api.step_bicycle_truth(x, v, dt)), ("oracle", o_step)]


def mirror(s):
    return np.array([s[0], -s[1], -s[2], s[3], s[4], -s[5], -s[6]])


@pytest.mark.parametrize("name,step", STEP)
def test_truth_model_pins(name, step, oracle):
    # straight-line coast advances only p_x
    x = np.zeros(7)
    x[4] = 5.0
    n = step(x, [0.0, 0.0], 0.025)
    assert n[0] == pytest.approx(5.0 * 0.025, rel=1e-15) and n[1] == 0 and n[2] == 0 and n[4] == 5.0
    assert n[5] == 0 and n[6] == 0
    # trajectories mirror under a left-right flip (200 steps)
    a = np.array([0.0, 0.4, 0.3, 0.0, 6.0, 0.2, 0.5])
    b = mirror(a)
    for t in range(200):
        steer, thr = 0.4 * math.sin(0.05 * t), 0.3 * math.cos(0.02 * t)
        a = step(a, [steer, thr], 0.025)
        b = step(b, [-steer, thr], 0.025)
    assert np.allclose(a, mirror(b), rtol=1e-12, atol=0)
    # the slow-speed guard avoids the division by v_x = 0
    x = np.zeros(7)
    x[5], x[6] = 0.3, 1.0
    n = step(x, [0.5, 0.2], 0.025)
    assert np.all(np.isfinite(n))
    ef = api.brush_tire_force(-P.steer_scale * 0.5, P.force_scale * 0.2)
    er = api.brush_tire_force(0.0, P.force_scale * 0.2)
    assert n[5] == pytest.approx(0.3 + ((ef + er) / P.mass - 1.0 * 0.0) * 0.025, rel=1e-12)


def test_library_plant_bit_identical_to_oracle(oracle):
    rng = np.random.default_rng(5)
    for _ in range(300):
        x = np.array([rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-3, 3), 0.0, rng.uniform(-1, 8),
                      rng.uniform(-1, 1), rng.uniform(-2, 2)])
        v = rng.uniform(-1, 1, 2)
        assert np.array_equal(api.step_bicycle_truth(x, v, 0.025), o_step(x, v, 0.025))


# ----------------------------------------------------------------- device --
def tiny_map(vals, w, h):
    return CostMap(np.asarray(vals, dtype=np.float64).reshape(h, w), 0.0, 0.0, 1.0)


def unit_costs():
    return CostParams(alpha_track=1.0, alpha_speed=1.0, alpha_stab=1.0, v_des=6.0)


def bicycle_ctrl(params, m, cost, prec="fp64", noise="injected", sg=None, **kw):
    c = Controller(params, ControlBounds(), sg, cost, precision=prec, noise=noise, system="vehicle_bicycle", **kw)
    c.set_bicycle(P)
    c.set_costmap(m)
    return c


def one_step_params(T, gamma):
    return SamplingParams(samples=1, horizon_steps=T, dt=0.025, sigma_diag=(0.0306, 0.0506), lambda_=12.5,
                          gamma=gamma)


def traj_cost(ctrl, x0, plan, eps):
    """trajectory_cost (costs.cpp:60-79) through the device rollout: one sample, injected noise."""
    T = plan.shape[0]
    ctrl.plan = plan
    e = np.ascontiguousarray(np.asarray(eps, dtype=np.float64).T.reshape(1, 2 * T))  # c-major per sample
    return float(ctrl.rollout_batch(x0, e)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["bicycle", "mlp"])
def test_gamma_zero_plan_matters_only_through_realized_inputs(model):
    m = tiny_map([0.0, 0.2, 0.4, 0.6, 0.8, 1.0, 0.9, 0.7, 0.5], 3, 3)
    sp = one_step_params(8, 0.0)
    if model == "bicycle":
        c = bicycle_ctrl(sp, m, unit_costs())
    else:
        c = Controller(sp, ControlBounds(), None, unit_costs(), precision="fp64", noise="injected")
        c.set_mlp(api.MlpWeights.xavier(32, 3, 0.1))
        c.set_costmap(m)
    x0 = np.zeros(7)
    x0[4] = 2.0
    plan_a = np.stack([0.05 * np.arange(8), np.full(8, 0.3)], axis=1)
    eps_a = np.tile([0.02, -0.1], (8, 1))
    a = traj_cost(c, x0, plan_a, eps_a)
    b = traj_cost(c, x0, np.zeros((8, 2)), plan_a + eps_a)
    assert a == pytest.approx(b, rel=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_preclamped_rollouts_equal_clamping_inside(prec):
    m = tiny_map([0.0, 0.2, 0.4, 0.6], 2, 2)
    sp = one_step_params(6, 0.0)  # gamma = 0: the coupling (unclamped inputs) drops
    c = bicycle_ctrl(sp, m, unit_costs(), prec=prec)
    x0 = np.zeros(7)
    x0[4] = 3.0
    plan = np.tile([0.9, 0.8], (6, 1))
    eps = np.tile([0.5, 0.6], (6, 1))  # drives the steer past the bound
    eps_c = np.clip(plan + eps, -1.0, 1.0) - plan
    inside, pre = traj_cost(c, x0, plan, eps), traj_cost(c, x0, plan, eps_c)
    assert inside == pytest.approx(pre, rel=1e-15 if prec == "fp64" else 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_device_bicycle_rollout_matches_oracle(prec):
    from paper_1707_02342_b200 import workload
    w = workload.make("c0", samples=512)
    g = Controller(w.params, w.bounds, w.sg, CostParams(), precision=prec, noise="ref_splitmix",
                   system="vehicle_bicycle")
    o = oracle.OracleController(w.params, w.bounds, w.sg, CostParams(), precision=prec, noise="ref_splitmix",
                                system="vehicle_bicycle")
    for c in (g, o):
        c.set_bicycle(P)
        c.set_costmap(w.costmap)
    U = np.random.default_rng(2).uniform(-0.4, 0.4, (w.params.horizon_steps, 2))
    g.plan, o.plan = U, U
    dc = g.rollout_batch(w.x0[0])
    oc = o.rollout_batch(w.x0[0], threads=8)
    if prec == "fp64":
        assert np.allclose(dc, oc, rtol=1e-12, atol=0)
        for k in (0, 17, 511):
            assert np.allclose(g.rollout_states(w.x0[0], k), o.rollout_states(w.x0[0], k), rtol=1e-12, atol=1e-12)
        u_d, u_o = g.mpc_step(w.x0[0]), o.mpc_step(w.x0[0], threads=8)
        assert np.allclose(u_d, u_o, atol=1e-10) and np.allclose(g.plan, o.plan, atol=1e-10)
    else:
        rel = np.abs(dc - oc) / np.abs(oc)
        assert (rel <= 1e-5).mean() >= 0.99


def corridor_map():
    W, Hh, res, x0, y0 = 240, 61, 0.25, -10.0, -7.5
    y = y0 + np.arange(Hh) * res
    v = np.minimum(np.abs(y) / 2.0, 2.5)[:, None] * np.ones((1, W))
    return CostMap(v, x0, y0, res)


def sim_params(seed, K=128, T=40):
    return SamplingParams(samples=K, horizon_steps=T, dt=0.025, sigma_diag=(0.0306, 0.0506), lambda_=12.5,
                          gamma=0.1, explore_fraction=0.01, seed=seed)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_straight_corridor_stays_inside_across_20_seeds(prec):
    """test_simulator.cpp:191-231: the bicycle model controls the bicycle plant."""
    m = corridor_map()
    for seed in range(1, 21):
        c = bicycle_ctrl(sim_params(seed), m, CostParams(v_des=5.0), prec=prec, noise="ref_splitmix",
                         sg=SGFilter(9, 3))
        start = np.zeros(7)
        start[0], start[4] = -8.0, 4.0
        tr = api.simulate_episode(c, SimConfig(episode_s=6.0, exec_noise=False, start_state=start))
        assert len(tr.time) == 240 and not tr.aborted
        assert np.all(np.abs(tr.state[:, 1]) < 2.0), (prec, seed)
        assert tr.state[-1, 0] > 0.0, (prec, seed)


def oval_setup(seed, episode_s=4.0, **kw):
    from paper_1707_02342_b200 import workload
    m = workload.track_map()
    c = bicycle_ctrl(sim_params(seed, K=192), m, CostParams(v_des=4.0), prec="fp64", noise="ref_splitmix",
                     sg=SGFilter(9, 3))
    start = workload.initial_states(1, seed, 40.0, 25.0, True, (3.0, 3.0), 0.0)[0]
    return c, SimConfig(episode_s=episode_s, start_state=start, **kw)


@pytest.mark.gpu
def test_same_seed_identical_different_seeds_differ():
    a = api.simulate_episode(*oval_setup(77))
    b = api.simulate_episode(*oval_setup(77))
    assert np.array_equal(a.state, b.state) and np.array_equal(a.commanded, b.commanded)
    assert np.array_equal(a.realized, b.realized)
    c = api.simulate_episode(*oval_setup(78))
    assert c.state[-1, 0] != a.state[-1, 0]


@pytest.mark.gpu
def test_noise_free_trace_replays_bitwise_through_truth_model(oracle):
    c, sim = oval_setup(5, exec_noise=False)
    tr = api.simulate_episode(c, sim)
    x = np.asarray(sim.start_state, dtype=np.float64)
    for i in range(len(tr.time)):
        assert np.array_equal(tr.state[i], x), i
        x = o_step(x, np.clip(tr.commanded[i], -1, 1), 0.025)  # the oracle's independent restatement


@pytest.mark.gpu
def test_disturbances_change_nothing_before_their_time():
    clean = api.simulate_episode(*oval_setup(9, episode_s=3.0))
    c, sim = oval_setup(9, episode_s=3.0, disturbances=[Disturbance(1.5, -1.0, 1.5, 3.0)])
    kicked = api.simulate_episode(c, sim)
    before = clean.time < 1.5
    assert np.array_equal(clean.state[before], kicked.state[before])
    assert not np.array_equal(clean.state[~before], kicked.state[~before])


@pytest.mark.gpu
def test_estimate_noise_and_trace_file(tmp_path):
    c, sim = oval_setup(3, episode_s=1.0, estimate_noise_std=[0.01] * 7)
    tr = api.simulate_episode(c, sim)
    clean = api.simulate_episode(*oval_setup(3, episode_s=1.0))
    assert np.array_equal(tr.state[0], clean.state[0]) and not np.array_equal(tr.commanded, clean.commanded)
    path = os.path.join(tmp_path, "trace.csv")
    api.save_trace(tr, path)
    lines = open(path).read().splitlines()
    assert lines[0] == ("time_s,p_x,p_y,theta,roll,v_x,v_y,theta_dot,steer_cmd,throttle_cmd,"
                        "steer_real,throttle_real,cost,map_h")
    assert len(lines) == 1 + len(tr.time) == 41
