"""Pin the oracle (CPU restatement of the reference hot path) against the
reference's own known-answer tests and the published generator vectors.

Each test names the reference test it ports (paths under /root/reference/proj).
"""
import json
import math
import os

import numpy as np
import pytest

from paper_1707_02342_b200.api import CostParams, MlpWeights

HERE = os.path.dirname(os.path.abspath(__file__))
PINS = json.load(open(os.path.join(HERE, "golden", "reference_pins.json")))
STREAM = 0x706572747572626F


def H(x):
    return int(x, 16)


# ---------------------------------------------------------------- generators
def test_splitmix64_vector(oracle):
    for c in PINS["splitmix64"]["cases"]:
        assert oracle.splitmix64(c["x"]) == H(c["out"])


def test_philox_kat(oracle):
    for c in PINS["philox4x32_10"]["cases"]:
        assert oracle.philox([H(x) for x in c["ctr"]], [H(x) for x in c["key"]]) == [H(x) for x in c["out"]]


# ------------------------------------------------------------------ sampler
def test_sampler_addressing_bitwise(oracle):
    """test_core.cpp:65-76."""
    pin = PINS["sampler_addressing"]
    eps, _ = oracle.sample_perturbations(pin["K"], pin["T"], pin["sigma_diag"], 0.0, pin["seed"], pin["iteration"])
    for k in range(pin["K"]):
        for t in range(pin["T"]):
            for c in range(2):
                z = oracle.counter_normal(pin["seed"], STREAM, pin["iteration"], k, t, c)
                assert eps[k, c, t] == math.sqrt(pin["sigma_diag"][c]) * z


def test_sampler_determinism(oracle):
    """test_core.cpp:53-63."""
    a, _ = oracle.sample_perturbations(16, 20, [0.0306, 0.0506], 0.0, 99, 7)
    b, _ = oracle.sample_perturbations(16, 20, [0.0306, 0.0506], 0.0, 99, 7)
    c, _ = oracle.sample_perturbations(16, 20, [0.0306, 0.0506], 0.0, 99, 8)
    assert np.array_equal(a, b)
    assert not np.array_equal(a[0], c[0])


def test_sampler_covariance(oracle):
    """test_core.cpp:78-92."""
    pin = PINS["sampler_covariance"]
    eps, _ = oracle.sample_perturbations(pin["K"], pin["T"], pin["sigma_diag"], 0.0, pin["seed"], 0)
    for c in range(2):
        x = eps[:, c, :].ravel()
        var = np.mean(x * x) - np.mean(x) ** 2
        assert var == pytest.approx(pin["sigma_diag"][c], rel=pin["rel_tol"])


def test_sampler_scalar_moments(oracle):
    """test_core.cpp:94-109 (m = 1)."""
    pin = PINS["sampler_scalar_moments"]
    eps, _ = oracle.sample_perturbations(pin["K"], 1, pin["sigma_diag"], 0.0, pin["seed"], 0)
    x = eps[:, 0, 0]
    n = x.size
    se = math.sqrt(0.25 / n)
    assert abs(x.mean()) <= pin["mean_se"] * se
    assert (np.mean(x * x) - x.mean() ** 2) == pytest.approx(0.25, rel=pin["var_rel_tol"])


def test_zero_mean_flags(oracle):
    """test_core.cpp:111-120."""
    pin = PINS["zero_mean_flags"]
    _, flags = oracle.sample_perturbations(pin["K"], pin["T"], [0.0306, 0.0506], pin["explore_fraction"], 1, 0)
    assert flags.sum() == pin["flagged"] and flags[-1] == 1 and flags[0] == 0


def test_sampler_rejects_bad_params(oracle):
    """test_core.cpp:122-133."""
    with pytest.raises(ValueError):
        oracle.sample_perturbations(0, 10, [0.0306, 0.0506], 0.0, 1, 0)
    with pytest.raises(ValueError):
        oracle.sample_perturbations(4, 10, [0.0306, 0.0], 0.0, 1, 0)
    with pytest.raises(ValueError):
        oracle.sample_perturbations(4, 10, [0.0306, 0.0506], 1.0, 1, 0)
    with pytest.raises(ValueError):
        oracle.sample_perturbations(4, 10, [0.0306, 0.0506], -0.1, 1, 0)


def test_philox_noise_moments(oracle):
    """Production stream: same statistical bar as test_core.cpp:78-92."""
    eps, _ = oracle.sample_perturbations(1200, 100, [0.09, 0.1225], 0.0, 2024, 0, mode=2)
    for c, s2 in enumerate([0.09, 0.1225]):
        x = eps[:, c, :].ravel()
        assert np.var(x) == pytest.approx(s2, rel=0.02)
        assert abs(x.mean()) < 4 * math.sqrt(s2 / x.size)
    # channels uncorrelated, timesteps uncorrelated
    assert abs(np.corrcoef(eps[:, 0, :].ravel(), eps[:, 1, :].ravel())[0, 1]) < 0.01
    assert abs(np.corrcoef(eps[:, 0, :-1].ravel(), eps[:, 0, 1:].ravel())[0, 1]) < 0.01


# ------------------------------------------------------------------ weights
def test_softmin_reference_values(oracle):
    """test_weights.cpp:17-24."""
    pin = PINS["softmin_values"]
    w, rho, eta = oracle.it_weights(pin["costs"], pin["lambda"])
    assert np.allclose(w, pin["weights"], rtol=pin["rel_tol"])
    assert w.sum() == pytest.approx(1.0, abs=1e-12)


def test_softmin_uniform_exact(oracle):
    """test_weights.cpp:9-15."""
    pin = PINS["softmin_uniform"]
    w, rho, eta = oracle.it_weights(pin["costs"], pin["lambda"])
    assert all(x == 1.0 / 7.0 for x in w) and rho == 123.25 and eta == 7.0


def test_softmin_shift_invariance(oracle):
    """test_weights.cpp:26-34."""
    pin = PINS["softmin_shift"]
    a, _, _ = oracle.it_weights(pin["costs"], pin["lambda"])
    b, rho, _ = oracle.it_weights(np.array(pin["costs"]) + pin["shift"], pin["lambda"])
    assert np.max(np.abs(a - b)) <= pin["abs_tol"] and rho == pin["shift"]


def test_softmin_monotone_and_limits(oracle):
    """test_weights.cpp:36-55."""
    pin = PINS["softmin_monotone"]
    c = np.array(pin["costs"])
    w, _, _ = oracle.it_weights(c, pin["lambda"])
    for i in range(5):
        for j in range(5):
            if c[i] < c[j]:
                assert w[i] > w[j]
    assert w[1] >= 1 / 5
    pin = PINS["softmin_temperature"]
    hot, _, _ = oracle.it_weights(pin["costs"], pin["hot_lambda"])
    assert np.max(np.abs(hot - 0.25)) <= pin["hot_tol"]
    cold, _, _ = oracle.it_weights(pin["costs"], pin["cold_lambda"])
    assert cold[0] == pytest.approx(1.0) and cold[1:].max() <= pin["cold_tail_max"]


def test_softmin_rejects_bad_input(oracle):
    """test_weights.cpp:57-63."""
    with pytest.raises(ValueError):
        oracle.it_weights([], 1.0)
    with pytest.raises(ValueError):
        oracle.it_weights([0.0, 0.0, 0.0], 0.0)
    with pytest.raises(ValueError):
        oracle.it_weights([0.0, float("nan"), 0.0], 1.0)


# ------------------------------------------------------------------------ SG
def per_timestep_fit(seq, j, window, degree):
    """Independent LSQ oracle of test_smoothing.cpp:11-34."""
    n, half = len(seq), window // 2

    def reflect(i):
        while i < 0 or i >= n:
            if i < 0:
                i = -i
            if i >= n:
                i = 2 * (n - 1) - i
        return i
    X = np.array([[(r - half) ** c for c in range(degree + 1)] for r in range(window)], dtype=float)
    y = np.array([seq[reflect(j + r - half)] for r in range(window)])
    return np.linalg.lstsq(X, y, rcond=None)[0][0]


def test_sg_kernels(oracle):
    """test_smoothing.cpp:38-62 (+ window 9, degree 2 == degree 3)."""
    pin = PINS["sg_kernels"]
    assert np.allclose(oracle.sg_coefficients(5, 2), pin["w5d2"], rtol=pin["rel_tol"])
    c3 = oracle.sg_coefficients(3, 2)
    assert abs(c3[0]) <= 1e-12 and c3[1] == pytest.approx(1.0, rel=1e-12) and abs(c3[2]) <= 1e-12
    assert np.allclose(oracle.sg_coefficients(9, 2) * 231, pin["w9d2_times_231"], rtol=1e-12, atol=1e-10)
    assert np.allclose(oracle.sg_coefficients(9, 3), oracle.sg_coefficients(9, 2), rtol=1e-12, atol=1e-14)
    for window in (3, 5, 7, 9, 11):
        for degree in range(window):
            c = oracle.sg_coefficients(window, degree)
            assert abs(c.sum() - 1.0) <= 1e-12
            assert np.allclose(c, c[::-1], rtol=1e-10, atol=1e-12)
    for bad in ((4, 2), (5, 5), (1, 0), (5, -1)):
        with pytest.raises(ValueError):
            oracle.sg_coefficients(*bad)


def test_sg_smoothing_properties(oracle):
    """test_smoothing.cpp:71-154."""
    c93 = oracle.sg_coefficients(9, 3)
    seq = np.full((25, 2), -0.75)
    assert np.max(np.abs(oracle.sg_smooth(seq, c93) - seq)) <= 1e-12
    c52 = oracle.sg_coefficients(5, 2)
    q = np.arange(30, dtype=float) ** 2
    out = oracle.sg_smooth(q, c52)[:, 0]
    assert np.allclose(out[2:-2], q[2:-2], rtol=1e-9)
    imp = np.zeros(11)
    imp[5] = 1.0
    out = oracle.sg_smooth(imp, c52)[:, 0]
    assert np.allclose(out[3:8], c52, rtol=1e-12) and out[0] == 0.0
    # per-timestep LSQ oracle with mirror padding
    h = 0x9E3779B97F4A7C15
    seq = []
    for _ in range(40):
        h ^= (h << 13) & (2**64 - 1)
        h ^= h >> 7
        h ^= (h << 17) & (2**64 - 1)
        seq.append((h % 1000) / 250.0 - 2.0)
    seq = np.array(seq)
    for window, degree in ((5, 2), (9, 3), (7, 4)):
        out = oracle.sg_smooth(seq, oracle.sg_coefficients(window, degree))[:, 0]
        ref = [per_timestep_fit(seq, j, window, degree) for j in range(40)]
        assert np.allclose(out, ref, rtol=1e-9, atol=1e-12)
    # linear, channel independent, overshoot bound, length-1 fixed point
    rng = np.random.default_rng(0)
    x, y = rng.uniform(-1, 1, (24, 2)), rng.uniform(-1, 1, (24, 2))
    lhs = oracle.sg_smooth(2.5 * x - 0.5 * y, c93)
    assert np.max(np.abs(lhs - (2.5 * oracle.sg_smooth(x, c93) - 0.5 * oracle.sg_smooth(y, c93)))) <= 1e-12
    z = rng.uniform(-1, 1, (50, 2))
    assert np.abs(oracle.sg_smooth(z, c93)).max() <= np.abs(c93).sum() * np.abs(z).max() + 1e-12
    one = oracle.sg_smooth(np.array([[0.3, -0.8]]), c52)
    assert np.allclose(one, [[0.3, -0.8]], rtol=1e-12)


# ---------------------------------------------------------------- dynamics
def test_clamp(oracle):
    """test_dynamics.cpp:40-63."""
    lo, hi = [-1.0, -1.0], [1.0, 1.0]
    assert list(oracle.clamp_controls([0.25, -0.5], lo, hi)) == [0.25, -0.5]
    assert list(oracle.clamp_controls([1.7, -3.0], lo, hi)) == [1.0, -1.0]
    for i in range(50):
        v = [3 * oracle.counter_normal(4242, 0x74657374, 0, i, 0, 0), 3 * oracle.counter_normal(4242, 0x74657374, 0, i, 0, 1)]
        once = oracle.clamp_controls(v, lo, hi)
        assert np.array_equal(once, oracle.clamp_controls(once, lo, hi)) and np.all(np.abs(once) <= 1)
    with pytest.raises(ValueError):
        oracle.clamp_controls([0.0, 0.0], [1.0, 1.0], [1.0, 1.0])


def test_kinematic_split(oracle):
    """test_dynamics.cpp:188-211 (advance_split with a zero dynamic derivative)."""
    x = [0.0, 0.0, 0.7, 0.02, 4.0, -0.5, 0.9]
    n = oracle.advance_split(x, [0, 0, 0, 0], 0.025)
    assert list(n[3:]) == x[3:]
    assert n[0] == pytest.approx((math.cos(0.7) * 4.0 - math.sin(0.7) * -0.5) * 0.025)
    assert n[2] == pytest.approx(0.7 + 0.9 * 0.025)
    n = oracle.advance_split([0, 0, math.pi / 2, 0, 1.0, 0, 0], [0, 0, 0, 0], 0.1)
    assert n[1] == pytest.approx(0.1, rel=1e-12) and abs(n[0]) <= 1e-15
    with pytest.raises(ValueError):
        oracle.advance_split(x, [0, 0, 0, 0], 0.0)


def test_mlp_forward_pins(oracle):
    """test_dynamics.cpp:340-378."""
    zero = MlpWeights.zeros(32)
    assert np.all(oracle.mlp_forward(zero, [1, 1, 1, 1], [0.5, 0.5]) == 0)
    biased = MlpWeights.zeros(32)
    biased.b3[:] = [0.1, -0.2, 0.3, -0.4]
    assert np.array_equal(oracle.mlp_forward(biased, [1, 1, 1, 1], [1, 1]), biased.b3)

    def g(k, t):
        return oracle.counter_normal(4242, 0x74657374, 0, k, t, 0)
    w = MlpWeights.zeros(32)
    for i in range(32):
        for j in range(6):
            w.w1[i, j] = 0.3 * g(700 + i, j)
        for j in range(32):
            w.w2[i, j] = 0.2 * g(740 + i, j)
        w.b1[i] = 0.1 * g(780, i)
        w.b2[i] = 0.1 * g(781, i)
    for i in range(4):
        for j in range(32):
            w.w3[i, j] = 0.2 * g(790 + i, j)
        w.b3[i] = 0.1 * g(795, i)
    x0 = np.array([0.05, 3.0, -0.4, 0.7])
    v = [0.2, -0.3]
    h = 1e-6
    for c in range(4):
        e = np.zeros(4)
        e[c] = h
        fd = (oracle.mlp_forward(w, x0 + e, v) - oracle.mlp_forward(w, x0 - e, v)) / (2 * h)
        lin = (oracle.mlp_forward(w, x0 + e, v) - oracle.mlp_forward(w, x0, v)) / h
        assert np.max(np.abs(fd - lin)) <= 1e-5


def test_mlp_file_format(tmp_path):
    """test_dynamics.cpp:380-400 (save_mlp / load_mlp; bad header rejected)."""
    w = MlpWeights.zeros(32)
    w.b3[:] = [1, 2, 3, 4]
    w.w1[0, 0] = 0.5
    path = str(tmp_path / "mlp.txt")
    w.save(path)
    back = MlpWeights.load(path, allowed_hidden=(32,))
    assert np.array_equal(back.b3, w.b3) and np.array_equal(back.w1, w.w1)
    with open(path, "w") as f:
        f.write("6 16 16 4\n")
    with pytest.raises(RuntimeError):
        MlpWeights.load(path, allowed_hidden=(32,))


# ------------------------------------------------------------------- costs
def test_costmap_lookup_pins(oracle):
    """test_costs.cpp:34-62."""
    pin = PINS["costmap_lookup"]
    for key in ("centres", "midpoint", "clamp"):
        case = pin[key]
        vals = np.array(case["values"]).reshape(case["h"], case["w"])
        for px, py, expect in case["queries"]:
            assert oracle.costmap_lookup(vals, 0.0, 0.0, 1.0, px, py) == pytest.approx(expect, rel=1e-15, abs=1e-15)
    vals = np.array([0.1, 0.9, 0.4, 0.3, 0.7, 0.2, 0.5, 0.6, 0.8]).reshape(3, 3)
    mid = oracle.costmap_lookup(vals, 0, 0, 1, 1.0, 0.5)
    for x in (0.999999, 1.000001):
        assert oracle.costmap_lookup(vals, 0, 0, 1, x, 0.5) == pytest.approx(mid, rel=1e-5)


def unit_costs(**kw):
    c = CostParams(alpha_track=1.0, alpha_speed=1.0, alpha_stab=1.0, v_des=6.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_state_cost_pins(oracle):
    """test_costs.cpp:64-128."""
    z = np.zeros((2, 2))
    assert oracle.state_cost([0, 0, 0, 0, 6.0, 0, 0], 0, z, 0, 0, 1, unit_costs()) == 0.0
    ones = np.ones((2, 2))
    cp = unit_costs(alpha_speed=0.0, alpha_stab=0.0)
    assert oracle.state_cost([0] * 7, 0, ones, 0, 0, 1, cp) == pytest.approx(1.0 + 10000.0)
    assert oracle.state_cost([0] * 7, 22, ones, 0, 0, 1, cp) == pytest.approx(1.0 + 0.9 ** 22 * 10000.0, rel=1e-12)
    assert oracle.state_cost([0] * 7, 0, np.full((2, 2), 0.99), 0, 0, 1, cp) == pytest.approx(0.99)
    prev = math.inf
    for t in range(40):
        c = oracle.state_cost([0] * 7, t, ones, 0, 0, 1, unit_costs())
        assert c < prev
        prev = c
    cp = unit_costs(alpha_speed=0.0)
    zeta = -math.atan(-2.0 / 4.0)
    assert oracle.state_cost([0, 0, 0, 0, 4.0, -2.0, 0], 0, z, 0, 0, 1, cp) == pytest.approx(zeta * zeta, rel=1e-12)
    assert oracle.state_cost([0, 0, 0, 0, 4.0, 6.0, 0], 0, z, 0, 0, 1, cp) >= 10000.0
    assert oracle.state_cost([0, 0, 0, 0, 0.005, 6.0, 0], 0, z, 0, 0, 1, cp) == 0.0
    assert oracle.side_slip(-4.0, -2.0) == pytest.approx(math.atan(2.0 / 4.0))
    m = np.array([[0.3, 1.2], [0.0, 2.5]])
    for vx in (-3.0, 0.0, 2.0, 9.0):
        assert oracle.state_cost([0.7, 0.2, 0, 0, vx, 1.0, 0], 3, m, 0, 0, 1, CostParams()) >= 0.0


def test_baseline_crash_cost(oracle):
    """BASELINE.json cost form: 200 h + (v_x - 6)^2 + 10000 [h > 1 or |roll| > 0.6]."""
    cp = CostParams.baseline()
    half = np.full((2, 2), 0.5)
    assert oracle.state_cost([0, 0, 0, 0.0, 5.0, 0, 0], 3, half, 0, 0, 1, cp) == pytest.approx(200 * 0.5 + 1.0)
    assert oracle.state_cost([0, 0, 0, 0.7, 5.0, 0, 0], 3, half, 0, 0, 1, cp) == pytest.approx(200 * 0.5 + 1.0 + 1e4)
    off = np.full((2, 2), 1.2)
    assert oracle.state_cost([0, 0, 0, 0.0, 6.0, 0, 0], 3, off, 0, 0, 1, cp) == pytest.approx(200 * 1.2 + 1e4)
