"""The reference's acceptance criteria that concern the hot path, on the device
(acceptance.cpp): 3 (softmin shift invariance), 10 (the basis-model rollout
throughput budget).  Criterion 1 (LQ convergence) is test_lq_verification.py;
8 (thread-count determinism) is the partition bit-identity of
test_multirank_device.py; 2 and 6 are the weight and SG pins of
test_gpu_parity.py / test_oracle_pins.py.
"""
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ACCEPT_SEED, ACCEPT_STREAM = 20240, 0x616363657074  # acceptance.cpp:44 (gauss)


def gauss(k, t, c):
    """acceptance.cpp:43-45: counter_normal(20240, "accept", 0, k, t, c)."""
    return oracle.counter_normal(ACCEPT_SEED, ACCEPT_STREAM, 0, k, t, c)


def test_criterion3_softmin_shift_invariance():
    """acceptance.cpp:103-121: 257 costs on a 2^-20 grid (so + 1e9 is exact in
    double), lambda 12.5: the device it_weights of costs and costs + 1e9 agree
    to 1e-12 relative."""
    from paper_1707_02342_b200.api import Controller, SamplingParams

    costs = np.array([np.round(40.0 * abs(gauss(k, 0, 0)) * 1048576.0) / 1048576.0 for k in range(257)])
    g = Controller(SamplingParams(samples=257, horizon_steps=4, lambda_=12.5), system="quadratic",
                   precision="fp64")
    a = g.compute_weights(costs).weights
    b = g.compute_weights(costs + 1e9).weights
    worst = float(np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)))
    print(f"criterion 3: max relative weight change {worst:.2e} under +1e9")
    assert worst <= 1e-12
    ref, _, _ = oracle.it_weights(costs, 12.5)
    assert np.allclose(a, ref, rtol=1e-12, atol=0)


def test_criterion10_basis_model_throughput():
    """acceptance.cpp:344-393: one K=1024, T=100 basis-model iteration
    (mpc_step), median of 7 steady-clock timed calls <= 100 ms — here through
    the C ABI on the device (the workload's Theta is the builder's seeded
    physical fit, workload.py ref10)."""
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller

    w = workload.make("ref10")
    g = Controller(w.params, w.bounds, w.sg, w.cost, system="vehicle_basis", precision="fp32", noise="philox")
    g.set_basis(w.theta)
    g.set_costmap(w.costmap)
    for _ in range(2):
        g.mpc_step(w.x0[0])
    times = []
    for _ in range(7):
        t0 = time.perf_counter()
        g.mpc_step(w.x0[0])
        times.append(time.perf_counter() - t0)
    median_ms = 1e3 * sorted(times)[3]
    print(f"criterion 10: K=1024, T=100 basis-model iteration, median {median_ms:.3f} ms (<= 100 ms)")
    assert median_ms <= 100.0
